O=gpurun_out/pp3; mkdir -p $O; rm -f $O/sweep.txt
V='"" 1,2,1,4,2,0 1,2,2,4,2,0 1,2,4,4,1,0 1,4,4,3,1,0 2,4,4,2,1,0 2,2,4,3,1,0 2,4,2,3,1,0 4,4,2,3,1,0 4,2,4,3,1,0 4,4,4,2,1,0 4,2,2,3,1,0 4,4,1,3,1,0'
for c in c3 c4 s27_16_k2; do
  eval timeout 600 python tools/probes/pp_sweep.py $c $V >> $O/sweep.txt 2>&1
done
timeout 300 python tools/probes/gpu_flow_trace.py c3 > $O/trace_c3.txt 2>&1
cat $O/sweep.txt; tail -30 $O/trace_c3.txt
