O=gpurun_out/tune1; mkdir -p $O; rm -f $O/tune.txt
for c in c3 c4; do
  for kbbo in 2:0 2:200 3:0 3:100 3:200 3:400 4:0 4:200; do
    kb=${kbbo%:*}; bo=${kbbo#*:}
    echo "kb=$kb bo=$bo $(TCG_FLOW_KB=$kb TCG_FLOW_BACKOFF=$bo timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/tune.txt
  done
done
timeout 600 python tools/probes/gpu_flow_trace.py c3 $O/trace_c3.npz > $O/trace_c3.txt 2>&1
cat $O/tune.txt
