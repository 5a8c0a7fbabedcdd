O=gpurun_out/sweep_trace; mkdir -p $O
for c in c3 c4; do timeout 600 python tools/probes/gpu_flow_trace.py $c > $O/trace_$c.txt 2>&1; done
grep -v "^  pos" $O/trace_c3.txt; grep -v "^  pos" $O/trace_c4.txt; grep "^  pos" $O/trace_c3.txt | tail -15
