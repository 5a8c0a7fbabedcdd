O=gpurun_out/r2ab1; mkdir -p $O
timeout 900 python tools/probes/gpu_flow_trace.py c3 > $O/trace_c3.txt 2>&1; echo trace=$?
for kb in 1 2 3 4; do for mb in 2 3 4; do
  echo "KB=$kb MINB=$mb $(TCG_FLOW_KB=$kb TCG_FLOW_MINB=$mb timeout 300 python tools/probes/time_cfg.py c3 2>&1 | tail -1)"
done; done > $O/ab_c3.txt 2>&1
cat $O/ab_c3.txt
