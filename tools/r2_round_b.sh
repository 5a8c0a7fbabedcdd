O=gpurun_out/r2b; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
for c in c3 c2 c4; do timeout 900 python tools/probes/gpu_flow_trace.py $c > $O/trace_$c.txt 2>&1; echo trace_$c=$?; done
