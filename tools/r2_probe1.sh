mkdir -p gpurun_out/r2p1
timeout 900 python tools/r2_devprog_probe.py > gpurun_out/r2p1/probe.jsonl 2> gpurun_out/r2p1/probe.err; echo rc=$?
tail -5 gpurun_out/r2p1/probe.err
cat gpurun_out/r2p1/probe.jsonl
