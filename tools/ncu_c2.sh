# ncu captures of the bench workload (run under gpurun; plain run first, per the recipe)
set -x
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow_pipe -s 3 -c 1 -o gpurun_out/prof_bench_c2 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
