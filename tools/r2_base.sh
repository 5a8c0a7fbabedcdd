set -x
O=gpurun_out/r2base; mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi -q | grep -i -A3 "L2\|Clocks" | head -40 > $O/smi.txt
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err; echo rc=$?
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow_pipe -s 3 -c 1 -o $O/prof_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu > $O/ncu_c3.log 2>&1; echo rc=$?
