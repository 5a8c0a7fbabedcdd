# The round's GPU check on one B200 (run through gpurun): tests, smoke, the
# bench lines (ours on C3 + the reference arm), the ncu launch list and one
# ncu --set full capture of the factor kernel. Output: gpurun_out/$R/.
R=${R:-round}
O=gpurun_out/$R
mkdir -p $O
set -x
nproc > $O/nproc.txt
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -2 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?; cat $O/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref_rc=$?; cat $O/bench_ref.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow -s 3 -c 1 -o $O/prof_bench_c3 python bench.py --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_full.log 2>&1; echo ncu2_rc=$?
