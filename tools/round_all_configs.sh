O=gpurun_out/${R:-all}; mkdir -p $O
R=$R bash tools/gpu_checked.sh
R=$R bash tools/gpu_round.sh
for c in c2 c4 c6 c5b c1 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow -s 3 -c 1 -o $O/prof_bench_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_full_c4.log 2>&1; echo ncu_c4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c6.csv python bench.py --config c6 --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_launch_c6.log 2>&1; echo launches_c6=$?
timeout 600 python tools/probes/oneshot_parts.py c2 c3 c6 > $O/oneshot.txt 2>&1
