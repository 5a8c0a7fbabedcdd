O=gpurun_out/${R:-r2d}; mkdir -p $O
R=$R bash tools/gpu_round.sh
for c in c2 c4 c6 c5b c1 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
done
for c in c2 c6 c4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow -s 3 -c 1 -o $O/prof_bench_$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_full_$c.log 2>&1; echo ncu_$c=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_launch_c2.log 2>&1; echo launches_c2=$?
