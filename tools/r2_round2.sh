O=gpurun_out/${R:-r2c}; mkdir -p $O
R=$R bash tools/gpu_checked.sh
R=$R bash tools/gpu_round.sh
for c in c2 c6; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_flow -s 3 -c 1 -o $O/prof_bench_$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-one-shot > $O/ncu_full_$c.log 2>&1; echo ncu_$c=$?
done
