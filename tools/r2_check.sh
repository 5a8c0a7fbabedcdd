# GPU tests + bench lines of the main configurations (one B200)
O=gpurun_out/${R:-check}; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
for c in ${CFGS:-c3 c2 c6 c5b c4}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['ms_per_step'], d['e2e']['ms_per_step'], d['config'].get('parity_vs_oracle'), d.get('one_shot',{}).get('ms'))"
done
