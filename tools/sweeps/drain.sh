O=gpurun_out/sweep_drain; mkdir -p $O; rm -f $O/t.txt
for c in c3 c4 c2 c6; do
  for d in 0 1; do
    echo "$c drain=$d $(TCG_DRAIN=$d timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-one-shot 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3), d["e2e"]["drain_ctas"])')" >> $O/t.txt
  done
done
cat $O/t.txt
