O=gpurun_out/sweep_pp; mkdir -p $O; rm -f $O/*.txt
V='"" 1,2,1,4,2,0 2,2,4,3,1,0 1,2,2,4,2,0 2,2,2,3,1,0 2,2,2,4,1,0 2,1,4,4,1,0 1,2,1,5,1,0 4,2,2,3,1,0'
for c in c6 c2 c5_m0 c1; do
  eval timeout 600 python tools/probes/pp_sweep.py $c $V >> $O/sweep.txt 2>&1
done
for v in "" 1,2,1,4,2,0 2,2,4,3,1,0 4,2,2,3,1,0; do
  echo "c5b pp=$v $(TCG_FLOW_PP=$v timeout 600 python bench.py --config c5b --steps 10 --warmup 3 --no-cpu --no-one-shot 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["e2e"]["ms_per_step"], d["config"].get("parity_vs_oracle"))')" >> $O/c5b.txt
done
cat $O/sweep.txt $O/c5b.txt
