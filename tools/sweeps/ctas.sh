O=gpurun_out/sweep_ctas; mkdir -p $O; rm -f $O/tune.txt
for c in c3 c4 s27_16_k2; do
  for ct in 3 2 1; do
    echo "ctas=$ct $(TCG_FLOW_CTAS=$ct timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/tune.txt
  done
done
for c in c2 c6; do
  for ct in 4 3 2; do
    echo "ctas=$ct $(TCG_FLOW_CTAS=$ct timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/tune.txt
  done
done
cat $O/tune.txt
