O=gpurun_out/sweep_backoff; mkdir -p $O; rm -f $O/tune.txt
for c in c3 c4 s27_16_k2; do
  for bo in 0 100 200 400 600 1000 2400; do
    echo "bo=$bo $(TCG_FLOW_BACKOFF=$bo timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/tune.txt
  done
done
for c in c2 c6 c1 c5_m0 elast6_k1; do echo "default $(timeout 300 python tools/probes/pp_sweep.py $c '' 0 2>&1 | tail -2 | tr '\n' ' ')" >> $O/tune.txt; done
cat $O/tune.txt
