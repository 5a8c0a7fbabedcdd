O=gpurun_out/tune2; mkdir -p $O; rm -f $O/tune.txt
for c in c3 c4 s27_16_k2; do
  for bo in 100 200 400 800 1600 -200 -400 -800 -1600; do
    echo "bo=$bo $(TCG_FLOW_BACKOFF=$bo timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/tune.txt
  done
done
for c in c3 c4 c6; do timeout 300 python tools/probes/oneshot_parts.py $c >> $O/oneshot.txt 2>&1; done
cat $O/tune.txt $O/oneshot.txt
