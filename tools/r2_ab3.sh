O=gpurun_out/r2ab3; mkdir -p $O
for c in c3 c4; do for bo in 0 100 200 400; do
  echo "$c BO=$bo $(TCG_FLOW_BACKOFF=$bo timeout 300 python tools/probes/time_cfg.py $c 2>&1 | tail -1)"
done; done > $O/ab.txt 2>&1
for c in c3 c4; do for bo in 0 200; do
  echo "$c BO=$bo $(TCG_FLOW_BACKOFF=$bo timeout 300 python tools/probes/time_cfg.py $c 2>&1 | tail -1)"
done; done >> $O/ab.txt 2>&1
cat $O/ab.txt
