O=gpurun_out/sweep_decouple; mkdir -p $O; rm -f $O/t.txt
for c in c3 c4 s27_16_k2 elast6_k1; do
  for d in 0 1; do
    echo "dec=$d $(TCG_FLOW_DECOUPLE=$d timeout 300 python tools/probes/pp_sweep.py $c "" 2>&1 | tail -1 | tr '\n' ' ')" >> $O/t.txt
  done
done
cat $O/t.txt
