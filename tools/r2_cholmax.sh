O=gpurun_out/cm2; mkdir -p $O; rm -f $O/cm.txt
for c in c3 c4 s27_16_k2 elast6_k1 c1 c5_m0; do
  for m in none 32 24 16 8; do
    if [ $m = none ]; then unset TCG_FLOW_CHOL_MAX; else export TCG_FLOW_CHOL_MAX=$m; fi
    echo "cholmax=$m $(timeout 600 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/cm.txt
  done
done
unset TCG_FLOW_CHOL_MAX
cat $O/cm.txt
