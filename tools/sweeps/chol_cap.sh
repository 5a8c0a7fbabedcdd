# Chol units capped at 8..32 coordinates (TCG_FLOW_CHOL_MAX, flow_plan.cpp): device ms and parity
O=gpurun_out/sweep_chol_cap; mkdir -p $O; rm -f $O/cm.txt
for c in c3 c4 s27_16_k2 elast6_k1; do
  for m in 32 24 16 12 8; do
    echo "cholmax=$m $(TCG_FLOW_CHOL_MAX=$m timeout 600 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/cm.txt
  done
done
cat $O/cm.txt
