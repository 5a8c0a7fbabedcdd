# diagonal-block slices cut at fixed column panels (TCG_FLOW_PANEL, flow_plan.cpp) vs the 32-entry Chol cap (0)
O=gpurun_out/sweep_panel; mkdir -p $O; rm -f $O/t.txt
for c in c3 c4 s27_16_k2 elast6_k1; do
  for pn in 0 32 24 16; do
    echo "panel=$pn $(TCG_FLOW_PANEL=$pn timeout 600 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/t.txt
  done
done
cat $O/t.txt
