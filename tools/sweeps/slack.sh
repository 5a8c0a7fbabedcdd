# schedule placement between a unit's earliest and latest level (TCG_FLOW_SLACK, percent of its slack)
O=gpurun_out/${R:-sweep_slack}; mkdir -p $O; rm -f $O/t.txt
for c in ${CFGS:-c3 c4 c2 c6 s27_16_k2}; do for sl in ${SLACKS:-0 10 25 50 75 100}; do
  echo "$c slack=$sl $(TCG_FLOW_SLACK=$sl timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/t.txt
done; done
cat $O/t.txt
