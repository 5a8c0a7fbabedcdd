# The schedule build (flow_frontiers) under different cooperative grids: TCG_SCHED_CTAS = CTAs per SM
for c in ${CFGS:-c4 c3}; do for ct in 0 1 2; do
  if [ $ct = 0 ]; then unset TCG_SCHED_CTAS; else export TCG_SCHED_CTAS=$ct; fi
  echo "== $c ctas=$ct $(TCG_PLAN_TIMES=1 timeout 300 python tools/probes/oneshot_parts.py $c 2>&1 | grep -E 'upload schedule' | tail -2 | tr '\n' ' ')"
done; done
