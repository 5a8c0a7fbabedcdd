# stale batch operands re-read together after a product waited (build/ab/refresh, NVEXTRA=-DTCG_FLOW_REFRESH=1)
O=gpurun_out/sweep_refresh; mkdir -p $O; rm -f $O/t.txt
for c in c3 c4 s27_16_k2 elast6_k1; do
  for lib in "" build/ab/refresh; do
    echo "lib=${lib:-default} $(TCG_LIB_DIR=$lib timeout 600 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/t.txt
  done
done
cat $O/t.txt
