# program pairs loaded with an L2 evict-first policy (build/ab/evf, make lib NVEXTRA=-DTCG_PROG_EVICT_FIRST) vs the default build
O=gpurun_out/sweep_evf; mkdir -p $O; rm -f $O/t.txt
for c in c3 c4 s27_16_k2; do
  for lib in "" build/ab/evf; do
    echo "lib=${lib:-default} $(TCG_LIB_DIR=$lib timeout 600 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1)" >> $O/t.txt
  done
done
cat $O/t.txt
