O=gpurun_out/pp2; mkdir -p $O; rm -f $O/sweep.txt
V='"" 1,2,1,4,2 1,2,2,4,2 1,2,4,4,1 1,4,4,3,1 2,4,4,2,1 2,2,4,3,1 2,4,2,3,1 4,4,2,3,1 4,4,2,3,1,200 4,2,4,3,1 4,4,4,2,1 4,2,2,3,1 4,4,1,3,1'
for c in ${CFGS:-c3 c4 s27_16_k2 elast6_k1 c2 c5_m0 c1}; do
  eval timeout 600 python tools/probes/pp_sweep.py $c $V >> $O/sweep.txt 2>&1
done
cat $O/sweep.txt
