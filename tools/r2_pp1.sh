O=gpurun_out/pp1; mkdir -p $O
V='"" 1,2,4,2,0 1,2,5,1,0 1,4,4,2,0 2,4,3,1,0 2,4,3,1,200 2,8,2,1,200 4,4,3,1,0 4,4,3,1,200 4,2,3,1,200 4,8,2,1,200'
for c in c1 elast6_k1 s27_16_k2 c5_m0 c2 c4 c3; do
  eval timeout 600 python tools/probes/pp_sweep.py $c $V >> $O/sweep.txt 2>&1
done
cat $O/sweep.txt
