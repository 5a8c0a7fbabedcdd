O=gpurun_out/sweep_pp_backoff; mkdir -p $O; rm -f $O/t.txt
for c in c6 c2 c5_m0 c1; do
  echo "$(timeout 300 python tools/probes/pp_sweep.py $c 1,2,1,4,2,0 1,2,1,4,2,50 1,2,1,4,2,100 1,2,1,4,2,200 2,2,2,3,1,0 2,2,2,3,1,100 2>&1)" >> $O/t.txt
done
cat $O/t.txt
