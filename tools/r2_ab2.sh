O=gpurun_out/r2ab2; mkdir -p $O
for c in c3 c4 c2; do
 for ns in 0 32 100 300 1000; do for af in 0 8; do
  echo "$c BACKOFF=$ns AFTER=$af $(TCG_FLOW_BACKOFF_NS=$ns TCG_FLOW_BACKOFF_AFTER=$af timeout 300 python tools/probes/time_cfg.py $c 2>&1 | tail -1)"
 done; done
done > $O/ab.txt 2>&1
cat $O/ab.txt
