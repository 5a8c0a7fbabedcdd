# compute-sanitizer evidence (memcheck, racecheck, synccheck) for the device
# paths on small cases; logs under gpurun_out/$R
O=gpurun_out/${R:-san}; mkdir -p $O
for c in c1 c5_m0; do
  for tool in memcheck racecheck synccheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/probes/sanitize_case.py $c > $O/sanitizer_${tool}_$c.txt 2>&1
    echo "$tool $c rc=$? $(grep -h 'ERROR SUMMARY\|SANITIZE_CASE\|RACECHECK SUMMARY' $O/sanitizer_${tool}_$c.txt | tr '\n' ' ')"
  done
done
