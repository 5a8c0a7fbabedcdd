# A/B of alternative builds in one session: bash tools/ab_probe.sh <dir under build/ab> ...
for round in 1 2; do
  for v in "$@"; do
    echo "== $v"
    TCG_LIB_DIR=build/ab/$v timeout 600 python tests/gpu_probe.py c5 c2 c4 c6 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+|bitwise=[A-Za-z]+' | paste - - -
    [ $round = 1 ] && TCG_LIB_DIR=build/ab/$v timeout 300 python tests/gpu_chain_probe.py 2>&1 | grep "mode=5" | head -2
  done
done
