# A/B of alternative builds: TCG_LIB_DIR=build/ab/<v> python tests/gpu_probe.py ...
for round in 1 2; do
  for v in "$@"; do
    echo "== $v"
    TCG_LIB_DIR=build/ab/$v timeout 600 python tests/gpu_probe.py c5 c2 c4 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+' | paste - -
  done
done
