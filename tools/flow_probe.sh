for r in 1 2; do
for cfg in "3 2" "5 2" "5 3" "6 2" "5 1"; do set -- $cfg
echo "minb=$1 kb=$2"; TCG_FLOW_MINB=$1 TCG_FLOW_KB=$2 timeout 600 python tests/gpu_probe.py c5 c2 c4 c6 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+|grid=[0-9]+' | paste - - - | tr '\n' ' '; echo
done; done
