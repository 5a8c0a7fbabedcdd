set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded or row_modes" 2>&1 | tail -2
for r in 1 2; do
timeout 600 python tests/gpu_probe.py c5 c2 c4 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+' | paste - -
TCG_FLOW_REMOTE=1 timeout 600 python tests/gpu_probe.py c5 c2 c4 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+' | paste - -
done
