timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for r in 1 2; do
for m in 0 1; do echo "merge=$m"; TCG_FLOW_MERGE_ROWS=$m timeout 900 python tests/gpu_probe.py c1 c5 c2 c3 c4 c6 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+|bitwise=[A-Za-z]+' | paste - - - | tr '\n' ' '; echo; done
done
