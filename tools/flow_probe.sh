for r in 1 2; do
for e in 0 1; do echo "extras=$e"; TCG_FLOW_EXTRAS=$e timeout 600 python tests/gpu_probe.py c5 c2 c4 c6 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+|bitwise=[A-Za-z]+' | paste - - - | tr '\n' ' '; echo; TCG_FLOW_EXTRAS=$e timeout 300 python tests/gpu_overhead_probe.py | tail -1; done
done
