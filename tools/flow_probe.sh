for r in 1 2; do
for o in "" "0.8,1.0,0.3" "1.5,1.0,0.3" "0.8,0.5,0.5" "2,1,0.2"; do echo "order=$o"; env ${o:+TCG_FLOW_ORDER=$o} timeout 600 python tests/gpu_probe.py c5 c2 c4 reps=5 mode=5 2>&1 | grep -oE '^c[0-9]|med_ms=[0-9.]+|bitwise=[A-Za-z]+' | paste - - - | tr '\n' ' '; echo; done
done
