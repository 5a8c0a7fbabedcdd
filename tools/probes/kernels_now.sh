# device ms of the default kernels on the long- and medium-program matrices (and the small ones)
for c in c3 c4 s27_16_k2 elast6_k1 grid20_k2_leaf4 c5; do timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1; done
for c in c2 c6; do TCG_FLOW_PP=0 timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1; timeout 300 python tools/probes/pp_sweep.py $c '' 2>&1 | tail -1; done
