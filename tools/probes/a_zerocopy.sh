# init_factor_values gathering A from pinned host memory (TCG_A_ZEROCOPY=1) against an H2D copy of all of A (0)
for z in 0 1; do echo "== TCG_A_ZEROCOPY=$z"; TCG_A_ZEROCOPY=$z timeout 300 python tools/probes/e2e_modes.py ${CFGS:-c3 c4 c2 c6} 2>&1 | grep -E "DRAIN=[012]"; done
