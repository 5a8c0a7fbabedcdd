set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "row_modes or flow or batch or known or breakdown or unit" 2>&1 | tail -2
bash tools/ab_probe.sh S0 S2
