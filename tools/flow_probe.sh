set -x
P="timeout 600 python tests/gpu_probe.py c1 c5 c2 c3 c4 reps=5 mode=5"
$P
TCG_FLOW_DYN=1 $P
