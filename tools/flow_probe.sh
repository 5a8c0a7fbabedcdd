set -x
P="timeout 600 python tests/gpu_probe.py c5 c2 c4 reps=5 mode=5"
$P
for b in 20 50 100 200 400; do TCG_FLOW_BACKOFF=$b $P; done
