"""Manual GPU probe: factor one config a few times (for ncu captures)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
threads = int(sys.argv[3]) if len(sys.argv) > 3 else 256
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
fz = T.GpuFactorizer(plan, T.GpuOptions(threads_per_cta=threads, timeout_s=60, mode=mode))
for r in range(reps):
    fz.restore()
    s = fz.factor()
    print(name, r, f"{s.device_ms:.3f} ms", flush=True)
