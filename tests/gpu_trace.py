"""Manual GPU probe: dump per-task device timestamps for critical-path analysis."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T

name = sys.argv[1]
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 256
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fz = T.GpuFactorizer(plan, T.GpuOptions(threads_per_cta=threads, timeout_s=20, trace=True, mode=mode))
for rep in range(2):
    fz.restore(); s = fz.factor()
tr, itr = fz.trace()
tab = plan.tables()
d = plan.dag()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"trace_{name}_{threads}.npz"), trace=tr, itrace=itr, task=tab["task"],
                    item=tab["item"][:, :6], efrom=d.edge_from, eto=d.edge_to, ms=s.device_ms)
print(name, threads, s.device_ms)
