"""Manual GPU probe: per-row stamps of the row-level mode."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T

name = sys.argv[1]
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=20, trace=True, mode=3))
for rep in range(2):
    fz.restore(); s = fz.factor()
_, itr = fz.trace()
ni = itr.shape[0]
st = itr.reshape(-1)[:2 * ni].reshape(-1, 2)
tab = plan.tables()
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"rows_{name}.npz"), stamps=st, rows=tab["row_rec"],
                    succ=tab["row_succ"], ms=s.device_ms)
print(name, s.device_ms)
