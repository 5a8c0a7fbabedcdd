"""Manual GPU probe (not collected): one factorization of the diagonal case, for ncu."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T
n = 1065600
a = T.CsrMatrix.from_arrays(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.full(n, 4.0))
fp = T.levelk_pattern(a, 0)
plan = T.Plan(a, fp, T.RangeList(np.array(list(range(0, n, 64)) + [n], np.int32)))
fz = T.GpuFactorizer(plan, T.GpuOptions(mode=5))
for _ in range(2):
    fz.restore()
    print(fz.factor().device_ms)
