"""Manual GPU probe (not collected): per-row cost with no dependences
(diagonal matrix: every row is a one-entry Chol row) -- the fixed cost of a
row in the value-flow kernel, rows per warp known."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T

for n in (355200, 1065600):
    a = T.CsrMatrix.from_arrays(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
                                np.full(n, 4.0))
    fp = T.levelk_pattern(a, 0)
    plan = T.Plan(a, fp, T.RangeList(np.array(list(range(0, n, 64)) + [n], np.int32)))
    fz = T.GpuFactorizer(plan, T.GpuOptions(mode=5))
    ts = []
    for _ in range(5):
        fz.restore()
        st = fz.factor()
        ts.append(st.device_ms)
    warps = st.grid_ctas * st.threads_per_cta // 32
    ms = float(np.median(ts))
    print(f"diagonal n={n}: {ms:.3f} ms, {n / warps:.0f} rows/warp -> {ms * 1e3 / (n / warps):.3f} us/row", flush=True)
