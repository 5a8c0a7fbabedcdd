"""Manual GPU probe (not collected): hop latency of a pure dependence chain
(tridiagonal 'path' matrix, IC(0): row t needs row t-1), with nothing else
running, per mode."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T

for n in (1000, 4000):
    a = T.generate("path", n)
    fp = T.levelk_pattern(a, 0)
    for bounds in ([0, n], list(range(0, n, 64)) + [n]):
        plan = T.Plan(a, fp, T.RangeList(np.array(bounds, np.int32)))
        s = plan.stats()
        for mode in (4, 5):
            fz = T.GpuFactorizer(plan, T.GpuOptions(mode=mode))
            ts = []
            for _ in range(5):
                fz.restore()
                ts.append(fz.factor().device_ms)
            fz.close()
            depth = s.flow_depth if mode == 5 else s.item_depth
            print(f"path n={n} ranges={len(bounds)-1} mode={mode} depth={depth} "
                  f"ms={np.median(ts):.3f} us/hop={np.median(ts) * 1e3 / depth:.3f}", flush=True)
