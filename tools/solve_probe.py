"""Device time of the preconditioner apply per config and direction (median of 7)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3", "c6"]:
    if name.startswith("path"):
        a, level = T.generate("path", int(name[4:])), 0
        an = T.analyze(a, level=0, leaf_size=int(name[4:]))  # one leaf: natural order, a pure chain
    else:
        a, level = T.config_matrix(name)
        an = T.analyze(a, level=level)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(plan)
    fz.factor()
    s = T.GpuTriSolve(fz)
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(a.nrows)).cuda()
    z = torch.empty_like(r)
    out = []
    for which in (1, 2, 3):
        ms = []
        for _ in range(7):
            ms.append(s.apply_device_ptr(r.data_ptr(), z.data_ptr(), which).device_ms)
        out.append(f"w{which}={statistics.median(ms):.3f}")
    st = s.stats()
    print(name, os.environ.get("TCG_SOLVE_CTAS", "-"), " ".join(out), "depth", st.depth_forward, st.depth_backward,
          "grid", st.grid_ctas, "factor_ms", (fz.restore(), round(fz.factor().device_ms, 3))[1], flush=True)
    s.close()
    fz.close()
