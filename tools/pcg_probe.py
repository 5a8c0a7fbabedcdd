"""IC(k)-preconditioned vs plain CG on the GPU (paper_1601_05871_b200.pcg):
iterations and wall time to a 1e-8 relative residual, b = ones, per
convergence-check interval (PCG_CHECK, default 1,8)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402

for name in sys.argv[1:] or ["c2", "c6"]:
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(plan)
    fz.factor()
    s = T.GpuTriSolve(fz)
    s.set_matrix(an.a_permuted)
    b = np.ones(a.nrows)
    for pre in (True, False):
      for ce in (int(c) for c in os.environ.get("PCG_CHECK", "1,8").split(",")):
        T.pcg(s, b, tol=1e-8, maxit=5, precondition=pre, check_every=ce)  # warm-up
        r = T.pcg(s, b, tol=1e-8, maxit=5000, precondition=pre, check_every=ce)
        print(f"{name} {'IC' if pre else 'plain'} check_every={ce}: {r.iterations} iterations, converged={r.converged}, "
              f"{r.seconds * 1e3:.1f} ms ({r.seconds * 1e3 / r.iterations:.3f} ms/iteration)", flush=True)
    s.close()
    fz.close()
