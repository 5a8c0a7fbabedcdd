"""GPU probe: the lean plan + device-built programs against the host-flattened
programs (same tables expected) and the golden factor hashes; plan, build
and factor times per configuration.  usage: r2_devprog_probe.py [names...]"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T  # noqa: E402
from checkers import Oracle  # noqa: E402

G = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
O = Oracle()
SMALL = {"c1": ("grid2d", 100, 100, 0, 0, 64), "grid20_k2_leaf4": ("grid2d", 20, 20, 0, 2, 4),
         "rand_spd_200": ("random_spd", 200, 20000, 7, 1, 8), "elast6_k1": ("elasticity", 6, 0, 3, 1, 16),
         "s27_16_k2": ("stencil27", 16, 0, 1, 2, 64)}
names = sys.argv[1:] or ["c1", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1", "s27_16_k2", "c5", "c2", "c3", "c4"]
for name in names:
    if name in SMALL:
        kind, p0, p1, seed, level, leaf = SMALL[name]
        a = T.generate(kind, p0, p1, seed)
        an = T.analyze(a, level=level, leaf_size=leaf)
        gname = name
    else:
        a, level = T.config_matrix(name)
        an = T.analyze(a, level=level)
        gname = "c5_m0" if name == "c5" else name
    t0 = time.perf_counter()
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    t_plan = time.perf_counter() - t0
    ps = plan.stats()
    t0 = time.perf_counter()
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=60))
    t_up = time.perf_counter() - t0
    slot, upd, build_ms = fz.flow_programs()
    ts = []
    for _ in range(5):
        fz.restore()
        ts.append(fz.factor().device_ms)
    vals = fz.download()
    fz.close()
    ok = O.hash(vals) == G[gname]["factor_values"]
    line = {"name": name, "nnz": int(an.pattern.pattern.nnz()), "plan_s": round(t_plan, 4),
            "plan_stats_s": round(ps.plan_seconds, 4), "block_s": round(ps.block_build_seconds, 4),
            "upload_s": round(t_up, 4), "build_ms": round(build_ms, 3), "units": int(ps.flow_rows),
            "depth": int(ps.flow_depth), "products": int(len(upd)), "factor_ms": round(statistics.median(ts), 4),
            "golden": ok}
    if an.pattern.pattern.nnz() <= 3_000_000 or "--host" in os.environ.get("PROBE", ""):
        t0 = time.perf_counter()
        ph = plan.problem_host_flow()
        t_full = time.perf_counter() - t0
        fh = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=60), problem=ph)
        s2, u2, _ = fh.flow_programs()
        th = []
        for _ in range(5):
            fh.restore()
            th.append(fh.factor().device_ms)
        fh.close()
        line.update({"same_slot": bool(np.array_equal(s2, slot)), "same_upd": bool(np.array_equal(u2, upd)),
                     "full_plan_s": round(t_full, 3), "host_flow_factor_ms": round(statistics.median(th), 4),
                     "host_flow_depth": int(plan.stats().host_flow_depth)})
    print(json.dumps(line), flush=True)
