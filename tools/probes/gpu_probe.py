"""Manual GPU probe: parity + timing over the configs (not collected by pytest).
usage: gpu_probe.py c2 [c3 ...] [threads=256] [ctas=0] [cap=0] [reps=6]"""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T
from checkers import Oracle

kv = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
names = [a for a in sys.argv[1:] if "=" not in a] or ["c1", "c2"]
threads, ctas, cap, reps, mode, lanes = (int(kv.get(k, d)) for k, d in
                            (("threads", 256), ("ctas", 0), ("cap", 0), ("reps", 6), ("mode", 0), ("lanes", 0)))
O = Oracle()
for name in names:
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    u = an.pattern.pattern
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    ref, st, _, _ = O.factor_serial(an.a_permuted, u)
    fz = T.GpuFactorizer(plan, T.GpuOptions(threads_per_cta=threads, ctas_per_sm=ctas,
                                            staging_cap=cap, timeout_s=20, mode=mode, lanes_per_row=lanes))
    times = []
    for rep in range(reps):
        fz.restore()
        s = fz.factor()
        times.append(s.device_ms)
    v = fz.download()
    bit = np.array_equal(v.view(np.int64), ref.view(np.int64))
    rel = float(np.max(np.abs(v - ref) / (np.abs(ref) + 1e-300)))
    print(f"{name} mode={s.mode} thr={threads} ctas/sm={ctas} grid={s.grid_ctas} cap={s.staging_cap} smem={s.smem_bytes} "
          f"lanes={s.lanes_per_row} helpers={s.helpers_run} med_ms={np.median(times):.3f} min_ms={min(times):.3f} "
          f"bitwise={bit} maxrel={rel:.2e}", flush=True)
    fz.close()
