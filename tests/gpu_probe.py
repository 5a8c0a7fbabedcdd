"""Manual GPU probe: parity + timing over the configs (not collected by pytest)."""
import sys, time, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T
from checkers import Oracle

O = Oracle()
names = sys.argv[1:] or ["c1", "c2"]
for name in names:
    threads = 256
    if ":" in name:
        name, threads = name.split(":"); threads = int(threads)
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    u = an.pattern.pattern
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    ref, st, _, _ = O.factor_serial(an.a_permuted, u)
    fz = T.GpuFactorizer(plan, T.GpuOptions(threads_per_cta=threads, timeout_s=20))
    times = []
    for rep in range(6):
        fz.restore()
        s = fz.factor()
        times.append(s.device_ms)
    v = fz.download()
    bit = np.array_equal(v.view(np.int64), ref.view(np.int64))
    rel = float(np.max(np.abs(v - ref) / (np.abs(ref) + 1e-300)))
    print(f"{name} thr={threads} nnz_u={u.nnz()} grid={s.grid_ctas} cap={s.staging_cap} smem={s.smem_bytes} "
          f"ms={['%.3f' % t for t in times]} bitwise={bit} maxrel={rel:.2e} executed={s.tasks_executed}", flush=True)
    fz.close()
