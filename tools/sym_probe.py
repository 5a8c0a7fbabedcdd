"""Device level-k symbolic vs the host implementation and the reference's
levelk_pattern_bfs (oracle/_ref), per config: device ms, slow rows, host s."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402
from checkers import Reference, reference_available  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5", "c6"]:
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    g = T.GpuSymbolic(an.a_permuted)
    fp, st = g.levelk(level)
    ms = []
    for _ in range(5):
        ms.append(g.levelk(level)[1].device_ms)
    g.close()
    ok = np.array_equal(fp.pattern.col_idx, an.pattern.pattern.col_idx) and \
        np.array_equal(fp.pattern.row_ptr, an.pattern.pattern.row_ptr)
    t0 = time.perf_counter()
    T.levelk_pattern(an.a_permuted, level, threads=1)
    host1 = time.perf_counter() - t0
    ref = None
    if reference_available():
        t0 = time.perf_counter()
        Reference().levelk(an.a_permuted, level)
        ref = time.perf_counter() - t0
    print(f"{name}: n={a.nrows} nnz_u={st.nnz_u} equal={ok} device_ms={sorted(ms)[2]:.3f} "
          f"launches={st.kernel_launches} slow_rows={st.slow_rows} grid={st.grid_ctas} "
          f"host_1t_s={host1:.3f} ref_s={ref}", flush=True)
