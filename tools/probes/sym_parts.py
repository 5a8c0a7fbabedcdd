"""The level-k symbolic end to end split into its parts: upload (host checks + H2D of PᵀAP's
pattern), the device search, the download and the Python arrays (4 calls, the last 3 shown)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T  # noqa: E402
from paper_1601_05871_b200 import _native as N  # noqa: E402
import ctypes as C  # noqa: E402
from conftest import analyzed  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    _, an = analyzed(name)
    ap, level = an.a_permuted, an.pattern.level_cap
    g = T.GpuSymbolic(ap)
    lib = g._lib
    for i in range(4):
        t = [time.perf_counter()]
        g.upload(ap)
        t.append(time.perf_counter())
        s = N.SymStats()
        g._check(lib.tcg_sym_levelk(g.h, level, 0, C.byref(s)))
        t.append(time.perf_counter())
        n = ap.nrows
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(max(int(s.nnz_u), 1), np.int32)
        g._check(lib.tcg_sym_download(g.h, rp.ctypes.data_as(N.i64p), ci.ctypes.data_as(N.i32p)))
        t.append(time.perf_counter())
        vals = np.ones(int(s.nnz_u))
        t.append(time.perf_counter())
        d = [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])]
        if i:
            print(f"{name}: upload {d[0]} levelk {d[1]} (device {s.device_ms:.3f}) download {d[2]} ones {d[3]} ms",
                  flush=True)
    g.close()
