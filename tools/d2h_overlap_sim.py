"""How much of the factor's D2H could overlap the kernel? One traced mode-5
factorization: per chunk of U (positions [c*S, (c+1)*S)), the time its last
row finished; then a serial copy engine at BW GB/s copying chunks as they
complete. Prints the simulated end of the last copy vs kernel end + full copy."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan, T.GpuOptions(mode=5, trace=True, timeout_s=60))
fz.factor()
fz.restore()
st = fz.factor()
_, items = fz.trace()
fz.close()
t = plan.tables()
rec, order = t["flow_rec"], t["flow_item"]
stamps = items[order].astype(np.int64)
t0 = stamps[:, 0].min()
e = stamps[:, 3] - t0
L = rec[:, 1] & ((1 << 30) - 1)
nnz = len(t["values"])
end_of = np.zeros(nnz, np.int64)
for q in range(len(rec)):
    end_of[rec[q, 0]:rec[q, 0] + L[q]] = e[q]
kend = e.max()
print(f"{name}: traced kernel span {kend / 1e3:.1f} us, nnz {nnz}")
for bw in (45.0, 52.0):
    full = kend + nnz * 8 / bw
    for S in (1 << 12, 1 << 14, 1 << 16):
        nch = (nnz + S - 1) // S
        ready = np.array([end_of[c * S:min(nnz, (c + 1) * S)].max() for c in range(nch)])
        sizes = np.array([min(nnz, (c + 1) * S) - c * S for c in range(nch)]) * 8
        tcopy = 0.0
        for c in np.argsort(ready, kind="stable"):
            tcopy = max(tcopy, ready[c]) + sizes[c] / bw + 3000.0  # ns; no per-copy overhead
        frac = np.mean(ready <= kend * 0.5)
        print(f"  bw {bw} GB/s chunk {S * 8 >> 10} KiB: overlapped end {tcopy / 1e3:.1f} us vs serial "
              f"{full / 1e3:.1f} us; chunks ready by half-time {frac:.2f}")
