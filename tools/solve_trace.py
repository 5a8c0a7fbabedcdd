"""Critical-path attribution of one traced preconditioner apply (TCG_SOLVE_TRACE=1)."""
import os
import sys

os.environ["TCG_SOLVE_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402
from paper_1601_05871_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
which = int(sys.argv[2]) if len(sys.argv) > 2 else 1
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan)
fz.factor()
s = T.GpuTriSolve(fz)
r = torch.from_numpy(np.random.default_rng(1).standard_normal(a.nrows)).cuda()
z = torch.empty_like(r)
for _ in range(3):
    st = s.apply_device_ptr(r.data_ptr(), z.data_ptr(), which)
n = a.nrows
stamps = np.zeros(6 * n, np.uint64)
recs = np.zeros((2 * n, 4), np.int32)
assert s._lib.tcg_solve_trace(s.h, stamps.ctypes.data_as(N.u64p), recs.ctypes.data_as(C.c_void_p)) == 0
lo, hi = (0, n) if which == 1 else (n, 2 * n) if which == 2 else (0, 2 * n)
S = stamps.reshape(-1, 3)[lo:hi].astype(np.int64)
R = recs[lo:hi]
t0 = S[:, 0].min()
S = S - t0
print(f"{name} which={which} device_ms={st.device_ms:.3f} span_us={S[:, 2].max() / 1e3:.1f}")
u = an.pattern.pattern
# per position: operand rows -> their positions
pos_of = {}
back = R[:, 1] < 0
rows = R[:, 3]
pos_row = np.full((2, n), -1)
pos_row[back.astype(int), rows] = np.arange(len(R))
# walk back from the last finisher
q = int(np.argmax(S[:, 2]))
tot = {"wait_prev_row": 0, "handoff": 0, "gather": 0, "chain_store": 0}
hops = 0
while True:
    b_ = R[q, 1] < 0
    row = R[q, 3]
    # operands
    if not b_:
        cols = np.nonzero(u.col_idx == row)[0]
        src_rows = np.searchsorted(u.row_ptr, cols, side="right") - 1
        src = [pos_row[0, i] for i in src_rows if i != row]
    else:
        js = u.col_idx[u.row_ptr[row] + 1:u.row_ptr[row + 1]]
        src = [pos_row[1, j] for j in js]
        if which == 3:
            src.append(pos_row[0, row])
    src = [p for p in src if p >= 0]
    start, ready, end = S[q]
    if src:
        p = max(src, key=lambda p: S[p, 2])
        pend = S[p, 2]
    else:
        p, pend = None, 0
    tot["chain_store"] += end - ready
    if pend > start:
        tot["handoff"] += ready - pend
        tot["wait_prev_row"] += 0
    else:
        tot["gather"] += ready - start
        tot["wait_prev_row"] += start - pend
    hops += 1
    if p is None:
        break
    q = p
print(f"hops={hops}", {k: round(v / 1e3, 1) for k, v in tot.items()}, "(us)")
