"""Manual GPU probe (not collected): where does the value-flow schedule lose
time? Runs one traced mode-5 factorization and attributes, along the
realised critical path, each step to either data (the row waited for an
operand) or the warp (the row's warp was still busy with its previous row).
usage: gpu_flow_trace.py c2 [out.npz]"""
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
rec, order, slot, upd = t["flow_rec"], t["flow_item"], t["flow_slot"], t["flow_upd"]
ni = len(t["row_rec"])
stamps = items.reshape(-1)[:2 * ni].reshape(-1, 2)[order].astype(np.int64)  # per position
t0 = stamps[:, 0].min()
s, e = stamps[:, 0] - t0, stamps[:, 1] - t0
npos = len(rec)
W = st.grid_ctas * st.threads_per_cta // 32
L = rec[:, 1] & ((1 << 30) - 1)
kind = (rec[:, 1] >> 30) & 3
owner = np.full(len(t["values"]), -1, np.int64)
for q in range(npos):
    owner[rec[q, 0]:rec[q, 0] + L[q]] = q
# ready time of each position: latest end among the positions it reads
ready = np.zeros(npos, np.int64)
src_of = np.full(npos, -1, np.int64)
for q in range(npos):
    tb = rec[q, 0]
    segs = [upd[u0:u1].ravel() for u0, u1 in slot[tb:tb + L[q], :2] if u1 > u0]
    srcs = owner[np.concatenate(segs)] if segs else np.zeros(0, np.int64)
    if kind[q] == 1:
        srcs = np.append(srcs, owner[rec[q, 2]])
    if len(srcs):
        m = srcs[np.argmax(e[srcs])]
        ready[q], src_of[q] = e[m], m
wp, order_w, makespan = plan.flow_schedule(W)  # the assignment tcg_factor laid out
prev = np.full(npos, -1, np.int64)  # previous position of the same warp
for w in range(W):
    seq = order_w[wp[w]:wp[w + 1]]
    prev[seq[1:]] = seq[:-1]
busy = np.where(prev >= 0, e[np.maximum(prev, 0)], 0)
print(f"simulated makespan {makespan:.1f} us")
print(f"{name}: kernel {st.device_ms:.3f} ms, {npos} rows, {W} warps, span {(e.max()) / 1e3:.1f} us")
dur = e - s
print(f"row time (start..end) us: median {np.median(dur) / 1e3:.2f}  p90 {np.percentile(dur, 90) / 1e3:.2f}  "
      f"mean {dur.mean() / 1e3:.2f}")
after_ready = e - np.maximum(ready, s)
print(f"end - max(ready, start) us: median {np.median(after_ready) / 1e3:.2f}  p90 "
      f"{np.percentile(after_ready, 90) / 1e3:.2f}")
# walk the realised critical path back from the last row
q = int(np.argmax(e))
data = warp = 0
tdata = twarp = 0
steps = []
while q >= 0:
    if src_of[q] >= 0 and ready[q] >= busy[q]:
        nq, kind_step = src_of[q], "data"
    elif prev[q] >= 0:
        nq, kind_step = prev[q], "warp"
    else:
        break
    dt = e[q] - e[nq]
    if kind_step == "data":
        data += 1
        tdata += dt
    else:
        warp += 1
        twarp += dt
    steps.append((kind_step, int(kind[q]), dt))
    q = nq
print(f"critical path: {data} data hops ({tdata / 1e3:.1f} us), {warp} warp-order hops ({twarp / 1e3:.1f} us)")
if len(sys.argv) > 2:
    np.savez_compressed(sys.argv[2], s=s, e=e, ready=ready, src=src_of, kind=kind, L=L, W=W)
