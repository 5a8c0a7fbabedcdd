"""Manual GPU probe (not collected): where does the value-flow schedule lose
time? Runs one traced mode-5 factorization and attributes, along the
realised critical path, each step to either data (the row waited for an
operand) or the warp (the row's warp was still busy with its previous row).
usage: gpu_flow_trace.py c2 [out.npz]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
slot, upd, _ = fz.flow_programs()
fz.close()
t = plan.flow_tables()
rec, order = t["flow_rec"], t["flow_item"]
stamps = items[order].astype(np.int64)  # per schedule position: start, operands final, -, end
t0 = stamps[:, 0].min()
s, r, e = stamps[:, 0] - t0, stamps[:, 1] - t0, stamps[:, 3] - t0
l0 = stamps[:, 2] - t0  # lane 0 (the diagonal of a Chol unit) done with its own program
npos = len(rec)
W = st.grid_ctas * st.threads_per_cta // 32
L = rec[:, 1] & ((1 << 30) - 1)
kind = (rec[:, 1] >> 30) & 3
owner = np.full(len(t["values"]), -1, np.int64)
for q in range(npos):
    owner[rec[q, 0]:rec[q, 0] + L[q]] = q
ready = np.zeros(npos, np.int64)  # latest end among the rows it reads
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
prev = np.arange(npos) - W
print(f"{name}: kernel {st.device_ms:.3f} ms, {npos} rows, {W} warps, span {e.max() / 1e3:.1f} us")
pct = lambda x: f"median {np.median(x) / 1e3:.2f} p90 {np.percentile(x, 90) / 1e3:.2f} us"
print("start -> operands final:", pct(r - s))
print("operands final -> end:  ", pct(e - r))
late = ready > s
print(f"rows whose last producer ended after they started: {late.mean():.1%}; "
      f"producer end -> operands final {pct((r - ready)[late])}")
# walk the realised critical path back from the last row
q = int(np.argmax(e))
acc = {"hop (producer end -> operands final)": 0, "row tail (operands final -> end)": 0,
       "gather after start (operands already final)": 0, "warp busy (previous row of the warp)": 0}
n = {k: 0 for k in acc}
while q >= 0:
    acc["row tail (operands final -> end)"] += e[q] - r[q]
    if src_of[q] >= 0 and ready[q] > s[q]:
        acc["hop (producer end -> operands final)"] += r[q] - ready[q]
        n["hop (producer end -> operands final)"] += 1
        q = src_of[q]
    else:
        acc["gather after start (operands already final)"] += r[q] - s[q]
        n["gather after start (operands already final)"] += 1
        if prev[q] >= 0 and e[prev[q]] <= s[q] + 2000:
            acc["warp busy (previous row of the warp)"] += s[q] - e[prev[q]]
            n["warp busy (previous row of the warp)"] += 1
            q = prev[q]
        else:
            break
for k in acc:
    print(f"  {k:48s} {acc[k] / 1e3:8.1f} us  ({n[k]} steps)")
if len(sys.argv) > 2:
    np.savez_compressed(sys.argv[2], s=s, r=r, e=e, l0=l0, ready=ready, src=src_of, kind=kind, L=L, W=W)
# the critical path row by row (the last 40 steps): length, products per
# coordinate (max), and where its time went
q = int(np.argmax(e))
path = []
while q >= 0 and len(path) < 100000:
    path.append(q)
    if src_of[q] >= 0 and ready[q] > s[q]:
        q = src_of[q]
    elif prev[q] >= 0 and e[prev[q]] <= s[q] + 2000:
        q = prev[q]
    else:
        break
print(f"critical path: {len(path)} rows")
prods = np.diff(slot[:, :2], axis=1).ravel()
for q in path[:40][::-1]:
    tb = rec[q, 0]
    pm = int(prods[tb:tb + L[q]].max()) if L[q] else 0
    ps = int(prods[tb:tb + L[q]].sum())
    print(f"  pos {q:7d} t={rec[q, 3]:7d} kind={kind[q]} L={L[q]:3d} prod max/sum {pm:4d}/{ps:6d} "
          f"start->final {(r[q] - s[q]) / 1e3:6.2f} final->end {(e[q] - r[q]) / 1e3:6.2f} "
          f"ready-start {(ready[q] - s[q]) / 1e3:7.2f} us")
# post-hop work of the critical rows: per lane (coordinate), the products whose
# operands were published in the last 5 us before the row's operands were
# final ("late"), and how many products follow the first late one in the
# lane's program (work that can only start after the hop)
late_n, after_n = [], []
for q in path[:60]:
    tb = rec[q, 0]
    for j in range(L[q]):
        u0, u1 = slot[tb + j, :2]
        if u1 <= u0:
            continue
        pr = upd[u0:u1]
        oe = np.maximum(e[owner[pr[:, 0]]], e[owner[pr[:, 1]]])
        late = oe > r[q] - 5000
        late_n.append(int(late.sum()))
        after_n.append(int(len(late) - np.argmax(late)) if late.any() else 0)
if late_n:
    print(f"critical rows, per coordinate: late products mean {np.mean(late_n):.1f} max {max(late_n)}; "
          f"products from the first late one on: mean {np.mean(after_n):.1f} p90 {np.percentile(after_n, 90):.0f} "
          f"max {max(after_n)}")
