"""Critical-path breakdown of a row-mode trace (gpurun_out/rows_*.npz)."""
import sys
import numpy as np

z = np.load(sys.argv[1])
st = z["stamps"].astype(np.int64)
rows, succ = z["rows"], z["succ"]
I = len(rows)
t0 = st[:, 0].min()
s, e = st[:, 0] - t0, st[:, 1] - t0
dur = e - s
kind = rows[:, 4]
print(f"rows={I} makespan={e.max()/1e3:.1f}us device_ms={float(z['ms']):.3f}")
names = ["CHOL", "TRSM", "HERK", "GEMM"]
for k in range(4):
    m = kind == k
    if m.any():
        print(f"  {names[k]}: n={m.sum()} dur med={np.median(dur[m]):.0f}ns mean={dur[m].mean():.0f} p99={np.percentile(dur[m],99):.0f}")
# predecessors from successor CSR
preds = [[] for _ in range(I)]
for k in range(I):
    for j in range(rows[k, 6], rows[k, 7]):
        preds[succ[j] & 0x3FFFFFFF].append(k)
cur = int(np.argmax(e)); path = []
while True:
    path.append(cur)
    if not preds[cur]:
        break
    cur = max(preds[cur], key=lambda p: e[p])
path = path[::-1]
busy = sum(dur[p] for p in path)
gaps = np.array([s[path[i]] - e[path[i - 1]] for i in range(1, len(path))])
print(f"critical path: {len(path)} rows, busy={busy/1e3:.1f}us gaps={gaps.sum()/1e3:.1f}us first_start={s[path[0]]/1e3:.1f}us")
print("  gap pct (10,50,90,99):", np.percentile(gaps, [10, 50, 90, 99]).astype(int))
print("  dur pct on path:", np.percentile([dur[p] for p in path], [10, 50, 90, 99]).astype(int))
# concurrency
ev = np.concatenate([np.stack([s, np.ones(I)], 1), np.stack([e, -np.ones(I)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
c = np.cumsum(ev[:, 1]); dt = np.diff(ev[:, 0], append=ev[-1, 0])
print(f"mean rows in flight={np.sum(c*dt)/e.max():.1f} max={c.max():.0f}")
hist = np.histogram(s, bins=10, range=(0, e.max()))[0]
print("row starts per decile:", hist.tolist())
