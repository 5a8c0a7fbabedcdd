"""Critical-path breakdown of a device trace (gpurun_out/trace_*.npz)."""
import sys
import numpy as np

z = np.load(sys.argv[1])
tr = z["trace"].astype(np.int64); task = z["task"]; item = z["item"]
ef, et = z["efrom"], z["eto"]
T = len(task)
t0 = tr[:, 0].min()
st, en = tr[:, 0] - t0, tr[:, 1] - t0
dur = en - st
kind = task[:, 0]
nitems = task[:, 3] - task[:, 2]
names = ["CHOL", "TRSM", "HERK", "GEMM"]
print(f"tasks={T} makespan={en.max()/1e3:.1f}us device_ms={float(z['ms']):.3f}")
for k in range(4):
    m = kind == k
    print(f"  {names[k]}: n={m.sum()} sum_dur={dur[m].sum()/1e3:.0f}us mean={dur[m].mean()/1e3:.2f}us max={dur[m].max()/1e3:.1f}us")
# critical path: walk back from the last-finishing task via latest-finishing predecessor
preds = [[] for _ in range(T)]
for a, b in zip(ef, et):
    preds[b].append(a)
cur = int(np.argmax(en))
path = []
while True:
    path.append(cur)
    if not preds[cur]:
        break
    cur = max(preds[cur], key=lambda p: en[p])
path = path[::-1]
busy = sum(dur[p] for p in path)
gaps = [st[path[0]]] + [st[path[i]] - en[path[i - 1]] for i in range(1, len(path))]
print(f"critical path: {len(path)} tasks, busy={busy/1e3:.1f}us gaps={sum(gaps)/1e3:.1f}us (mean gap {np.mean(gaps)/1e3:.2f}us)")
for k in range(4):
    sel = [p for p in path if kind[p] == k]
    print(f"  {names[k]}: {len(sel)} on path, busy={sum(dur[p] for p in sel)/1e3:.1f}us items={sum(nitems[p] for p in sel)}")
top = sorted(path, key=lambda p: -dur[p])[:12]
for p in top:
    print(f"   task {p} {names[kind[p]]} rows={task[p][1]} items={nitems[p]} dur={dur[p]/1e3:.1f}us")
# concurrency profile
ev = np.concatenate([np.stack([st, np.ones(T)], 1), np.stack([en, -np.ones(T)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
c = np.cumsum(ev[:, 1]); dt = np.diff(ev[:, 0], append=ev[-1, 0])
print(f"mean concurrency={np.sum(c*dt)/en.max():.1f} max={c.max():.0f}")
print("top tasks by duration (width, nlevels, items):")
for p in sorted(range(T), key=lambda p: -dur[p])[:8]:
    print(f"   task {p} {names[kind[p]]} width={task[p][1]} nlev={task[p][7]} items={nitems[p]} dur={dur[p]/1e3:.1f}us per-level={dur[p]/1e3/max(1,task[p][7]):.2f}us")
if "itrace" in z.files:
    it = z["itrace"].astype(np.int64) - t0
    ok = it[:, 3] > 0
    d_wait = it[:, 1] - it[:, 0]; d_merge = it[:, 2] - it[:, 1]; d_pub = it[:, 3] - it[:, 2]
    print("per-item phases (ns) over all items: wait/ready med %.0f  merge med %.0f  publish med %.0f" %
          (np.median(d_wait[ok]), np.median(d_merge[ok]), np.median(d_pub[ok])))
    for k in range(4):
        m = ok & np.isin(np.arange(len(it)), np.concatenate([np.arange(task[p][2], task[p][3]) for p in np.where(kind == k)[0]]) if (kind == k).any() else [])
        if m.any():
            print(f"  {names[k]}: items={m.sum()} ready-claim med={np.median(d_wait[m]):.0f} mean={d_wait[m].mean():.0f}  merge med={np.median(d_merge[m]):.0f} mean={d_merge[m].mean():.0f}  publish med={np.median(d_pub[m]):.0f} mean={d_pub[m].mean():.0f}")
    big = int(np.argmax(np.where(kind == 0, dur, 0)))
    ib, ie = task[big][2], task[big][3]
    seg = it[ib:ie]
    print(f"largest CHOL task {big}: items={ie-ib} dur={dur[big]/1e3:.1f}us")
    print("   first 12 items (claim, ready, merged, published) relative to task start:")
    for r in seg[:12]:
        print("     ", (r - st[big]).tolist())
    dw = seg[:, 1] - seg[:, 0]; dm = seg[:, 2] - seg[:, 1]; dp = seg[:, 3] - seg[:, 2]
    print(f"   med wait={np.median(dw):.0f} merge={np.median(dm):.0f} publish={np.median(dp):.0f} ns")
