"""Manual GPU probe (not collected): where the end-to-end time goes."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1601_05871_b200 as T

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan, T.GpuOptions())
vals = plan.tables()["values"]
hin = torch.from_numpy(vals.copy()).pin_memory()
hout = torch.empty(len(vals), dtype=torch.float64).pin_memory()
dev = torch.empty(len(vals), dtype=torch.float64, device="cuda")

def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return np.median(ts)

print(name, "nnz", len(vals), "MB", len(vals) * 8 / 1e6)
print("torch H2D pinned  ms", t(lambda: dev.copy_(hin, non_blocking=True)))
print("torch D2H pinned  ms", t(lambda: hout.copy_(dev, non_blocking=True)))
print("set_values (H2D+D2D) ms", t(lambda: fz.set_values_ptr(hin.data_ptr())))
def fac():
    fz.restore()
    return fz.factor()
print("factor (device ev)  ms", np.median([fac().device_ms for _ in range(10)]))
print("restore+factor wall ms", t(fac))
print("restore wall        ms", t(lambda: fz.restore()))
print("download            ms", t(lambda: fz.download_ptr(hout.data_ptr())))
print("factor_host         ms", t(lambda: fz.factor_host_ptr(hin.data_ptr(), hout.data_ptr())))
print("factor_host dev ev  ms", fz.last.device_ms)
