"""End-to-end (tcg_factor_host_a, pinned buffers) with and without the in-kernel
drain: wall ms and device ms (H2D + init + prelude + factor [+ drain tail]), median of 9."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan)
a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
out = torch.empty(fz.nnz, dtype=torch.float64).pin_memory()
fz.restore()
plain = statistics.median([(fz.restore(), fz.factor().device_ms)[1] for _ in range(9)])
print(f"{name}: factor only {plain:.3f} ms (device)")
settings = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "4", "8", "16"]
for dr in settings:
    if dr == "0":
        os.environ["TCG_DRAIN"] = "0"
    else:
        os.environ.pop("TCG_DRAIN", None)
        os.environ["TCG_DRAIN_CTAS"] = dr
    wall, dev = [], []
    for _ in range(9):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(st.device_ms)
    print(f"  drain_ctas={st.drain_ctas:2d} wall {statistics.median(wall):.3f} ms, device {statistics.median(dev):.3f} ms",
          flush=True)
