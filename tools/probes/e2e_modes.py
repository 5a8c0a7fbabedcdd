"""End to end (tcg_factor_host_a, pinned buffers) under each way the factor can
leave -- TCG_DRAIN=0 a copy after the launch, 1 the drain CTAs, 2 chunked copies
beside the launch -- wall ms (median of 10 after 3) and the factor's bits
against the device-only result."""
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402

for name in sys.argv[1:] or ["c3"]:
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    fz.restore()
    dev_ms = fz.factor().device_ms
    ref = fz.download().copy()
    hin = torch.from_numpy(np.ascontiguousarray(an.a_permuted.values)).pin_memory()
    hout = torch.empty(len(ref), dtype=torch.float64).pin_memory()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for mode in ("0", "1", "2"):
        os.environ["TCG_DRAIN"] = mode
        ts = []
        for i in range(14):
            if i == 13:  # only the last, untimed call starts from a cleared buffer (CPU-written
                hout.fill_(-1.0)  # lines make the DMA slower; a stale factor would pass the check otherwise)
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st = fz.factor_host_a_ptr(hin.data_ptr(), hout.data_ptr())
            ts.append((time.perf_counter() - t0) * 1e3)
        same = np.array_equal(hout.numpy().view(np.int64), ref.view(np.int64))
        print(f"{name} TCG_DRAIN={mode} e2e ms {statistics.median(ts[3:13]):.3f} min {min(ts[:13]):.3f} device {st.device_ms:.3f} "
              f"(device-only {dev_ms:.3f}) drain_ctas {st.drain_ctas} bitwise={same}", flush=True)
    del os.environ["TCG_DRAIN"]
    fz.close()
