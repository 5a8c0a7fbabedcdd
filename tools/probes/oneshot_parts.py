"""Where a one-shot factor_by_blocks_gpu call spends its wall time: plan,
context + upload (incl. the device-built programs), factor, download, close;
4 calls in one warm process."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T  # noqa: E402
from conftest import analyzed  # noqa: E402

for name in sys.argv[1:] or ["c3"]:
    _, an = analyzed(name)
    for i in range(4):
        t = [time.perf_counter()]
        plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
        t.append(time.perf_counter())
        fz = T.GpuFactorizer(plan)
        t.append(time.perf_counter())
        st = fz.factor()
        t.append(time.perf_counter())
        fz.download()
        t.append(time.perf_counter())
        fz.close()
        t.append(time.perf_counter())
        d = [round((b - a) * 1e3, 1) for a, b in zip(t, t[1:])]
        print(f"{name} call {i}: plan {d[0]} ctx+upload {d[1]} factor {d[2]} (device {st.device_ms:.2f}) "
              f"download {d[3]} close {d[4]} total {round((t[-1] - t[0]) * 1e3, 1)} ms", flush=True)
