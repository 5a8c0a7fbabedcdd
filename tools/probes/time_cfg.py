"""Device ms of the default factorization of one configuration (median of 7,
L2 not flushed), for quick A/B runs under environment overrides."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
a, level = T.config_matrix(name)
an = T.analyze(a, level=level)
plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=60))
ts = []
for _ in range(9):
    fz.restore()
    ts.append(fz.factor().device_ms)
st = fz.last
print(f"{name} ms {statistics.median(ts[2:]):.4f} grid {st.grid_ctas} threads {st.threads_per_cta}")
