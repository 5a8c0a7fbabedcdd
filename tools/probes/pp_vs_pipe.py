"""Per-lane kernel (TCG_FLOW_PP=0) against the product-parallel variants on 7-point Laplacians of
growing size (IC(1), short programs): device ms, median of 7. TCG_FLOW_SLACK applies to all."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T  # noqa: E402

MODES = (("pipe", "0"), ("pp2x", "2,2,2,3,1"), ("pp1x", "1,2,1,4,2"), ("auto", None))
for m in [int(x) for x in sys.argv[1:]] or [40, 56, 64, 80, 96, 112]:
    a = T.generate("lap7", m)
    an = T.analyze(a, level=1)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    out = []
    for name, pp in MODES:
        if pp is None:
            os.environ.pop("TCG_FLOW_PP", None)
        else:
            os.environ["TCG_FLOW_PP"] = pp
        fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=60))
        ts = []
        for _ in range(9):
            fz.restore()
            ts.append(fz.factor().device_ms)
        st = fz.last
        out.append(f"{name} {statistics.median(ts[2:]):.4f} (k{st.row_kernel})")
        fz.close()
    print(f"lap7 {m}^3 rows {a.nrows}: " + "  ".join(out), flush=True)
