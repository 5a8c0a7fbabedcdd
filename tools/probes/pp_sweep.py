"""A/B of the value-flow row kernels on one configuration in one process:
for each TCG_FLOW_PP setting ("" = the per-lane pipelined kernel), the
median device ms of 7 factorizations (L2 not flushed) and whether the factor
hashes to the reference's golden factor_serial hash.

    python tools/probes/pp_sweep.py c3 "" 4,4,3,1,200 2,4,3,1,200 ...
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T  # noqa: E402
from checkers import Oracle  # noqa: E402
from conftest import analyzed, planned  # noqa: E402
import json  # noqa: E402

name = sys.argv[1]
specs = sys.argv[2:] or [""]
golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))[name]["factor_values"]
orc = Oracle()
plan = planned(name)
fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=20))
for spec in specs:
    if spec:
        os.environ["TCG_FLOW_PP"] = spec
    else:
        os.environ.pop("TCG_FLOW_PP", None)
    ts = []
    ok = "?"
    try:
        for i in range(9):
            fz.restore()
            st = fz.factor()
            ts.append(st.device_ms)
            if i == 0:
                ok = "bitwise" if orc.hash(fz.download()) == golden else "MISMATCH"
        print(f"{name} pp={spec or '-':16s} ms {statistics.median(ts[2:]):.4f} min {min(ts):.4f} "
              f"grid {st.grid_ctas} lanes {st.lanes_per_row} {ok}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name} pp={spec or '-':16s} FAILED {type(e).__name__}: {e}", flush=True)
        fz.close()
        fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=20))
fz.close()
