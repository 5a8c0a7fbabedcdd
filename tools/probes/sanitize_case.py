"""One small run of each device path, for compute-sanitizer (memcheck,
racecheck, synccheck): the value-flow factorization with both row kernels
(product-parallel groups of 1 and 2 warps, and one lane per coordinate), a
batch of members, the end-to-end drain, the triangular solves, the level-k
symbolic pattern. Checks every factor against the reference's golden hash.

    compute-sanitizer --tool racecheck python tools/probes/sanitize_case.py c1
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1601_05871_b200 as T  # noqa: E402
from checkers import Oracle  # noqa: E402
from conftest import analyzed, planned  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))[name]
orc = Oracle()
plan = planned(name)
_, an = analyzed(name)
ok = True
for spec in ("1,2,1,4,2,0", "2,2,2,3,1,0", "0"):
    os.environ["TCG_FLOW_PP"] = spec
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=600))
    st = fz.factor()
    v = fz.download()
    good = orc.hash(v) == golden["factor_values"]
    ok &= good
    print(f"factor pp={spec} kernel={st.row_kernel} bitwise={good}", flush=True)
    if spec == "0":
        # end to end with the drain CTAs copying the factor out during the launch
        import torch
        os.environ["TCG_DRAIN"] = "1"
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        out = torch.zeros(fz.nnz, dtype=torch.float64).pin_memory()
        st = fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
        good = orc.hash(out.numpy().copy()) == golden["factor_values"] and st.drain_ctas > 0
        ok &= good
        print(f"factor_host_a drain bitwise={good}", flush=True)
        os.environ.pop("TCG_DRAIN")
        s = T.GpuTriSolve(fz)
        b = np.random.default_rng(3).standard_normal(an.a_permuted.nrows)
        x = s.apply(b)
        good = np.array_equal(x.view(np.int64), orc.trisolve(an.pattern.pattern, v, b, 3).view(np.int64))
        ok &= good
        print(f"trisolve bitwise={good}", flush=True)
        s.close()
    fz.close()
os.environ.pop("TCG_FLOW_PP")
# a batch of 3 members with the default (product-parallel) kernel
fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=600))
init = plan.flow_tables()["values"]
fz.set_batch(np.stack([init, init, init]))
fz.factor()
out = fz.download_batch()
good = all(orc.hash(out[i]) == golden["factor_values"] for i in range(3))
ok &= good
print(f"batch of 3 bitwise={good}", flush=True)
fz.close()
fp = T.levelk_pattern_gpu(an.a_permuted, golden["level"])
good = np.array_equal(fp.pattern.col_idx, an.pattern.pattern.col_idx)
ok &= good
print(f"symbolic pattern equal={good}", flush=True)
print("SANITIZE_CASE", "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
