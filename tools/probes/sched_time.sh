# device schedule time inside tcg_upload (TCG_PLAN_TIMES) for C6 and C3, 3 uploads each
for c in c6 c3; do TCG_PLAN_TIMES=1 timeout 120 python - <<PY 2>&1 | grep -v "flow plan"
import sys, time; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_1601_05871_b200 as T
from conftest import analyzed
_,an=analyzed('$c')
for i in range(3):
    p=T.Plan(an.a_permuted, an.pattern, an.ranges)
    t0=time.perf_counter(); fz=T.GpuFactorizer(p); t1=time.perf_counter()
    print('$c upload total ms', round((t1-t0)*1e3,1), 'depth', fz.flow_records()[2], flush=True)
    fz.close()
PY
done
