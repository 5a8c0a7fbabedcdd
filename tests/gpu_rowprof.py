"""Manual GPU probe: per-phase warp-cycle breakdown of the row kernel."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1601_05871_b200 as T
kv = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
for name in [a for a in sys.argv[1:] if "=" not in a]:
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=20, trace=True, mode=3,
                                            threads_per_cta=int(kv.get("threads", 256)),
                                            ctas_per_sm=int(kv.get("ctas", 0))))
    for rep in range(3):
        fz.restore(); s = fz.factor()
    fz2 = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=20, mode=3, threads_per_cta=int(kv.get("threads", 256)),
                                             ctas_per_sm=int(kv.get("ctas", 0))))
    for rep in range(3):
        fz2.restore(); s2 = fz2.factor()
    p = list(s.profile)
    rows, pops, pushes = p[4], p[5], p[6]
    tot = sum(p[:4])
    print(f"{name}: ms(trace)={s.device_ms:.3f} ms(plain)={s2.device_ms:.3f} grid={s.grid_ctas} rows={rows} pops={pops} pushes={pushes}")
    for i, nm in enumerate(["pop/idle", "row body", "fence", "release"]):
        print(f"   {nm:9s} {100*p[i]/tot:5.1f}%  {p[i]/max(rows,1):8.0f} cyc/row")
