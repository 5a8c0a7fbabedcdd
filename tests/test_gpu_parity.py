"""GPU parity: the sm_100a factorization through the C ABI against the CPU
oracle (itself pinned to the reference, tests/test_oracle.py).

Bar (BASELINE.json north_star): pattern and DAG bit-exact, values within
1e-12 relative (fp64) -- these kernels are in fact bitwise equal to
factor_serial, which is asserted -- and the pattern-restricted residual
||A - UᵀU||_P / max|A| equal to the reference's.
"""
import math
import os

import numpy as np
import pytest

from conftest import analyzed, bitwise_equal, max_rel_diff, planned

pytestmark = pytest.mark.gpu

TOL = 1e-12  # relative, fp64 (north_star)


def gpu_factor(T, plan, **opt):
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30, **opt))
    try:
        st = fz.factor()
        return fz.download(), st
    finally:
        fz.close()


def check_against_oracle(name, vals, golden, oracle):
    _, an = analyzed(name)
    ref, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert st == 0
    assert max_rel_diff(vals, ref) <= TOL
    assert bitwise_equal(vals, ref), "expected bitwise equality with factor_serial"
    assert oracle.hash(vals) == golden[name]["factor_values"]
    res = oracle.residual(an.a_permuted, an.pattern.pattern, vals)
    assert res == pytest.approx(golden[name]["residual"], rel=1e-9, abs=1e-18)


@pytest.mark.parametrize("name", ["c1", "c5_m0", "c5_m63", "s27_16_k2", "grid20_k2_leaf4",
                                  "rand_spd_200", "elast6_k1", "c2", "c3", "c4"])
def test_configs_value_flow(T, golden, oracle, name):  # noqa: D103
    vals, st = gpu_factor(T, planned(name), mode=5)
    assert st.mode == 5
    check_against_oracle(name, vals, golden, oracle)


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "elast6_k1", "grid20_k2_leaf4", "rand_spd_200",
                                  "c2", "c3", "c4"])
def test_device_schedule_equals_the_host_schedule(T, name):
    # flow_schedule.cu (levels and heights by polling dry runs, a radix sort,
    # the records) against flow_plan_schedule on the host: record for record
    _, an = analyzed(name)
    fresh = T.Plan(an.a_permuted, an.pattern, an.ranges)  # no host schedule: the device builds it
    assert fresh.stats().flow_depth == 0
    fz = T.GpuFactorizer(fresh, T.GpuOptions(timeout_s=30))
    try:
        rec, item, depth = fz.flow_records()
    finally:
        fz.close()
    host = T.Plan(an.a_permuted, an.pattern, an.ranges).schedule()
    f = host.flow_tables()
    assert np.array_equal(rec, f["flow_rec"]) and np.array_equal(item, f["flow_item"])
    assert depth == host.stats().flow_depth > 0


@pytest.mark.parametrize("name,slack", [("c1", "100"), ("s27_16_k2", "60"), ("c2", "100")])
def test_slack_placed_device_schedule(T, golden, oracle, name, slack, monkeypatch):
    # TCG_FLOW_SLACK: the device and the host place the units alike, and the
    # factor is the golden one under either row kernel
    monkeypatch.setenv("TCG_FLOW_SLACK", slack)
    _, an = analyzed(name)
    fresh = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(fresh, T.GpuOptions(timeout_s=30))
    try:
        rec, item, depth = fz.flow_records()
        for pp in ("0", "1,2,1,4,2"):
            monkeypatch.setenv("TCG_FLOW_PP", pp)
            fz.restore()
            fz.factor()
            check_against_oracle(name, fz.download(), golden, oracle)
    finally:
        fz.close()
    f = T.Plan(an.a_permuted, an.pattern, an.ranges).schedule().flow_tables()
    assert np.array_equal(rec, f["flow_rec"]) and np.array_equal(item, f["flow_item"])


def test_default_row_kernel_follows_program_length(T):
    # product-parallel rows where programs are short and the matrix small (C1, C5;
    # large ones too: C6), one lane per coordinate where programs are long (s27,
    # C3: 24.8 products per coordinate) and on mid-size matrices (C2: 262 K units)
    for name, want in (("c1", 2), ("c5_m0", 2), ("c2", 1), ("s27_16_k2", 1)):
        _, st = gpu_factor(T, planned(name), mode=5)
        assert st.row_kernel == want, name


@pytest.mark.parametrize("name,spec", [("c3", "1,2,1,4,2,0"), ("s27_16_k2", "4,2,4,3,1,0"),
                                       ("elast6_k1", "2,2,2,3,1,0"), ("c2", "2,1,4,4,1,0"),
                                       ("c1", "1,2,2,4,2,0"), ("rand_spd_200", "4,4,4,2,1,0"),
                                       ("c4", "2,2,2,3,1,0"), ("grid20_k2_leaf4", "1,2,1,4,2,0")])
def test_product_parallel_variants(T, golden, oracle, name, spec, monkeypatch):
    # flow_pp_kernel.cu: rows longer than the group (passes), programs longer
    # than a chunk (several chunks, prefetched one ahead), one to four warps
    # per row: every variant bitwise equal to factor_serial
    monkeypatch.setenv("TCG_FLOW_PP", spec)
    vals, st = gpu_factor(T, planned(name), mode=5)
    assert st.row_kernel == 2 and st.lanes_per_row == 32 * int(spec.split(",")[0])
    check_against_oracle(name, vals, golden, oracle)


@pytest.mark.parametrize("name,decouple", [("c3", "100"), ("s27_16_k2", "20"), ("c4", "100"), ("elast6_k1", "400")])
def test_pivot_through_shared_memory(T, golden, oracle, name, decouple, monkeypatch):
    # per-lane kernel: the Chol pivot handed to the other lanes through shared
    # memory (each lane publishes as soon as its program and the pivot are
    # ready) or by a warp shuffle (0); bitwise either way
    monkeypatch.setenv("TCG_FLOW_DECOUPLE", decouple)
    monkeypatch.setenv("TCG_FLOW_PP", "0")
    vals, st = gpu_factor(T, planned(name), mode=5)
    assert st.row_kernel == 1
    check_against_oracle(name, vals, golden, oracle)


@pytest.mark.parametrize("name,cap", [("c3", "8"), ("elast6_k1", "16"), ("s27_16_k2", "24"), ("c4", "1000")])
def test_chol_unit_caps(T, golden, oracle, name, cap, monkeypatch):
    # units of the value flow with Chol units capped at 8..1000 coordinates
    # (the rest of a wide diagonal slice as chunks dividing by U(t,t)): a
    # different schedule, the same factor bit for bit
    monkeypatch.setenv("TCG_FLOW_CHOL_MAX", cap)
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    f = plan.flow_tables()
    L = f["flow_rec"][:, 1] & ((1 << 30) - 1)
    chol = ((f["flow_rec"][:, 1] >> 30) & 1) == 0
    long_rows = np.diff(f["row_ptr"])[f["flow_rec"][chol, 3]] > 32
    assert L[chol][long_rows].max() <= int(cap)
    vals, _ = gpu_factor(T, plan, mode=5)
    check_against_oracle(name, vals, golden, oracle)


@pytest.mark.parametrize("name,spec", [("c3", "1,2,1,4,2,0"), ("s27_16_k2", "1,2,2,4,2,0"),
                                       ("elast6_k1", "1,2,1,4,2,0")])
def test_product_parallel_passes_over_wide_units(T, golden, oracle, name, spec, monkeypatch):
    # Chol units up to 64-81 coordinates (TCG_FLOW_CHOL_MAX=128) on groups of
    # 32 or 64 threads: the product-parallel kernel's later passes over a unit
    # (coordinates past the group, the pivot kept from pass 0)
    monkeypatch.setenv("TCG_FLOW_CHOL_MAX", "128")
    monkeypatch.setenv("TCG_FLOW_PP", spec)
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    L = plan.flow_tables()["flow_rec"][:, 1] & ((1 << 30) - 1)
    assert L.max() > 32 * int(spec.split(",")[0])
    vals, st = gpu_factor(T, plan, mode=5)
    assert st.row_kernel == 2
    check_against_oracle(name, vals, golden, oracle)


def test_empty_matrix(T):
    # n = 0: nothing to factor, an empty factor back (factorize.hpp:134-235 with no ranges)
    a = T.CsrMatrix.from_arrays(0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    fp = T.levelk_pattern(a, 0)
    res = T.factor_by_blocks_gpu(a, fp, T.RangeList(np.array([0], np.int32)))
    assert res.factor.values.size == 0 and res.factor.nrows == 0


@pytest.mark.parametrize("name", ["c1", "c5_m0", "c2", "rand_spd_200"])
def test_per_lane_kernel_on_short_programs(T, golden, oracle, name, monkeypatch):
    monkeypatch.setenv("TCG_FLOW_PP", "0")
    vals, st = gpu_factor(T, planned(name), mode=5)
    assert st.row_kernel == 1
    check_against_oracle(name, vals, golden, oracle)


@pytest.mark.parametrize("name", ["c1", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1", "c5_m0"])
def test_device_programs_equal_the_cpu_restatement(T, name):
    # flow_program.cu (transposed index by a radix sort, count, scan, fill)
    # against checkers.flow_programs, table for table
    from checkers import flow_programs
    plan = planned(name)
    f = plan.flow_tables()
    want_slot, want_upd = flow_programs(f["row_ptr"], f["cols"])
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    try:
        slot, upd, ms = fz.flow_programs()
    finally:
        fz.close()
    assert ms > 0
    assert np.array_equal(slot, want_slot) and np.array_equal(upd, want_upd)


def test_default_mode_is_value_flow(T):
    _, st = gpu_factor(T, planned("c1"))
    assert st.mode == 5


@pytest.mark.parametrize("name", ["c5_m0", "elast6_k1", "s27_16_k2"])
def test_flow_trace_is_sound(T, name):
    # acceptance.cpp:285-316 for the value flow: the stamps bracket every row
    # ({start, operands final, -, end}), and a row's operands become final only
    # after every row it reads had its own operands final (the producer
    # computes its values after that stamp, the reader sees them before its
    # own). Readers: rows of <= 32 entries, whose stamp covers all of them.
    from checkers import flow_programs
    plan = planned(name)
    fz = T.GpuFactorizer(plan, T.GpuOptions(mode=5, trace=True, timeout_s=30))
    try:
        fz.factor()
        _, units = fz.trace()
    finally:
        fz.close()
    f = plan.flow_tables()
    rec, unit = f["flow_rec"], f["flow_item"]
    st = units[unit]  # per schedule position
    assert np.all(st[:, 0] > 0) and np.all(st[:, 0] <= st[:, 1]) and np.all(st[:, 1] <= st[:, 3])
    L = rec[:, 1] & ((1 << 30) - 1)
    owner = np.empty(len(f["cols"]), np.int64)
    for q, (tb, l) in enumerate(zip(rec[:, 0], L)):
        owner[tb:tb + l] = q
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    checked = 0
    for q in range(len(rec)):
        if L[q] > 32:
            continue
        tb = rec[q, 0]
        deps = {owner[x] for ub, ue in slot[tb:tb + L[q], :2] for x in upd[ub:ue].ravel()}
        if (rec[q, 1] >> 30) & 1:
            deps.add(owner[rec[q, 2]])
        for d in deps:
            assert st[d, 1] <= st[q, 1], (q, d)
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "elast6_k1", "c2", "c3", "c4"])
def test_configs_task_modes(T, golden, oracle, name, mode):
    # the literal task executors (device ready queue + dependence counters
    # over the reference's Chol/Trsm/Herk/Gemm DAG) on the task-DAG plan
    vals, st = gpu_factor(T, planned(name), mode=mode)
    assert st.mode == mode
    assert st.tasks_completed == sum(planned(name).stats().tasks)
    check_against_oracle(name, vals, golden, oracle)


def test_c6_full_size(T, golden, oracle):
    # 128^3 IC(1): 16.4 M factor entries, 1.48 M tasks, through the drop-in
    _, an = analyzed("c6")
    res = T.factor_by_blocks_gpu(an.a_permuted, an.pattern, an.ranges)
    assert oracle.hash(res.factor.values) == golden["c6"]["factor_values"]
    assert res.stats.total_tasks() == golden["c6"]["dag"]["nodes"]


def test_drop_in_api_matches_reference_result_semantics(T, oracle):
    a, an = analyzed("c1")
    res = T.factor_by_blocks_gpu(an.a_permuted, an.pattern, an.ranges)
    u = an.pattern.pattern
    assert np.array_equal(res.factor.row_ptr, u.row_ptr) and np.array_equal(res.factor.col_idx, u.col_idx)
    assert res.stats.backend == "gpu" and res.stats.nnz_u == u.nnz()
    assert (res.stats.chol_tasks, res.stats.trsm_tasks, res.stats.herk_tasks, res.stats.gemm_tasks) == \
        (353, 807, 807, 331)
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, u)
    assert bitwise_equal(res.factor.values, ref)


def small(T, n, entries, level=0, bounds=None):
    ti, tj, tv = (np.array(x) for x in zip(*entries))
    order = np.lexsort((tj, ti))
    ti, tj, tv = ti[order], tj[order], tv[order]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ptr, ti + 1, 1)
    a = T.CsrMatrix.from_arrays(n, np.cumsum(ptr), tj, tv)
    fp = T.levelk_pattern(a, level)
    rl = T.RangeList(np.array(bounds if bounds is not None else [0, n], dtype=np.int32))
    return a, fp, rl


def sym(entries):
    return entries + [(j, i, v) for i, j, v in entries if i != j]


@pytest.mark.parametrize("mode", [1, 2, 5])
def test_known_answers(T, mode):
    # test_factorize.cpp:78-97 and test_kernels.cpp:36-57
    opt = T.GpuOptions(mode=mode)
    a, fp, rl = small(T, 3, [(0, 0, 4.0), (1, 1, 9.0), (2, 2, 16.0)], bounds=[0, 1, 3])
    assert list(T.factor_by_blocks_gpu(a, fp, rl, opt).factor.values) == [2.0, 3.0, 4.0]
    p = T.generate("path", 3)
    fp = T.levelk_pattern(p, 0)
    v = T.factor_by_blocks_gpu(p, fp, T.RangeList(np.array([0, 1, 2, 3], np.int32)), opt).factor.values
    want = [math.sqrt(2.0), -1.0 / math.sqrt(2.0), math.sqrt(1.5), -math.sqrt(2.0 / 3.0),
            math.sqrt(4.0 / 3.0)]
    assert np.allclose(v, want, rtol=1e-15, atol=0)
    a, fp, rl = small(T, 2, sym([(0, 0, 4.0), (0, 1, 2.0), (1, 1, 3.0)]))
    v = T.factor_by_blocks_gpu(a, fp, rl, opt).factor.values
    assert v[0] == 2.0 and v[1] == 1.0 and v[2] == math.sqrt(2.0)


@pytest.mark.parametrize("mode", [1, 2, 5])
def test_breakdown_reports_row_and_pivot(T, mode):
    # test_factorize.cpp:99-108,157-165 and test_kernels.cpp:62-76
    opt = T.GpuOptions(mode=mode)
    a, fp, rl = small(T, 2, sym([(0, 0, 1.0), (0, 1, 2.0), (1, 1, 1.0)]))
    with pytest.raises(T.BreakdownError) as e:
        T.factor_by_blocks_gpu(a, fp, rl, opt)
    assert e.value.row == 1 and e.value.pivot < 0.0
    a, fp, rl = small(T, 4, sym([(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 3, 4.0), (3, 3, 1.0)]),
                      bounds=[0, 2, 4])
    with pytest.raises(T.BreakdownError) as e:
        T.factor_by_blocks_gpu(a, fp, rl, opt)
    assert e.value.row == 3


@pytest.mark.parametrize("seed", range(5))
def test_random_spd_many_blockings(T, oracle, seed):
    # test_factorize.cpp:125-155 / acceptance c3: by-blocks == serial for any blocking
    rng = np.random.default_rng(seed)
    a = T.generate("random_spd", int(rng.integers(30, 160)), int(rng.integers(20000, 80000)), seed)
    k = int(rng.integers(0, 4))
    an = T.analyze(a, level=k, leaf_size=int(rng.integers(2, 16)))
    ref, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert st == 0
    n = a.nrows
    for nr in (1, 3, 7, n):
        step = max(1, -(-n // nr))
        b = np.array(list(range(0, n, step)) + [n], dtype=np.int32)
        plan = T.Plan(an.a_permuted, an.pattern, T.RangeList(b))
        for mode in (1, 2, 5):
            vals, _ = gpu_factor(T, plan, mode=mode)
            assert bitwise_equal(vals, ref), (nr, mode)


@pytest.mark.parametrize("g", [8, 14])
def test_complete_fill_reconstructs(T, oracle, g):
    # acceptance c5: complete fill, residual <= 1e-10
    a = T.generate("grid2d", g, g)
    an = T.analyze(a, level=g * g, leaf_size=4, treecut=1)
    res = T.factor_by_blocks_gpu(an.a_permuted, an.pattern, an.ranges)
    assert oracle.residual(an.a_permuted, an.pattern.pattern, res.factor.values) <= 1e-10


def test_edge_cases_single_row_and_diagonal_blocks(T, oracle):
    a, fp, rl = small(T, 1, [(0, 0, 9.0)])
    assert list(T.factor_by_blocks_gpu(a, fp, rl).factor.values) == [3.0]
    d = T.generate("grid2d", 1, 40)
    fp = T.levelk_pattern(d, 2)
    for b in ([0, 40], list(range(41)), [0, 7, 8, 30, 40]):
        res = T.factor_by_blocks_gpu(d, fp, T.RangeList(np.array(b, np.int32)))
        ref, _, _, _ = oracle.factor_serial(d, fp.pattern)
        assert bitwise_equal(res.factor.values, ref)


def test_task_trace_respects_every_dag_edge(T):
    # acceptance c7 (soundness): finish[pred] <= start[succ] for every edge
    plan = planned("c5_m0")
    fz = T.GpuFactorizer(plan, T.GpuOptions(mode=2, trace=True))
    fz.factor()
    tasks, _ = fz.trace()
    fz.close()
    d = plan.dag()
    assert np.all(tasks[:, 0] <= tasks[:, 1])
    assert np.all(tasks[d.edge_from, 1] <= tasks[d.edge_to, 0])


def test_refactor_with_new_values_and_determinism(T, oracle):
    # C5-style reuse: one plan, several value sets (same pattern and DAG)
    name = "c5_m0"
    plan = planned(name)
    fz = T.GpuFactorizer(plan, T.GpuOptions())
    try:
        fz.factor()
        first = fz.download()
        fz.restore()
        fz.factor()
        assert bitwise_equal(fz.download(), first)
        for member in (5, 17):
            a, _ = T.config_matrix("c5", member)
            _, an = analyzed(name)
            ap = T.CsrMatrix.from_arrays(a.nrows, an.a_permuted.row_ptr, an.a_permuted.col_idx,
                                         None)
            # permute the member's values with the shared ordering
            ap_vals = T.analyze(a, level=1).a_permuted
            assert np.array_equal(ap_vals.col_idx, ap.col_idx)
            init = T.init_factor_values(ap_vals, an.pattern)
            fz.set_values(init)
            fz.factor()
            ref, st, _, _ = oracle.factor_serial(ap_vals, an.pattern.pattern)
            assert bitwise_equal(fz.download(), ref)
    finally:
        fz.close()


@pytest.mark.parametrize("threads", [128, 512])
def test_cta_sizes_agree(T, threads):
    plan = planned("s27_16_k2")
    base, _ = gpu_factor(T, plan)
    for mode in (1, 2, 5):
        vals, st = gpu_factor(T, plan, mode=mode, threads_per_cta=threads)
        assert st.threads_per_cta == (256 if mode == 5 else threads)  # the value flow: 256 always
        assert bitwise_equal(vals, base)


def test_cpp_dropin_with_reference_types():
    # include/tacho_b200.hpp called with taskchol::CsrMatrix/FillPattern/
    # RangeList/FactorResult (binary built from the unmodified reference
    # headers by `make -C oracle ref`); compares with the reference's own
    # factor_serial bit for bit
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_with_reference_types")
    if not os.path.exists(exe):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bitwise=1" in r.stdout


def c5_members(T, members):
    """Initial U values of C5 members (shared ordering, pattern and plan)."""
    _, an = analyzed("c5_m0")
    vals, perms = [], []
    for m in members:
        a, _ = T.config_matrix("c5", m)
        ap = T.analyze(a, level=1).a_permuted
        assert np.array_equal(ap.col_idx, an.a_permuted.col_idx)
        vals.append(T.init_factor_values(ap, an.pattern))
        perms.append(ap)
    return an, np.stack(vals), perms


def test_c5_batch_one_launch_bitwise(T, oracle):
    # C5: many matrices with one structure, factored in one launch (mode 5)
    members = list(range(6))
    an, vals, perms = c5_members(T, members)
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_batch(vals)
        assert fz.batch == len(members)
        st = fz.factor()
        assert st.mode == 5 and st.batch == len(members) and st.kernel_launches == 2
        out = fz.download_batch()
        for i, ap in enumerate(perms):
            ref, status, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert status == 0
            assert bitwise_equal(out[i], ref), i
        rows, _ = fz.batch_breakdown()
        assert np.all(rows == -1)
        # refactor after restore gives the same bits; back to one matrix works
        fz.restore()
        fz.factor()
        assert bitwise_equal(fz.download_batch(), out)
        fz.set_batch(vals[:1])
        assert fz.batch == 1
        fz.factor()
        assert bitwise_equal(fz.download(), out[0])
    finally:
        fz.close()


def test_c5_batch_breakdown_is_per_member(T, oracle):
    an, vals, perms = c5_members(T, [0, 1, 2])
    u = an.pattern.pattern
    row = 1000
    vals[1, u.row_ptr[row]] = -1.0  # member 1: negative pivot at `row`
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_batch(vals)
        with pytest.raises(T.BreakdownError) as e:
            fz.factor()
        assert e.value.row == row and fz.last.breakdown_member == 1
        rows, piv = fz.batch_breakdown()
        assert list(rows) == [-1, row, -1] and piv[1] < 0
        out = fz.download_batch()
        for i in (0, 2):
            ref, _, _, _ = oracle.factor_serial(perms[i], u)
            assert bitwise_equal(out[i], ref), i
    finally:
        fz.close()


@pytest.mark.parametrize("name", ["c1", "c5_m0", "c2", "c4"])
def test_factor_host_overlapped_upload(T, golden, oracle, name):
    # tcg_factor_host: the input copy runs beside the mode-5 kernel, which
    # polls the inputs; the result is the same bits
    import torch
    plan = planned(name)
    vals = plan.flow_tables()["values"]
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    try:
        host_in = torch.from_numpy(vals.copy()).pin_memory()
        host_out = torch.empty(len(vals), dtype=torch.float64).pin_memory()
        for _ in range(2):
            host_out.fill_(0.0)
            st = fz.factor_host_ptr(host_in.data_ptr(), host_out.data_ptr())
            check_against_oracle(name, host_out.numpy(), golden, oracle)
        assert st.mode == 5
        out = fz.factor_host(vals)  # pageable buffers work too
        check_against_oracle(name, out, golden, oracle)
    finally:
        fz.close()


def test_factor_host_batch(T, oracle):
    an, vals, perms = c5_members(T, [0, 3, 9])
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_batch(vals)
        out = fz.factor_host(vals)
        for i, ap in enumerate(perms):
            ref, _, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert bitwise_equal(out[i], ref), i
    finally:
        fz.close()


@pytest.mark.parametrize("name,nparts", [("c5_m0", 2), ("c5_m0", 4), ("c2", 8)])
def test_sharded_parts_through_peer_pointers(T, golden, oracle, name, nparts):
    # C6's sharded path on one GPU, made sequential: parts 0..n-1 own the ND
    # subtrees (independent of each other), part n the separators above them,
    # which read the subtree parts' U through the peer-pointer table exactly as
    # they would across GPUs. Each launch only reads parts that have finished,
    # so no kernel waits on another.
    _, an = analyzed(name)
    plan = planned(name)
    owners = an.subtree_owners(nparts, separators=nparts)
    total = nparts + 1
    fzs = [T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30), problem=plan.part_problem(total, owners, k))
           for k in range(total)]
    try:
        ptrs = [f.values_device_ptr() for f in fzs]
        for f in fzs:
            f.set_peers(ptrs)
        for f in fzs:
            st = f.factor()
            assert st.mode == 5
        full = np.full(an.pattern.pattern.nnz(), np.nan)
        own_pos = np.repeat(owners, np.diff(an.pattern.pattern.row_ptr))  # owner of every U entry
        for k, f in enumerate(fzs):
            v = f.download()
            full[own_pos == k] = v[own_pos == k]
        check_against_oracle(name, full, golden, oracle)
    finally:
        for f in fzs:
            f.close()


def _ipc_owner(q_out, q_in, name, nparts):
    """Process A: owns the subtree parts, factors them, exports its U by IPC."""
    import sys as _s
    _s.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import paper_1601_05871_b200 as T
    from conftest import analyzed, planned
    _, an = analyzed(name)
    plan = planned(name)
    owners = an.subtree_owners(nparts, separators=nparts)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30),
                         problem=plan.part_problem(nparts + 1, owners, 0))
    fz.set_peers([fz.values_device_ptr()] * (nparts + 1))
    fz.factor()
    q_out.put((fz.ipc_handle(), fz.download()))
    q_in.get()  # keep the allocation alive until the reader is done
    fz.close()


def test_ipc_peer_values_across_processes(T, golden, oracle):
    # the multi-process path of bench.py run_sharded on one GPU, made
    # sequential: a second process owns part 0 (one ND subtree) and exports
    # its U by CUDA IPC; this process runs the other parts, whose separator
    # rows read part 0's values through the IPC mapping
    import multiprocessing as mp
    name, nparts = "c5_m0", 2
    ctx = mp.get_context("spawn")
    q_out, q_in = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_owner, args=(q_out, q_in, name, nparts))
    p.start()
    try:
        (handle, offset), part0 = q_out.get(timeout=300)
        _, an = analyzed(name)
        plan = planned(name)
        owners = an.subtree_owners(nparts, separators=nparts)
        fzs = [T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30), problem=plan.part_problem(nparts + 1, owners, k))
               for k in range(1, nparts + 1)]
        remote0 = fzs[0].ipc_open(handle, offset)
        ptrs = [remote0] + [f.values_device_ptr() for f in fzs]
        for f in fzs:
            f.set_peers(ptrs)
            f.factor()
        own_pos = np.repeat(owners, np.diff(an.pattern.pattern.row_ptr))
        full = np.where(own_pos == 0, part0, np.nan)
        for k, f in enumerate(fzs, start=1):
            v = f.download()
            full[own_pos == k] = v[own_pos == k]
        check_against_oracle(name, full, golden, oracle)
        for f in fzs:
            f.close()
    finally:
        q_in.put(1)
        p.join(timeout=120)


@pytest.mark.parametrize("name", ["c1", "c5_m0", "c2", "elast6_k1"])
def test_device_init_factor_values(T, golden, oracle, name):
    # init_factor_values on the device from PᵀAP's values equals the host one
    # bit for bit, and the factor from it equals the golden factor
    _, an = analyzed(name)
    plan = planned(name)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    try:
        fz.set_a_values(an.a_permuted.values)
        fz.restore()
        init = fz.download()
        assert bitwise_equal(init, plan.flow_tables()["values"])
        fz.factor()
        check_against_oracle(name, fz.download(), golden, oracle)
    finally:
        fz.close()


def test_device_init_batch(T, oracle):
    an, vals, perms = c5_members(T, [0, 5])
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_a_values(np.stack([ap.values for ap in perms]))
        assert fz.batch == 2
        fz.factor()
        out = fz.download_batch()
        for i, ap in enumerate(perms):
            ref, _, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert bitwise_equal(out[i], ref), i
    finally:
        fz.close()


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "c2"])
def test_factor_host_a_end_to_end(T, golden, oracle, name):
    # PᵀAP's values in, factor out in one call (tcg_factor_host_a): the
    # reference's factor_by_blocks inputs, bitwise the golden factor
    _, an = analyzed(name)
    fz = T.GpuFactorizer(planned(name), T.GpuOptions(timeout_s=30))
    try:
        for _ in range(2):  # the restore copy it leaves behind is the initialised U
            out = fz.factor_host_a(an.a_permuted.values)
            check_against_oracle(name, out, golden, oracle)
        assert fz.last.kernel_launches == 3
        fz.restore()
        assert bitwise_equal(fz.download(), planned(name).flow_tables()["values"])
    finally:
        fz.close()


def test_factor_host_a_batch(T, oracle):
    an, vals, perms = c5_members(T, [0, 3, 7])
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_a_values(np.stack([ap.values for ap in perms]))
        out = fz.factor_host_a(np.stack([ap.values for ap in perms]).ravel())
        for i, ap in enumerate(perms):
            ref, _, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert bitwise_equal(out[i * fz.nnz:(i + 1) * fz.nnz], ref), i
    finally:
        fz.close()


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "elast6_k1", "c2", "c4"])
def test_drained_end_to_end(T, golden, oracle, name, monkeypatch):
    # pinned host output: CTAs of the launch copy the factor out while the rows
    # run (tcg_factor_host[_a] drain); the result is the golden factor bit for bit
    import torch
    _, an = analyzed(name)
    plan = planned(name)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    try:
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        u_in = torch.from_numpy(plan.flow_tables()["values"]).pin_memory()
        monkeypatch.setenv("TCG_DRAIN", "1")  # forced: no calibration
        for ctas in ("1", "2", "4"):
            monkeypatch.setenv("TCG_DRAIN_CTAS", ctas)
            out = torch.full((fz.nnz,), float("nan"), dtype=torch.float64).pin_memory()
            st = fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
            assert st.drain_ctas == int(ctas)
            check_against_oracle(name, out.numpy().copy(), golden, oracle)
            out.fill_(float("nan"))
            st = fz.factor_host_ptr(u_in.data_ptr(), out.data_ptr())
            assert st.drain_ctas == int(ctas)
            check_against_oracle(name, out.numpy().copy(), golden, oracle)
        monkeypatch.setenv("TCG_DRAIN", "0")
        out = torch.zeros(fz.nnz, dtype=torch.float64).pin_memory()
        assert fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr()).drain_ctas == 0
        check_against_oracle(name, out.numpy().copy(), golden, oracle)
        # pageable output: no drain, a copy after the launch
        monkeypatch.delenv("TCG_DRAIN")
        assert fz.factor_host_a(an.a_permuted.values) is not None and fz.last.drain_ctas == 0
        # a pinned buffer 8 bytes off 16-byte alignment: no drain either, same factor
        big = torch.zeros(fz.nnz + 1, dtype=torch.float64).pin_memory()
        assert fz.factor_host_a_ptr(a_in.data_ptr(), big.data_ptr() + 8).drain_ctas == 0
        check_against_oracle(name, big.numpy()[1:].copy(), golden, oracle)
    finally:
        fz.close()


@pytest.mark.parametrize("name,kb", [("c2", None), ("c4", None), ("c1", "16"), ("elast6_k1", "1"), ("s27_16_k2", "64")])
def test_chunked_copies_end_to_end(T, golden, oracle, name, kb, monkeypatch):
    # TCG_DRAIN=2: U in chunks cut at unit starts; the unit that completes a chunk
    # flags it and the host's copy engine takes it out beside the rest of the
    # launch (run_flow, chunk_count). Bitwise the golden factor, call after call.
    import torch
    monkeypatch.setenv("TCG_DRAIN", "2")
    if kb:
        monkeypatch.setenv("TCG_D2H_CHUNK_KB", kb)  # small matrices: small chunks
    _, an = analyzed(name)
    plan = planned(name)
    fz = T.GpuFactorizer(plan, T.GpuOptions(timeout_s=30))
    try:
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        u_in = torch.from_numpy(plan.flow_tables()["values"]).pin_memory()
        for _ in range(3):
            out = torch.full((fz.nnz,), float("nan"), dtype=torch.float64).pin_memory()
            st = fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
            assert st.drain_ctas <= -4  # (minus the number of chunks)
            check_against_oracle(name, out.numpy().copy(), golden, oracle)
        out.fill_(float("nan"))
        assert fz.factor_host_ptr(u_in.data_ptr(), out.data_ptr()).drain_ctas <= -4
        check_against_oracle(name, out.numpy().copy(), golden, oracle)
        # pageable output: a copy after the launch
        assert fz.factor_host_a(an.a_permuted.values) is not None and fz.last.drain_ctas == 0
    finally:
        fz.close()


@pytest.mark.parametrize("name", ["c1", "elast6_k1", "c4"])
def test_pinned_input_gathered_in_place(T, golden, oracle, name, monkeypatch):
    # tcg_factor_host_a with a pinned input: the device init gathers the entries U
    # starts from straight out of host memory (TCG_A_ZEROCOPY=1; the default for
    # long rows) instead of copying all of A first (0); the same factor bit for bit
    import torch
    _, an = analyzed(name)
    fz = T.GpuFactorizer(planned(name), T.GpuOptions(timeout_s=30))
    try:
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        for z in ("1", "0", None):
            if z is None:
                monkeypatch.delenv("TCG_A_ZEROCOPY")
            else:
                monkeypatch.setenv("TCG_A_ZEROCOPY", z)
            out = torch.full((fz.nnz,), float("nan"), dtype=torch.float64).pin_memory()
            fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
            check_against_oracle(name, out.numpy().copy(), golden, oracle)
        # a pageable input is copied (no device address to gather from)
        monkeypatch.setenv("TCG_A_ZEROCOPY", "1")
        check_against_oracle(name, fz.factor_host_a(an.a_permuted.values), golden, oracle)
    finally:
        fz.close()


def test_chunked_copies_breakdown_and_calibration(T, golden, oracle, monkeypatch):
    import torch
    _, an = analyzed("c2")
    fz = T.GpuFactorizer(planned("c2"), T.GpuOptions(timeout_s=30))
    try:
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        out = torch.zeros(fz.nnz, dtype=torch.float64).pin_memory()
        # without TCG_DRAIN the three ways out take turns for nine calls, then the fastest stays
        monkeypatch.delenv("TCG_DRAIN", raising=False)
        seen = []
        for _ in range(12):
            seen.append(fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr()).drain_ctas)
            check_against_oracle("c2", out.numpy().copy(), golden, oracle)
        assert all(x == 0 for x in seen[0:9:3]) and all(x > 0 for x in seen[1:9:3]) and all(x < 0 for x in seen[2:9:3])
        assert len(set(seen[9:])) == 1
        # an indefinite matrix: the rows after the failing pivot keep their inputs and still
        # count towards their chunks, so every chunk leaves; BreakdownError as usual
        monkeypatch.setenv("TCG_DRAIN", "2")
        bad = an.a_permuted.values.copy()
        r = an.a_permuted.nrows // 2
        b0, b1 = int(an.a_permuted.row_ptr[r]), int(an.a_permuted.row_ptr[r + 1])
        bad[b0 + int(np.flatnonzero(an.a_permuted.col_idx[b0:b1] == r)[0])] = -1.0
        a_bad = torch.from_numpy(bad).pin_memory()
        with pytest.raises(T.BreakdownError) as e:
            fz.factor_host_a_ptr(a_bad.data_ptr(), out.data_ptr())
        assert e.value.row == r and fz.last.drain_ctas < 0
        # and the context is good for the next call
        fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
        check_against_oracle("c2", out.numpy().copy(), golden, oracle)
    finally:
        fz.close()


def test_drained_end_to_end_breakdown(T, monkeypatch):
    # an indefinite matrix: the rows after the failing pivot are skipped and
    # keep their inputs, so the drain still finishes; BreakdownError as usual
    import torch
    monkeypatch.setenv("TCG_DRAIN", "1")
    a, fp, rl = small(T, 4, sym([(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 3, 4.0), (3, 3, 1.0)]),
                      bounds=[0, 2, 4])
    fz = T.GpuFactorizer(T.Plan(a, fp, rl), T.GpuOptions(timeout_s=30))
    try:
        u_in = torch.from_numpy(T.init_factor_values(a, fp)).pin_memory()
        out = torch.zeros(fz.nnz, dtype=torch.float64).pin_memory()
        with pytest.raises(T.BreakdownError) as e:
            fz.factor_host_ptr(u_in.data_ptr(), out.data_ptr())
        assert e.value.row == 3 and fz.last.drain_ctas > 0
    finally:
        fz.close()


def test_drained_batch_end_to_end(T, oracle, monkeypatch):
    # a C5 batch through tcg_factor_host_a into a pinned buffer: the drain
    # copies every member's factor during the launch; bitwise per member
    import torch
    monkeypatch.setenv("TCG_DRAIN", "1")
    an, vals, perms = c5_members(T, [0, 9, 21])
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_a_values(np.stack([ap.values for ap in perms]))
        a_in = torch.from_numpy(np.stack([ap.values for ap in perms]).ravel().copy()).pin_memory()
        out = torch.full((3 * fz.nnz,), float("nan"), dtype=torch.float64).pin_memory()
        st = fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
        assert st.drain_ctas > 0 and st.batch == 3
        got = out.numpy().reshape(3, fz.nnz)
        for i, ap in enumerate(perms):
            ref, _, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert bitwise_equal(got[i], ref), i
    finally:
        fz.close()


def test_drain_calibrates_per_problem(T, golden, oracle, monkeypatch):
    # without TCG_DRAIN: the first six calls alternate between a copy after
    # the launch and the drain, later calls keep the faster; every result bitwise
    import torch
    monkeypatch.delenv("TCG_DRAIN", raising=False)
    _, an = analyzed("c5_m0")
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        a_in = torch.from_numpy(an.a_permuted.values.copy()).pin_memory()
        seen = []
        for _ in range(9):
            out = torch.zeros(fz.nnz, dtype=torch.float64).pin_memory()
            seen.append(fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr()).drain_ctas)
            check_against_oracle("c5_m0", out.numpy().copy(), golden, oracle)
        assert seen[:6:2] == [0, 0, 0] and min(seen[1:6:2]) > 0  # alternating probe calls
        assert len(set(seen[6:])) == 1 and seen[6] in (0, seen[1])
    finally:
        fz.close()


@pytest.mark.parametrize("chunks", ["4", "3", "1"])
def test_pipelined_batch_end_to_end(T, oracle, chunks, monkeypatch):
    # 10 C5 members through tcg_factor_host_a, pipelined over member chunks
    # (uploads and downloads beside the launches); member 6 made indefinite:
    # it breaks down at the oracle's row, the others stay bitwise
    import torch
    monkeypatch.setenv("TCG_CHUNKS", chunks)
    monkeypatch.setenv("TCG_DRAIN", "0")
    members = list(range(10))
    an, vals, perms = c5_members(T, members)
    a_vals = np.stack([ap.values.copy() for ap in perms])
    ap6 = perms[6]
    b0, b1 = int(ap6.row_ptr[100]), int(ap6.row_ptr[101])
    d = b0 + int(np.flatnonzero(ap6.col_idx[b0:b1] == 100)[0])  # the (100, 100) entry
    a_vals[6, d] = -1.0
    fz = T.GpuFactorizer(planned("c5_m0"), T.GpuOptions(timeout_s=30))
    try:
        fz.set_a_values(a_vals)
        a_in = torch.from_numpy(a_vals.ravel().copy()).pin_memory()
        out = torch.full((10 * fz.nnz,), float("nan"), dtype=torch.float64).pin_memory()
        with pytest.raises(T.BreakdownError) as e:
            fz.factor_host_a_ptr(a_in.data_ptr(), out.data_ptr())
        assert fz.last.chunks == (int(chunks) if chunks != "1" else 0)
        bad = T.CsrMatrix(ap6.nrows, ap6.ncols, ap6.row_ptr, ap6.col_idx, a_vals[6])
        _, st, row, _ = oracle.factor_serial(bad, an.pattern.pattern)
        assert st == 1 and e.value.row == row and fz.last.breakdown_member == 6
        got = out.numpy().reshape(10, fz.nnz)
        for i, ap in enumerate(perms):
            if i == 6:
                continue
            ref, _, _, _ = oracle.factor_serial(ap, an.pattern.pattern)
            assert bitwise_equal(got[i], ref), i
        rows, _ = fz.batch_breakdown()
        assert [int(r) for r in rows] == [row if i == 6 else -1 for i in range(10)]
    finally:
        fz.close()


def test_forced_backoff_without_a_variant_is_an_error(T, monkeypatch):
    # a sweep value that has no compiled kernel variant must not run silently
    # without a back-off (that once made every value above 400 ns measure as 0)
    monkeypatch.setenv("TCG_FLOW_BACKOFF", "777")
    fz = T.GpuFactorizer(planned("s27_16_k2"), T.GpuOptions(timeout_s=30))
    try:
        with pytest.raises(ValueError, match="back-off"):
            fz.factor()
        monkeypatch.setenv("TCG_FLOW_BACKOFF", "600")
        fz.restore()
        assert fz.factor().row_kernel == 1
    finally:
        fz.close()
