"""Host plans. The lean value-flow plan (tcg_plan_build): task counts equal
the reference DAG's, and its schedule -- replayed on the CPU with the
programs the device builds (restated in checkers.flow_programs) -- gives
factor_serial bit for bit, in schedule order and in row order. The task-DAG
plan (tcg_plan_expand): the DAG is bit-exact with the reference's
export_task_dag, the block structure with build_block_matrix, and its work
tables replay to factor_serial in task order."""
import numpy as np
import pytest

from checkers import Reference, emulate_flow, emulate_plan, emulate_program, flow_programs, reference_available
from conftest import analyzed, bitwise_equal, planned

FAST = ["c1", "c5_m0", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1"]


def an_perm(name):
    return analyzed(name)[1].perm


@pytest.mark.parametrize("name", FAST + ["c2", "c3", "c4", pytest.param("c6", marks=pytest.mark.slow)])
def test_plan_dag_and_blocks_match_reference(name, golden, oracle):
    # c6: 1,479,042 tasks and 3,003,864 edges, bit-exact with export_task_dag
    g = golden[name]
    plan = planned(name)
    d = plan.dag()
    assert len(d.kind) == g["dag"]["nodes"] and len(d.edge_from) == g["dag"]["edges"]
    for arr, key in ((d.kind, "kind"), (d.block_row, "block_row"), (d.block_col, "block_col"),
                     (d.edge_from, "edge_from"), (d.edge_to, "edge_to")):
        assert oracle.hash(arr) == g["dag"][key], key
    bp, bc = plan.blocks()
    assert len(bc) == g["blocks"]["nblocks"]
    assert oracle.hash(bp) == g["blocks"]["brow_ptr"]
    assert oracle.hash(bc) == g["blocks"]["bcol_idx"]
    s = plan.stats()
    assert list(s.tasks) == g["dag"]["tasks"]
    assert oracle.hash(an_perm(name)) == g["perm"]


@pytest.mark.parametrize("name", ["c1", "elast6_k1", "grid20_k2_leaf4", "rand_spd_200"])
def test_replays_are_bitwise_serial(name, golden, oracle):
    plan = planned(name)
    _, an = analyzed(name)
    ref, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert oracle.hash(ref) == golden[name]["factor_values"]
    assert bitwise_equal(emulate_plan(plan), ref)       # device merge mode, task order
    assert bitwise_equal(emulate_program(plan), ref)    # update programs, task order


def test_dag_edges_point_forward_and_task_count_formula(T):
    # test_factorize.cpp:262-311
    a = T.generate("grid2d", 6, 6)
    an = T.analyze(a, level=1, leaf_size=3, treecut=1)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    d = plan.dag()
    assert np.all(d.edge_from < d.edge_to)
    bp, bc = plan.blocks()
    present = {(i, int(c)) for i in range(len(bp) - 1) for c in bc[bp[i]:bp[i + 1]]}
    expected = 0
    for p in range(len(bp) - 1):
        cols = bc[bp[p]:bp[p + 1]]
        expected += 1 + (len(cols) - 1)
        for x in range(1, len(cols)):
            for y in range(x, len(cols)):
                expected += (int(cols[x]), int(cols[y])) in present
    assert len(d.kind) == expected
    # every TRSM(p, j) has CHOL(p, p) among its ancestors (direct edge here)
    chol_of = {int(d.block_row[t]): t for t in range(len(d.kind)) if d.kind[t] == 0}
    preds = {}
    for f, t in zip(d.edge_from, d.edge_to):
        preds.setdefault(int(t), set()).add(int(f))
    for t in range(len(d.kind)):
        if d.kind[t] == 1:
            assert chol_of[int(d.block_row[t])] in preds[t]


def test_flow_depth_is_below_the_task_dag_depth(T):
    # value flow follows the rows that interact, not the blocks: much shallower
    _, an = analyzed("c5_m0")
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    s = plan.schedule().stats()
    assert s.full_plan == 0 and s.flow_depth > 0
    plan.expand()
    s = plan.stats()
    assert s.full_plan == 1 and s.flow_depth < s.dag_depth


def test_single_range_and_diagonal_only(T, oracle):
    a = T.generate("grid2d", 5, 5)
    fp = T.levelk_pattern(a, 1)
    one = T.RangeList(np.array([0, 25], dtype=np.int32))
    plan = T.Plan(a, fp, one)
    assert list(plan.stats().tasks) == [1, 0, 0, 0]
    ref, _, _, _ = oracle.factor_serial(a, fp.pattern)
    assert bitwise_equal(replay_lean(plan), ref)
    d = T.generate("grid2d", 1, 8)  # path-like, blocks of one vertex each
    fp = T.levelk_pattern(d, 0)
    plan = T.Plan(d, fp, T.RangeList(np.arange(9, dtype=np.int32)))
    assert plan.stats().tasks[0] == 8


def test_invalid_inputs_raise(T):
    a = T.generate("grid2d", 4, 4)
    an = T.analyze(a)
    with pytest.raises(ValueError):
        T.Plan(an.a_permuted, an.pattern, T.RangeList(np.array([0, 5, 5, 16], dtype=np.int32)))
    # missing diagonal entry in the pattern (kernels.hpp:46-48)
    u = an.pattern.pattern
    cut = T.CsrMatrix.from_arrays(16, np.concatenate([[0], u.row_ptr[1:] - 1]), u.col_idx[1:])
    with pytest.raises(ValueError):
        T.Plan(an.a_permuted, T.FillPattern(cut), an.ranges)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(4))
def test_random_blockings_against_live_reference(T, oracle, seed):
    # test_factorize.cpp:125-155 style: several blockings of one matrix
    R = Reference()
    rng = np.random.default_rng(seed)
    a = T.generate("random_spd", int(rng.integers(40, 120)), 60000, seed + 3)
    an = T.analyze(a, level=int(rng.integers(0, 3)), leaf_size=4)
    n = a.nrows
    for nr in (1, 3, 7):
        step = max(1, -(-n // nr))
        b = np.array(list(range(0, n, step)) + [n], dtype=np.int32)
        plan = T.Plan(an.a_permuted, an.pattern, T.RangeList(b))
        kinds, bi, bj, ef, et = R.export_dag(an.pattern.pattern, b)
        d = plan.dag()
        assert np.array_equal(d.kind, kinds) and np.array_equal(d.edge_from, ef)
        assert np.array_equal(d.edge_to, et) and np.array_equal(d.block_row, bi)
        vals, st, _, _, _, _ = R.factor_by_blocks(an.a_permuted, an.pattern.pattern, b, workers=2)
        assert st == 0
        assert list(plan.stats().tasks) == [int((kinds == k).sum()) for k in range(4)]
        assert bitwise_equal(replay_lean(plan), vals)


def replay_lean(plan, order=None):
    f = plan.flow_tables()
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    return emulate_flow(f["flow_rec"], f["values"], slot, upd, order)


@pytest.mark.parametrize("name", ["c1", "rand_spd_200", "grid20_k2_leaf4", "elast6_k1", "c5_m0"])
def test_flow_schedule_partitions_u_and_replays_bitwise(T, name, golden, oracle):
    # mode 5: the rows of the schedule own every coordinate once -- whole
    # matrix rows of <= 32 entries, longer ones the diagonal-block slice +
    # chunks of <= 32; with the device-built programs the replay equals
    # factor_serial, in schedule order and in any order that reads only
    # written values (matrix-row order is one)
    _, an = analyzed(name)
    plan = planned(name)
    f = plan.flow_tables()
    s = plan.stats()
    rec = f["flow_rec"]
    L = rec[:, 1] & ((1 << 30) - 1)
    assert s.flow_rows == len(rec) and int(L.sum()) == len(f["values"])
    cover = np.zeros(len(f["values"]), np.int64)
    for tb, l in zip(rec[:, 0], L):
        cover[tb:tb + l] += 1
    assert np.all(cover == 1)  # a partition of U
    u = an.pattern.pattern
    lens = np.diff(u.row_ptr)
    assert int((lens <= 32).sum()) <= s.flow_rows
    assert np.array_equal(np.sort(f["flow_item"]), np.arange(len(rec)))
    assert list(s.tasks) == golden[name]["dag"]["tasks"]  # counted without the DAG walk
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, u)
    assert bitwise_equal(replay_lean(plan), ref)
    assert bitwise_equal(replay_lean(plan, np.argsort(f["flow_item"])), ref)


@pytest.mark.parametrize("name", ["c1", "rand_spd_200", "elast6_k1"])
def test_flow_programs_equal_the_task_dag_merges(T, name):
    # the per-coordinate programs (restated from the device builder) hold the
    # same products, in the same order, as the task-DAG plan's per-item
    # programs taken in generation order: the reference's kernels'
    # pattern-restricted merges (kernels.hpp:55-65, 85-89, 104-108, 125-129)
    plan = planned(name)
    f = plan.flow_tables()
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    t = plan.tables()
    per = [[] for _ in range(len(f["cols"]))]
    for rec in t["task"]:
        for it in range(rec[2], rec[3]):
            tb, te, _, _, _, _, soff, _ = t["item"][it]
            for k in range(te - tb):
                ub, ue = t["slot_rec"][soff + k, :2]
                per[tb + k].extend(map(tuple, t["upd"][ub:ue]))
    flat = [mo for p in per for mo in p]
    assert len(flat) == len(upd)
    assert np.array_equal(np.array(flat, np.int32).reshape(-1, 2), upd)


def part_tables(p):
    """The schedule rows of one part (tcg_plan_part_problem)."""
    from paper_1601_05871_b200.core import _copy
    return {"rec": _copy(p.flow_rec, 4 * p.nflow, np.int32).reshape(-1, 4),
            "unit": _copy(p.flow_item, p.nflow, np.int32)}


def part_programs(slot, upd, rowid, owners, part):
    """The device rewrite of a part's programs (flow_program.cu): operands in
    rows another part owns become 0x80000000 | owner << 25 | position."""
    s, u = slot.copy(), upd.astype(np.int64).copy()
    for x in range(len(slot)):
        if owners[rowid[x]] != part:
            continue
        for e in range(slot[x, 0], slot[x, 1]):
            ow = owners[rowid[u[e, 0]]]
            if ow != part:
                u[e] |= 0x80000000 | (int(ow) << 25)
        if slot[x, 0] < slot[x, 1]:
            s[x, 2:] = u[slot[x, 0]]
    return s, u


def replay_parts(f, slot, upd, parts, owners):
    """Sharded value flow on the CPU: every part's rows in the global order,
    each part with its own copy of U, remote operands read from their owner's
    copy. Returns (assembled factor, remote operand count, rows read remotely,
    rows flagged exported)."""
    total = len(parts)
    pos_of_unit = {int(g): q for q, g in enumerate(f["flow_item"])}
    order = sorted((pos_of_unit[int(g)], k, i) for k, p in enumerate(parts) for i, g in enumerate(p["unit"]))
    a = f["values"]
    rowid = np.repeat(np.arange(len(f["row_ptr"]) - 1), np.diff(f["row_ptr"]))
    progs = [part_programs(slot, upd, rowid, owners, k) for k in range(total)]
    out = [np.full(len(a), np.nan) for _ in range(total)]
    done = [np.zeros(len(a), bool) for _ in range(total)]
    remote = 0
    exported, read_remotely = set(), set()
    for _, k, i in order:
        tb, lk, dpos, trow = (int(x) for x in parts[k]["rec"][i])
        assert owners[trow] == k
        L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 1
        if lk < 0:
            exported.add((k, trow))
        v = a[tb:tb + L].copy()
        ps, pu = progs[k]
        for j in range(L):
            ub, ue = ps[tb + j, :2]
            for m, o in pu[ub:ue]:
                vals = []
                for x in (int(m), int(o)):
                    if x & 0x80000000:
                        ow, pos = (x >> 25) & 63, x & 0x1FFFFFF
                        assert ow != k
                        remote += 1
                        read_remotely.add((ow, int(rowid[pos])))
                    else:
                        ow, pos = k, x
                    assert done[ow][pos], "read before written"
                    vals.append(out[ow][pos])
                v[j] = v[j] - vals[0] * vals[1]
        if kind == 0:
            d = np.sqrt(v[0])
            v[1:] = v[1:] / d
            v[0] = d
        else:
            assert done[k][dpos]
            v = v / out[k][dpos]
        out[k][tb:tb + L] = v
        done[k][tb:tb + L] = True
    full = np.full(len(a), np.nan)
    for k in range(total):
        full[done[k]] = out[k][done[k]]
    assert all(not (done[i] & done[j]).any() for i in range(total) for j in range(i + 1, total))
    return full, remote, read_remotely, exported


@pytest.mark.parametrize("name,nparts,extra", [("c5_m0", 2, False), ("c5_m0", 4, True),
                                               ("elast6_k1", 2, True), ("c1", 8, False)])
def test_sharded_parts_replay_bitwise(T, name, nparts, extra, oracle):
    # C6-style sharding: each part owns the rows of its ND subtree (separators
    # to part 0, or to an extra last part); every part has its own copy of U
    # and reads other parts' values through remote (peer) operands
    _, an = analyzed(name)
    plan = planned(name)
    owners = an.subtree_owners(nparts, separators=nparts if extra else 0)
    total = nparts + (1 if extra else 0)
    parts = []
    for k in range(total):
        p = plan.part_problem(total, owners, k)
        assert p.flow_devprog == 1 and p.flow_part == k
        parts.append(part_tables(p))
    f = plan.flow_tables()
    assert sum(len(p["unit"]) for p in parts) == len(f["flow_item"])
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    full, remote, read_remotely, exported = replay_parts(f, slot, upd, parts, owners)
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(full, ref)
    assert remote > 0
    assert read_remotely <= exported  # every row another part reads publishes at system scope


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "elast6_k1", "rand_spd_200"])
def test_init_factor_map_reproduces_host_init(name):
    # device init_factor_values (tcg_set_a_values) is a gather through this map
    _, an = analyzed(name)
    t = planned(name).flow_tables()
    m = t["a_map"]
    assert len(m) == len(t["values"])
    got = np.where(m >= 0, 0.0 + an.a_permuted.values[np.maximum(m, 0)], 0.0)
    assert bitwise_equal(got, t["values"])
    assert len(np.unique(m[m >= 0])) == int((m >= 0).sum())  # every A entry feeds one slot at most


@pytest.mark.parametrize("name,cap", [("elast6_k1", "1"), ("elast6_k1", "8"), ("grid20_k2_leaf4", "4"),
                                      ("s27_16_k2", "16"), ("elast6_k1", "1000")])
def test_chol_cap_schedules_replay_bitwise(T, name, cap, oracle, monkeypatch):
    # Chol units capped at `cap` coordinates (flow_plan.cpp; the default is
    # 32): still a partition of U, in an order where every read follows its
    # write (emulate_flow asserts it), and the replay is factor_serial's bits
    from checkers import emulate_flow, flow_programs
    monkeypatch.setenv("TCG_FLOW_CHOL_MAX", cap)
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    f = plan.flow_tables()
    rec = f["flow_rec"]
    L = rec[:, 1] & ((1 << 30) - 1)
    chol = ((rec[:, 1] >> 30) & 1) == 0
    lens = np.diff(f["row_ptr"])
    assert np.all(L[chol & (lens[rec[:, 3]] > 32)] <= int(cap))
    assert np.all(L <= np.maximum(32, int(cap)))
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(emulate_flow(rec, f["values"], slot, upd), ref)


@pytest.mark.parametrize("name,slack", [("elast6_k1", "100"), ("grid20_k2_leaf4", "50"), ("s27_16_k2", "100"),
                                        ("c1", "100"), ("c1", "37")])
def test_slack_placed_schedules_replay_bitwise(T, name, slack, oracle, monkeypatch):
    # units placed between their earliest and latest level (flow_slack_pct: the
    # default for large short-row matrices is as late as possible): still an
    # order where every read follows its write, and factor_serial's bits
    from checkers import emulate_flow, flow_programs
    _, an = analyzed(name)
    base = T.Plan(an.a_permuted, an.pattern, an.ranges).flow_tables()["flow_rec"]
    monkeypatch.setenv("TCG_FLOW_SLACK", slack)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    f = plan.flow_tables()
    rec = f["flow_rec"]
    assert rec.shape == base.shape and not np.array_equal(rec, base)  # a different order of the same units
    assert np.array_equal(np.sort(rec[:, 0]), np.sort(base[:, 0]))
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(emulate_flow(rec, f["values"], slot, upd), ref)


@pytest.mark.parametrize("name,panel", [("elast6_k1", "32"), ("elast6_k1", "8"), ("s27_16_k2", "16"),
                                        ("grid20_k2_leaf4", "4")])
def test_panel_schedules_replay_bitwise(T, name, panel, oracle, monkeypatch):
    # diagonal-block slices cut at fixed column panels (TCG_FLOW_PANEL): every
    # unit of a long row stays inside one panel of its block, U is still
    # partitioned, reads follow writes, and the replay is factor_serial's bits
    from checkers import emulate_flow, flow_programs
    monkeypatch.setenv("TCG_FLOW_PANEL", panel)
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    f = plan.flow_tables()
    rec, cols = f["flow_rec"], f["cols"]
    L = rec[:, 1] & ((1 << 30) - 1)
    b = an.ranges.bounds
    lens = np.diff(f["row_ptr"])
    for tb, ln, t in zip(rec[:, 0], L, rec[:, 3]):
        if lens[t] <= 32:
            continue
        k = int(np.searchsorted(b, t, side="right")) - 1  # t's block [b[k], b[k+1])
        c = cols[tb:tb + ln]
        if c[-1] < b[k + 1]:  # inside the diagonal block: one panel
            assert len(set(((c - b[k]) // int(panel)).tolist())) == 1
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(emulate_flow(rec, f["values"], slot, upd), ref)
