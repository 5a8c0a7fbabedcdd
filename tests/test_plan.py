"""Host flattener (tcg_plan_build): the DAG is bit-exact with the reference's
export_task_dag, the block structure with build_block_matrix, and the work
tables reproduce factor_serial bit for bit when replayed on the CPU in any
order the dependences allow (task order, row order, random row orders)."""
import numpy as np
import pytest

from checkers import Reference, emulate_plan, emulate_program, emulate_rows, reference_available
from conftest import analyzed, bitwise_equal, planned

FAST = ["c1", "c5_m0", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1"]


@pytest.mark.parametrize("name", FAST + ["c2", "c3", "c4"])
def test_plan_dag_and_blocks_match_reference(name, golden, oracle):
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


@pytest.mark.parametrize("name", ["c1", "elast6_k1", "grid20_k2_leaf4", "rand_spd_200"])
def test_replays_are_bitwise_serial(name, golden, oracle):
    plan = planned(name)
    _, an = analyzed(name)
    ref, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert oracle.hash(ref) == golden[name]["factor_values"]
    assert bitwise_equal(emulate_plan(plan), ref)       # device merge mode, task order
    assert bitwise_equal(emulate_program(plan), ref)    # update programs, task order
    for seed in range(3):                               # row-level DAG, random orders
        assert bitwise_equal(emulate_rows(plan, seed), ref)


@pytest.mark.parametrize("name", ["c1", "s27_16_k2", "rand_spd_200"])
def test_static_schedule_is_topological_and_replays_bitwise(name, oracle):
    # mode 4: rows in position order; every predecessor sits at an earlier position
    plan = planned(name)
    t = plan.tables()
    order, pos, extra = t["row_order"], t["pos_rec"], t["pos_pred"]
    pos_of = np.empty(len(order), np.int64)
    pos_of[order] = np.arange(len(order))
    for q in range(len(order)):
        rec = pos[q]
        assert rec[12] == order[q]
        preds = [p for p in rec[8:8 + min(4, rec[6])]] + list(extra[rec[7]:rec[7] + max(0, rec[6] - 4)])
        assert len(preds) == rec[6]
        assert all(pos_of[p] < q for p in preds)
    # replay in position order == serial
    _, an = analyzed(name)
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    vals = t["values"].copy()
    srec, upd, rows = t["slot_rec"], t["upd"], t["row_rec"]
    for k in order:
        tb, te, dpos, soff, kind = rows[k][:5]
        tv = vals[tb:te].copy()
        for j in range(te - tb):
            ub, ue, _, _ = srec[soff + j]
            for u in range(ub, ue):
                tv[j] = tv[j] - vals[upd[u][0]] * vals[upd[u][1]]
        if kind == 0:
            d = np.sqrt(tv[0])
            tv[1:] = tv[1:] / d
            tv[0] = d
        elif kind == 1:
            tv = tv / vals[dpos]
        vals[tb:te] = tv
    assert bitwise_equal(vals, ref)


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


def test_row_dependences_are_acyclic_and_shorter(T):
    plan = planned("c5_m0")
    s = plan.stats()
    assert s.item_depth < s.dag_depth  # rows shorten the critical path
    t = plan.tables()
    rows, succ = t["row_rec"], t["row_succ"] & 0x3FFFFFFF
    for k in range(0, len(rows), 97):
        assert np.all(succ[rows[k, 6]:rows[k, 7]] > k)  # generation order is topological
    assert t["row_indeg"].sum() == len(succ)


def test_single_range_and_diagonal_only(T, oracle):
    a = T.generate("grid2d", 5, 5)
    fp = T.levelk_pattern(a, 1)
    one = T.RangeList(np.array([0, 25], dtype=np.int32))
    plan = T.Plan(a, fp, one)
    assert list(plan.stats().tasks) == [1, 0, 0, 0]
    ref, _, _, _ = oracle.factor_serial(a, fp.pattern)
    assert bitwise_equal(emulate_rows(plan), ref)
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
        assert bitwise_equal(emulate_rows(plan, seed), vals)


def replay_flow(t, order=None):
    """Mode 5 on the CPU: finalising rows in schedule order (or `order`), each
    coordinate applying its merged program once, reading only final values."""
    rec, slot, upd = t["flow_rec"], t["flow_slot"], t["flow_upd"]
    a = t["values"]
    out = np.full(len(a), np.nan)
    done = np.zeros(len(a), bool)
    for q in (range(len(rec)) if order is None else order):
        tb, lk, dpos, _ = rec[q]
        L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 3
        v = a[tb:tb + L].copy()
        for j in range(L):
            ub, ue = slot[tb + j, :2]
            for m, o in upd[ub:ue]:
                assert done[m] and done[o], "read before written"
                v[j] = v[j] - out[m] * out[o]
        if kind == 0:
            d = np.sqrt(v[0])
            v[1:] = v[1:] / d
            v[0] = d
        else:
            assert done[dpos]
            v = v / out[dpos]
        assert not done[tb:tb + L].any(), "written twice"
        out[tb:tb + L] = v
        done[tb:tb + L] = True
    assert done.all()
    return out


@pytest.mark.parametrize("merge", [True, False])
@pytest.mark.parametrize("name", ["c1", "rand_spd_200", "grid20_k2_leaf4", "elast6_k1"])
def test_flow_schedule_partitions_u_and_replays_bitwise(T, name, merge, oracle, monkeypatch):
    # mode 5: the rows of the schedule own every coordinate once -- whole
    # matrix rows of <= 32 entries (merge) or one Chol/Trsm item each; merged
    # programs keep the per-coordinate product order, so replays equal
    # factor_serial
    monkeypatch.setenv("TCG_FLOW_MERGE_ROWS", "1" if merge else "0")
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    t = plan.tables()
    s = plan.stats()
    fin = int((t["row_rec"][:, 4] <= 1).sum())
    rec = t["flow_rec"]
    L = rec[:, 1] & ((1 << 30) - 1)
    assert s.flow_rows == len(rec) and int(L.sum()) == len(t["values"])  # a partition of U
    u = an.pattern.pattern
    if merge:  # rows of <= 32 entries whole; longer ones: the diagonal-block slice + chunks of <= 32
        assert s.flow_rows <= fin
        assert int((np.diff(u.row_ptr) <= 32).sum()) <= s.flow_rows
    else:
        assert s.flow_rows == fin
        assert np.array_equal(np.sort(t["flow_item"]), np.flatnonzero(t["row_rec"][:, 4] <= 1))
    assert len(t["flow_upd"]) == len(t["upd"])  # every product folded in exactly once
    assert s.flow_depth <= s.item_depth
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(replay_flow(t), ref)
    # any order that respects "reads only written values" gives the same bits:
    # matrix-row order is one
    assert bitwise_equal(replay_flow(t, np.lexsort(((rec[:, 1] >> 30) & 1, rec[:, 3]))), ref)


LOCAL = 0x80000000


def replay_units(t):
    """Mode 6 on the CPU: units and rows in the joint schedule order; a unit
    runs its rows level by level with its own values in a local array
    (operands flagged LOCAL), everything else reads the global factor."""
    rows, rows_item = t["m6_row_rec"], t["m6_row_item"]
    units, urec, ulb, ulev = t["m6_unit_rec"], t["m6_urow_rec"], t["m6_urow_lbase"], t["m6_ulev"]
    slot, upd = t["m6_slot"], t["m6_upd"]
    a = t["values"]
    out = np.full(len(a), np.nan)
    done = np.zeros(len(a), bool)
    m6_node = t["m6_row_node"] if "m6_row_node" in t else None

    def run_row(rec, local=None, lb=None):
        tb, lk, dpos, _ = rec
        L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 3
        v = a[tb:tb + L].copy()
        for j in range(L):
            ub, ue = slot[tb + j, :2]
            for m, o in upd[ub:ue]:
                vals = []
                for x in (int(m) & 0xFFFFFFFF, int(o) & 0xFFFFFFFF):
                    if x & LOCAL:
                        assert local is not None and not np.isnan(local[x & ~LOCAL]), "local read before written"
                        vals.append(local[x & ~LOCAL])
                    else:
                        assert done[x], "read before written"
                        vals.append(out[x])
                v[j] = v[j] - vals[0] * vals[1]
        if kind == 0:
            d = np.sqrt(v[0])
            v[1:] = v[1:] / d
            v[0] = d
        else:
            assert done[dpos]
            v = v / out[dpos]
        assert not done[tb:tb + L].any(), "written twice"
        out[tb:tb + L] = v
        done[tb:tb + L] = True
        if local is not None:
            local[lb:lb + L] = v

    # joint order: unit k sits at order position units[k, 3]; rows fill the rest in order
    nodes = len(rows) + len(units)
    unit_at = {int(u[3]): k for k, u in enumerate(units)}
    r = 0
    for pos in range(nodes):
        if pos in unit_at:
            lb, le, rb, _ = units[unit_at[pos]]
            n_local = 0
            start = rb
            bounds = []
            for s in range(lb, le):
                bounds.append((start, ulev[s]))
                start = ulev[s]
            for b0, b1 in bounds:
                for q in range(b0, b1):
                    n_local = max(n_local, ulb[q] + (urec[q, 1] & ((1 << 30) - 1)))
            local = np.full(n_local, np.nan)
            for b0, b1 in bounds:
                # rows of one level are independent: run them in reverse to prove it
                for q in reversed(range(b0, b1)):
                    run_row(urec[q], local, ulb[q])
        else:
            run_row(rows[r])
            r += 1
    assert r == len(rows) and done.all()
    return out


@pytest.mark.parametrize("name,min_rows,merge", [("c5_m0", 64, 0), ("c5_m0", 16, 0), ("grid20_k2_leaf4", 8, 0),
                                                 ("elast6_k1", 32, 0), ("rand_spd_200", 4, 0),
                                                 # merged rows: units only where a block's rows are all
                                                 # diagonal-block slices; long rows' chunks share an item
                                                 ("s27_16_k2", 16, 1), ("elast6_k1", 16, 1)])
def test_unit_schedule_replays_bitwise(T, name, min_rows, merge, oracle, monkeypatch):
    monkeypatch.setenv("TCG_UNIT_MIN_ROWS", str(min_rows))
    monkeypatch.setenv("TCG_FLOW_MERGE_ROWS", str(merge))
    _, an = analyzed(name)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    t = plan.tables()
    s = plan.stats()
    if merge and s.unit_count == 0:
        pytest.skip("every large block has merged whole rows")
    assert s.unit_count == len(t["m6_unit_rec"]) > 0
    assert len(t["m6_row_rec"]) + s.unit_rows == s.flow_rows
    assert sorted(np.concatenate([t["m6_row_item"], t["m6_urow_item"]])) == sorted(t["flow_item"])
    assert t["m6_smem"] <= 72 * 1024
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(replay_units(t), ref)


def part_tables(p):
    from paper_1601_05871_b200.core import _copy
    n = int(p.nflow)
    return {"rec": _copy(p.flow_rec, 4 * n, np.int32).reshape(-1, 4), "item": _copy(p.flow_item, n, np.int32),
            "slot": _copy(p.flow_slot, 4 * p.nnz, np.int32).reshape(-1, 4),
            "upd": _copy(p.flow_upd, 2 * p.nflow_upd, np.int32).reshape(-1, 2)}


def replay_parts(t, parts, owners):
    """Sharded value flow on the CPU: every part's rows in the global order,
    each part with its own copy of U, remote operands read from their owner's
    copy. Returns (assembled factor, remote operand count, rows read remotely,
    rows flagged exported)."""
    total = len(parts)
    pos_of_item = {int(it): q for q, it in enumerate(t["flow_item"])}
    order = sorted((pos_of_item[int(it)], k, i) for k, p in enumerate(parts) for i, it in enumerate(p["item"]))
    a = t["values"]
    out = [np.full(len(a), np.nan) for _ in range(total)]
    done = [np.zeros(len(a), bool) for _ in range(total)]
    remote = 0
    exported, read_remotely = set(), set()
    row_start = {}  # U position -> (part, first position of its row slice)
    for k, p in enumerate(parts):
        for tb, lk, _, _ in p["rec"]:
            for x in range(tb, tb + (lk & ((1 << 30) - 1))):
                row_start[x] = (k, int(tb))
    for _, k, i in order:
        tb, lk, dpos, trow = parts[k]["rec"][i]
        assert owners[trow] == k
        L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 1
        if lk < 0:
            exported.add((k, int(tb)))
        v = a[tb:tb + L].copy()
        for j in range(L):
            ub, ue = parts[k]["slot"][tb + j, :2]
            for m, o in parts[k]["upd"][ub:ue]:
                vals = []
                for x in (int(m) & 0xFFFFFFFF, int(o) & 0xFFFFFFFF):
                    if x & 0x80000000:
                        ow, pos = (x >> 25) & 63, x & 0x1FFFFFF
                        assert ow != k
                        remote += 1
                        read_remotely.add(row_start[pos])
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
    parts = [part_tables(plan.part_problem(total, owners, k)) for k in range(total)]
    t = plan.tables()
    assert sum(len(p["item"]) for p in parts) == len(t["flow_item"])
    full, remote, read_remotely, exported = replay_parts(t, parts, owners)
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(full, ref)
    assert remote > 0
    assert read_remotely <= exported  # every row another part reads publishes at system scope


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2", "elast6_k1", "rand_spd_200"])
def test_init_factor_map_reproduces_host_init(name):
    # device init_factor_values (tcg_set_a_values) is a gather through this map
    _, an = analyzed(name)
    t = planned(name).tables()
    m = t["a_map"]
    assert len(m) == len(t["values"])
    got = np.where(m >= 0, 0.0 + an.a_permuted.values[np.maximum(m, 0)], 0.0)
    assert bitwise_equal(got, t["values"])
    assert len(np.unique(m[m >= 0])) == int((m >= 0).sum())  # every A entry feeds one slot at most
