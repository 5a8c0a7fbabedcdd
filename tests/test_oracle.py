"""The plain-C oracle (oracle/oracle.c) pinned against the reference:
golden hashes of the reference's factor_serial / export_task_dag /
build_block_matrix, plus the known-answer tests of the reference's suites
(proj/tests/test_kernels.cpp, test_factorize.cpp, acceptance.cpp)."""
import math

import numpy as np
import pytest

from conftest import analyzed, bitwise_equal

FAST = ["c1", "c5_m0", "c5_m63", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1"]


@pytest.mark.parametrize("name", FAST + ["c2"])
def test_oracle_factor_matches_reference_hash(name, golden, oracle):
    g = golden[name]
    _, an = analyzed(name)
    vals, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert st == g["factor_status"] == 0
    assert oracle.hash(vals) == g["factor_values"]
    res = oracle.residual(an.a_permuted, an.pattern.pattern, vals)
    assert res == pytest.approx(g["residual"], rel=1e-9, abs=1e-18)


@pytest.mark.parametrize("name", FAST + ["c2"])
def test_oracle_dag_matches_reference_hash(name, golden, oracle):
    g = golden[name]["dag"]
    _, an = analyzed(name)
    k, bi, bj, ef, et = oracle.export_dag(an.pattern.pattern, an.ranges.bounds)
    assert len(k) == g["nodes"] and len(ef) == g["edges"]
    assert [int((k == t).sum()) for t in range(4)] == g["tasks"]
    for arr, key in ((k, "kind"), (bi, "block_row"), (bj, "block_col"), (ef, "edge_from"),
                     (et, "edge_to")):
        assert oracle.hash(arr) == g[key], key


@pytest.mark.parametrize("name", FAST)
def test_oracle_by_blocks_is_bitwise_serial(name, oracle):
    # the reference's own claim (factorize.hpp:15-19, README.md:93-96)
    _, an = analyzed(name)
    s, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    b, st2, _, _ = oracle.factor_by_blocks(an.a_permuted, an.pattern.pattern, an.ranges.bounds)
    assert st == st2 == 0
    assert bitwise_equal(s, b)


def csr(T, n, entries):
    ti, tj, tv = zip(*entries)
    import numpy as np
    order = np.lexsort((np.array(tj), np.array(ti)))
    ti, tj, tv = (np.array(x)[order] for x in (ti, tj, tv))
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ptr, ti + 1, 1)
    return T.CsrMatrix.from_arrays(n, np.cumsum(ptr), tj, tv)


def sym(entries):
    out = []
    for i, j, v in entries:
        out.append((i, j, v))
        if i != j:
            out.append((j, i, v))
    return out


def test_kat_diagonal_and_tridiagonal(T, oracle):
    # test_factorize.cpp:78-97
    d = csr(T, 3, [(0, 0, 4.0), (1, 1, 9.0), (2, 2, 16.0)])
    fp = T.levelk_pattern(d, 0)
    v, st, _, _ = oracle.factor_serial(d, fp.pattern)
    assert st == 0 and list(v) == [2.0, 3.0, 4.0]
    p = T.generate("path", 3)
    fp = T.levelk_pattern(p, 0)
    v, st, _, _ = oracle.factor_serial(p, fp.pattern)
    want = [math.sqrt(2.0), -1.0 / math.sqrt(2.0), math.sqrt(1.5), -math.sqrt(2.0 / 3.0),
            math.sqrt(4.0 / 3.0)]
    assert np.allclose(v, want, rtol=1e-15, atol=0)


def test_kat_chol_2x2_and_breakdown_rows(T, oracle):
    # test_kernels.cpp:36-77: [[4,2],[.,3]] -> [[2,1],[.,sqrt 2]]; breakdown row/pivot
    a = csr(T, 2, sym([(0, 0, 4.0), (0, 1, 2.0), (1, 1, 3.0)]))
    v, st, _, _ = oracle.factor_serial(a, T.levelk_pattern(a, 0).pattern)
    assert st == 0 and v[0] == 2.0 and v[1] == 1.0 and v[2] == math.sqrt(2.0)
    bad = csr(T, 2, sym([(0, 0, 1.0), (0, 1, 2.0), (1, 1, 1.0)]))
    _, st, row, piv = oracle.factor_serial(bad, T.levelk_pattern(bad, 0).pattern)
    assert st == 1 and row == 1 and piv < 0.0
    # a breakdown in the second block reports the global row (test_kernels.cpp:62-76)
    b4 = csr(T, 4, sym([(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 3, 4.0), (3, 3, 1.0)]))
    _, st, row, _ = oracle.factor_by_blocks(b4, T.levelk_pattern(b4, 0).pattern, [0, 2, 4])
    assert st == 1 and row == 3


def five_block_matrix(T):
    # test_factorize.cpp:40-53: one vertex per block, canonical 5x5 block structure
    ent = [(i, i, 4.0) for i in range(5)]
    ent += [(0, 4, -1.0), (1, 3, -1.0), (1, 4, -1.0), (2, 3, -1.0), (2, 4, -1.0), (3, 4, -1.0)]
    return csr(T, 5, sym(ent))


def test_five_range_dag_facts(T, oracle):
    # test_factorize.cpp:167-241 and acceptance c6
    a = five_block_matrix(T)
    fp = T.levelk_pattern(a, 0)
    k, bi, bj, ef, et = oracle.export_dag(fp.pattern, [0, 1, 2, 3, 4, 5])
    assert len(k) == 19
    assert [int((k == t).sum()) for t in range(4)] == [5, 6, 6, 2]
    per_iter = np.diff(np.append(np.where(k == 0)[0], len(k))).tolist()
    assert per_iter == [3, 6, 6, 3, 1]
    chol22 = int(np.where((k == 0) & (bi == 2))[0][0])
    assert chol22 not in set(et.tolist())
    # exact edge set, recomputed by replaying the generation walk
    blocks = {(0, 0), (0, 4), (1, 1), (1, 3), (1, 4), (2, 2), (2, 3), (2, 4), (3, 3), (3, 4), (4, 4)}
    writer, expected, nid = {}, set(), 0

    def emit(reads, write):
        nonlocal nid
        for blk in reads:
            if blk in writer:
                expected.add((writer[blk], nid))
        writer[write] = nid
        nid += 1

    for p in range(5):
        emit([(p, p)], (p, p))
        off = [j for j in range(p + 1, 5) if (p, j) in blocks]
        for j in off:
            emit([(p, p), (p, j)], (p, j))
        for x in range(len(off)):
            for y in range(x, len(off)):
                i, j = off[x], off[y]
                if (i, j) in blocks:
                    emit([(p, i), (p, j), (i, j)], (i, j))
    assert nid == 19
    assert set(zip(ef.tolist(), et.tolist())) == expected


def test_degenerate_dags(T, oracle):
    # test_factorize.cpp:243-260
    g = T.generate("grid2d", 3, 3)
    k, *_, ef, et = oracle.export_dag(T.levelk_pattern(g, 0).pattern, [0, 9])
    assert list(k) == [0] and len(ef) == 0
    d = csr(T, 8, [(i, i, 4.0) for i in range(8)])
    k, *_, ef, et = oracle.export_dag(T.levelk_pattern(d, 0).pattern, [0, 2, 4, 6, 8])
    assert len(k) == 4 and len(ef) == 0


@pytest.mark.parametrize("g", [4, 6])
def test_complete_fill_reconstructs(T, oracle, g):
    # test_factorize.cpp:314-331 / acceptance c5: complete fill reproduces A
    a = T.generate("grid2d", g, g)
    an = T.analyze(a, level=g * g, leaf_size=4, treecut=1)
    v, st, _, _ = oracle.factor_by_blocks(an.a_permuted, an.pattern.pattern, an.ranges.bounds)
    assert st == 0
    assert oracle.residual(an.a_permuted, an.pattern.pattern, v) <= 1e-10
