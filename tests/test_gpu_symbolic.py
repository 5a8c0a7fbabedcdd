"""Level-k symbolic on the GPU (tcg_sym_*) against the
reference's levelk_pattern_bfs (symbolic.hpp:57-120): the golden pattern hashes
the unmodified reference produced (tests/golden/golden.json), the oracle's
dense level recurrence (oracle.c orc_levelk_dense, symbolic.hpp:125-160) and
the host implementation; the reference's own symbolic facts
(test_symbolic.cpp:61-81). Bit-exact: integer work."""
import numpy as np
import pytest

from conftest import analyzed

pytestmark = pytest.mark.gpu

GOLDEN = ["c1", "c5_m0", "c5_m63", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1", "c2", "c3", "c4"]


def gpu_levelk(T, a, k, all_slow=False):
    g = T.GpuSymbolic(a)
    try:
        return g.levelk(k, all_slow=all_slow)
    finally:
        g.close()


def same_pattern(p, q):
    return np.array_equal(p.row_ptr, q.row_ptr) and np.array_equal(p.col_idx, q.col_idx)


def count_upper(a):
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))
    return int(np.count_nonzero(a.col_idx >= rows))


@pytest.mark.parametrize("name", GOLDEN)
def test_gpu_pattern_matches_reference_golden(T, golden, oracle, name):
    g = golden[name]
    _, an = analyzed(name)
    fp, st = gpu_levelk(T, an.a_permuted, g["level"])
    assert oracle.hash(fp.pattern.row_ptr) == g["pattern"]["row_ptr"]
    assert oracle.hash(fp.pattern.col_idx) == g["pattern"]["col_idx"]
    assert fp.pattern.nnz() == g["nnz_u"]
    assert fp.nnz_triu_input == count_upper(an.a_permuted)
    assert same_pattern(fp.pattern, an.pattern.pattern)


def test_gpu_pattern_c6_matches_reference_golden(T, golden, oracle):
    g = golden["c6"]
    _, an = analyzed("c6")
    fp, st = gpu_levelk(T, an.a_permuted, g["level"])
    assert oracle.hash(fp.pattern.row_ptr) == g["pattern"]["row_ptr"]
    assert oracle.hash(fp.pattern.col_idx) == g["pattern"]["col_idx"]
    assert st.slow_rows == 0


@pytest.mark.parametrize("name", ["c1", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1"])
def test_slow_path_equals_fast_path(T, name):
    _, an = analyzed(name)
    k = 2
    fast, sf = gpu_levelk(T, an.a_permuted, k)
    slow, ss = gpu_levelk(T, an.a_permuted, k, all_slow=True)
    assert ss.slow_rows == an.a_permuted.nrows
    assert same_pattern(fast.pattern, slow.pattern)
    assert same_pattern(fast.pattern, T.levelk_pattern(an.a_permuted, k).pattern)


@pytest.mark.parametrize("seed", range(6))
def test_gpu_levelk_equals_dense_dp_oracle(T, oracle, seed):
    # acceptance c1 (symbolic oracle), on the device
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 90))
    a = T.generate("random_spd", n, int(rng.integers(10000, 60000)), seed + 11)
    g = T.GpuSymbolic(a)
    try:
        for k in range(0, 5):
            for all_slow in (False, True):
                pat = g.levelk(k, all_slow=all_slow)[0].pattern
                dense = np.zeros((n, n), dtype=np.uint8)
                for i in range(n):
                    dense[i, pat.col_idx[pat.row_ptr[i]:pat.row_ptr[i + 1]]] = 1
                assert np.array_equal(dense, oracle.levelk_dense(a, k)), (n, k, all_slow)
    finally:
        g.close()


def test_grid3_fill_counts_and_level1_fill_set(T):
    # test_symbolic.cpp:61-81: 3x3 grid nnz 21/25/27/29, k=1 fill {(1,3),(2,4),(4,6),(5,7)}
    a = T.generate("grid2d", 3, 3)
    for k, nnz in ((0, 21), (1, 25), (2, 27), (9, 29)):
        assert gpu_levelk(T, a, k)[0].pattern.nnz() == nnz
    p0 = gpu_levelk(T, a, 0)[0].pattern
    p1 = gpu_levelk(T, a, 1)[0].pattern
    fill = [(i, int(c)) for i in range(9) for c in p1.col_idx[p1.row_ptr[i]:p1.row_ptr[i + 1]]
            if not p0.has_entry(i, int(c))]
    assert fill == [(1, 3), (2, 4), (4, 6), (5, 7)]


def test_edge_cases_match_host(T):
    C = T.CsrMatrix.from_arrays
    cases = {
        "empty": C(0, [0], []),
        "single": C(1, [0, 1], [0]),
        "no_diagonal": C(3, [0, 1, 3, 4], [1, 0, 2, 1]),
        "diagonal_only": C(4, [0, 1, 2, 3, 4], [0, 1, 2, 3]),
        "disconnected": C(4, [0, 2, 4, 6, 8], [0, 1, 0, 1, 2, 3, 2, 3]),
    }
    for name, a in cases.items():
        for k in (-1, 0, 1, 2, 50):
            fp, st = gpu_levelk(T, a, k)
            host = T.levelk_pattern(a, k).pattern
            assert same_pattern(fp.pattern, host), (name, k)


def test_large_level_searches_overflow_to_slow_path(T, oracle):
    # level >= n on a sparse random graph: late rows reach most of the graph,
    # far beyond a warp's shared-memory table
    a = T.generate("random_spd", 1500, 2500, 7)
    fp, st = gpu_levelk(T, a, 5000)
    assert st.tier2_rows > 0
    assert same_pattern(fp.pattern, T.levelk_pattern(a, 5000).pattern)
    a = T.generate("random_spd", 4000, 1000, 5)
    fp, st = gpu_levelk(T, a, 5000)
    assert st.slow_rows > 0
    assert same_pattern(fp.pattern, T.levelk_pattern(a, 5000).pattern)
    # and against the dense recurrence on a smaller one
    b = T.generate("random_spd", 300, 12000, 3)
    fb, sb = gpu_levelk(T, b, 300)
    dense = np.zeros((300, 300), dtype=np.uint8)
    for i in range(300):
        dense[i, fb.pattern.col_idx[fb.pattern.row_ptr[i]:fb.pattern.row_ptr[i + 1]]] = 1
    assert np.array_equal(dense, oracle.levelk_dense(b, 300))


def star(T, n):
    # vertex 0 adjacent to all others
    rows, cols = [], []
    for i in range(n):
        for c in (range(n) if i == 0 else (0, i)):
            rows.append(i)
            cols.append(c)
    ptr = np.zeros(n + 1, np.int64)
    np.add.at(ptr, np.asarray(rows) + 1, 1)
    return T.CsrMatrix.from_arrays(n, np.cumsum(ptr), cols)


@pytest.mark.parametrize("n,tier", [(1001, 2), (3001, 3)])
def test_star_hub_row_moves_through_the_tiers(T, n, tier):
    # row 0 has n - 1 targets at k = 0: beyond the 384-key tables (tier 2,
    # 1,536 keys) and beyond those too (global-memory path)
    a = star(T, n)
    for k in (0, 1):
        fp, st = gpu_levelk(T, a, k)
        assert st.tier2_rows >= 1
        assert (st.slow_rows >= 1) == (tier == 3)
        assert same_pattern(fp.pattern, T.levelk_pattern(a, k).pattern)


def test_reupload_reuses_the_handle(T):
    # a smaller matrix, then a larger one, through the same handle
    g = T.GpuSymbolic(analyzed("c5_m0")[1].a_permuted)
    try:
        for name in ("c1", "s27_16_k2", "c1"):
            _, an = analyzed(name)
            g.upload(an.a_permuted)
            fp, _ = g.levelk(an.pattern.level_cap)
            assert same_pattern(fp.pattern, an.pattern.pattern), name
    finally:
        g.close()


def test_invalid_input_raises(T):
    a = T.CsrMatrix.from_arrays(2, [0, 1, 2], [0, 5])
    with pytest.raises(ValueError, match="out of range"):
        T.GpuSymbolic(a)


def test_scratch_grows_to_a_single_pass(T):
    # level 40 on a random graph fills far more than the first scratch guess:
    # the short rows are searched again, scratch grows, the next call is one pass
    a = T.generate("random_spd", 900, 6000, 2)
    g = T.GpuSymbolic(a)
    try:
        first, s1 = g.levelk(40)
        second, s2 = g.levelk(40)
        assert s1.single_pass == 0 and s2.single_pass == 1
        host = T.levelk_pattern(a, 40).pattern
        assert same_pattern(first.pattern, host) and same_pattern(second.pattern, host)
        small, s3 = g.levelk(1)  # and back to a small level on the grown scratch
        assert s3.single_pass == 1 and same_pattern(small.pattern, T.levelk_pattern(a, 1).pattern)
    finally:
        g.close()
