"""File formats either side of the path: Matrix Market
input and factor output, imported orderings, analyze() with an imported
ordering. Checked against the unmodified reference (oracle/_ref: the same
bytes written, the same matrices and errors read) and against the
reference's own unit-test facts (test_matrix_market.cpp, test_ordering.cpp)."""
import os

import numpy as np
import pytest

from checkers import Oracle, Reference, reference_available
from conftest import analyzed, bitwise_equal

needs_ref = pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built (no /root/reference)")


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


# -- reference facts (test_matrix_market.cpp) ---------------------------------

def test_symmetric_storage_is_mirrored(T, tmp_path):
    p = write(tmp_path, "sym2.mtx", "%%MatrixMarket matrix coordinate real symmetric\n% comment line\n"
                                    "2 2 3\n1 1 4\n2 1 2\n2 2 3\n")
    m = T.load_matrix_market(p)
    assert m.nnz() == 4
    assert (m.at(0, 0), m.at(0, 1), m.at(1, 0), m.at(1, 1)) == (4.0, 2.0, 2.0, 3.0)


def test_pattern_files_and_empty_pattern(T, tmp_path):
    m = T.load_matrix_market(write(tmp_path, "pat.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                                                        "3 3 2\n1 1\n3 1\n"))
    assert m.nnz() == 3 and m.at(0, 0) == m.at(0, 2) == m.at(2, 0) == 1.0
    e = T.load_matrix_market(write(tmp_path, "empty3.mtx", "%%MatrixMarket matrix coordinate pattern general\n"
                                                           "3 3 0\n"))
    assert e.nrows == 3 and e.nnz() == 0 and list(e.row_ptr) == [0, 0, 0, 0]


def test_duplicates_are_summed(T, tmp_path):
    m = T.load_matrix_market(write(tmp_path, "dup.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                        "2 2 3\n1 1 1.5\n1 1 2.5\n2 2 1\n"))
    assert m.nnz() == 2 and m.at(0, 0) == 4.0


MALFORMED = {
    "cx.mtx": ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "complex"),
    "rect.mtx": ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", "square"),
    "trunc.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n", "expected 3 entries"),
    "badidx.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n5 1 1\n", "out of range"),
    "arr.mtx": ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "coordinate"),
    "skew.mtx": ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n", "symmetry"),
    "nobanner.mtx": ("2 2 1\n1 1 1\n", "not a Matrix Market"),
    "nosize.mtx": ("%%MatrixMarket matrix coordinate real general\n% only comments\n", "missing size"),
    "badsize.mtx": ("%%MatrixMarket matrix coordinate real general\n2 x 1\n", "malformed size"),
    "badval.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n", "malformed value"),
    "badent.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 1\n", "malformed entry"),
    "empty.mtx": ("", "empty file"),
}


@pytest.mark.parametrize("name", sorted(MALFORMED))
def test_malformed_inputs_are_rejected_with_context(T, tmp_path, name):
    text, needle = MALFORMED[name]
    p = write(tmp_path, name, text)
    with pytest.raises(T.MatrixMarketError, match=needle):
        T.load_matrix_market(p)
    if reference_available():  # the same message as the reference
        with pytest.raises(RuntimeError) as ref:
            Reference().load_mm(p)
        with pytest.raises(T.MatrixMarketError) as ours:
            T.load_matrix_market(p)
        assert str(ours.value) == str(ref.value)


def test_missing_file(T):
    with pytest.raises(T.MatrixMarketError, match="cannot open"):
        T.load_matrix_market("/nonexistent/file.mtx")


# -- against the reference ------------------------------------------------------

def factor_matrix(T, oracle):
    """U of C1 with factor_serial's values: many distinct doubles to print."""
    _, an = analyzed("c1")
    vals, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    u = an.pattern.pattern
    return T.CsrMatrix(u.nrows, u.ncols, u.row_ptr, u.col_idx, vals)


@needs_ref
def test_writer_bytes_equal_the_reference(T, tmp_path):
    R = Reference()
    rng = np.random.default_rng(3)
    cases = {"factor_c1": factor_matrix(T, Oracle()), "c5_m0": analyzed("c5_m0")[1].a_permuted}
    odd = T.generate("random_spd", 40, 200000, 9)
    odd.values[:12] = [0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 1e22, 1e-7,
                       0.1, 1.0 / 3.0, -123456789.125, 2.0 ** 53 + 2, np.nextafter(1.0, 2.0)]
    odd.values[12:] = rng.standard_normal(odd.nnz() - 12) * 10.0 ** rng.integers(-30, 30, odd.nnz() - 12)
    cases["odd_values"] = odd
    for name, m in cases.items():
        ours, ref = tmp_path / f"{name}_ours.mtx", tmp_path / f"{name}_ref.mtx"
        T.write_matrix_market(m, str(ours))
        R.write_mm(m, str(ref))
        assert ours.read_bytes() == ref.read_bytes(), name


@needs_ref
def test_reader_equals_the_reference(T, tmp_path):
    R = Reference()
    texts = {
        "general": "%%MatrixMarket matrix coordinate real general\n% c\n\n3 3 5\n3 1 -2.5e-3\n1 1 4\n"
                   "1 3 -2.5e-3\n3 3 7\n2 2 1e300\n",
        "symmetric_int": "%%MatrixMarket matrix coordinate integer symmetric\n4 4 5\n1 1 2\n2 1 -1\n"
                         "2 2 2\n4 3 -1\n4 4 2\n",
        "upper_case": "%%MATRIXMARKET MATRIX COORDINATE REAL GENERAL\n2 2 2\n1 1 1\n2 2 2\n",
        "dups_sym": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n2 1 0.1\n2 1 0.2\n1 2 0.3\n3 3 1\n",
    }
    for name, text in texts.items():
        p = write(tmp_path, name + ".mtx", text)
        m = T.load_matrix_market(p)
        rp, rc, rv = R.load_mm(p)
        assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, rc), name
        assert bitwise_equal(m.values, rv), name
    # a written factor reads back bit for bit (shortest round-trip printing)
    u = factor_matrix(T, Oracle())
    p = str(tmp_path / "u.mtx")
    T.write_matrix_market(u, p)
    back = T.load_matrix_market(p)
    assert bitwise_equal(back.values, u.values) and np.array_equal(back.col_idx, u.col_idx)


# -- orderings (test_ordering.cpp "ordering import") ---------------------------

def test_ordering_import_reference_facts(T, tmp_path):
    perm, b = T.load_ordering(write(tmp_path, "ord_ok.txt", "3\n0\n1\n2\n1\n0 3\n"), 3)
    assert list(perm) == [0, 1, 2] and list(b) == [0, 3]
    with pytest.raises(RuntimeError, match="bijection"):
        T.load_ordering(write(tmp_path, "ord_dup.txt", "3\n0\n0\n2\n1\n0 3\n"), 3)
    with pytest.raises(RuntimeError, match="contiguous"):
        T.load_ordering(write(tmp_path, "ord_gap.txt", "4\n0\n1\n2\n3\n2\n0 2\n3 4\n"), 4)
    with pytest.raises(RuntimeError):
        T.load_ordering(write(tmp_path, "ord_n.txt", "5\n0\n1\n2\n3\n4\n1\n0 5\n"), 3)


ORDERING_ERRORS = {
    "range.txt": ("3\n0\n1\n7\n1\n0 3\n", 3),
    "trunc_perm.txt": ("3\n0\n1\n", 3),
    "no_count.txt": ("3\n0\n1\n2\n", 3),
    "neg_count.txt": ("3\n0\n1\n2\n-1\n", 3),
    "trunc_ranges.txt": ("3\n2\n1\n0\n2\n0 1\n", 3),
    "cover.txt": ("3\n2\n1\n0\n1\n0 2\n", 3),
    "empty.txt": ("", 3),
}


@pytest.mark.parametrize("name", sorted(ORDERING_ERRORS))
def test_ordering_errors_match_the_reference(T, tmp_path, name):
    text, n = ORDERING_ERRORS[name]
    p = write(tmp_path, name, text)
    with pytest.raises(RuntimeError) as ours:
        T.load_ordering(p, n)
    if reference_available():
        with pytest.raises(RuntimeError) as ref:
            Reference().load_ordering(p, n)
        assert str(ours.value) == str(ref.value)


def write_ordering(path, perm, bounds):
    with open(path, "w") as f:
        f.write(f"{len(perm)}\n" + "".join(f"{int(v)}\n" for v in perm))
        f.write(f"{len(bounds) - 1}\n" + "".join(f"{int(b)} {int(e)}\n" for b, e in zip(bounds[:-1], bounds[1:])))


@pytest.mark.parametrize("name", ["c1", "c5_m0", "s27_16_k2"])
def test_analyze_with_imported_ordering_reproduces_nd(T, tmp_path, name, golden, oracle):
    # the ND ordering written out and imported gives the same analysis (and
    # therefore the reference's golden pattern and factor)
    a, an = analyzed(name)
    p = str(tmp_path / "ord.txt")
    write_ordering(p, an.perm, an.ranges.bounds)
    if reference_available():
        rp, rb = Reference().load_ordering(p, a.nrows)
        assert np.array_equal(rp, an.perm) and np.array_equal(rb, an.ranges.bounds)
    im = T.analyze(a, level=golden[name]["level"], ordering_path=p)
    assert np.array_equal(im.perm, an.perm) and np.array_equal(im.ranges.bounds, an.ranges.bounds)
    assert np.array_equal(im.a_permuted.col_idx, an.a_permuted.col_idx)
    assert bitwise_equal(im.a_permuted.values, an.a_permuted.values)
    assert oracle.hash(im.pattern.pattern.col_idx) == golden[name]["pattern"]["col_idx"]


def test_analyze_with_a_coarse_imported_ordering(T, tmp_path, oracle):
    # an external ordering (reverse numbering, two ranges): PᵀAP, pattern and
    # the factor by blocks on it agree with factor_serial
    a = T.generate("grid2d", 12, 12)
    n = a.nrows
    perm = np.arange(n)[::-1].astype(np.int32)
    p = str(tmp_path / "rev.txt")
    write_ordering(p, perm, [0, 50, n])
    an = T.analyze(a, level=1, ordering_path=p)
    assert list(an.ranges.bounds) == [0, 50, n]
    assert an.a_permuted.at(int(perm[0]), int(perm[1])) == a.at(0, 1)
    ref, st, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    blk, st2, _, _ = oracle.factor_by_blocks(an.a_permuted, an.pattern.pattern, an.ranges.bounds)
    assert st == st2 == 0 and bitwise_equal(ref, blk)
