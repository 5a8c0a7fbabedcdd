"""Test-only bindings of the CPU checkers (oracle/ and oracle/_ref).

``Oracle``    the plain-C restatement (oracle/_build/liboracle.so)
``Reference`` the unmodified reference headers behind an extern "C" shim
              (oracle/_ref/libtaskchol_ref.so); available only where it was
              built (the dev container, and the GPU box via the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtaskchol_ref.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


def _p(a, t):
    return a.ctypes.data_as(t)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle`")
        L = C.CDLL(path)
        L.orc_hash_f64.restype = C.c_uint64
        L.orc_hash_f64.argtypes = [f64p, C.c_int64]
        L.orc_hash_i32.restype = C.c_uint64
        L.orc_hash_i32.argtypes = [i32p, C.c_int64]
        L.orc_hash_i64.restype = C.c_uint64
        L.orc_hash_i64.argtypes = [i64p, C.c_int64]
        L.orc_init_factor_values.argtypes = [C.c_int32, i64p, i32p, f64p, i64p, i32p, f64p]
        L.orc_factor_serial.argtypes = [C.c_int32, i64p, i32p, f64p, i32p, f64p]
        L.orc_export_dag.argtypes = [C.c_int32, i64p, i32p, C.c_int32, i32p, i64p, i64p,
                                     i32p, i32p, i32p, i32p, i32p]
        L.orc_factor_by_blocks.argtypes = [C.c_int32, i64p, i32p, f64p, C.c_int32, i32p, i32p, f64p]
        L.orc_pattern_residual.restype = C.c_double
        L.orc_pattern_residual.argtypes = [C.c_int32, i64p, i32p, f64p, i64p, i32p, f64p]
        L.orc_levelk_dense.argtypes = [C.c_int32, i64p, i32p, C.c_int32, u8p]
        L.orc_trisolve.argtypes = [C.c_int32, i64p, i32p, f64p, f64p, C.c_int32, f64p]
        L.orc_trisolve.restype = C.c_int
        self.L = L

    # hashes ---------------------------------------------------------------
    def hash(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        if a.dtype == np.float64:
            h = self.L.orc_hash_f64(_p(a, f64p), a.size)
        elif a.dtype == np.int32:
            h = self.L.orc_hash_i32(_p(a, i32p), a.size)
        elif a.dtype == np.int64:
            h = self.L.orc_hash_i64(_p(a, i64p), a.size)
        else:
            raise TypeError(a.dtype)
        return f"{h:016x}"

    # numeric --------------------------------------------------------------
    def init_values(self, a, u) -> np.ndarray:
        out = np.zeros(u.nnz(), dtype=np.float64)
        self.L.orc_init_factor_values(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p),
                                      _p(a.values, f64p), _p(u.row_ptr, i64p), _p(u.col_idx, i32p),
                                      _p(out, f64p))
        return out

    def factor_serial(self, a, u):
        """Returns (values, status, row, pivot)."""
        vals = self.init_values(a, u)
        row, piv = C.c_int32(-1), C.c_double(0.0)
        st = self.L.orc_factor_serial(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p),
                                      _p(vals, f64p), C.byref(row), C.byref(piv))
        return vals, st, row.value, piv.value

    def factor_by_blocks(self, a, u, bounds):
        vals = self.init_values(a, u)
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        row, piv = C.c_int32(-1), C.c_double(0.0)
        st = self.L.orc_factor_by_blocks(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p),
                                         _p(vals, f64p), b.size - 1, _p(b, i32p), C.byref(row),
                                         C.byref(piv))
        return vals, st, row.value, piv.value

    def export_dag(self, u, bounds):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        nn, ne = C.c_int64(), C.c_int64()
        null = C.cast(None, i32p)
        st = self.L.orc_export_dag(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), b.size - 1,
                                   _p(b, i32p), C.byref(nn), C.byref(ne), null, null, null, null,
                                   null)
        if st:
            raise ValueError(f"orc_export_dag status {st}")
        k = np.zeros(nn.value, np.int32)
        bi, bj = np.zeros_like(k), np.zeros_like(k)
        ef, et = np.zeros(ne.value, np.int32), np.zeros(ne.value, np.int32)
        self.L.orc_export_dag(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), b.size - 1,
                              _p(b, i32p), C.byref(nn), C.byref(ne), _p(k, i32p), _p(bi, i32p),
                              _p(bj, i32p), _p(ef, i32p), _p(et, i32p))
        return k, bi, bj, ef, et

    def residual(self, a, u, vals) -> float:
        v = np.ascontiguousarray(vals, dtype=np.float64)
        return self.L.orc_pattern_residual(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p),
                                           _p(a.values, f64p), _p(u.row_ptr, i64p),
                                           _p(u.col_idx, i32p), _p(v, f64p))

    def trisolve(self, u, vals, b, which=3) -> np.ndarray:
        """x with Uᵀ y = b (which & 1) and U x = y (which & 2), oracle order."""
        v = np.ascontiguousarray(vals, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(u.nrows, np.float64)
        st = self.L.orc_trisolve(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), _p(v, f64p),
                                 _p(bb, f64p), which, _p(x, f64p))
        if st != 0:
            raise ValueError(f"orc_trisolve status {st}")
        return x

    def levelk_dense(self, a, k) -> np.ndarray:
        m = np.zeros(a.nrows * a.nrows, dtype=np.uint8)
        self.L.orc_levelk_dense(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p), k, _p(m, u8p))
        return m.reshape(a.nrows, a.nrows)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The reference's own code, compiled unmodified (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make ref` where /root/reference exists")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_error.restype = C.c_char_p
        L.ref_analyze.restype = vp
        L.ref_analyze.argtypes = [C.c_int32, i64p, i32p, f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.ref_analysis_free.argtypes = [vp]
        for name, rt in [("perm", i32p), ("bounds", i32p), ("u_ptr", i64p), ("u_col", i32p),
                         ("a_ptr", i64p), ("a_col", i32p), ("a_val", f64p)]:
            f = getattr(L, "ref_analysis_" + name)
            f.restype = rt
            f.argtypes = [vp]
        for name in ("nranges",):
            f = getattr(L, "ref_analysis_" + name)
            f.restype = C.c_int32
            f.argtypes = [vp]
        for name in ("nnz_u", "nnz_a"):
            f = getattr(L, "ref_analysis_" + name)
            f.restype = C.c_int64
            f.argtypes = [vp]
        L.ref_analysis_seconds.restype = C.c_double
        L.ref_analysis_seconds.argtypes = [vp, C.c_int]
        L.ref_levelk.restype = C.c_int64
        L.ref_levelk.argtypes = [C.c_int32, i64p, i32p, C.c_int32, i64p, i32p, C.c_int64]
        L.ref_factor_serial.argtypes = [C.c_int32, i64p, i32p, f64p, i64p, i32p, f64p, f64p, i32p, f64p]
        L.ref_factor_by_blocks.argtypes = [C.c_int32, i64p, i32p, f64p, i64p, i32p, C.c_int32, i32p,
                                           C.c_int32, f64p, f64p, f64p, i64p, i32p, f64p]
        L.ref_write_mm.argtypes = [C.c_int32, i64p, i32p, f64p, C.c_char_p]
        L.ref_load_mm.restype = vp
        L.ref_load_mm.argtypes = [C.c_char_p]
        L.ref_csr_free.argtypes = [vp]
        L.ref_csr_n.restype = C.c_int32
        L.ref_csr_nnz.restype = C.c_int64
        for name, rt in (("ptr", i64p), ("col", i32p), ("val", f64p)):
            getattr(L, "ref_csr_" + name).restype = rt
        for name in ("n", "nnz", "ptr", "col", "val"):
            getattr(L, "ref_csr_" + name).argtypes = [vp]
        L.ref_generate.restype = vp
        L.ref_generate.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64]
        L.ref_load_ordering.restype = C.c_int32
        L.ref_load_ordering.argtypes = [C.c_char_p, C.c_int32, i32p, C.c_int32, i32p]
        L.ref_export_dag.restype = vp
        L.ref_export_dag.argtypes = [C.c_int32, i64p, i32p, C.c_int32, i32p]
        L.ref_dag_free.argtypes = [vp]
        for name in ("nnodes", "nedges"):
            f = getattr(L, "ref_dag_" + name)
            f.restype = C.c_int64
            f.argtypes = [vp]
        for name in ("kind", "bi", "bj", "from", "to"):
            f = getattr(L, "ref_dag_" + name)
            f.restype = i32p
            f.argtypes = [vp]
        L.ref_blocks.restype = C.c_int64
        L.ref_blocks.argtypes = [C.c_int32, i64p, i32p, C.c_int32, i32p, i64p, i32p, C.c_int64]
        self.L = L

    @staticmethod
    def _arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dt, copy=True)

    def analyze(self, a, level=0, treecut=0, leaf=64, max_depth=100) -> dict:
        h = self.L.ref_analyze(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p), _p(a.values, f64p),
                               level, treecut, leaf, max_depth)
        if not h:
            raise ValueError(self.L.ref_error().decode())
        try:
            n = a.nrows
            nr = self.L.ref_analysis_nranges(h)
            nu = self.L.ref_analysis_nnz_u(h)
            na = self.L.ref_analysis_nnz_a(h)
            return {
                "perm": self._arr(self.L.ref_analysis_perm(h), n, np.int32),
                "bounds": self._arr(self.L.ref_analysis_bounds(h), nr + 1, np.int32),
                "u_ptr": self._arr(self.L.ref_analysis_u_ptr(h), n + 1, np.int64),
                "u_col": self._arr(self.L.ref_analysis_u_col(h), nu, np.int32),
                "a_ptr": self._arr(self.L.ref_analysis_a_ptr(h), n + 1, np.int64),
                "a_col": self._arr(self.L.ref_analysis_a_col(h), na, np.int32),
                "a_val": self._arr(self.L.ref_analysis_a_val(h), na, np.float64),
                "ordering_seconds": self.L.ref_analysis_seconds(h, 0),
                "symbolic_seconds": self.L.ref_analysis_seconds(h, 1),
            }
        finally:
            self.L.ref_analysis_free(h)

    def write_mm(self, m, path) -> None:
        if self.L.ref_write_mm(m.nrows, _p(m.row_ptr, i64p), _p(m.col_idx, i32p), _p(m.values, f64p),
                               str(path).encode()) != 0:
            raise RuntimeError(self.L.ref_error().decode())

    def load_mm(self, path):
        """(row_ptr, col_idx, values) or raises RuntimeError(reference message)."""
        h = self.L.ref_load_mm(str(path).encode())
        if not h:
            raise RuntimeError(self.L.ref_error().decode())
        try:
            n, nnz = self.L.ref_csr_n(h), self.L.ref_csr_nnz(h)
            return (self._arr(self.L.ref_csr_ptr(h), n + 1, np.int64), self._arr(self.L.ref_csr_col(h), nnz, np.int32),
                    self._arr(self.L.ref_csr_val(h), nnz, np.float64))
        finally:
            self.L.ref_csr_free(h)

    def generate(self, kind, p0, p1=0, seed=0):
        """The repo's seeded config generators, compiled into the shim: (row_ptr, col_idx, values)."""
        h = self.L.ref_generate(kind.encode(), p0, p1, seed)
        if not h:
            raise ValueError(self.L.ref_error().decode())
        try:
            n, nnz = self.L.ref_csr_n(h), self.L.ref_csr_nnz(h)
            return (self._arr(self.L.ref_csr_ptr(h), n + 1, np.int64), self._arr(self.L.ref_csr_col(h), nnz, np.int32),
                    self._arr(self.L.ref_csr_val(h), nnz, np.float64))
        finally:
            self.L.ref_csr_free(h)

    def test_matrix(self, kind, p0, p1=0, seed=0):
        """The reference's own test generators (tests/support/test_matrices.hpp): (row_ptr, col_idx, values)."""
        self.L.ref_test_matrix.restype = C.c_void_p
        self.L.ref_test_matrix.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64]
        h = self.L.ref_test_matrix(kind.encode(), p0, p1, seed)
        if not h:
            raise ValueError(self.L.ref_error().decode())
        try:
            n, nnz = self.L.ref_csr_n(h), self.L.ref_csr_nnz(h)
            return (self._arr(self.L.ref_csr_ptr(h), n + 1, np.int64), self._arr(self.L.ref_csr_col(h), nnz, np.int32),
                    self._arr(self.L.ref_csr_val(h), nnz, np.float64))
        finally:
            self.L.ref_csr_free(h)

    def load_ordering(self, path, n):
        perm = np.zeros(max(n, 1), np.int32)
        cnt = self.L.ref_load_ordering(str(path).encode(), n, _p(perm, i32p), 0, C.cast(None, i32p))
        if cnt < 0:
            raise RuntimeError(self.L.ref_error().decode())
        b = np.zeros(cnt + 1, np.int32)
        self.L.ref_load_ordering(str(path).encode(), n, _p(perm, i32p), cnt, _p(b, i32p))
        return perm[:n], b

    def levelk(self, a, k):
        nnz = self.L.ref_levelk(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p), k,
                                C.cast(None, i64p), C.cast(None, i32p), 0)
        ptr = np.zeros(a.nrows + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        self.L.ref_levelk(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p), k, _p(ptr, i64p),
                          _p(col, i32p), nnz)
        return ptr, col

    def factor_serial(self, a, u):
        out = np.zeros(u.nnz(), np.float64)
        secs, row, piv = C.c_double(), C.c_int32(-1), C.c_double()
        st = self.L.ref_factor_serial(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p),
                                      _p(a.values, f64p), _p(u.row_ptr, i64p), _p(u.col_idx, i32p),
                                      _p(out, f64p), C.byref(secs), C.byref(row), C.byref(piv))
        return out, st, secs.value, row.value, piv.value

    def factor_by_blocks(self, a, u, bounds, workers=0, want_values=True):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        out = np.zeros(u.nnz(), np.float64) if want_values else None
        secs, bsecs, tasks = C.c_double(), C.c_double(), C.c_int64()
        row, piv = C.c_int32(-1), C.c_double()
        st = self.L.ref_factor_by_blocks(a.nrows, _p(a.row_ptr, i64p), _p(a.col_idx, i32p),
                                         _p(a.values, f64p), _p(u.row_ptr, i64p), _p(u.col_idx, i32p),
                                         b.size - 1, _p(b, i32p), workers,
                                         _p(out, f64p) if out is not None else C.cast(None, f64p),
                                         C.byref(secs), C.byref(bsecs), C.byref(tasks), C.byref(row),
                                         C.byref(piv))
        return out, st, secs.value, tasks.value, row.value, piv.value

    def export_dag(self, u, bounds):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        h = self.L.ref_export_dag(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), b.size - 1,
                                  _p(b, i32p))
        if not h:
            raise ValueError(self.L.ref_error().decode())
        try:
            nn, ne = self.L.ref_dag_nnodes(h), self.L.ref_dag_nedges(h)
            return (self._arr(self.L.ref_dag_kind(h), nn, np.int32),
                    self._arr(self.L.ref_dag_bi(h), nn, np.int32),
                    self._arr(self.L.ref_dag_bj(h), nn, np.int32),
                    self._arr(self.L.ref_dag_from(h), ne, np.int32),
                    self._arr(self.L.ref_dag_to(h), ne, np.int32))
        finally:
            self.L.ref_dag_free(h)

    def blocks(self, u, bounds):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        nb = self.L.ref_blocks(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), b.size - 1,
                               _p(b, i32p), C.cast(None, i64p), C.cast(None, i32p), 0)
        bp = np.zeros(b.size, np.int64)
        bc = np.zeros(nb, np.int32)
        self.L.ref_blocks(u.nrows, _p(u.row_ptr, i64p), _p(u.col_idx, i32p), b.size - 1, _p(b, i32p),
                          _p(bp, i64p), _p(bc, i32p), nb)
        return bp, bc


def emulate_plan(plan) -> np.ndarray:
    """Sequential host replay of the device algorithm over a plan's tables.

    Tasks in generation order; items in order; sources in order; for every
    source entry the product is subtracted from the matching target slot
    (absent columns dropped); Chol rows take sqrt/scale, Trsm rows divide by
    U(t,t). This checks the flattener's work tables without a GPU; it is
    slow and meant for small matrices only.
    """
    T = plan.tables()
    vals = T["values"].copy()
    cols = T["cols"]
    items, srcs = T["item"], T["src"]
    for rec in T["task"]:
        kind, _, ib, ie = rec[0], rec[1], rec[2], rec[3]
        for it in range(ib, ie):
            tb, te, local, dpos, sb_, se_ = items[it][:6]
            tcols = cols[tb:te]
            tv = vals[tb:te].copy()
            for s in range(sb_, se_):
                _, pos_rt, sb, se = srcs[s]
                v1 = vals[pos_rt]
                for pos in range(sb, se):
                    k = int(np.searchsorted(tcols, cols[pos]))
                    if k < len(tcols) and tcols[k] == cols[pos]:
                        tv[k] = tv[k] - v1 * vals[pos]
            if kind == 0:
                d = np.sqrt(tv[0])
                tv[1:] = tv[1:] / d
                tv[0] = d
            elif kind == 1:
                tv = tv / vals[dpos]
            vals[tb:te] = tv
    return vals


def emulate_program(plan) -> np.ndarray:
    """Sequential host replay of the update-program mode (small matrices)."""
    T = plan.tables()
    vals = T["values"].copy()
    srec, upd = T["slot_rec"], T["upd"]
    items = T["item"]
    for rec in T["task"]:
        kind, ib, ie = rec[0], rec[2], rec[3]
        for it in range(ib, ie):
            tb, te, _, dpos, _, _, soff, _ = items[it]
            L = te - tb
            tv = vals[tb:te].copy()
            for k in range(L):
                ub, ue, m0, o0 = srec[soff + k]
                assert ub == ue or (upd[ub][0] == m0 and upd[ub][1] == o0)
                for u in range(ub, ue):
                    m, o = upd[u]
                    tv[k] = tv[k] - vals[m] * vals[o]
            if kind == 0:
                d = np.sqrt(tv[0])
                tv[1:] = tv[1:] / d
                tv[0] = d
            elif kind == 1:
                tv = tv / vals[dpos]
            vals[tb:te] = tv
    return vals


def flow_programs(row_ptr, cols):
    """CPU restatement of the device program builder (flow_program.cu): per
    coordinate (t, c) of U, the (m, o) positions of U(r,t), U(r,c) over the
    rows r < t holding both, ascending r (the per-coordinate order of
    factor_serial, factorize.hpp:113-123). Returns (slot [nnz, 4] = {u_b,
    u_e, m0, o0}, upd [k, 2]). Pure Python: small matrices only."""
    row_ptr = np.asarray(row_ptr, np.int64)
    cols = np.asarray(cols, np.int64)
    n, nnz = len(row_ptr) - 1, len(cols)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    off = np.ones(nnz, bool)
    off[row_ptr[:-1]] = False
    m_all = np.flatnonzero(off)
    m_all = m_all[np.argsort(cols[m_all], kind="stable")]  # by column, rows ascending
    col_ptr = np.searchsorted(cols[m_all], np.arange(n + 1))
    progs = [[] for _ in range(nnz)]
    for t in range(n):
        tb, te = int(row_ptr[t]), int(row_ptr[t + 1])
        where = {int(c): tb + j for j, c in enumerate(cols[tb:te])}
        for m in m_all[col_ptr[t]:col_ptr[t + 1]]:
            r = rows[m]
            for q in range(int(m), int(row_ptr[r + 1])):
                x = where.get(int(cols[q]))
                if x is not None:
                    progs[x].append((int(m), q))
    cnt = np.array([len(p) for p in progs], np.int64)
    ub = np.concatenate([[0], np.cumsum(cnt)])
    slot = np.zeros((nnz, 4), np.int32)
    slot[:, 0], slot[:, 1] = ub[:-1], ub[1:]
    upd = np.array([mo for p in progs for mo in p], np.int32).reshape(-1, 2)
    has = cnt > 0
    slot[has, 2:] = upd[ub[:-1][has]]
    return slot, upd


def emulate_flow(rec, values, slot, upd, order=None) -> np.ndarray:
    """Replay of the value-flow schedule: rows of `rec` ({tb, L | kind << 30,
    dpos, t}) in `order` (default: schedule order), each coordinate taking its
    program's products in order; a read of a value not yet written fails."""
    out = np.full(len(values), np.nan)
    done = np.zeros(len(values), bool)
    for q in (range(len(rec)) if order is None else order):
        tb, lk, dpos, _ = (int(x) for x in rec[q])
        L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 1
        v = values[tb:tb + L].copy()
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
