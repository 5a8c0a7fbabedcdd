"""Python mirror of the reference's factorization interface, over the C ABI.

Names follow the reference (`taskchol`, /root/reference/proj/include):
``CsrMatrix``, ``RangeList``, ``FillPattern``, ``FactorStats``,
``FactorResult``, ``BreakdownError``, ``analyze``, ``export_task_dag`` and
the drop-in ``factor_by_blocks_gpu`` (the GPU replacement of
``factor_by_blocks(a_permuted, fp, ranges, policy)``, factorize.hpp:134-137).
Every numeric call runs on the GPU through libtacho_b200.so; nothing here
computes a factor on the CPU.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N

KIND_NAMES = ("CHOL", "TRSM", "HERK", "GEMM")


class BreakdownError(RuntimeError):
    """Non-positive pivot (reference kernels.hpp:21-36)."""

    def __init__(self, row: int, pivot: float, msg: str = ""):
        super().__init__(msg or f"factorization breakdown at row {row}: pivot {pivot} is not positive")
        self.row = row
        self.pivot = pivot


class SchedulerError(RuntimeError):
    """Stalled task graph (reference scheduler.hpp:298-309); here the device watchdog."""


class DeviceError(RuntimeError):
    """CUDA runtime failure inside the C ABI."""


@dataclass
class CsrMatrix:
    nrows: int
    ncols: int
    row_ptr: np.ndarray  # int64, nrows + 1
    col_idx: np.ndarray  # int32
    values: np.ndarray   # float64

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def view(self) -> N.CsrView:
        v = N.CsrView()
        v.n = self.nrows
        v.nnz = self.nnz()
        v.row_ptr = self.row_ptr.ctypes.data_as(N.i64p)
        v.col_idx = self.col_idx.ctypes.data_as(N.i32p)
        vals = self.values
        if vals.ndim == 1 and vals.size > 1 and vals.strides[0] == 0:
            # a pattern's broadcast 1.0 values (levelk_pattern_gpu): dense only when C needs them
            dense = getattr(self, "_dense_values", None)
            if dense is None or dense.size != vals.size:
                dense = np.ascontiguousarray(vals)
                self._dense_values = dense
            vals = dense
        v.values = vals.ctypes.data_as(N.f64p)
        return v

    @staticmethod
    def from_arrays(n: int, row_ptr, col_idx, values=None) -> "CsrMatrix":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = (np.ones(ci.shape[0]) if values is None
              else np.ascontiguousarray(values, dtype=np.float64))
        return CsrMatrix(int(n), int(n), rp, ci, va)

    def at(self, i: int, j: int) -> float:
        b, e = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        k = b + int(np.searchsorted(self.col_idx[b:e], j))
        return float(self.values[k]) if k < e and self.col_idx[k] == j else 0.0

    def has_entry(self, i: int, j: int) -> bool:
        b, e = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        k = b + int(np.searchsorted(self.col_idx[b:e], j))
        return k < e and self.col_idx[k] == j


@dataclass
class RangeList:
    bounds: np.ndarray  # int32, count + 1 ascending row bounds

    @staticmethod
    def from_ranges(ranges: List[Tuple[int, int]]) -> "RangeList":
        if not ranges:
            return RangeList(np.zeros(1, dtype=np.int32))
        b = [ranges[0][0]] + [r[1] for r in ranges]
        # keep malformed lists (gaps, inversions) visible to the validator
        if any(ranges[k][0] != ranges[k - 1][1] for k in range(1, len(ranges))):
            raise ValueError("ranges not contiguous")
        return RangeList(np.asarray(b, dtype=np.int32))

    def count(self) -> int:
        return int(self.bounds.shape[0]) - 1

    @property
    def ranges(self) -> List[Tuple[int, int]]:
        return [(int(self.bounds[k]), int(self.bounds[k + 1])) for k in range(self.count())]


@dataclass
class FillPattern:
    pattern: CsrMatrix
    level_cap: int = 0
    nnz_triu_input: int = 0


@dataclass
class Analysis:
    perm: np.ndarray
    iperm: np.ndarray
    ranges: RangeList
    a_permuted: CsrMatrix
    pattern: FillPattern
    ordering_seconds: float = 0.0
    symbolic_seconds: float = 0.0
    # ND subtree row spans per depth (0..6): {depth: (lo, hi)}; rows outside
    # every span at a depth are the separators above it
    subtree_spans: Optional[dict] = None

    def subtree_owners(self, nparts: int, separators=0) -> np.ndarray:
        """Owner part of every row for a sharded run over `nparts` (a power of
        two): the depth-log2(nparts) subtrees in order; the separators above
        them to part `separators` (an extra part when it equals nparts), or
        with separators="spread" each separator to the middle part among the
        parts its subtree covers (depth 0 -> part N/2, depth 1 -> N/4 and 3N/4,
        ...), so no part holds more than one separator and the critical
        separator chain crosses GPUs once per ND level (ordering.hpp:68-86)."""
        depth = max(0, int(nparts).bit_length() - 1)
        if 1 << depth != nparts or depth not in (self.subtree_spans or {}):
            raise ValueError("subtree_owners: nparts must be a power of two up to 64")
        spread = separators == "spread"
        lo, hi = self.subtree_spans[depth]
        owners = np.full(self.perm.shape[0], -1 if spread else separators, dtype=np.int32)
        # more subtrees than parts (nodes with several children): contiguous groups
        for i, (a, b) in enumerate(zip(lo, hi)):
            owners[a:b] = i * nparts // len(lo)
        if spread:
            for d in range(depth - 1, -1, -1):  # deeper separators first
                for a, b in zip(*self.subtree_spans[d]):
                    seg = owners[a:b]
                    parts = np.unique(seg[seg >= 0])
                    seg[seg < 0] = parts[len(parts) // 2] if len(parts) else 0
            owners[owners < 0] = 0
        return owners


@dataclass
class FactorStats:
    """Reference FactorStats (factorize.hpp:37-54) plus device figures."""
    ordering_seconds: float = 0.0
    symbolic_seconds: float = 0.0
    block_build_seconds: float = 0.0
    numeric_seconds: float = 0.0
    chol_tasks: int = 0
    trsm_tasks: int = 0
    herk_tasks: int = 0
    gemm_tasks: int = 0
    workers: int = 0
    backend: str = "gpu"
    nnz_u: int = 0
    relative_overhead: Optional[float] = None
    device_ms: float = 0.0
    plan_seconds: float = 0.0
    grid_ctas: int = 0
    threads_per_cta: int = 0

    def total_tasks(self) -> int:
        return self.chol_tasks + self.trsm_tasks + self.herk_tasks + self.gemm_tasks


@dataclass
class FactorResult:
    factor: CsrMatrix
    stats: FactorStats


@dataclass
class TaskDag:
    """Static DAG in generation order (reference factorize.hpp:240-302)."""
    kind: np.ndarray
    block_row: np.ndarray
    block_col: np.ndarray
    edge_from: np.ndarray
    edge_to: np.ndarray

    @property
    def labels(self) -> List[str]:
        return [f"{KIND_NAMES[k]}({i},{j})" for k, i, j in zip(self.kind, self.block_row, self.block_col)]

    def to_dot(self) -> str:
        out = ["digraph tasks {"]
        out += [f'  t{i} [label="{lab}"];' for i, lab in enumerate(self.labels)]
        out += [f"  t{a} -> t{b};" for a, b in zip(self.edge_from, self.edge_to)]
        return "\n".join(out) + "\n}\n"


def _lib():
    return N.load()


def _copy(ptr, n, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True)


def _from_view(v: N.CsrView) -> CsrMatrix:
    n = int(v.n)
    return CsrMatrix(n, n, _copy(v.row_ptr, n + 1, np.int64), _copy(v.col_idx, v.nnz, np.int32),
                     _copy(v.values, v.nnz, np.float64))


# ------------------------------------------------------------------ inputs --

def generate(kind: str, p0: int, p1: int = 0, seed: int = 0) -> CsrMatrix:
    """Seeded synthetic matrices; see tacho_b200.h."""
    lib = _lib()
    h = lib.tch_generate(kind.encode(), int(p0), int(p1), int(seed))
    if not h:
        raise ValueError(lib.tch_error().decode())
    try:
        v = N.CsrView()
        lib.tch_matrix_view(h, C.byref(v))
        return _from_view(v)
    finally:
        lib.tch_matrix_free(h)


CONFIGS = {
    # name: (generator kind, p0, p1, seed, level)  — BASELINE.json configs
    "c1": ("grid2d", 100, 100, 0, 0),
    "c2": ("lap7", 64, 0, 0, 1),
    "c3": ("stencil27", 48, 0, 1, 2),
    "c4": ("elasticity", 40, 0, 1, 0),
    "c5": ("diffusion", 32, 1000, 1, 1),   # batch member b uses seed b + 1
    "c6": ("lap7", 128, 0, 0, 1),
}


def config_matrix(name: str, member: int = 0) -> Tuple[CsrMatrix, int]:
    kind, p0, p1, seed, level = CONFIGS[name]
    if name == "c5":
        seed = member + 1
    return generate(kind, p0, p1, seed), level


def analyze(a: CsrMatrix, level: int = 0, treecut: int = 0, leaf_size: int = 64,
            max_depth: int = 100, threads: int = 0, ordering_path: Optional[str] = None) -> Analysis:
    """ND ordering -> prune -> PᵀAP -> level-k pattern (reference pipeline.hpp:35-55);
    with ``ordering_path`` the ordering and ranges are imported instead
    (load_ordering, pipeline.hpp:39-44)."""
    lib = _lib()
    m = lib.tch_matrix_from_csr(C.byref(a.view()))
    if not m:
        raise ValueError(lib.tch_error().decode())
    try:
        if ordering_path is not None:
            perm_in, b_in = load_ordering(ordering_path, a.nrows)
            h = lib.tch_analyze_with_ordering(m, perm_in.ctypes.data_as(N.i32p), int(b_in.shape[0]) - 1,
                                              b_in.ctypes.data_as(N.i32p), level, threads)
        else:
            h = lib.tch_analyze(m, level, treecut, leaf_size, max_depth, threads)
        if not h:
            raise ValueError(lib.tch_error().decode())
        try:
            perm, iperm = N.i32p(), N.i32p()
            lib.tch_analysis_perm(h, C.byref(perm), C.byref(iperm))
            bounds = N.i32p()
            cnt = lib.tch_analysis_ranges(h, C.byref(bounds))
            ap, pat = N.CsrView(), N.CsrView()
            lib.tch_analysis_permuted(h, C.byref(ap))
            lib.tch_analysis_pattern(h, C.byref(pat))
            t_ord, t_sym = C.c_double(), C.c_double()
            lib.tch_analysis_times(h, C.byref(t_ord), C.byref(t_sym))
            a_perm = _from_view(ap)
            pattern = _from_view(pat)
            nnz_triu = int(np.count_nonzero(
                a_perm.col_idx >= np.repeat(np.arange(a_perm.nrows, dtype=np.int64),
                                            np.diff(a_perm.row_ptr))))
            spans = {}
            for depth in range(7):
                k = lib.tch_analysis_subtrees(h, depth, 0, None, None)
                lo = np.zeros(max(k, 1), np.int32)
                hi = np.zeros(max(k, 1), np.int32)
                lib.tch_analysis_subtrees(h, depth, k, lo.ctypes.data_as(N.i32p), hi.ctypes.data_as(N.i32p))
                spans[depth] = (lo[:k].copy(), hi[:k].copy())
            return Analysis(perm=_copy(perm, a.nrows, np.int32), iperm=_copy(iperm, a.nrows, np.int32),
                            ranges=RangeList(_copy(bounds, cnt + 1, np.int32)), a_permuted=a_perm,
                            pattern=FillPattern(pattern, level, nnz_triu),
                            ordering_seconds=t_ord.value, symbolic_seconds=t_sym.value,
                            subtree_spans=spans)
        finally:
            lib.tch_analysis_free(h)
    finally:
        lib.tch_matrix_free(m)


class MatrixMarketError(RuntimeError):
    """Reference MatrixMarketError (matrix_market.hpp:24-27)."""


def load_matrix_market(path: str) -> CsrMatrix:
    """Reference load_matrix_market (matrix_market.hpp:61-157)."""
    lib = _lib()
    h = lib.tch_load_matrix_market(str(path).encode())
    if not h:
        raise MatrixMarketError(lib.tch_error().decode())
    try:
        v = N.CsrView()
        lib.tch_matrix_view(h, C.byref(v))
        return _from_view(v)
    finally:
        lib.tch_matrix_free(h)


def write_matrix_market(m: CsrMatrix, path: str) -> None:
    """Reference write_matrix_market (matrix_market.hpp:159-176): the same bytes."""
    lib = _lib()
    if lib.tch_write_matrix_market(C.byref(m.view()), str(path).encode()) != N.TCG_OK:
        raise MatrixMarketError(lib.tch_error().decode())


def load_ordering(path: str, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Reference load_ordering (ordering.hpp:355-399): (perm, range bounds)."""
    lib = _lib()
    perm = np.zeros(max(n, 1), np.int32)
    cnt = lib.tch_load_ordering(str(path).encode(), n, perm.ctypes.data_as(N.i32p), 0, None)
    if cnt < 0:
        raise RuntimeError(lib.tch_error().decode())
    bounds = np.zeros(cnt + 1, np.int32)
    lib.tch_load_ordering(str(path).encode(), n, perm.ctypes.data_as(N.i32p), cnt, bounds.ctypes.data_as(N.i32p))
    return perm[:n].copy(), bounds


def levelk_pattern(a_permuted: CsrMatrix, level: int, threads: int = 0) -> FillPattern:
    lib = _lib()
    m = lib.tch_matrix_from_csr(C.byref(a_permuted.view()))
    if not m:
        raise ValueError(lib.tch_error().decode())
    try:
        h = lib.tch_levelk_pattern(m, level, threads)
        if not h:
            raise ValueError(lib.tch_error().decode())
        try:
            v = N.CsrView()
            lib.tch_matrix_view(h, C.byref(v))
            return FillPattern(_from_view(v), level)
        finally:
            lib.tch_matrix_free(h)
    finally:
        lib.tch_matrix_free(m)


@dataclass
class SymbolicStats:
    device_ms: float
    host_ms: float
    nnz_u: int
    nnz_triu_input: int
    slow_rows: int
    tier2_rows: int
    kernel_launches: int
    grid_ctas: int
    single_pass: int = 1


class GpuSymbolic:
    """levelk_pattern_bfs (reference symbolic.hpp:57-120) on the device, one
    warp per source row: upload PᵀAP's pattern once, compute the level-k
    pattern for any k, download it as the reference's FillPattern."""

    def __init__(self, a_permuted: CsrMatrix, device: int = 0):
        self._lib = _lib()
        h = C.c_void_p()
        if self._lib.tcg_sym_create(device, C.byref(h)) != N.TCG_OK:
            raise DeviceError("tcg_sym_create failed (no CUDA device?)")
        self.h = h
        self.upload(a_permuted)

    def upload(self, a_permuted: CsrMatrix):
        """Copy PᵀAP's pattern to the device (buffers are reused when large enough)."""
        self.a = a_permuted
        self._check(self._lib.tcg_sym_upload(self.h, C.byref(a_permuted.view())))

    def _check(self, st):
        if st == N.TCG_OK:
            return
        msg = self._lib.tcg_sym_error(self.h).decode()
        if st == N.TCG_INVALID:
            raise ValueError(msg)
        raise DeviceError(msg)

    def levelk(self, level: int, all_slow: bool = False) -> Tuple[FillPattern, SymbolicStats]:
        s = N.SymStats()
        self._check(self._lib.tcg_sym_levelk(self.h, level, N.TCG_SYM_ALL_SLOW if all_slow else 0, C.byref(s)))
        n, nnz = self.a.nrows, int(s.nnz_u)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int32)
        self._check(self._lib.tcg_sym_download(self.h, rp.ctypes.data_as(N.i64p), ci.ctypes.data_as(N.i32p)))
        # the pattern's values are 1.0 and unused (symbolic.hpp:118): a read-only broadcast,
        # made dense only if the pattern is handed to C as a matrix (CsrMatrix.view)
        pat = CsrMatrix(n, n, rp, ci[:nnz], np.broadcast_to(np.float64(1.0), (nnz,)))
        st = SymbolicStats(s.device_ms, s.host_ms, int(s.nnz_u), int(s.nnz_triu_input), int(s.slow_rows), int(s.tier2_rows),
                           int(s.kernel_launches), int(s.grid_ctas), int(s.single_pass))
        return FillPattern(pat, level, int(s.nnz_triu_input)), st

    def close(self):
        if self.h:
            self._lib.tcg_sym_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def levelk_pattern_gpu(a_permuted: CsrMatrix, level: int, device: int = 0) -> FillPattern:
    """The level-k fill pattern computed on the GPU; same arrays as
    levelk_pattern / the reference's levelk_pattern_bfs."""
    g = GpuSymbolic(a_permuted, device)
    try:
        return g.levelk(level)[0]
    finally:
        g.close()


def init_factor_values(a_permuted: CsrMatrix, fp: FillPattern) -> np.ndarray:
    lib = _lib()
    out = np.zeros(fp.pattern.nnz(), dtype=np.float64)
    st = lib.tch_init_values(C.byref(a_permuted.view()), C.byref(fp.pattern.view()),
                             out.ctypes.data_as(N.f64p))
    if st != N.TCG_OK:
        raise ValueError(lib.tch_error().decode())
    return out


# -------------------------------------------------------------------- plan --

class Plan:
    """Host-flattened DAG + work tables (tcg_plan)."""

    def __init__(self, a_permuted: CsrMatrix, fp: FillPattern, ranges: RangeList):
        lib = _lib()
        self._lib = lib
        h = C.c_void_p()
        b = np.ascontiguousarray(ranges.bounds, dtype=np.int32)
        t0 = time.perf_counter()
        st = lib.tcg_plan_build(C.byref(a_permuted.view()), C.byref(fp.pattern.view()),
                                ranges.count(), b.ctypes.data_as(N.i32p), C.byref(h))
        self.build_seconds = time.perf_counter() - t0
        if st != N.TCG_OK:
            msg = lib.tcg_plan_error().decode()
            if "diagonal block missing" in msg:
                raise RuntimeError(msg)  # reference: std::logic_error
            raise ValueError(msg)
        self.handle = h
        self.n = a_permuted.nrows
        self.pattern = fp.pattern

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self._lib.tcg_plan_free(h)
            self.handle = None

    def stats(self) -> N.PlanStats:
        s = N.PlanStats()
        self._lib.tcg_plan_get_stats(self.handle, C.byref(s))
        return s

    def problem(self) -> N.Problem:
        """The upload image: the value-flow schedule (update programs built on the
        device), plus the task executors' tables once the plan is expanded."""
        p = N.Problem()
        self._lib.tcg_plan_problem(self.handle, C.byref(p))
        return p

    def expand(self) -> "Plan":
        """Build the task-DAG plan (the reference's generation walk, flattened)."""
        if self._lib.tcg_plan_expand(self.handle) != N.TCG_OK:
            raise ValueError(self._lib.tcg_plan_error().decode())
        return self

    def schedule(self) -> "Plan":
        """The value-flow schedule on the host (tcg_plan_schedule); without it the device
        builds the schedule at upload."""
        if self._lib.tcg_plan_schedule(self.handle) != N.TCG_OK:
            raise ValueError(self._lib.tcg_plan_error().decode())
        return self

    def flow_tables(self) -> dict:
        """The lean value-flow plan's host arrays (the schedule, U, initial values)."""
        self.schedule()
        p = self.problem()
        return {
            "flow_rec": _copy(p.flow_rec, 4 * p.nflow, np.int32).reshape(-1, 4),
            "flow_item": _copy(p.flow_item, p.nflow, np.int32),
            "row_ptr": _copy(p.u_row_ptr, p.n + 1, np.int32),
            "a_map": _copy(p.a_map, p.nnz, np.int32) if p.a_map else np.zeros(0, np.int32),
            "values": _copy(p.values, p.nnz, np.float64),
            "cols": _copy(p.col_idx, p.nnz, np.int32),
        }

    def part_problem(self, nparts: int, owners: np.ndarray, part: int) -> N.Problem:
        """The rows of one part of a sharded run (tcg_plan_part_problem, mode 5)."""
        own = np.ascontiguousarray(owners, dtype=np.int32)
        p = N.Problem()
        remote = C.c_int64()
        rc = self._lib.tcg_plan_part_problem(self.handle, nparts, own.ctypes.data_as(N.i32p), part,
                                             C.byref(p), C.byref(remote))
        if rc != 0:
            raise ValueError(self._lib.tcg_plan_error().decode())
        p.remote_operands = remote.value  # python-side annotation
        return p

    def dag(self) -> TaskDag:
        nn, ne = C.c_int64(), C.c_int64()
        k, bi, bj, ef, et = N.i32p(), N.i32p(), N.i32p(), N.i32p(), N.i32p()
        self._lib.tcg_plan_dag(self.handle, C.byref(nn), C.byref(k), C.byref(bi), C.byref(bj),
                               C.byref(ne), C.byref(ef), C.byref(et))
        return TaskDag(_copy(k, nn.value, np.int32), _copy(bi, nn.value, np.int32),
                       _copy(bj, nn.value, np.int32), _copy(ef, ne.value, np.int32),
                       _copy(et, ne.value, np.int32))

    def blocks(self) -> Tuple[np.ndarray, np.ndarray]:
        m, nb = C.c_int32(), C.c_int64()
        bp, bc = N.i64p(), N.i32p()
        self._lib.tcg_plan_blocks(self.handle, C.byref(m), C.byref(bp), C.byref(nb), C.byref(bc))
        return _copy(bp, m.value + 1, np.int64), _copy(bc, nb.value, np.int32)

    def tables(self) -> dict:
        """Copies of the task-DAG plan's tables (for host-side inspection in
        tests; expands the plan and builds the host schedule)."""
        self.expand()
        self.schedule()
        p = self.problem()
        return {
            "task": _copy(p.task_rec, 12 * p.ntasks, np.int32).reshape(-1, 12),
            "item": _copy(p.item_rec, 8 * p.nitems, np.int32).reshape(-1, 8),
            "src": _copy(p.src_rec, 4 * p.nsources, np.int32).reshape(-1, 4),
            "succ": _copy(p.succ, p.nedges, np.int32),
            "indeg": _copy(p.indeg, p.ntasks, np.int32),
            "roots": _copy(p.roots, p.nroots, np.int32),
            "values": _copy(p.values, p.nnz, np.float64),
            "cols": _copy(p.col_idx, p.nnz, np.int32),
            "slot_rec": _copy(p.slot_rec, 4 * p.nslots, np.int32).reshape(-1, 4),
            "upd": _copy(p.upd, 2 * p.nupdates, np.int32).reshape(-1, 2),
            "flow_rec": _copy(p.flow_rec, 4 * p.nflow, np.int32).reshape(-1, 4),
            "flow_item": _copy(p.flow_item, p.nflow, np.int32),
            "a_map": _copy(p.a_map, p.nnz, np.int32) if p.a_map else np.zeros(0, np.int32),
        }


def export_task_dag(fp: FillPattern, ranges: RangeList) -> TaskDag:
    """Dry-run DAG (no execution), as export_task_dag (factorize.hpp:260-302)."""
    a = CsrMatrix(fp.pattern.nrows, fp.pattern.ncols, fp.pattern.row_ptr, fp.pattern.col_idx,
                  np.ones(fp.pattern.nnz()))
    return Plan(a, fp, ranges).dag()


# ------------------------------------------------------------------ device --

@dataclass
class GpuOptions:
    device: int = 0
    threads_per_cta: int = 0
    ctas_per_sm: int = 0
    staging_cap: int = 0
    timeout_s: float = 0.0
    trace: bool = False
    mode: int = 0  # 0 auto (5); task DAG (expands the plan): 1 device merge, 2 update programs;
    #                5 static value flow (finalising rows, the values are their own flags)
    lanes_per_row: int = 0  # ignored (ABI field): mode 5 picks whole warps or warp groups per row


class GpuFactorizer:
    """A device context holding one uploaded plan (tcg_ctx)."""

    def __init__(self, plan: Plan, options: Optional[GpuOptions] = None, problem: Optional[N.Problem] = None):
        self.opt = options or GpuOptions()
        lib = _lib()
        self._lib = lib
        h = C.c_void_p()
        st = lib.tcg_create(self.opt.device, C.byref(h))
        if st != N.TCG_OK:
            raise DeviceError(lib.tcg_last_error(None).decode())
        self.ctx = h
        o = N.Options(self.opt.threads_per_cta, self.opt.ctas_per_sm, self.opt.staging_cap,
                      self.opt.timeout_s, 1 if self.opt.trace else 0, self.opt.mode,
                      self.opt.lanes_per_row)
        self._check(lib.tcg_set_options(self.ctx, C.byref(o)))
        self.plan = plan
        if problem is None and self.opt.mode not in (0, 5):
            plan.expand()  # the task executors run the task-DAG plan's tables
        self._problem = problem if problem is not None else plan.problem()
        self.nnz = int(self._problem.nnz)
        self.ntasks = int(self._problem.ntasks)
        self._ntab = self.ntasks if self._problem.task_rec else 0
        self._check(lib.tcg_upload(self.ctx, C.byref(self._problem)))
        self.last = N.Stats()

    def close(self):
        if getattr(self, "ctx", None):
            self._lib.tcg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def _check(self, st):
        if st == N.TCG_OK:
            return
        msg = self._lib.tcg_last_error(self.ctx).decode()
        if st == N.TCG_BREAKDOWN:
            raise BreakdownError(self.last.breakdown_row, self.last.breakdown_pivot, msg)
        if st == N.TCG_TIMEOUT:
            raise SchedulerError(msg)
        if st == N.TCG_INVALID:
            raise ValueError(msg)
        raise DeviceError(msg)

    def set_values(self, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self._lib.tcg_set_values(self.ctx, v.ctypes.data_as(N.f64p)))

    def set_values_ptr(self, host_ptr: int):
        self._check(self._lib.tcg_set_values(self.ctx, C.cast(C.c_void_p(host_ptr), N.f64p)))

    def restore(self):
        self._check(self._lib.tcg_restore(self.ctx))

    def factor(self) -> N.Stats:
        self.last = N.Stats()
        st = self._lib.tcg_factor(self.ctx, C.byref(self.last))
        self._check(st)
        return self.last

    def factor_host_a_ptr(self, a_ptr: int, out_ptr: int) -> N.Stats:
        """PᵀAP's values in (nnz(A) x batch doubles, a_permuted's CSR order),
        factor out (nnz x batch), through tcg_factor_host_a: upload, device
        init_factor_values, factor, download in one call. Pinned memory."""
        self.last = N.Stats()
        st = self._lib.tcg_factor_host_a(self.ctx, C.cast(C.c_void_p(a_ptr), N.f64p),
                                         C.cast(C.c_void_p(out_ptr), N.f64p), C.byref(self.last))
        self._check(st)
        return self.last

    def factor_host_a(self, a_values: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """factor_host_a_ptr with numpy arrays (one member: a_permuted.values)."""
        v = np.ascontiguousarray(a_values, dtype=np.float64)
        if out is None:
            out = np.empty(self.nnz * max(1, v.size // max(1, self._problem.nnz_a)), np.float64)
        self.factor_host_a_ptr(v.ctypes.data, out.ctypes.data)
        return out

    def factor_host_ptr(self, in_ptr: int, out_ptr: int) -> N.Stats:
        """Host buffers in, factor out (tcg_factor_host): upload, factor and
        download on one stream. Pointers to nnz x batch doubles (pinned)."""
        self.last = N.Stats()
        st = self._lib.tcg_factor_host(self.ctx, C.cast(C.c_void_p(in_ptr), N.f64p),
                                       C.cast(C.c_void_p(out_ptr), N.f64p), C.byref(self.last))
        self._check(st)
        return self.last

    def factor_host(self, values: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64)
        if out is None:
            out = np.empty_like(v)
        self.factor_host_ptr(v.ctypes.data, out.ctypes.data)
        return out

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.nnz, dtype=np.float64)
        self._check(self._lib.tcg_download(self.ctx, out.ctypes.data_as(N.f64p)))
        return out

    def download_ptr(self, host_ptr: int):
        self._check(self._lib.tcg_download(self.ctx, C.cast(C.c_void_p(host_ptr), N.f64p)))

    # ---- batch of value sets sharing the pattern (mode 5; C5) ----
    def set_batch(self, values: np.ndarray):
        """values: [nbatch, nnz] initial U values, one row per member."""
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.ndim != 2 or v.shape[1] != self.nnz:
            raise ValueError(f"batch values must be [nbatch, {self.nnz}]")
        self._check(self._lib.tcg_set_batch(self.ctx, v.shape[0], v.ctypes.data_as(N.f64p)))

    def set_a_values(self, a_values: np.ndarray):
        """init_factor_values on the device: PᵀAP's values (a_permuted CSR order),
        one row per member ([nbatch, nnz_A] or [nnz_A])."""
        v = np.ascontiguousarray(a_values, dtype=np.float64)
        nb = 1 if v.ndim == 1 else v.shape[0]
        self._check(self._lib.tcg_set_a_values(self.ctx, nb, v.ctypes.data_as(N.f64p)))

    def set_batch_values_ptr(self, host_ptr: int):
        self._check(self._lib.tcg_set_batch_values(self.ctx, C.cast(C.c_void_p(host_ptr), N.f64p)))

    @property
    def batch(self) -> int:
        return int(self._lib.tcg_batch_size(self.ctx))

    def download_batch(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.batch, self.nnz), dtype=np.float64)
        self._check(self._lib.tcg_download_batch(self.ctx, out.ctypes.data_as(N.f64p)))
        return out

    def download_batch_ptr(self, host_ptr: int):
        self._check(self._lib.tcg_download_batch(self.ctx, C.cast(C.c_void_p(host_ptr), N.f64p)))

    def batch_breakdown(self):
        """Per member of the last factor: (row or -1, pivot)."""
        b = self.batch
        rows = np.zeros(b, np.int32)
        piv = np.zeros(b, np.float64)
        self._check(self._lib.tcg_batch_breakdown(self.ctx, rows.ctypes.data_as(N.i32p),
                                                  piv.ctypes.data_as(N.f64p)))
        return rows, piv

    def trace(self):
        """(task stamps [ntasks, 2], item stamps [nitems, 4]) of the last traced factor."""
        ni = max(int(self._problem.nitems), int(self._problem.nflow))
        out = np.zeros(2 * self._ntab + 4 * ni, dtype=np.uint64)
        self._check(self._lib.tcg_download_trace(self.ctx, out.ctypes.data_as(N.u64p)))
        return out[:2 * self._ntab].reshape(-1, 2), out[2 * self._ntab:].reshape(-1, 4)

    # ---- sharded runs (C6): other parts' U through peer memory ----
    def factor_phase(self, phase: int) -> N.Stats:
        """1: reset the output; 2: launch (after every part finished phase 1)."""
        self.last = N.Stats()
        self._check(self._lib.tcg_factor_phase(self.ctx, phase, C.byref(self.last)))
        return self.last

    def flow_records(self):
        """The schedule the device runs: (records [nflow, 4], unit ids, depth built on the device)."""
        n = int(self._problem.nflow)
        rec = np.zeros((n, 4), np.int32)
        item = np.zeros(n, np.int32)
        depth = C.c_int32()
        self._check(self._lib.tcg_flow_records(self.ctx, rec.ctypes.data_as(N.i32p), item.ctypes.data_as(N.i32p),
                                               C.byref(depth)))
        return rec, item, int(depth.value)

    def flow_programs(self):
        """(slot [nnz, 4], upd [n, 2], build ms) of the uploaded value-flow programs."""
        n, ms = C.c_int64(), C.c_double()
        self._check(self._lib.tcg_flow_programs(self.ctx, C.cast(None, N.i32p), C.cast(None, N.i32p),
                                                C.byref(n), C.byref(ms)))
        slot = np.zeros((self.nnz, 4), np.int32)
        upd = np.zeros((n.value, 2), np.int32)
        self._check(self._lib.tcg_flow_programs(self.ctx, slot.ctypes.data_as(N.i32p), upd.ctypes.data_as(N.i32p),
                                                C.byref(n), C.byref(ms)))
        return slot, upd, ms.value

    def values_device_ptr(self) -> int:
        d = N.f64p()
        n = C.c_int64()
        self._check(self._lib.tcg_device_values(self.ctx, C.byref(d), C.byref(n)))
        return C.cast(d, C.c_void_p).value or 0

    def set_peers(self, ptrs):
        arr = (C.c_uint64 * len(ptrs))(*[int(x) for x in ptrs])
        self._check(self._lib.tcg_set_peers(self.ctx, len(ptrs), arr))

    def ipc_handle(self):
        h = (C.c_char * 64)()
        off = C.c_int64()
        self._check(self._lib.tcg_ipc_values_handle(self.ctx, h, C.byref(off)))
        return bytes(h), off.value

    def ipc_open(self, handle: bytes, offset: int) -> int:
        h = (C.c_char * 64).from_buffer_copy(handle)
        ptr = C.c_uint64()
        self._check(self._lib.tcg_ipc_open(self.ctx, h, offset, C.byref(ptr)))
        return ptr.value

    def arena_bytes(self) -> int:
        return int(self._lib.tcg_arena_bytes(self.ctx))


@dataclass
class SolveStats:
    device_ms: float
    depth_forward: int
    depth_backward: int
    grid_ctas: int
    kernel_launches: int


class GpuTriSolve:
    """Triangular solves with the factor a GpuFactorizer holds (tcg_solve_*):
    ``apply(b)`` = (UᵀU)⁻¹ b, the IC(k) preconditioner apply; ``forward(b)``
    solves Uᵀ y = b, ``backward(y)`` solves U x = y. Fixed operation order
    (oracle.c orc_trisolve), bitwise reproducible."""

    def __init__(self, fz: "GpuFactorizer"):
        self._lib = _lib()
        self.fz = fz
        self.n = fz.plan.n
        h = C.c_void_p()
        st = self._lib.tcg_solve_create(fz.ctx, C.byref(fz.plan.pattern.view()), C.byref(h))
        if st != N.TCG_OK:
            raise (DeviceError if st == N.TCG_CUDA else ValueError)(
                self._lib.tcg_solve_error(h).decode() if h else "tcg_solve_create: invalid context or pattern")
        self.h = h
        self.last = N.SolveStats()

    def _run(self, b, which) -> np.ndarray:
        bb = np.ascontiguousarray(b, dtype=np.float64)
        if bb.shape != (self.n,):
            raise ValueError(f"expected a vector of {self.n} values")
        x = np.empty(self.n, np.float64)
        st = self._lib.tcg_solve_apply(self.h, bb.ctypes.data_as(N.f64p), x.ctypes.data_as(N.f64p), which,
                                       C.byref(self.last))
        if st != N.TCG_OK:
            msg = self._lib.tcg_solve_error(self.h).decode()
            raise (SchedulerError if st == N.TCG_TIMEOUT else ValueError if st == N.TCG_INVALID
                   else DeviceError)(msg)
        return x

    def apply(self, b) -> np.ndarray:
        return self._run(b, N.TCG_SOLVE_BOTH)

    def forward(self, b) -> np.ndarray:
        return self._run(b, N.TCG_SOLVE_FORWARD)

    def backward(self, y) -> np.ndarray:
        return self._run(y, N.TCG_SOLVE_BACKWARD)

    def apply_device_ptr(self, b_ptr: int, x_ptr: int, which: int = 3) -> SolveStats:
        """Device vectors (e.g. torch CUDA tensors' data_ptr()), on the context's stream."""
        st = self._lib.tcg_solve_apply_device(self.h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), which,
                                              C.byref(self.last))
        if st != N.TCG_OK:
            raise (SchedulerError if st == N.TCG_TIMEOUT else DeviceError)(self._lib.tcg_solve_error(self.h).decode())
        return self.stats()

    def apply_async_ptr(self, b_ptr: int, x_ptr: int, which: int = 3):
        """apply_device_ptr without the host wait; errors surface at sync()."""
        st = self._lib.tcg_solve_apply_async(self.h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), which)
        if st != N.TCG_OK:
            raise (ValueError if st == N.TCG_INVALID else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def sync(self):
        """Wait for the context's stream; raise SchedulerError if an apply's watchdog expired."""
        st = self._lib.tcg_solve_sync(self.h)
        if st != N.TCG_OK:
            raise (SchedulerError if st == N.TCG_TIMEOUT else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def apply_host_ptr(self, b_ptr: int, x_ptr: int, which: int = 3) -> SolveStats:
        """Host vectors by address (pinned memory for full PCIe speed)."""
        st = self._lib.tcg_solve_apply(self.h, C.cast(b_ptr, N.f64p), C.cast(x_ptr, N.f64p), which,
                                       C.byref(self.last))
        if st != N.TCG_OK:
            raise (SchedulerError if st == N.TCG_TIMEOUT else DeviceError)(self._lib.tcg_solve_error(self.h).decode())
        return self.stats()

    def set_matrix(self, a: CsrMatrix):
        """The system matrix (PᵀAP) for spmv_ptr, uploaded once."""
        st = self._lib.tcg_solve_set_matrix(self.h, C.byref(a.view()))
        if st != N.TCG_OK:
            raise (ValueError if st == N.TCG_INVALID else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def cg_step_ptr(self, x: int, r: int, p: int, ap: int, state: int, hist: int, it: int):
        """tcg_solve_cg_step on device vectors (asynchronous, the context's stream)."""
        st = self._lib.tcg_solve_cg_step(self.h, C.c_void_p(x), C.c_void_p(r), C.c_void_p(p), C.c_void_p(ap),
                                         C.c_void_p(state), C.c_void_p(hist), it)
        if st != N.TCG_OK:
            raise (ValueError if st == N.TCG_INVALID else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def cg_direction_ptr(self, r: int, z: int, p: int, state: int):
        """tcg_solve_cg_direction on device vectors (asynchronous, the context's stream)."""
        st = self._lib.tcg_solve_cg_direction(self.h, C.c_void_p(r), C.c_void_p(z), C.c_void_p(p),
                                              C.c_void_p(state))
        if st != N.TCG_OK:
            raise (ValueError if st == N.TCG_INVALID else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def spmv_ptr(self, x_ptr: int, y_ptr: int):
        """y = A x on device vectors, on the context's stream (asynchronous)."""
        st = self._lib.tcg_solve_spmv(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr))
        if st != N.TCG_OK:
            raise (ValueError if st == N.TCG_INVALID else DeviceError)(self._lib.tcg_solve_error(self.h).decode())

    def stream_ptr(self) -> int:
        out = C.c_void_p()
        if self._lib.tcg_solve_stream(self.h, C.byref(out)) != N.TCG_OK:
            raise ValueError("tcg_solve_stream failed")
        return int(out.value or 0)

    def stats(self) -> SolveStats:
        s = self.last
        return SolveStats(s.device_ms, int(s.depth_forward), int(s.depth_backward), int(s.grid_ctas),
                          int(s.kernel_launches))

    def close(self):
        if getattr(self, "h", None):
            self._lib.tcg_solve_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    relative_residual: float
    seconds: float


def pcg(solver: "GpuTriSolve", b, tol: float = 1e-8, maxit: int = 1000, precondition: bool = True,
        device: int = 0, check_every: int = 8) -> PcgResult:
    """Conjugate gradients on PᵀAP x = b on the GPU, preconditioned with the
    IC(k) factor the solver's context holds (z = (UᵀU)⁻¹ r through
    tcg_solve_apply_device) -- the caller of the factorization. The system
    matrix must be set (solver.set_matrix). Vectors and the dots live on the
    device (torch, on the context's stream); the applies are queued without a
    host wait (tcg_solve_apply_async).

    Converged means ‖r‖ <= tol·‖b‖. The test runs on the device: a 0/1 mask
    (1 until the first converged iteration) scales every later step, so x and
    r freeze at that iteration, and the host reads the residual history once
    every ``check_every`` iterations instead of syncing on each one. The
    iterates, the iteration count and x are the same for any check_every (at
    most check_every - 1 frozen iterations run after convergence)."""
    import torch
    if check_every < 1:
        raise ValueError("check_every must be >= 1")
    dev = torch.device("cuda", device)
    stream = torch.cuda.ExternalStream(solver.stream_ptr(), device=dev)
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        bd = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64)).to(dev, non_blocking=False)
        x = torch.zeros_like(bd)
        r = bd.clone()
        z = torch.empty_like(bd)
        ap = torch.empty_like(bd)

        def prec(src, dst):
            if precondition:
                solver.apply_async_ptr(src.data_ptr(), dst.data_ptr(), N.TCG_SOLVE_BOTH)
            else:
                dst.copy_(src)

        bnorm = float(torch.linalg.vector_norm(bd).item())
        if bnorm == 0.0:
            return PcgResult(np.zeros(bd.numel()), 0, True, 0.0, time.perf_counter() - t0)
        thr = tol * bnorm
        hist = torch.empty(max(maxit, 1), dtype=torch.float64, device=dev)
        prec(r, z)
        p = z.clone()
        # {rz, live, threshold} on the device: the vector updates are two fused kernels per
        # iteration (tcg_solve_cg_step / cg_direction, deterministic dots)
        state = torch.stack([torch.dot(r, z), torch.ones((), dtype=torch.float64, device=dev),
                             torch.full((), thr, dtype=torch.float64, device=dev)])
        done, it, rel, converged = 0, 0, 1.0, False
        while done < maxit and not converged:
            k = min(check_every, maxit - done)
            for _ in range(k):
                solver.spmv_ptr(p.data_ptr(), ap.data_ptr())
                # alpha = rz / (p.ap); where live: x += alpha p, r -= alpha ap (a frozen step
                # may carry 0/0); hist[done] = ||r||; live = 0 once ||r|| <= thr (NaN stays live)
                solver.cg_step_ptr(x.data_ptr(), r.data_ptr(), p.data_ptr(), ap.data_ptr(), state.data_ptr(),
                                   hist.data_ptr(), done)
                done += 1
                prec(r, z)
                solver.cg_direction_ptr(r.data_ptr(), z.data_ptr(), p.data_ptr(), state.data_ptr())
            h = hist[done - k:done].cpu().numpy()
            solver.sync()  # a watchdog expiry in any of the k applies raises here
            hit = np.nonzero(h <= thr)[0]
            if hit.size:
                it = done - k + int(hit[0]) + 1
                rel, converged = float(h[hit[0]]) / bnorm, True
            else:
                it, rel = done, float(h[-1]) / bnorm
        out = x.cpu().numpy()
    torch.cuda.synchronize(dev)
    return PcgResult(out, it, converged, rel, time.perf_counter() - t0)


def factor_by_blocks_gpu(a_permuted: CsrMatrix, fp: FillPattern, ranges: RangeList,
                         options: Optional[GpuOptions] = None) -> FactorResult:
    """GPU drop-in for ``factor_by_blocks`` (reference factorize.hpp:134-235).

    Same inputs and result semantics: a fresh factor on ``fp.pattern``'s
    arrays; ``BreakdownError(row, pivot)`` on a non-positive pivot;
    ``ValueError`` for invalid ranges / missing diagonals and
    ``RuntimeError`` for a missing diagonal block (logic_error).
    """
    plan = Plan(a_permuted, fp, ranges)
    ps = plan.stats()
    fz = GpuFactorizer(plan, options)
    try:
        st = fz.factor()
        vals = fz.download()
    finally:
        fz.close()
    stats = FactorStats(
        block_build_seconds=ps.block_build_seconds, numeric_seconds=st.device_ms / 1e3,
        chol_tasks=ps.tasks[0], trsm_tasks=ps.tasks[1], herk_tasks=ps.tasks[2], gemm_tasks=ps.tasks[3],
        workers=int(st.grid_ctas), backend="gpu", nnz_u=fp.pattern.nnz(), device_ms=st.device_ms,
        plan_seconds=ps.plan_seconds, grid_ctas=int(st.grid_ctas), threads_per_cta=int(st.threads_per_cta))
    factor = CsrMatrix(fp.pattern.nrows, fp.pattern.ncols, fp.pattern.row_ptr.copy(),
                       fp.pattern.col_idx.copy(), vals)
    return FactorResult(factor, stats)
