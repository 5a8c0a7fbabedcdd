"""ctypes binding of the C ABI in include/tacho_b200.h.

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build()``)
into ``paper_1601_05871_b200/lib/libtacho_b200.so``. There is no fallback:
if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TCG_LIB_DIR: load an alternative in-tree build (A/B experiments under tools/)
LIB_PATH = os.path.join(os.environ.get("TCG_LIB_DIR") or os.path.join(_HERE, "lib"), "libtacho_b200.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)

TCG_OK, TCG_BREAKDOWN, TCG_INVALID, TCG_CUDA, TCG_TIMEOUT = range(5)


class CsrView(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("nnz", C.c_int64),
        ("row_ptr", i64p),
        ("col_idx", i32p),
        ("values", f64p),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("nnz", C.c_int64),
        ("col_idx", i32p),
        ("values", f64p),
        ("ntasks", C.c_int64),
        ("task_rec", i32p),
        ("nitems", C.c_int64),
        ("item_rec", i32p),
        ("nsources", C.c_int64),
        ("src_rec", i32p),
        ("nedges", C.c_int64),
        ("succ", i32p),
        ("succ_rec", i32p),
        ("indeg", i32p),
        ("nroots", C.c_int64),
        ("roots", i32p),
        ("max_target_len", C.c_int32),
        ("max_flag_rows", C.c_int32),
        ("nhelpers", C.c_int64),
        ("nslots", C.c_int64),
        ("slot_rec", i32p),
        ("nupdates", C.c_int64),
        ("upd", i32p),
        ("nflow", C.c_int64),
        ("flow_rec", i32p),
        ("flow_item", i32p),
        ("flow_slot", i32p),
        ("nflow_upd", C.c_int64),
        ("flow_upd", i32p),
        ("nnz_a", C.c_int64),
        ("a_map", i32p),
        ("flow_devprog", C.c_int32),
        ("u_row_ptr", i32p),
        ("flow_part", C.c_int32),
        ("part_of_row", i32p),
        ("u_first", i32p),
        ("u_tb", i32p),
        ("u_len", i32p),
        ("u_row", i32p),
    ]


class Options(C.Structure):
    _fields_ = [
        ("threads_per_cta", C.c_int32),
        ("ctas_per_sm", C.c_int32),
        ("staging_cap", C.c_int32),
        ("timeout_s", C.c_double),
        ("trace", C.c_int32),
        ("mode", C.c_int32),
        ("lanes_per_row", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("device_ms", C.c_double),
        ("tasks_completed", C.c_int64),
        ("tasks_executed", C.c_int64),
        ("breakdown_row", C.c_int32),
        ("breakdown_pivot", C.c_double),
        ("grid_ctas", C.c_int32),
        ("threads_per_cta", C.c_int32),
        ("staging_cap", C.c_int32),
        ("smem_bytes", C.c_int64),
        ("kernel_launches", C.c_int32),
        ("helpers_run", C.c_int64),
        ("mode", C.c_int32),
        ("profile", C.c_uint64 * 7),
        ("lanes_per_row", C.c_int32),
        ("batch", C.c_int32),
        ("breakdown_member", C.c_int32),
        ("drain_ctas", C.c_int32),
        ("chunks", C.c_int32),
        ("row_kernel", C.c_int32),
        ("flow_depth", C.c_int32),
    ]


class PlanStats(C.Structure):
    _fields_ = [
        ("tasks", C.c_int64 * 4),
        ("nblocks_rows", C.c_int32),
        ("nblocks", C.c_int64),
        ("block_build_seconds", C.c_double),
        ("plan_seconds", C.c_double),
        ("flow_rows", C.c_int64),
        ("flow_depth", C.c_int32),
        ("host_threads", C.c_int32),
        ("full_plan", C.c_int32),
        ("full_plan_seconds", C.c_double),
        ("edges", C.c_int64),
        ("items", C.c_int64),
        ("sources", C.c_int64),
        ("pairs", C.c_int64),
        ("empty_tasks", C.c_int64),
        ("max_target_len", C.c_int32),
        ("max_flag_rows", C.c_int32),
        ("dag_depth", C.c_int32),
        ("max_width", C.c_int32),
        ("helpers", C.c_int64),
        ("updates", C.c_int64),
    ]


class SymStats(C.Structure):
    _fields_ = [
        ("device_ms", C.c_double),
        ("host_ms", C.c_double),
        ("nnz_u", C.c_int64),
        ("nnz_triu_input", C.c_int64),
        ("slow_rows", C.c_int64),
        ("tier2_rows", C.c_int64),
        ("kernel_launches", C.c_int32),
        ("grid_ctas", C.c_int32),
        ("single_pass", C.c_int32),
    ]


TCG_SYM_ALL_SLOW = 1


class SolveStats(C.Structure):
    _fields_ = [
        ("device_ms", C.c_double),
        ("depth_forward", C.c_int32),
        ("depth_backward", C.c_int32),
        ("grid_ctas", C.c_int32),
        ("kernel_launches", C.c_int32),
    ]


TCG_SOLVE_FORWARD, TCG_SOLVE_BACKWARD, TCG_SOLVE_BOTH = 1, 2, 3

# (name, restype, argtypes) for every symbol declared in include/tacho_b200.h
SIGNATURES = [
    ("tcg_plan_build", C.c_int, [C.POINTER(CsrView), C.POINTER(CsrView), C.c_int32, i32p, C.POINTER(C.c_void_p)]),
    ("tcg_plan_free", None, [C.c_void_p]),
    ("tcg_plan_error", C.c_char_p, []),
    ("tcg_plan_problem", C.c_int, [C.c_void_p, C.POINTER(Problem)]),
    ("tcg_plan_expand", C.c_int, [C.c_void_p]),
    ("tcg_plan_schedule", C.c_int, [C.c_void_p]),
    ("tcg_plan_get_stats", C.c_int, [C.c_void_p, C.POINTER(PlanStats)]),
    ("tcg_plan_part_problem", C.c_int, [C.c_void_p, C.c_int32, i32p, C.c_int32, C.POINTER(Problem), i64p]),
    ("tcg_plan_dag", C.c_int, [C.c_void_p, i64p, C.POINTER(i32p), C.POINTER(i32p), C.POINTER(i32p),
                                i64p, C.POINTER(i32p), C.POINTER(i32p)]),
    ("tcg_plan_blocks", C.c_int, [C.c_void_p, i32p, C.POINTER(i64p), i64p, C.POINTER(i32p)]),
    ("tcg_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("tcg_destroy", None, [C.c_void_p]),
    ("tcg_last_error", C.c_char_p, [C.c_void_p]),
    ("tcg_set_options", C.c_int, [C.c_void_p, C.POINTER(Options)]),
    ("tcg_upload", C.c_int, [C.c_void_p, C.POINTER(Problem)]),
    ("tcg_set_values", C.c_int, [C.c_void_p, f64p]),
    ("tcg_restore", C.c_int, [C.c_void_p]),
    ("tcg_factor", C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    ("tcg_download", C.c_int, [C.c_void_p, f64p]),
    ("tcg_factor_host", C.c_int, [C.c_void_p, f64p, f64p, C.c_void_p]),
    ("tcg_factor_host_a", C.c_int, [C.c_void_p, f64p, f64p, C.c_void_p]),
    ("tcg_download_trace", C.c_int, [C.c_void_p, u64p]),
    ("tcg_set_batch", C.c_int, [C.c_void_p, C.c_int32, f64p]),
    ("tcg_set_batch_values", C.c_int, [C.c_void_p, f64p]),
    ("tcg_set_a_values", C.c_int, [C.c_void_p, C.c_int32, f64p]),
    ("tcg_batch_size", C.c_int32, [C.c_void_p]),
    ("tcg_download_batch", C.c_int, [C.c_void_p, f64p]),
    ("tcg_batch_breakdown", C.c_int, [C.c_void_p, i32p, f64p]),
    ("tcg_flow_records", C.c_int, [C.c_void_p, i32p, i32p, i32p]),
    ("tcg_flow_programs", C.c_int, [C.c_void_p, i32p, i32p, i64p, f64p]),
    ("tcg_device_values", C.c_int, [C.c_void_p, C.POINTER(f64p), i64p]),
    ("tcg_arena_bytes", C.c_int64, [C.c_void_p]),
    ("tcg_set_peers", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64)]),
    ("tcg_factor_phase", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("tcg_ipc_values_handle", C.c_int, [C.c_void_p, C.c_void_p, i64p]),
    ("tcg_ipc_open", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_uint64)]),
    ("tcg_sym_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("tcg_sym_destroy", None, [C.c_void_p]),
    ("tcg_sym_error", C.c_char_p, [C.c_void_p]),
    ("tcg_sym_upload", C.c_int, [C.c_void_p, C.POINTER(CsrView)]),
    ("tcg_sym_levelk", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(SymStats)]),
    ("tcg_sym_nnz", C.c_int64, [C.c_void_p]),
    ("tcg_sym_download", C.c_int, [C.c_void_p, i64p, i32p]),
    ("tcg_solve_create", C.c_int, [C.c_void_p, C.POINTER(CsrView), C.POINTER(C.c_void_p)]),
    ("tcg_solve_destroy", None, [C.c_void_p]),
    ("tcg_solve_error", C.c_char_p, [C.c_void_p]),
    ("tcg_solve_apply", C.c_int, [C.c_void_p, f64p, f64p, C.c_int32, C.POINTER(SolveStats)]),
    ("tcg_solve_trace", C.c_int, [C.c_void_p, u64p, C.c_void_p]),
    ("tcg_solve_set_matrix", C.c_int, [C.c_void_p, C.POINTER(CsrView)]),
    ("tcg_solve_cg_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int32]),
    ("tcg_solve_cg_direction", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tcg_solve_spmv", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tcg_solve_stream", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tcg_solve_apply_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(SolveStats)]),
    ("tcg_solve_apply_async", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    ("tcg_solve_sync", C.c_int, [C.c_void_p]),
    ("tch_generate", C.c_void_p, [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64]),
    ("tch_matrix_from_csr", C.c_void_p, [C.POINTER(CsrView)]),
    ("tch_matrix_free", None, [C.c_void_p]),
    ("tch_matrix_view", None, [C.c_void_p, C.POINTER(CsrView)]),
    ("tch_analyze", C.c_void_p, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("tch_analysis_free", None, [C.c_void_p]),
    ("tch_error", C.c_char_p, []),
    ("tch_analysis_perm", None, [C.c_void_p, C.POINTER(i32p), C.POINTER(i32p)]),
    ("tch_analysis_ranges", C.c_int32, [C.c_void_p, C.POINTER(i32p)]),
    ("tch_analysis_subtrees", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, i32p, i32p]),
    ("tch_analysis_permuted", None, [C.c_void_p, C.POINTER(CsrView)]),
    ("tch_analysis_pattern", None, [C.c_void_p, C.POINTER(CsrView)]),
    ("tch_analysis_times", None, [C.c_void_p, f64p, f64p]),
    ("tch_levelk_pattern", C.c_void_p, [C.c_void_p, C.c_int32, C.c_int32]),
    ("tch_init_values", C.c_int, [C.POINTER(CsrView), C.POINTER(CsrView), f64p]),
    ("tch_load_matrix_market", C.c_void_p, [C.c_char_p]),
    ("tch_write_matrix_market", C.c_int, [C.POINTER(CsrView), C.c_char_p]),
    ("tch_load_ordering", C.c_int32, [C.c_char_p, C.c_int32, i32p, C.c_int32, i32p]),
    ("tch_analyze_with_ordering", C.c_void_p, [C.c_void_p, i32p, C.c_int32, i32p, C.c_int32, C.c_int32]),
]

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make lib` or __graft_entry__.build(); "
            "there is no CPU fallback for the factorization path")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
