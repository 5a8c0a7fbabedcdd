"""B200-native numeric IC(k) Cholesky-by-blocks (arXiv 1601.05871, "Tacho").

The hot path — the reference's ``factor_by_blocks`` — runs as one
persistent sm_100a kernel behind the C ABI in ``include/tacho_b200.h``.
"""
from .core import (  # noqa: F401
    Analysis,
    BreakdownError,
    CONFIGS,
    CsrMatrix,
    DeviceError,
    FactorResult,
    FactorStats,
    FillPattern,
    GpuFactorizer,
    GpuOptions,
    GpuSymbolic,
    GpuTriSolve,
    KIND_NAMES,
    MatrixMarketError,
    Plan,
    RangeList,
    SchedulerError,
    TaskDag,
    analyze,
    config_matrix,
    export_task_dag,
    factor_by_blocks_gpu,
    generate,
    init_factor_values,
    levelk_pattern,
    levelk_pattern_gpu,
    pcg,
    load_matrix_market,
    load_ordering,
    write_matrix_market,
)
