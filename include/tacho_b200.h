/*
 * tacho_b200.h — C ABI of the B200-native numeric IC(k) Cholesky-by-blocks.
 *
 * The reference (arXiv 1601.05871, "Tacho" re-implementation `taskchol`) has
 * no FFI: its replaceable unit on the hot path is the C++ function
 *
 *   FactorResult factor_by_blocks(const CsrMatrix& a_permuted,
 *                                 const FillPattern& fp,
 *                                 const RangeList& ranges,
 *                                 TaskPolicy& policy);
 *   (reference proj/include/taskchol/factorize.hpp:134-137)
 *
 * This header is the plain-pointer boundary below a C++ drop-in with the same
 * semantics (include/tacho_b200.hpp: factor_by_blocks_gpu). No exception
 * crosses it; every call returns a tcg_status. One context per host thread.
 *
 * Entry points and the reference interface each one replaces:
 *   tcg_plan_build    the host side of factor_by_blocks before its numeric
 *                     region: init_factor_values (factorize.hpp:71-89), the
 *                     block layout's task counts (block_layout.hpp:98-181,
 *                     factorize.hpp:177-224) and the value-flow schedule of
 *                     the finalising rows, O(nnz) host work
 *   tcg_plan_expand   the full generation walk of factor_by_blocks /
 *                     export_task_dag, flattened (factorize.hpp:169-225,
 *                     260-302): the DAG contract and the task executors
 *   tcg_upload        the one-arena upload of U values and the schedule;
 *                     the update programs (the pattern-restricted merges of
 *                     kernels.hpp:40-132, per coordinate) are built on the
 *                     device (replaces the TaskView/Future state,
 *                     block_layout.hpp:66-93)
 *   tcg_factor        spawn-all + wait(policy) over the whole DAG, executing
 *                     chol/trsm/herk/gemm_block (kernels.hpp:40-132) on the
 *                     GPU; breakdown latch and rethrow (factorize.hpp:146-167,229)
 *   tcg_download      the factored FactorResult::factor.values
 *   tcg_last_error    message of BreakdownError / invalid_argument / CUDA
 */
#ifndef TACHO_B200_H_
#define TACHO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TCG_OK = 0,
  TCG_BREAKDOWN = 1,   /* non-positive pivot: reference BreakdownError(row, pivot) */
  TCG_INVALID = 2,     /* malformed input: reference std::invalid_argument / logic_error */
  TCG_CUDA = 3,        /* CUDA runtime failure */
  TCG_TIMEOUT = 4      /* device watchdog expired (stalled DAG; reference SchedulerError) */
} tcg_status;

typedef enum { TCG_CHOL = 0, TCG_TRSM = 1, TCG_HERK = 2, TCG_GEMM = 3 } tcg_task_kind;

typedef struct tcg_ctx tcg_ctx;
typedef struct tcg_plan tcg_plan;

/* CSR view with the reference's index types (csr_matrix.hpp:16-28). */
typedef struct {
  int32_t n;
  int64_t nnz;
  const int64_t* row_ptr; /* n + 1 */
  const int32_t* col_idx; /* nnz, strictly increasing per row */
  const double* values;   /* nnz (may be NULL for a pattern) */
} tcg_csr_view;

/* Flattened problem image (what tcg_upload copies into the device arena). */
typedef struct {
  int32_t n;
  int64_t nnz;
  const int32_t* col_idx;      /* U columns */
  const double* values;        /* initialised U values (init_factor_values) */
  int64_t ntasks;
  const int32_t* task_rec;     /* 12 words per task */
  int64_t nitems;
  const int32_t* item_rec;     /* 8 words per item */
  int64_t nsources;
  const int32_t* src_rec;      /* 4 words per source */
  int64_t nedges;
  const int32_t* succ;         /* successor lists, grouped per task */
  const int32_t* succ_rec;     /* per edge 16 words: successor, 0, 0, 0, its task record */
  const int32_t* indeg;        /* dependence counters per task */
  int64_t nroots;
  const int32_t* roots;        /* tasks with no predecessor, ascending */
  int32_t max_target_len;
  int32_t max_flag_rows;
  int64_t nhelpers;            /* extra ready-queue entries of multi-CTA tasks */
  int64_t nslots;              /* update programs (optional; 0 when absent): */
  const int32_t* slot_rec;     /*   per target slot {u_b, u_e, m0, o0}; item word 6 = first slot */
  int64_t nupdates;
  const int32_t* upd;          /*   (m, o) pairs: U[tb+k] -= U[m] * U[o] */
  /* value-flow execution (mode 5): the finalising rows of U (whole rows of up to 32 entries;
   * else a row's diagonal-block slice and warp-wide chunks of the rest), each applying every
   * update of its coordinates, in a static (level, falling height) order */
  int64_t nflow;
  const int32_t* flow_rec;     /*   4 words per position: tb, L | kind << 30, dpos, t */
  const int32_t* flow_item;    /*   per position: its unit id (trace stamps are per unit) */
  const int32_t* flow_slot;    /*   host-built programs (flow_devprog = 0): 4 words per coordinate */
  int64_t nflow_upd;           /*   of U {u_b, u_e, m0, o0} and nflow_upd (m, o) pairs */
  const int32_t* flow_upd;
  /* device init_factor_values (optional): per U slot, the position in a_permuted's values it
   * starts from (-1 = fill, starts at 0.0); absent when A has duplicate entries */
  int64_t nnz_a;
  const int32_t* a_map;
  /* value flow with device-built programs (the default, tcg_plan_build): nflow / flow_rec /
   * flow_item are the schedule, flow_slot / flow_upd stay NULL -- tcg_upload builds U's
   * transposed index and the update programs on the device from U's pattern */
  int32_t flow_devprog;        /* 1: u_row_ptr is set */
  const int32_t* u_row_ptr;    /*   n + 1 positions of U's rows (int32) */
  /* a part of a sharded run (tcg_plan_part_problem): the schedule holds the part's rows; the
   * device programs read operands of rows other parts own from their U (tcg_set_peers) */
  int32_t flow_part;           /* -1: the whole matrix */
  const int32_t* part_of_row;  /*   owner part of every row (n) */
  /* the schedule built on the device (flow_devprog = 1 and flow_rec = NULL, the default of
   * tcg_plan_build): the nflow units in natural order, from which tcg_upload computes the
   * levels, heights, order and records on the device (tcg_plan_schedule builds them on the
   * host instead) */
  const int32_t* u_first;      /*   n + 1: first unit of every row */
  const int32_t* u_tb;         /*   per unit: first position in U */
  const int32_t* u_len;        /*   per unit: coordinates */
  const int32_t* u_row;        /*   per unit: its row */
} tcg_problem;

typedef struct {
  int32_t threads_per_cta;  /* task executors (modes 1/2): 128, 256 or 512; 0 = default (256);
                               mode 5 always runs 256-thread CTAs */
  int32_t ctas_per_sm;      /* 0 = occupancy maximum */
  int32_t staging_cap;      /* target-row entries staged per warp; 0 = auto */
  double timeout_s;         /* device watchdog; 0 = default (30 s) */
  int32_t trace;            /* 1 = record per-task start/end globaltimer stamps */
  int32_t mode;             /* 0 = auto (5), task-level DAG execution (the reference's
                               Chol/Trsm/Herk/Gemm tasks, device ready queue + dependence
                               counters; needs tcg_plan_expand) with 1 = device merge of
                               sorted indices or 2 = precomputed update programs; 5 = static
                               schedule of the finalising rows, readers polling the values
                               themselves (no flags, no fences) */
  int32_t lanes_per_row;    /* ignored (kept for the ABI): mode 5 runs whole warps or
                               groups of warps per row, chosen by program length */
} tcg_options;

typedef struct {
  double device_ms;          /* persistent kernel, CUDA events on the launch stream */
  int64_t tasks_completed;
  int64_t tasks_executed;    /* bodies run (a breakdown skips the rest) */
  int32_t breakdown_row;     /* -1 when none */
  double breakdown_pivot;
  int32_t grid_ctas;
  int32_t threads_per_cta;
  int32_t staging_cap;
  int64_t smem_bytes;
  int32_t kernel_launches;   /* device launches issued by the call */
  int64_t helpers_run;       /* helper tickets that joined a multi-CTA task */
  int32_t mode;              /* execution mode used (1, 2 or 5, see tcg_options.mode) */
  uint64_t profile[7];       /* trace mode, rows: SM cycles in {pop wait, row body, publish
                                fence, release} summed over warps; rows, pops, pushes */
  int32_t lanes_per_row;     /* mode 5: lanes per row used */
  int32_t batch;             /* mode 5: value sets factored by the call */
  int32_t breakdown_member;  /* batch: member of breakdown_row (-1 when none) */
  int32_t drain_ctas;        /* end to end: CTAs that copied the factor to the host during the
                                launch; negative: minus the number of chunks the copy engine took
                                out beside the launch as they became final; 0: a D2H copy after it */
  int32_t chunks;            /* end to end, batches: member chunks pipelined with the copies
                                (0: one launch) */
  int32_t row_kernel;        /* mode 5: 1 = one lane per coordinate (factor_flow_pipe),
                                2 = product-parallel row groups (factor_flow_pp) */
  int32_t flow_depth;        /* mode 5: longest chain of the schedule when the device built it
                                (0 when the plan brought a host schedule: tcg_plan_get_stats) */
} tcg_stats;

typedef struct {
  int64_t tasks[4];          /* chol, trsm, herk, gemm (counted from the block layout) */
  int32_t nblocks_rows;      /* block rows m (= number of ranges) */
  int64_t nblocks;
  double block_build_seconds, plan_seconds;
  int64_t flow_rows;         /* value-flow rows (mode 5) */
  int32_t flow_depth;        /* longest value-flow chain, in rows */
  int32_t host_threads;      /* host threads the plan used */
  /* the task-DAG plan (tcg_plan_expand; 0 until it exists) */
  int32_t full_plan;         /* 1 when it exists */
  double full_plan_seconds;  /* its host time */
  int64_t edges, items, sources, pairs, empty_tasks;
  int32_t max_target_len, max_flag_rows, dag_depth;
  int32_t max_width;         /* most CTAs cooperating on one task */
  int64_t helpers;           /* helper tickets over all multi-CTA tasks */
  int64_t updates;           /* products in the task executors' update programs */
} tcg_plan_stats;

/* ---- host flattener ---------------------------------------------------- */
/* a_permuted: PᵀAP (full symmetric CSR with values); pattern: fp.pattern
 * (upper, full diagonal); range_bounds: nranges + 1 ascending row bounds. */
tcg_status tcg_plan_build(const tcg_csr_view* a_permuted, const tcg_csr_view* pattern,
                          int32_t nranges, const int32_t* range_bounds, tcg_plan** out);
void tcg_plan_free(tcg_plan* plan);
const char* tcg_plan_error(void); /* message of the last failed tcg_plan_build (thread-local) */
/* The upload image: U, its initial values and the value-flow schedule (programs built on the
 * device); with the task-DAG plan (tcg_plan_expand) also the task executors' tables. */
tcg_status tcg_plan_problem(const tcg_plan* plan, tcg_problem* out);
/* The value-flow schedule (levels, heights, order, records) on the host threads, if it does
 * not exist yet; tcg_upload otherwise builds it on the device. tcg_plan_part_problem calls it. */
tcg_status tcg_plan_schedule(tcg_plan* plan);
/* Builds the task-DAG plan (the reference's generation walk, flattened) if it does not exist
 * yet; tcg_plan_dag, tcg_plan_blocks and tcg_plan_part_problem do so on first use. */
tcg_status tcg_plan_expand(tcg_plan* plan);
tcg_status tcg_plan_get_stats(const tcg_plan* plan, tcg_plan_stats* out);
/* DAG in generation order, the export_task_dag contract (factorize.hpp:260-302):
 * node kind/block_row/block_col and edges (before, after) in emission order.
 * Pointers stay valid until tcg_plan_free. */
tcg_status tcg_plan_dag(const tcg_plan* plan, int64_t* nnodes, const int32_t** kind,
                        const int32_t** block_row, const int32_t** block_col, int64_t* nedges,
                        const int32_t** edge_from, const int32_t** edge_to);
/* Block structure (brow_ptr m+1, bcol_idx nblocks), reference BlockMatrix. */
tcg_status tcg_plan_blocks(const tcg_plan* plan, int32_t* m, const int64_t** brow_ptr,
                           int64_t* nblocks, const int32_t** bcol_idx);

/* Sharded value flow (C6: ND subtrees on different GPUs). part_of_row: owner part of every
 * row of U (n entries, < nparts <= 64). Fills `out` like tcg_plan_problem but with only the
 * rows of `part` (mode 5 only); operands owned by other parts are read from their copies of
 * U, set with tcg_set_peers. Valid until the next call for the same part or tcg_plan_free. */
tcg_status tcg_plan_part_problem(tcg_plan* plan, int32_t nparts, const int32_t* part_of_row, int32_t part,
                                 tcg_problem* out, int64_t* remote_operands);

/* ---- device context ---------------------------------------------------- */
tcg_status tcg_create(int device, tcg_ctx** out);
void tcg_destroy(tcg_ctx* ctx);
const char* tcg_last_error(const tcg_ctx* ctx);
tcg_status tcg_set_options(tcg_ctx* ctx, const tcg_options* opt);
/* One cudaMalloc arena; replaces any previous upload. */
tcg_status tcg_upload(tcg_ctx* ctx, const tcg_problem* problem);
/* Replace the initial values (host pointer, nnz doubles) of the uploaded problem. */
tcg_status tcg_set_values(tcg_ctx* ctx, const double* values);
/* Restore the working values from the device copy of the initial values. */
tcg_status tcg_restore(tcg_ctx* ctx);
/* Factor the working values in place. TCG_BREAKDOWN sets stats->breakdown_*. */
tcg_status tcg_factor(tcg_ctx* ctx, tcg_stats* stats);
tcg_status tcg_download(tcg_ctx* ctx, double* values);
/* End-to-end refactorization from host buffers (nnz x nbatch doubles each; pinned memory for
 * full PCIe speed): upload the initial values, factor, download the factor, stream-ordered
 * in one call. The device copy of the initial values (tcg_restore) is not updated. */
tcg_status tcg_factor_host(tcg_ctx* ctx, const double* values_in, double* values_out, tcg_stats* stats);
/* End to end from the matrix, as the reference's call takes it: PᵀAP's values (host,
 * nbatch x nnz(a_permuted) in a_permuted's CSR order) are uploaded, scattered into U on the
 * device (init_factor_values, factorize.hpp:71-89; needs the A -> U map, see
 * tcg_set_a_values), factored, and the factor downloaded -- one stream-ordered call. The
 * restore copy is updated too. */
tcg_status tcg_factor_host_a(tcg_ctx* ctx, const double* a_values, double* values_out, tcg_stats* stats);
/* Stamps of the last traced factor: per task {start, end} (2*ntasks words), then per
 * item {claimed, sources ready, merged, published} (4*nitems words); globaltimer ns. */
tcg_status tcg_download_trace(tcg_ctx* ctx, uint64_t* stamps);
/* Device pointer to the working values and their count (for in-process users
 * that keep U resident, e.g. a preconditioner apply on the same stream). */
tcg_status tcg_device_values(tcg_ctx* ctx, double** dptr, int64_t* nnz);
/* The value-flow schedule on the device (nflow records of 4 words, nflow unit ids; depth =
 * its longest chain when the device built it, else 0); for checks against tcg_plan_schedule. */
tcg_status tcg_flow_records(tcg_ctx* ctx, int32_t* rec, int32_t* item, int32_t* depth);
/* The value-flow update programs on the device (slot: 4 * nnz ints {u_b, u_e, m0, o0}; upd:
 * 2 * nupd ints (m, o); either may be NULL) and the device time of their build (ms). */
tcg_status tcg_flow_programs(tcg_ctx* ctx, int32_t* slot, int32_t* upd, int64_t* nupd, double* build_ms);
/* Batch of value sets sharing the uploaded pattern (mode 5; C5-style refactorization of
 * many matrices with one structure). `values`: nbatch x nnz host doubles, member-major.
 * nbatch = 1 returns to the single-matrix state. tcg_factor then factors every member in
 * one launch; a breakdown skips the rest of that member only (TCG_BREAKDOWN reports the
 * first; tcg_batch_breakdown gives each member's row, -1 = none, and pivot). */
tcg_status tcg_set_batch(tcg_ctx* ctx, int32_t nbatch, const double* values);
/* init_factor_values on the device (reference factorize.hpp:71-89): `a_values` holds nbatch x
 * nnz(a_permuted) values of PᵀAP in a_permuted's CSR order (host); they are uploaded and
 * scattered into U (fill = 0.0, bitwise as the host init). Sets the batch size to nbatch. */
tcg_status tcg_set_a_values(tcg_ctx* ctx, int32_t nbatch, const double* a_values);
tcg_status tcg_set_batch_values(tcg_ctx* ctx, const double* values); /* same nbatch */
int32_t tcg_batch_size(const tcg_ctx* ctx);
tcg_status tcg_download_batch(tcg_ctx* ctx, double* values);
tcg_status tcg_batch_breakdown(tcg_ctx* ctx, int32_t* rows, double* pivots);
/* Mode 5 in two steps (sharded runs): phase 1 resets the output (and waits for it), phase 2
 * launches the factorization; 0 = both, as tcg_factor. Between them the caller makes sure
 * every part has finished phase 1, since parts read each other's U. */
tcg_status tcg_factor_phase(tcg_ctx* ctx, int32_t phase, tcg_stats* stats);
/* Sharded runs: device pointers of every part's working values (index = part; own included,
 * from tcg_device_values, or tcg_ipc_open for parts in other processes). */
tcg_status tcg_set_peers(tcg_ctx* ctx, int32_t nparts, const uint64_t* values_ptrs);
/* CUDA IPC of the working values: a 64-byte handle of the arena plus the values' offset. */
tcg_status tcg_ipc_values_handle(tcg_ctx* ctx, void* handle, int64_t* offset);
tcg_status tcg_ipc_open(tcg_ctx* ctx, const void* handle, int64_t offset, uint64_t* values_ptr);
/* Bytes of the device arena. */
int64_t tcg_arena_bytes(const tcg_ctx* ctx);

/* ---- level-k symbolic on the device ------------------------------------- */
/* The fill pattern of U, levelk_pattern_bfs (reference symbolic.hpp:57-120), one warp per
 * source row: same FillPattern.pattern arrays as the reference
 * (row i = {i} then its targets ascending), bit-exact. Separate handle: it needs no plan. */
typedef struct tcg_sym tcg_sym;
typedef struct {
  double device_ms;          /* search (rows into scratch) + scan + copy, CUDA events on the handle's stream */
  double host_ms;            /* wall time of tcg_sym_levelk (includes the nnz_u readback) */
  int64_t nnz_u;             /* FillPattern.pattern.nnz() */
  int64_t nnz_triu_input;    /* FillPattern.nnz_triu_input (count_upper, csr_matrix.hpp:219-225) */
  int64_t slow_rows;         /* rows whose search outgrew shared memory (global-memory path) */
  int64_t tier2_rows;        /* rows that outgrew the 512-slot tables (then 2,048 slots) */
  int32_t kernel_launches;
  int32_t grid_ctas;
  int32_t single_pass;       /* 1: every shared-memory row was searched once (its row copied from
                                scratch); 0: scratch was short and rows were searched again
                                (scratch then grows for the next call) */
} tcg_sym_stats;
enum { TCG_SYM_ALL_SLOW = 1 };  /* tcg_sym_levelk flag: every row on the global-memory path */
tcg_status tcg_sym_create(int device, tcg_sym** out);
void tcg_sym_destroy(tcg_sym* s);
const char* tcg_sym_error(const tcg_sym* s);
/* a_permuted: PᵀAP's pattern (values unused); square, row_ptr 0..nnz, columns in range. */
tcg_status tcg_sym_upload(tcg_sym* s, const tcg_csr_view* a_permuted);
tcg_status tcg_sym_levelk(tcg_sym* s, int32_t level, int32_t flags, tcg_sym_stats* stats);
int64_t tcg_sym_nnz(const tcg_sym* s); /* nnz of the last pattern, -1 before the first */
/* row_ptr: n + 1, col_idx: tcg_sym_nnz entries (host). */
tcg_status tcg_sym_download(tcg_sym* s, int64_t* row_ptr, int32_t* col_idx);

/* ---- triangular solves with the factor ----------------------------------- */
/* The preconditioner apply of IC(k)-preconditioned CG: with the
 * factor U held by a context (after tcg_factor), forward Uᵀ y = b and backward U x = y on
 * the device, one warp per unknown in a static level order, operands polled in place
 * (no per-level launches). The reference has no solve; the order of
 * operations is fixed: per unknown, products in ascending source index subtracted in that
 * order, then one division (oracle.c orc_trisolve), so results are reproducible bitwise. */
typedef struct tcg_solve tcg_solve;
typedef struct {
  double device_ms;          /* marker reset + solve kernel + result copy, CUDA events */
  int32_t depth_forward;     /* longest dependence chain of Uᵀ y = b, in unknowns */
  int32_t depth_backward;    /* ... of U x = y */
  int32_t grid_ctas;
  int32_t kernel_launches;
} tcg_solve_stats;
enum { TCG_SOLVE_FORWARD = 1, TCG_SOLVE_BACKWARD = 2, TCG_SOLVE_BOTH = 3 };
/* u_pattern: the factor's pattern (FillPattern.pattern of the uploaded problem); the values
 * are read from the context at every apply, so a refactorization is picked up (with a batch,
 * member 0's factor). Destroy the solve handle before its context. */
tcg_status tcg_solve_create(tcg_ctx* ctx, const tcg_csr_view* u_pattern, tcg_solve** out);
void tcg_solve_destroy(tcg_solve* s);
const char* tcg_solve_error(const tcg_solve* s);
/* host vectors of n doubles (b and x may alias); which: TCG_SOLVE_* */
tcg_status tcg_solve_apply(tcg_solve* s, const double* b, double* x, int32_t which, tcg_solve_stats* stats);
/* device vectors (b_dev and x_dev may alias), on the context's stream */
tcg_status tcg_solve_apply_device(tcg_solve* s, const double* b_dev, double* x_dev, int32_t which,
                                  tcg_solve_stats* stats);
/* The same apply without a host wait (for iterative callers that queue many steps):
 * enqueued on the context's stream, returns at once. A watchdog expiry is sticky and is
 * reported by the next tcg_solve_sync (or synchronous apply), which waits for the stream. */
tcg_status tcg_solve_apply_async(tcg_solve* s, const double* b_dev, double* x_dev, int32_t which);
tcg_status tcg_solve_sync(tcg_solve* s);
/* The caller's other step per CG iteration: y = A x with the system matrix (PᵀAP), set once
 * (host CSR with values, n x n), applied to device vectors on the context's stream; per row
 * the products are summed in column order. */
tcg_status tcg_solve_set_matrix(tcg_solve* s, const tcg_csr_view* a);
tcg_status tcg_solve_spmv(tcg_solve* s, const double* x_dev, double* y_dev);
/* Conjugate-gradient vector updates on the context's stream (device vectors of n doubles;
 * state = {rz, live (1/0), threshold} in device memory; dots summed in a fixed order, so
 * the iterates are the same in every run). cg_step: alpha = rz / (p . ap); where live,
 * x += alpha p and r -= alpha ap; hist[it] = ||r||; live = 0 once ||r|| <= threshold.
 * cg_direction: rz' = r . z; p = p (rz' / rz) + z; rz = rz'. */
tcg_status tcg_solve_cg_step(tcg_solve* s, double* x, double* r, const double* p, const double* ap, double* state,
                             double* hist, int32_t it);
tcg_status tcg_solve_cg_direction(tcg_solve* s, const double* r, const double* z, double* p, double* state);
/* The context's stream (cudaStream_t): everything above is ordered on it. */
tcg_status tcg_solve_stream(tcg_solve* s, void** stream);
/* With TCG_SOLVE_TRACE=1 in the environment: per schedule position (2 n) the globaltimer
 * stamps {start, operands final, end} of the last apply, and (recs != NULL) the position
 * records {entry begin, length | backward << 31, diagonal position, row} (16 bytes each). */
tcg_status tcg_solve_trace(tcg_solve* s, uint64_t* stamps, void* recs);

/* ---- host input side (analysis) ---------------------------------------- */
/* Own implementations of the reference's analysis chain (pipeline.hpp:35-55),
 * kept bit-exact with it; they produce the inputs of tcg_plan_build. */
typedef struct tch_matrix tch_matrix;
typedef struct tch_analysis tch_analysis;

/* kind: "grid2d" (p0 x p1), "lap7" (p0^3), "stencil27" (p0^3, seed),
 * "elasticity" (p0^3 x 3, seed), "diffusion" (p0^3, seed, sigma = p1 / 1000),
 * "path" (p0, diag = 2), "random_spd" (p0, density = p1 / 1e6, seed). */
tch_matrix* tch_generate(const char* kind, int64_t p0, int64_t p1, uint64_t seed);
tch_matrix* tch_matrix_from_csr(const tcg_csr_view* view);
void tch_matrix_free(tch_matrix* m);
void tch_matrix_view(const tch_matrix* m, tcg_csr_view* out);

tch_analysis* tch_analyze(const tch_matrix* a, int32_t level, int32_t treecut,
                          int32_t leaf_size, int32_t max_depth, int32_t threads);
void tch_analysis_free(tch_analysis* an);
const char* tch_error(void); /* thread-local message of the last tch_* failure */
void tch_analysis_perm(const tch_analysis* an, const int32_t** perm, const int32_t** iperm);
int32_t tch_analysis_ranges(const tch_analysis* an, const int32_t** bounds); /* returns count */
/* Row spans [lo, hi) of the ND subtrees at `depth` (a shallower leaf stands for itself);
 * writes at most `cap` of them and returns their count. Rows outside every span are the
 * separators above them. */
int32_t tch_analysis_subtrees(const tch_analysis* an, int32_t depth, int32_t cap, int32_t* lo, int32_t* hi);
void tch_analysis_permuted(const tch_analysis* an, tcg_csr_view* out);
void tch_analysis_pattern(const tch_analysis* an, tcg_csr_view* out);
void tch_analysis_times(const tch_analysis* an, double* ordering_s, double* symbolic_s);
/* Fill pattern for an arbitrary permuted matrix (levelk_pattern_bfs). */
tch_matrix* tch_levelk_pattern(const tch_matrix* a_permuted, int32_t level, int32_t threads);
/* File formats. Matrix Market coordinate files, reference
 * matrix_market.hpp:61-176: real/integer/pattern, general/symmetric (mirrored), duplicates
 * summed; NULL / TCG_INVALID with tch_error() = the reference's MatrixMarketError text. The
 * writer emits the reference's bytes (general storage, shortest round-trip values). */
tch_matrix* tch_load_matrix_market(const char* path);
tcg_status tch_write_matrix_market(const tcg_csr_view* m, const char* path);
/* Ordering file, reference load_ordering (ordering.hpp:355-399): n, perm (new index of old),
 * range count, "begin end" per range. Writes perm (n) and, when cap >= count, count + 1
 * bounds; returns the range count, or -1 (tch_error() = the reference's message). */
int32_t tch_load_ordering(const char* path, int32_t n, int32_t* perm, int32_t cap, int32_t* bounds);
/* analyze() with an imported ordering (reference pipeline.hpp:39-44): PᵀAP and the
 * level-k pattern for the given permutation and ranges. */
tch_analysis* tch_analyze_with_ordering(const tch_matrix* a, const int32_t* perm, int32_t nranges,
                                        const int32_t* bounds, int32_t level, int32_t threads);
/* init_factor_values (factorize.hpp:71-89): out has pattern->nnz doubles. */
tcg_status tch_init_values(const tcg_csr_view* a_permuted, const tcg_csr_view* pattern, double* out);

#ifdef __cplusplus
}
#endif

#endif /* TACHO_B200_H_ */
