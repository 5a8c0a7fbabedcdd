// Lean host plan of the value-flow factorization (the default executor).
//
// Everything here is O(nnz(U)) host work, spread over the host threads
// where rows are independent: the initial values (init_factor_values,
// factorize.hpp:71-89), the reference DAG's task counts, and the schedule of
// the finalising rows. U's transposed index and the per-coordinate update
// programs -- the sorted-index merges of kernels.hpp:55-65, :85-89,
// :104-108, :125-129, folded per coordinate -- are built on the device from
// U's pattern (csrc/device/flow_program.cu), so the host never walks the
// products. The full task-DAG plan (plan.hpp) is built only when the DAG
// itself is asked for (export_task_dag parity, the task executors, sharded
// parts).
//
// Units ("rows" of the schedule), per matrix row t in ascending order:
//   * a U row of at most 32 entries is one unit (one warp pass);
//   * a longer row is its diagonal-block slice (the Chol item of block
//     (p,p), block_layout.hpp:98-181; entries with column < range_end(t)),
//     then warp-wide chunks of the rest that divide by U(t,t).
// Every coordinate of U belongs to exactly one unit, which writes it once.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "sparse.hpp"

namespace tcb {

// std::vector storage whose resize() leaves new elements default-initialised
// (no zero fill): the plan's arrays are written in full by the host threads,
// so a single-threaded memset before that would only add time.
template <class T>
struct uninit_alloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = uninit_alloc<U>;
  };
  uninit_alloc() = default;
  template <class U>
  uninit_alloc(const uninit_alloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using hvec = std::vector<T, uninit_alloc<T>>;

// A borrowed CSR matrix (the caller's arrays; values may be null for a pattern).
struct CsrRef {
  index_t n = 0;
  offset_t nnz = 0;
  const offset_t* row_ptr = nullptr;
  const index_t* col_idx = nullptr;
  const double* values = nullptr;
};

struct FlowPlanStats {
  std::int64_t tasks[4] = {0, 0, 0, 0};  // Chol/Trsm/Herk/Gemm of the reference's DAG (counted)
  std::int32_t nblock_rows = 0;
  std::int64_t nblocks = 0;
  std::int64_t units = 0;      // schedule rows
  std::int32_t depth = 0;      // longest chain of units (levels)
  int threads = 1;             // host threads used
  double block_build_seconds = 0.0;
  double plan_seconds = 0.0;
};

struct FlowPlan {
  index_t n = 0;
  std::int64_t nnz = 0;
  std::int64_t nnz_a = 0;             // entries of a_permuted
  hvec<std::int32_t> cols;     // U column indices
  hvec<std::int32_t> row_ptr;  // n + 1 positions (int32: nnz < 2^31)
  hvec<double> values;         // initialised U values (init_factor_values)
  hvec<std::int32_t> a_map;    // U slot -> a_permuted position, -1 = fill (empty: A has duplicates)
  // units in natural order (row ascending; a row's Chol unit, then its chunks)
  hvec<std::int32_t> ufirst;   // n + 1: first unit of every row
  hvec<std::int32_t> u_tb;     // per unit: first position in U
  hvec<std::int32_t> u_len;    // per unit: coordinates
  hvec<std::int32_t> u_row;    // per unit: its row
  // the schedule (flow_plan_schedule on the host, or built on the device at
  // upload, flow_schedule.cu): empty until scheduled
  bool scheduled = false;
  hvec<std::int32_t> rec;      // 4 words per schedule position: tb, L | kind << 30, dpos, t
  hvec<std::int32_t> unit;     // per schedule position: unit id (natural order)
  FlowPlanStats stats;
};

// Validates both matrices as csr_from_view did (validate_csr), then the
// ranges (ordering.hpp:43-55) and the leading diagonal of every U row
// (kernels.hpp:46-48); std::invalid_argument on failure.
// schedule = false leaves the schedule to the device (tcg_upload) or to a
// later flow_plan_schedule.
FlowPlan build_flow_plan(const CsrRef& a_permuted, const CsrRef& pattern, const RangeList& ranges,
                         bool schedule = true);

// The schedule on the host threads: every unit's level (longest chain from a
// source) and height (longest chain to a sink), the order (level ascending,
// height descending, unit id ascending), the records; stats.depth. Idempotent.
void flow_plan_schedule(FlowPlan& P);

// Where a unit goes between its earliest level and its latest (depth + 1 -
// height), in percent of its slack; host and device schedules alike. 0: as
// soon as possible, the placement of the latency-bound runs (any later costs
// them: C3 2.17 -> 2.80 ms at 100, C2 0.33 -> 0.38). 100: as late as possible,
// for large matrices with short rows, which run the product-parallel kernel
// throughput-bound: a value is then produced shortly before its readers run
// and is still in L2 when they do (B200: C6 1.43 -> 1.15 ms, 7-point 80^3 /
// 96^3 / 112^3 0.53 / 0.75 / 1.05 -> 0.43 / 0.60 / 0.83). TCG_FLOW_SLACK overrides.
int flow_slack_pct(std::int64_t n, std::int64_t nnz, std::int64_t units);

// The pattern as an owning CsrMatrix (values 1.0), for the full plan.
CsrMatrix flow_plan_pattern(const FlowPlan& P);

// One part of a sharded value-flow factorization (C6: ND subtrees on
// different GPUs). The part runs the units of the rows t with
// part_of_row[t] == part, in the global schedule order (the union of the
// parts' lists is one topological order, so no part can deadlock while the
// others run). Its programs are the device-built ones with every operand of
// a row another part owns rewritten to kRemoteBit | owner << kRemoteShift |
// position (flow_program.cu), read from the owner's copy of U through peer
// memory. A unit of a row some other part reads (a source of one of its
// rows) carries bit 31 in its length word and publishes at system scope.
constexpr std::uint32_t kRemoteBit = 0x80000000u;
constexpr int kRemoteShift = 25;  // positions below 2^25, owners below 64
struct FlowPart {
  std::vector<std::int32_t> rec, unit;  // 4 words per schedule row, global order
  std::int64_t rows = 0;
  std::int64_t exported_rows = 0;     // units publishing at system scope
  std::int64_t remote_sources = 0;    // entries U(r,t), t of the part, r of another part
};
FlowPart build_flow_part(const FlowPlan& P, const std::vector<std::int32_t>& part_of_row, std::int32_t nparts,
                         std::int32_t part);

}  // namespace tcb
