// Flattened, device-ready image of one Cholesky-by-blocks factorization.
//
// The reference's factor_by_blocks (factorize.hpp:134-235) builds the 2D
// block layout (block_layout.hpp:98-181), then walks block rows emitting
// Chol/Trsm/Herk/Gemm tasks whose dependences are the previous writer of
// every block they touch (export_task_dag, factorize.hpp:260-302 is the
// static form of the same walk). A `Plan` holds that exact DAG (same node
// order, same edge list) plus, per task, the precomputed gather work the
// device kernel executes:
//
//   item   = one target row of the task's output block
//            {tb, te}   : the row's slice of U (positions) inside the block
//            local      : row index inside the diagonal range (Chol/Trsm flags)
//            dpos       : position of U(t,t) (Trsm divisor; Chol pivot)
//            [sbeg,send): its source list
//   source = one row r of the task's panel that couples to t through U(r,t)
//            {r_local, pos_rt, sb, se}: wait flag (Chol/Trsm, else -1), the
//            multiplier's position, and the slice of row r whose entries
//            update row t (sorted columns; entries absent from the target
//            are dropped by the device merge).
// Items are stored in ascending t and sources in ascending r, which is the
// per-coordinate order that makes the result bitwise equal to factor_serial.
#pragma once

#include <cstdint>
#include <vector>

#include "sparse.hpp"

namespace tcb {

enum TaskKind : std::int32_t { kChol = 0, kTrsm = 1, kHerk = 2, kGemm = 3 };

// Integer words per record in the device tables.
constexpr int kTaskWords = 8;  // kind, flag_rows, item_b, item_e, succ_b, succ_e, row_begin, out_block
constexpr int kItemWords = 8;  // tb, te, local, dpos, src_b, src_e, 0, 0
constexpr int kSrcWords = 4;   // r_local, pos_rt, sb, se

struct BlockLayout {
  index_t m = 0;
  std::vector<offset_t> brow_ptr;  // m + 1
  std::vector<index_t> bcol_idx;   // sorted within a block row
  std::vector<offset_t> span_off;  // per block: first row slot (nblocks + 1)
  std::vector<std::int32_t> span_b, span_e;  // per (block, local row): slice of U
  offset_t nblocks() const { return static_cast<offset_t>(bcol_idx.size()); }
  offset_t find(index_t i, index_t j) const;
};

struct PlanStats {
  std::int64_t tasks[4] = {0, 0, 0, 0};
  std::int64_t edges = 0;
  std::int64_t items = 0;
  std::int64_t sources = 0;
  std::int64_t pairs = 0;          // source entries visited by the device merge
  std::int64_t empty_tasks = 0;    // Herk/Gemm tasks with no work items
  std::int32_t max_target_len = 0; // longest target row slice
  std::int32_t max_flag_rows = 0;  // largest Chol/Trsm diagonal range
  std::int32_t dag_depth = 0;      // longest path, in tasks
  double block_build_seconds = 0.0;
  double plan_seconds = 0.0;
};

struct Plan {
  index_t n = 0;
  std::int64_t nnz = 0;
  std::vector<std::int32_t> cols;     // U column indices (int32 positions)
  std::vector<double> values;         // initialised U values
  BlockLayout blocks;
  // DAG in generation order (export_task_dag contract)
  std::vector<std::int32_t> node_kind, node_i, node_j;
  std::vector<std::int32_t> edge_from, edge_to;  // emission order
  // device tables
  std::vector<std::int32_t> task_rec, item_rec, src_rec;
  std::vector<std::int32_t> succ;      // successors grouped per task
  std::vector<std::int32_t> indeg;     // predecessors per task (edge multiplicity)
  std::vector<std::int32_t> roots;     // tasks with indeg 0, ascending
  PlanStats stats;
};

BlockLayout build_block_layout(const CsrMatrix& u, const RangeList& ranges);

// Throws std::invalid_argument on inconsistent inputs (reference
// block_layout.hpp:100, kernels.hpp:46-48) and std::logic_error when a
// diagonal block is missing (factorize.hpp:173-174).
Plan build_plan(const CsrMatrix& pattern, const std::vector<double>& init_values,
                const RangeList& ranges, bool with_work = true);

}  // namespace tcb
