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
//            local      : row index inside the diagonal range (breakdown row)
//            dpos       : position of U(t,t) (Trsm divisor; Chol pivot)
//            [sbeg,send): its source list
//   source = one row r of the task's panel that couples to t through U(r,t)
//            {dep, pos_rt, sb, se}: item position to wait for (Chol/Trsm, else -1), the
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
// task: kind, width, item_b, item_e | succ_b, succ_e, row_begin, nlevels |
//       src_b, src_e, out_block, 0   (three int4 loads)
constexpr int kTaskWords = 12;
constexpr int kItemWords = 8;  // tb, te, local, dpos, src_b, src_e, slot_off, 0
constexpr int kSrcWords = 4;   // dep (item position in task, Chol/Trsm; else -1), pos_rt, sb, se
constexpr int kSuccWords = 16; // successor id, 0, 0, 0, then its 12-word task record
// value-flow schedule record per position: tb, L | kind << 30, dpos, t
constexpr int kFlowWords = 4;
constexpr int kFlowKindShift = 30;

struct PlanOptions {
  double cta_cost = 64.0;  // estimated warp-steps one CTA should get before a helper joins
  int max_width = 64;      // most CTAs cooperating on one task
  double dep_wide_cost = 64.0;  // Chol/Trsm go multi-CTA only above this cost per level
  bool programs = true;    // precompute per-row update programs (slot_rec / upd, mode 2)
  int threads = 0;         // host threads for the program build (0 = all)
};

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
  std::int32_t max_width = 1;      // widest task, in CTAs
  std::int64_t helpers = 0;        // extra queue entries for multi-CTA tasks
  std::int64_t updates = 0;        // (m, o) products in the update programs
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
  std::vector<std::int32_t> task_blk;  // per task: target, multiplier, operand block, 0
  std::vector<std::int32_t> slot_rec;  // update-program slots {u_b, u_e, m0, o0} (per item: L)
  std::vector<std::int32_t> upd;       // update-program (m, o) pairs
  std::vector<std::int32_t> succ;      // successors grouped per task
  std::vector<std::int32_t> succ_rec;  // per edge: successor + copy of its task record
  std::vector<std::int32_t> indeg;     // predecessors per task (edge multiplicity)
  std::vector<std::int32_t> roots;     // tasks with indeg 0, ascending
  PlanStats stats;
};

BlockLayout build_block_layout(const CsrMatrix& u, const RangeList& ranges);

// Throws std::invalid_argument on inconsistent inputs (reference
// block_layout.hpp:100, kernels.hpp:46-48) and std::logic_error when a
// diagonal block is missing (factorize.hpp:173-174).
Plan build_plan(const CsrMatrix& pattern, const std::vector<double>& init_values,
                const RangeList& ranges, bool with_work = true,
                const PlanOptions& opt = PlanOptions());

}  // namespace tcb
