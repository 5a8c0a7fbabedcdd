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
constexpr int kRowWords = 8;   // row-level record: tb, te, dpos, slot_off | kind, t, succ_b, succ_e
constexpr std::int32_t kRowHot = 0x40000000;  // row_succ flag: push to the priority queue
// static schedule record per position: tb, L, dpos, slot_off | kind, t, npred, pred_off |
// first kPosInline predecessor items (-1 = none) | item id, 0, 0, 0
constexpr int kPosWords = 16;
constexpr int kPosInline = 4;
// value-flow schedule (mode 5) record per position: tb, L | kind << 30, dpos, t
constexpr int kFlowWords = 4;
constexpr int kFlowKindShift = 30;
// mode 6: operand positions with this bit index the unit's shared-memory values
constexpr std::uint32_t kLocalBit = 0x80000000u;

struct PlanOptions {
  double cta_cost = 64.0;  // estimated warp-steps one CTA should get before a helper joins
  int max_width = 64;      // most CTAs cooperating on one task
  double dep_wide_cost = 64.0;  // Chol/Trsm go multi-CTA only above this cost per level
  double hot_fraction = 0.6;    // rows with height >= this fraction of the max are "hot"
  bool programs = true;    // precompute per-row update programs (slot_rec / upd)
  bool flow_merge_rows = true;  // mode 5: one unit per matrix row when its U row has <= 32 entries
  int unit_min_rows = 64;  // mode 6: diagonal blocks above this many rows become units
  std::int64_t unit_smem_cap = 72 * 1024;  // ... if their values fit in this many bytes
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
  std::int64_t item_edges = 0;     // row-level dependences
  std::int32_t item_depth = 0;     // longest row-level chain, in items
  std::int64_t flow_rows = 0;      // value-flow rows (Chol/Trsm items; they partition U)
  std::int32_t flow_depth = 0;     // longest value-flow chain, in rows
  std::int64_t unit_count = 0;     // mode 6 block units
  std::int64_t unit_rows = 0;      // rows inside units
  std::int32_t unit_depth = 0;     // longest chain of units and rows
  std::int32_t unit_max_levels = 0;  // most intra-unit levels
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
  // row-level execution: per item, the items it must follow (rows it reads
  // and the previous writer of its own row), derived from the same walk
  std::vector<std::int64_t> item_dep_ptr;
  std::vector<std::int32_t> item_dep;
  std::vector<std::int32_t> row_rec;    // kRowWords per item
  std::vector<std::int32_t> row_succ;   // successor items, grouped per item
  std::vector<std::int32_t> row_indeg;  // dependence counters per item
  std::vector<std::int32_t> row_roots;  // items with no dependence, by falling height
  std::vector<std::int32_t> row_height; // longest row chain from an item to the end
  std::vector<std::int32_t> row_level;  // longest row chain from a root to the item (1-based)
  std::vector<std::int32_t> row_order;  // static schedule: rows by (level, falling height)
  std::vector<std::int32_t> row_pred_ptr;  // int32 copy of item_dep_ptr (preds = item_dep)
  std::vector<std::int32_t> pos_rec;   // kPosWords per schedule position
  std::vector<std::int32_t> pos_pred;  // predecessor items beyond the inline ones
  // value-flow schedule (mode 5): every coordinate of U is written once, by
  // the Chol/Trsm item owning it, which applies all of its updates (the
  // Herk/Gemm items' products folded in, generation order kept)
  std::vector<std::int32_t> flow_rec;   // kFlowWords per schedule position
  std::vector<std::int32_t> flow_item;  // per schedule position: its item
  std::vector<std::int32_t> flow_slot;  // per coordinate of U: {u_b, u_e, m0, o0}
  std::vector<std::int32_t> flow_upd;   // (m, o) pairs
  std::vector<std::int32_t> flow_owner; // per coordinate of U: the item writing it
  std::vector<std::int32_t> flow_pos;   // per coordinate of U: the schedule position writing it
  // mode 6 (block units): rows outside units in schedule order; units with
  // their rows by intra-unit level; programs with local operands rewritten
  std::vector<std::int32_t> m6_row_rec;   // kFlowWords per row
  std::vector<std::int32_t> m6_row_item;
  std::vector<std::int32_t> m6_row_node;  // position of the row in the joint order
  std::vector<std::int32_t> m6_unit_rec;  // per unit: level slot begin/end, first row, node position
  std::vector<std::int32_t> m6_urow_rec;  // kFlowWords per unit row
  std::vector<std::int32_t> m6_urow_lbase;  // first shared-memory index of the row's values
  std::vector<std::int32_t> m6_urow_item;
  std::vector<std::int32_t> m6_ulev;      // per level slot: end of its rows
  std::vector<std::int32_t> m6_slot;      // like flow_slot / flow_upd, local operands rewritten
  std::vector<std::int32_t> m6_upd;
  std::int32_t m6_units = 0;
  std::int64_t m6_smem = 0;               // largest unit, bytes
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

// One part of a sharded value-flow factorization (C6: ND subtrees on
// different GPUs). The part runs the rows t with part_of_row[t] == part, in
// the global schedule order; an operand owned by another part is encoded as
// kRemoteBit | (owner << kRemoteShift) | position and read from the owner's
// copy of U (peer memory). Programs are compacted to the part's coordinates.
// A row some other part reads carries bit 31 in its length word and
// publishes its values at system scope.
constexpr std::uint32_t kRemoteBit = 0x80000000u;
constexpr int kRemoteShift = 25;  // positions below 2^25, owners below 64
struct FlowPart {
  std::vector<std::int32_t> rec, item;   // kFlowWords per row, schedule order
  std::vector<std::int32_t> slot;        // 4 per coordinate of U (zero outside the part)
  std::vector<std::int32_t> upd;         // the part's products
  std::int64_t remote_operands = 0;      // products reading another part
  std::int64_t exported_rows = 0;        // rows another part reads (rec word 1, bit 31)
  std::int64_t rows = 0;
};
FlowPart build_flow_part(const Plan& P, const std::vector<std::int32_t>& part_of_row, std::int32_t nparts,
                         std::int32_t part);

}  // namespace tcb
