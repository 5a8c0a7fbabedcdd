// Host flattener: block layout, task DAG and per-task gather work.
#include "plan.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <atomic>
#include <limits>
#include <thread>
#include <stdexcept>

namespace tcb {

namespace {
double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

offset_t BlockLayout::find(index_t i, index_t j) const {
  const auto b = bcol_idx.begin() + brow_ptr[i];
  const auto e = bcol_idx.begin() + brow_ptr[i + 1];
  const auto it = std::lower_bound(b, e, j);
  return (it == e || *it != j) ? -1 : static_cast<offset_t>(it - bcol_idx.begin());
}

BlockLayout build_block_layout(const CsrMatrix& u, const RangeList& ranges) {
  // Block (I, J), I <= J, exists iff U has an entry in rows ranges[I] x
  // columns ranges[J] (reference block_layout.hpp:71-72, :98-181). Each
  // U row is cut at range borders; every slice lands in exactly one block.
  validate_ranges(ranges, u.nrows);
  if (u.nnz() > std::numeric_limits<std::int32_t>::max())
    throw std::invalid_argument("factor has more than 2^31-1 entries");
  const index_t m = ranges.count();
  std::vector<index_t> owner(u.nrows);
  for (index_t r = 0; r < m; ++r)
    for (index_t c = ranges.ranges[r].begin; c < ranges.ranges[r].end; ++c) owner[c] = r;

  BlockLayout bl;
  bl.m = m;
  bl.brow_ptr.assign(static_cast<std::size_t>(m) + 1, 0);
  std::vector<index_t> stamp(m, -1);
  std::vector<index_t> present;
  for (index_t bi = 0; bi < m; ++bi) {
    present.clear();
    for (index_t i = ranges.ranges[bi].begin; i < ranges.ranges[bi].end; ++i) {
      for (offset_t q = u.row_begin(i); q < u.row_end(i);) {
        const index_t bj = owner[u.col_idx[q]];
        if (stamp[bj] != bi) {
          stamp[bj] = bi;
          present.push_back(bj);
        }
        const index_t stop = ranges.ranges[bj].end;
        while (q < u.row_end(i) && u.col_idx[q] < stop) ++q;
      }
    }
    std::sort(present.begin(), present.end());
    bl.bcol_idx.insert(bl.bcol_idx.end(), present.begin(), present.end());
    bl.brow_ptr[bi + 1] = static_cast<offset_t>(bl.bcol_idx.size());
  }

  const offset_t nb = bl.nblocks();
  bl.span_off.assign(static_cast<std::size_t>(nb) + 1, 0);
  for (index_t bi = 0; bi < m; ++bi)
    for (offset_t q = bl.brow_ptr[bi]; q < bl.brow_ptr[bi + 1]; ++q)
      bl.span_off[q + 1] = bl.span_off[q] + ranges.ranges[bi].size();
  bl.span_b.assign(static_cast<std::size_t>(bl.span_off[nb]), 0);
  bl.span_e.assign(static_cast<std::size_t>(bl.span_off[nb]), 0);
  // anchor every slice at its row start; non-empty ones are overwritten
  for (index_t bi = 0; bi < m; ++bi)
    for (offset_t q = bl.brow_ptr[bi]; q < bl.brow_ptr[bi + 1]; ++q)
      for (index_t r = 0; r < ranges.ranges[bi].size(); ++r) {
        const auto anchor = static_cast<std::int32_t>(u.row_begin(ranges.ranges[bi].begin + r));
        bl.span_b[bl.span_off[q] + r] = anchor;
        bl.span_e[bl.span_off[q] + r] = anchor;
      }
  for (index_t bi = 0; bi < m; ++bi) {
    const index_t rb = ranges.ranges[bi].begin;
    offset_t blk = bl.brow_ptr[bi];
    for (index_t i = rb; i < ranges.ranges[bi].end; ++i) {
      blk = bl.brow_ptr[bi];
      for (offset_t q = u.row_begin(i); q < u.row_end(i);) {
        const index_t bj = owner[u.col_idx[q]];
        const index_t stop = ranges.ranges[bj].end;
        const offset_t s = q;
        while (q < u.row_end(i) && u.col_idx[q] < stop) ++q;
        while (bl.bcol_idx[blk] != bj) ++blk;  // block columns ascend along the row
        bl.span_b[bl.span_off[blk] + (i - rb)] = static_cast<std::int32_t>(s);
        bl.span_e[bl.span_off[blk] + (i - rb)] = static_cast<std::int32_t>(q);
      }
    }
  }
  return bl;
}

namespace {

// Per-block transposed index: for every block, its non-empty columns t
// (ascending) with the slice of U's column t that falls in the block's rows.
struct BlockColumns {
  std::vector<offset_t> ptr;          // per block into col/slice arrays
  std::vector<std::int32_t> col;      // t
  std::vector<std::int32_t> cb, ce;   // slice [cb, ce) of the CSC arrays
  std::vector<std::int32_t> csc_row;  // r, ascending per column
  std::vector<std::int32_t> csc_pos;  // position of U(r, t)
};

BlockColumns transpose_blocks(const CsrMatrix& u, const RangeList& ranges,
                              const BlockLayout& bl) {
  const index_t n = u.nrows;
  BlockColumns bc;
  std::vector<std::int64_t> cptr(static_cast<std::size_t>(n) + 1, 0);
  for (offset_t q = 0; q < u.nnz(); ++q) ++cptr[u.col_idx[q] + 1];
  for (index_t t = 0; t < n; ++t) cptr[t + 1] += cptr[t];
  bc.csc_row.resize(static_cast<std::size_t>(u.nnz()));
  bc.csc_pos.resize(static_cast<std::size_t>(u.nnz()));
  {
    std::vector<std::int64_t> fill(cptr.begin(), cptr.end() - 1);
    for (index_t r = 0; r < n; ++r)
      for (offset_t q = u.row_begin(r); q < u.row_end(r); ++q) {
        const std::int64_t at = fill[u.col_idx[q]]++;
        bc.csc_row[at] = r;
        bc.csc_pos[at] = static_cast<std::int32_t>(q);
      }
  }
  std::vector<index_t> owner(n);
  for (index_t r = 0; r < ranges.count(); ++r)
    for (index_t c = ranges.ranges[r].begin; c < ranges.ranges[r].end; ++c) owner[c] = r;

  const offset_t nb = bl.nblocks();
  std::vector<std::int64_t> count(static_cast<std::size_t>(nb), 0);
  // pass 1: count column runs per block
  for (index_t t = 0; t < n; ++t) {
    const index_t bj = owner[t];
    for (std::int64_t h = cptr[t]; h < cptr[t + 1];) {
      const index_t bi = owner[bc.csc_row[h]];
      const index_t stop = ranges.ranges[bi].end;
      while (h < cptr[t + 1] && bc.csc_row[h] < stop) ++h;
      ++count[bl.find(bi, bj)];
    }
  }
  bc.ptr.assign(static_cast<std::size_t>(nb) + 1, 0);
  for (offset_t b = 0; b < nb; ++b) bc.ptr[b + 1] = bc.ptr[b] + count[b];
  bc.col.resize(static_cast<std::size_t>(bc.ptr[nb]));
  bc.cb.resize(bc.col.size());
  bc.ce.resize(bc.col.size());
  std::vector<std::int64_t> fill(bc.ptr.begin(), bc.ptr.end() - 1);
  for (index_t t = 0; t < n; ++t) {
    const index_t bj = owner[t];
    for (std::int64_t h = cptr[t]; h < cptr[t + 1];) {
      const index_t bi = owner[bc.csc_row[h]];
      const index_t stop = ranges.ranges[bi].end;
      const std::int64_t s = h;
      while (h < cptr[t + 1] && bc.csc_row[h] < stop) ++h;
      const offset_t b = bl.find(bi, bj);
      const std::int64_t at = fill[b]++;
      bc.col[at] = t;
      bc.cb[at] = static_cast<std::int32_t>(s);
      bc.ce[at] = static_cast<std::int32_t>(h);
    }
  }
  return bc;
}

// Update programs: the sorted-index merge of every (item, source) pair done
// once on the host. For item i with target slice [tb, te) (L slots), slot k
// has the record slot_rec[off_i + k] = {u_b, u_e, m0, o0}: its updates are
// the (m, o) position pairs upd[u_b .. u_e), each meaning U[tb + k] -= U[m] *
// U[o], in ascending source row (the reference's per-coordinate order), and
// (m0, o0) repeats the first of them so the device can start gathering right
// after one load. Entries whose column is absent from the target row are
// dropped here (kernels.hpp:62-63).
void build_programs(Plan& P, int threads) {
  const std::size_t I = P.item_rec.size() / kItemWords;
  std::vector<std::int64_t> slot_off(I + 1, 0), upd_off(I + 1, 0);
  for (std::size_t i = 0; i < I; ++i) {
    const std::int32_t* r = &P.item_rec[i * kItemWords];
    slot_off[i + 1] = slot_off[i] + (r[1] - r[0]);
  }
  if (slot_off[I] > std::numeric_limits<std::int32_t>::max())
    throw std::invalid_argument("plan: update-program slot table exceeds 2^31 entries");
  const int nt = std::max(1, threads > 0 ? threads
                                         : static_cast<int>(std::thread::hardware_concurrency()));
  auto parallel = [&](auto&& body) {
    std::atomic<std::size_t> next{0};
    auto run = [&]() {
      constexpr std::size_t kChunk = 512;
      while (true) {
        const std::size_t b = next.fetch_add(kChunk);
        if (b >= I) break;
        for (std::size_t i = b; i < std::min(I, b + kChunk); ++i) body(i);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(run);
    run();
    for (auto& th : pool) th.join();
  };
  // merge one item: calls hit(slot, m, o) for every surviving update, in order
  auto merge_item = [&](std::size_t i, auto&& hit) {
    const std::int32_t* r = &P.item_rec[i * kItemWords];
    const std::int32_t* tc = P.cols.data() + r[0];
    const std::int32_t L = r[1] - r[0];
    for (std::int32_t s = r[4]; s < r[5]; ++s) {
      const std::int32_t* sr = &P.src_rec[static_cast<std::size_t>(s) * kSrcWords];
      std::int32_t k = 0;
      for (std::int32_t e = sr[2]; e < sr[3] && k < L; ++e) {
        k = static_cast<std::int32_t>(std::lower_bound(tc + k, tc + L, P.cols[e]) - tc);
        if (k < L && tc[k] == P.cols[e]) hit(k, sr[1], e);
      }
    }
  };
  std::vector<std::int64_t> count(I, 0);
  parallel([&](std::size_t i) {
    std::int64_t c = 0;
    merge_item(i, [&](std::int32_t, std::int32_t, std::int32_t) { ++c; });
    count[i] = c;
  });
  for (std::size_t i = 0; i < I; ++i) upd_off[i + 1] = upd_off[i] + count[i];
  if (upd_off[I] > std::numeric_limits<std::int32_t>::max())
    throw std::invalid_argument("plan: update program exceeds 2^31 updates");
  P.slot_rec.assign(static_cast<std::size_t>(4 * slot_off[I]), 0);
  P.upd.assign(static_cast<std::size_t>(2 * upd_off[I]), 0);
  parallel([&](std::size_t i) {
    std::int32_t* r = &P.item_rec[i * kItemWords];
    const std::int32_t L = r[1] - r[0];
    std::vector<std::int32_t> sp(static_cast<std::size_t>(L) + 1, 0);
    merge_item(i, [&](std::int32_t k, std::int32_t, std::int32_t) { ++sp[k + 1]; });
    for (std::int32_t k = 0; k < L; ++k) sp[k + 1] += sp[k];
    std::vector<std::int32_t> fill(sp.begin(), sp.end() - 1);
    const std::int64_t base = upd_off[i];
    merge_item(i, [&](std::int32_t k, std::int32_t m, std::int32_t o) {
      const std::int64_t at = base + fill[k]++;
      P.upd[2 * at] = m;
      P.upd[2 * at + 1] = o;
    });
    std::int32_t* sr = &P.slot_rec[static_cast<std::size_t>(4 * slot_off[i])];
    for (std::int32_t k = 0; k < L; ++k) {
      const std::int64_t ub = base + sp[k], ue = base + sp[k + 1];
      sr[4 * k] = static_cast<std::int32_t>(ub);
      sr[4 * k + 1] = static_cast<std::int32_t>(ue);
      sr[4 * k + 2] = ub < ue ? P.upd[2 * ub] : 0;
      sr[4 * k + 3] = ub < ue ? P.upd[2 * ub + 1] : 0;
    }
    r[6] = static_cast<std::int32_t>(slot_off[i]);
  });
  P.stats.updates = upd_off[I];
}

// Row-level dependences. Every coordinate of U receives its updates in
// ascending source row as long as (a) the items writing the same (block,
// row) slice run in generation order and (b) an item reads only slices that
// are final. So an item follows: the previous item writing its own slice,
// and the last writer of every slice it reads (multipliers U(r,t), operand
// rows U(r,:), the Trsm divisor U(t,t)). These are exactly the block-level
// edges of the generation walk (factorize.hpp:175-224) restricted to the
// rows that actually interact.
void build_item_deps(Plan& P, const RangeList& ranges, double opt_hot_fraction) {
  const BlockLayout& bl = P.blocks;
  const std::size_t I = P.item_rec.size() / kItemWords;
  const std::size_t T = P.node_kind.size();
  std::vector<std::int32_t> row0(static_cast<std::size_t>(bl.nblocks()));
  for (index_t bi = 0; bi < bl.m; ++bi)
    for (offset_t q = bl.brow_ptr[bi]; q < bl.brow_ptr[bi + 1]; ++q) row0[q] = ranges.ranges[bi].begin;
  std::vector<std::int32_t> last(static_cast<std::size_t>(bl.span_off.back()), -1);
  auto slot = [&](std::int32_t blk, std::int32_t row) -> std::int32_t& {
    return last[static_cast<std::size_t>(bl.span_off[blk] + (row - row0[blk]))];
  };
  P.item_dep_ptr.assign(I + 1, 0);
  P.item_dep.clear();
  P.item_dep.reserve(3 * I);
  std::vector<std::int32_t> depth(I, 1), deps;
  for (std::size_t tk = 0; tk < T; ++tk) {
    const std::int32_t* rec = &P.task_rec[tk * kTaskWords];
    const std::int32_t kind = rec[0], ib = rec[2], ie = rec[3];
    const std::int32_t tgt = P.task_blk[4 * tk], mult = P.task_blk[4 * tk + 1],
                       oper = P.task_blk[4 * tk + 2];
    for (std::int32_t k = ib; k < ie; ++k) {
      const std::int32_t* it = &P.item_rec[static_cast<std::size_t>(k) * kItemWords];
      const std::int32_t t = it[7];
      deps.clear();
      if (slot(tgt, t) >= 0) deps.push_back(slot(tgt, t));
      if (kind == kTrsm) deps.push_back(slot(mult, t));  // U(t,t)
      for (std::int32_t s = it[4]; s < it[5]; ++s) {
        const std::int32_t d = P.src_rec[static_cast<std::size_t>(s) * kSrcWords];
        if (kind == kChol) {
          deps.push_back(ib + d);
        } else if (kind == kTrsm) {
          const std::int32_t r = row0[mult] + P.item_rec[static_cast<std::size_t>(ib + d) * kItemWords + 2];
          deps.push_back(slot(mult, r));  // U(r,t), written by Chol(p)
          deps.push_back(ib + d);         // row r of this panel
        } else {
          const std::int32_t rg = row0[oper] + d;  // d: row within block row p
          deps.push_back(slot(mult, rg));
          if (oper != mult) deps.push_back(slot(oper, rg));
        }
      }
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      std::int32_t dp = 1;
      for (std::int32_t d : deps) {
        if (d < 0 || d >= k) throw std::logic_error("plan: row dependence out of order");
        P.item_dep.push_back(d);
        dp = std::max(dp, depth[d] + 1);
      }
      depth[k] = dp;
      P.item_dep_ptr[k + 1] = static_cast<std::int64_t>(P.item_dep.size());
      slot(tgt, t) = k;
    }
  }
  P.stats.item_edges = static_cast<std::int64_t>(P.item_dep.size());
  P.stats.item_depth = I ? *std::max_element(depth.begin(), depth.end()) : 0;
  P.row_level = depth;

  // device tables of the row-level mode: successor CSR, counters, roots and
  // a self-contained record per row {tb, te, dpos, slot_off | kind, t, succ_b, succ_e}
  std::vector<std::int32_t> cnt(I + 1, 0);
  for (std::int32_t d : P.item_dep) ++cnt[d + 1];
  for (std::size_t k = 0; k < I; ++k) cnt[k + 1] += cnt[k];
  P.row_succ.assign(P.item_dep.size(), 0);
  P.row_indeg.assign(I, 0);
  std::vector<std::int32_t> fill(cnt.begin(), cnt.end() - 1);
  for (std::size_t k = 0; k < I; ++k)
    for (std::int64_t e = P.item_dep_ptr[k]; e < P.item_dep_ptr[k + 1]; ++e) {
      P.row_succ[fill[P.item_dep[e]]++] = static_cast<std::int32_t>(k);
      ++P.row_indeg[k];
    }
  // Scheduling priority: the height of a row (longest chain of rows still
  // to run after it). Successor lists are sorted by falling height so that
  // the continuation a warp keeps is the most critical ready row, and rows
  // in the top part of the height range are flagged (kRowHot) for the
  // device's priority queue.
  P.row_height.assign(I, 1);
  for (std::size_t k = I; k-- > 0;)
    for (std::int32_t e = cnt[k]; e < cnt[k + 1]; ++e)
      P.row_height[k] = std::max(P.row_height[k], P.row_height[P.row_succ[e]] + 1);
  const std::int32_t hmax = I ? *std::max_element(P.row_height.begin(), P.row_height.end()) : 0;
  const std::int32_t hot = std::max<std::int32_t>(1, static_cast<std::int32_t>(hmax * opt_hot_fraction));
  for (std::size_t k = 0; k < I; ++k) {
    std::sort(P.row_succ.begin() + cnt[k], P.row_succ.begin() + cnt[k + 1],
              [&](std::int32_t x, std::int32_t y) {
                return P.row_height[x] != P.row_height[y] ? P.row_height[x] > P.row_height[y] : x < y;
              });
    for (std::int32_t e = cnt[k]; e < cnt[k + 1]; ++e)
      if (P.row_height[P.row_succ[e]] >= hot) P.row_succ[e] |= kRowHot;
  }
  P.row_rec.assign(I * kRowWords, 0);
  P.row_roots.clear();
  for (std::size_t tk = 0; tk < T; ++tk) {
    const std::int32_t* rec = &P.task_rec[tk * kTaskWords];
    for (std::int32_t k = rec[2]; k < rec[3]; ++k) {
      const std::int32_t* it = &P.item_rec[static_cast<std::size_t>(k) * kItemWords];
      std::int32_t* r = &P.row_rec[static_cast<std::size_t>(k) * kRowWords];
      r[0] = it[0];
      r[1] = it[1];
      r[2] = it[3];
      r[3] = it[6];
      r[4] = rec[0];
      r[5] = it[7];
      r[6] = cnt[k];
      r[7] = cnt[k + 1];
      if (P.row_indeg[k] == 0) P.row_roots.push_back(k);
    }
  }
  std::stable_sort(P.row_roots.begin(), P.row_roots.end(), [&](std::int32_t x, std::int32_t y) {
    return P.row_height[x] > P.row_height[y];
  });

  // static schedule (mode 4): rows by level (a topological order), most
  // critical first within a level; warp w of W takes positions w, w+W, ...
  P.row_order.resize(I);
  for (std::size_t k = 0; k < I; ++k) P.row_order[k] = static_cast<std::int32_t>(k);
  std::stable_sort(P.row_order.begin(), P.row_order.end(), [&](std::int32_t x, std::int32_t y) {
    if (P.row_level[x] != P.row_level[y]) return P.row_level[x] < P.row_level[y];
    return P.row_height[x] > P.row_height[y];
  });
  P.row_pred_ptr.resize(I + 1);
  for (std::size_t k = 0; k <= I; ++k) P.row_pred_ptr[k] = static_cast<std::int32_t>(P.item_dep_ptr[k]);

  // Position-ordered records for the static schedule: everything a warp
  // needs for the row at position q in one 64-byte record. Predecessors are
  // named by item id (the first kPosInline inline, the rest in pos_pred):
  // the row stamps are indexed by item, which scatters the stamps of rows
  // that run at the same time over different cache lines (positions would
  // pack 32 concurrently written stamps into one line).
  std::vector<std::int32_t> pos_of(I);
  for (std::size_t q = 0; q < I; ++q) pos_of[P.row_order[q]] = static_cast<std::int32_t>(q);
  P.pos_rec.assign(I * kPosWords, -1);
  P.pos_pred.clear();
  for (std::size_t q = 0; q < I; ++q) {
    const std::int32_t k = P.row_order[q];
    const std::int32_t* r = &P.row_rec[static_cast<std::size_t>(k) * kRowWords];
    std::int32_t* o = &P.pos_rec[q * kPosWords];
    o[0] = r[0];
    o[1] = r[1] - r[0];
    o[2] = r[2];
    o[3] = r[3];
    o[4] = r[4];
    o[5] = r[5];
    const std::int64_t pb = P.item_dep_ptr[k], pe = P.item_dep_ptr[k + 1];
    o[6] = static_cast<std::int32_t>(pe - pb);
    o[7] = static_cast<std::int32_t>(P.pos_pred.size());
    o[12] = k;
    for (std::int64_t e = pb; e < pe; ++e) {
      const std::int32_t d = P.item_dep[e];
      if (pos_of[d] >= static_cast<std::int32_t>(q)) throw std::logic_error("plan: schedule not topological");
      if (e - pb < kPosInline)
        o[8 + (e - pb)] = d;
      else
        P.pos_pred.push_back(d);
    }
  }
}

// Value-flow schedule (mode 5). The Chol/Trsm items partition U: each
// coordinate is finalised by exactly one of them, and every Herk/Gemm item
// on the same slice runs before it (the own-slice chain above). Folding the
// Herk/Gemm products into the finaliser's program, in item (generation)
// order, keeps the per-coordinate product order ascending in source row, so
// the result stays bitwise equal to factor_serial while every coordinate is
// written once. A reader then needs no flag: it polls the value itself
// until the writer has replaced the "not yet written" marker (flow_kernel.cu).
// Schedule: finalisers by (level, falling height) over the dependences
// "reads a coordinate owned by", which point to earlier items.
//
// (Measured alternative, not kept: cutting the chains into several
// segments that hand partial values on through scratch, so heavy Herk/Gemm
// work runs early. On B200 it lost on every acceptance config -- C2 0.69 ->
// 0.83 ms, C3 7.6 -> 17 ms -- the extra rows cost more than the shorter
// finaliser programs saved.)
void build_flow(Plan& P, const CsrMatrix& u, bool merge_rows) {
  const std::size_t I = P.item_rec.size() / kItemWords;
  const std::size_t N = static_cast<std::size_t>(P.nnz);
  auto R = [&](std::size_t k, int w) { return P.row_rec[k * kRowWords + w]; };
  // every coordinate's finalising item, and per matrix row its Chol item
  std::vector<std::int32_t> fin_item(N, -1), chol_of_row(static_cast<std::size_t>(P.n), -1);
  for (std::size_t k = 0; k < I; ++k)
    if (R(k, 4) <= kTrsm) {
      if (R(k, 4) == kChol) chol_of_row[R(k, 5)] = static_cast<std::int32_t>(k);
      for (std::int32_t x = R(k, 0); x < R(k, 1); ++x) {
        if (fin_item[x] >= 0) throw std::logic_error("flow: coordinate finalised twice");
        fin_item[x] = static_cast<std::int32_t>(k);
      }
    }
  for (std::size_t x = 0; x < N; ++x)
    if (fin_item[x] < 0) throw std::logic_error("flow: coordinate without a finaliser");
  // The rows the schedule runs ("units"). The Chol and Trsm items of a
  // matrix row share the divisor U(t,t) and nearly all their sources (every
  // coordinate (t,c) takes U(r,t)*U(r,c) over the same rows r), so with
  // merge_rows a U row of at most 32 entries is one unit (one warp pass, the
  // per-row cost paid once); a longer row keeps its diagonal-block slice (the
  // Chol item, which the next rows of the block chain read) and cuts the rest
  // into warp-wide chunks that divide by U(t,t). Without merge_rows, one unit
  // per Chol/Trsm item. Units are in (row, Chol first) order, which is
  // topological: every operand comes from a row above.
  struct Unit {
    std::int32_t tb, L, dpos, kind, t, item;
  };
  std::vector<Unit> units;
  std::vector<std::int32_t> unit_of(N, -1);
  std::vector<std::vector<std::int32_t>> items_of_row(static_cast<std::size_t>(P.n));
  for (std::size_t k = 0; k < I; ++k)
    if (R(k, 4) == kTrsm) items_of_row[R(k, 5)].push_back(static_cast<std::int32_t>(k));
  for (index_t t = 0; t < P.n; ++t) {
    const std::int32_t ck = chol_of_row[t];
    if (ck < 0) throw std::logic_error("flow: row without a Chol item");
    const auto rb = static_cast<std::int32_t>(u.row_begin(t)), re = static_cast<std::int32_t>(u.row_end(t));
    if (merge_rows && re - rb <= 32) {  // the whole row in one warp pass
      units.push_back({rb, re - rb, rb, kChol, static_cast<std::int32_t>(t), ck});
      continue;
    }
    if (merge_rows) {  // the diagonal-block slice, then the rest of the row in warp-wide chunks
      units.push_back({R(ck, 0), R(ck, 1) - R(ck, 0), R(ck, 2), kChol, static_cast<std::int32_t>(t), ck});
      for (std::int32_t c0 = R(ck, 1); c0 < re; c0 += 32)
        units.push_back({c0, std::min(re - c0, 32), R(ck, 2), kTrsm, static_cast<std::int32_t>(t),
                         fin_item[static_cast<std::size_t>(c0)]});
      continue;
    }
    units.push_back({R(ck, 0), R(ck, 1) - R(ck, 0), R(ck, 2), kChol, static_cast<std::int32_t>(t), ck});
    for (std::int32_t k : items_of_row[t])
      units.push_back({R(k, 0), R(k, 1) - R(k, 0), R(k, 2), kTrsm, static_cast<std::int32_t>(t), k});
  }
  const std::size_t U = units.size();
  for (std::size_t g = 0; g < U; ++g)
    for (std::int32_t x = units[g].tb; x < units[g].tb + units[g].L; ++x) {
      if (unit_of[x] >= 0) throw std::logic_error("flow: coordinate in two units");
      unit_of[x] = static_cast<std::int32_t>(g);
    }
  // flow_owner (per coordinate): the item representing its unit (build_units / build_flow_part)
  P.flow_owner.assign(N, -1);
  for (std::size_t x = 0; x < N; ++x) P.flow_owner[x] = units[unit_of[x]].item;
  // merged programs: per coordinate, the products of every item on it in item order
  std::vector<std::int64_t> cnt(N + 1, 0);
  for (std::size_t k = 0; k < I; ++k)
    for (std::int32_t j = 0; j < R(k, 1) - R(k, 0); ++j) {
      const std::int32_t* s = &P.slot_rec[static_cast<std::size_t>(R(k, 3) + j) * 4];
      cnt[R(k, 0) + j + 1] += s[1] - s[0];
    }
  for (std::size_t x = 0; x < N; ++x) cnt[x + 1] += cnt[x];
  if (cnt[N] > 0x7fffffffLL) throw std::length_error("flow: more than 2^31 products");
  P.flow_upd.assign(static_cast<std::size_t>(2 * cnt[N]), 0);
  std::vector<std::int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (std::size_t k = 0; k < I; ++k)
    for (std::int32_t j = 0; j < R(k, 1) - R(k, 0); ++j) {
      const std::int32_t* s = &P.slot_rec[static_cast<std::size_t>(R(k, 3) + j) * 4];
      std::int64_t& f = fill[R(k, 0) + j];
      for (std::int32_t u = s[0]; u < s[1]; ++u, ++f) {
        P.flow_upd[2 * f] = P.upd[2 * static_cast<std::size_t>(u)];
        P.flow_upd[2 * f + 1] = P.upd[2 * static_cast<std::size_t>(u) + 1];
      }
    }
  P.flow_slot.assign(4 * N, 0);
  for (std::size_t x = 0; x < N; ++x) {
    std::int32_t* s = &P.flow_slot[4 * x];
    s[0] = static_cast<std::int32_t>(cnt[x]);
    s[1] = static_cast<std::int32_t>(cnt[x + 1]);
    if (s[0] < s[1]) {
      s[2] = P.flow_upd[2 * static_cast<std::size_t>(s[0])];
      s[3] = P.flow_upd[2 * static_cast<std::size_t>(s[0]) + 1];
    }
  }
  // levels (forward) and heights (backward) over "reads a coordinate owned by"
  std::vector<std::int32_t> level(U, 0), height(U, 0);
  auto each_src = [&](std::size_t g, auto&& fn) {
    if (units[g].kind == kTrsm) fn(unit_of[units[g].dpos]);  // divisor U(t,t)
    for (std::int32_t x = units[g].tb; x < units[g].tb + units[g].L; ++x)
      for (std::int64_t e = cnt[x]; e < cnt[x + 1]; ++e) {
        fn(unit_of[P.flow_upd[2 * e]]);
        fn(unit_of[P.flow_upd[2 * e + 1]]);
      }
  };
  std::int32_t depth = 0;
  for (std::size_t g = 0; g < U; ++g) {
    std::int32_t lv = 1;
    each_src(g, [&](std::int32_t sidx) {
      if (sidx < 0 || static_cast<std::size_t>(sidx) >= g) throw std::logic_error("flow: dependence out of order");
      lv = std::max(lv, level[sidx] + 1);
    });
    level[g] = lv;
    depth = std::max(depth, lv);
  }
  for (std::size_t g = U; g-- > 0;) {
    height[g] = std::max(height[g], 1);
    const std::int32_t h = height[g] + 1;
    each_src(g, [&](std::int32_t sidx) { height[sidx] = std::max(height[sidx], h); });
  }
  std::vector<std::int32_t> order(U);
  for (std::size_t g = 0; g < U; ++g) order[g] = static_cast<std::int32_t>(g);
  std::stable_sort(order.begin(), order.end(), [&](std::int32_t x, std::int32_t y) {
    if (level[x] != level[y]) return level[x] < level[y];
    return height[x] > height[y];
  });
  P.flow_rec.assign(U * kFlowWords, 0);
  P.flow_item.assign(U, 0);
  for (std::size_t q = 0; q < U; ++q) {
    const Unit& un = units[static_cast<std::size_t>(order[q])];
    if (un.L >= (1 << kFlowKindShift)) throw std::length_error("flow: row slice too long");
    std::int32_t* o = &P.flow_rec[q * kFlowWords];
    o[0] = un.tb;
    o[1] = un.L | (un.kind << kFlowKindShift);
    o[2] = un.dpos;
    o[3] = un.t;
    P.flow_item[q] = un.item;
  }
  // the schedule position writing each coordinate (a long item's chunks share
  // the item, so the item alone does not name the writing row)
  std::vector<std::int32_t> pos_of_unit(U);
  for (std::size_t q = 0; q < U; ++q) pos_of_unit[static_cast<std::size_t>(order[q])] = static_cast<std::int32_t>(q);
  P.flow_pos.assign(N, -1);
  for (std::size_t x = 0; x < N; ++x) P.flow_pos[x] = pos_of_unit[static_cast<std::size_t>(unit_of[x])];
  const std::int64_t nfin = static_cast<std::int64_t>(U);
  P.stats.flow_rows = nfin;
  P.stats.flow_depth = depth;
}

// Block units (mode 6). A chain of Chol rows inside one large diagonal
// block (an ND separator) is most of the critical path in mode 5: every link
// costs a cross-SM hand-off through L2 (C2: ~190 of the 214 steps of the
// longest chain sit in diagonal blocks of 114-3,072 rows). Here such a block
// becomes a unit executed by one CTA: its rows in intra-block level order,
// one __syncthreads between levels, and the block's own values kept in shared
// memory, so an intra-block operand costs a shared-memory load instead of a
// hand-off. Operands from other blocks are still polled in global memory.
// Programs are the mode-5 merged programs with every intra-unit operand
// position rewritten to kLocalBit | (its index in the unit's shared array).
// Everything that is not in a unit runs as in mode 5. The schedule orders
// units and rows by level over "reads a value written by" (a unit counts as
// one node); unit CTAs take the units and the other warps the rows, each
// list in that topological order, which keeps the launch deadlock-free.
void build_units(Plan& P, const RangeList& ranges, std::int32_t min_rows, std::int64_t smem_cap) {
  const std::size_t R = P.flow_item.size();
  const std::size_t N = static_cast<std::size_t>(P.nnz);
  auto F = [&](std::size_t q, int w) { return P.flow_rec[q * kFlowWords + w]; };
  auto len = [&](std::size_t q) { return F(q, 1) & ((1 << kFlowKindShift) - 1); };
  auto kind = [&](std::size_t q) { return static_cast<std::int32_t>(static_cast<std::uint32_t>(F(q, 1)) >> kFlowKindShift); };
  std::vector<std::int32_t> range_of(static_cast<std::size_t>(P.n));
  for (index_t r = 0; r < ranges.count(); ++r)
    for (index_t c = ranges.ranges[r].begin; c < ranges.ranges[r].end; ++c) range_of[c] = r;
  // candidate units: Chol rows of large diagonal blocks whose values fit
  // (only blocks whose Chol rows are the diagonal-block slices: a whole
  // matrix row run as one flow row, build_flow merge_rows, reaches into
  // blocks other rows of the chain read, which would tie a unit into a cycle)
  std::vector<std::int64_t> nloc(static_cast<std::size_t>(ranges.count()), 0);
  std::vector<char> whole_rows(static_cast<std::size_t>(ranges.count()), 0);
  for (std::size_t q = 0; q < R; ++q)
    if (kind(q) == kChol) {
      nloc[range_of[F(q, 3)]] += len(q);
      const std::size_t it = static_cast<std::size_t>(P.flow_item[q]);
      if (len(q) != P.row_rec[it * kRowWords + 1] - P.row_rec[it * kRowWords]) whole_rows[range_of[F(q, 3)]] = 1;
    }
  std::vector<std::int32_t> unit_of_range(static_cast<std::size_t>(ranges.count()), -1);
  std::int32_t nunits = 0;
  for (index_t r = 0; r < ranges.count(); ++r)
    if (min_rows > 0 && ranges.ranges[r].size() > min_rows && nloc[r] > 0 && nloc[r] * 8 <= smem_cap &&
        !whole_rows[r])
      unit_of_range[r] = nunits++;
  std::vector<std::int32_t> unit_of_pos(R, -1);
  for (std::size_t q = 0; q < R; ++q)
    if (kind(q) == kChol) unit_of_pos[q] = unit_of_range[range_of[F(q, 3)]];
  // local indices: unit rows in flow order, coordinates consecutive
  std::vector<std::int32_t> loc_of(N, -1), lbase(R, -1);
  std::vector<std::int64_t> ucount(static_cast<std::size_t>(nunits), 0);
  for (std::size_t q = 0; q < R; ++q) {
    const std::int32_t u = unit_of_pos[q];
    if (u < 0) continue;
    lbase[q] = static_cast<std::int32_t>(ucount[u]);
    for (std::int32_t j = 0; j < len(q); ++j) loc_of[F(q, 0) + j] = static_cast<std::int32_t>(ucount[u] + j);
    ucount[u] += len(q);
  }
  // programs with intra-unit operands rewritten
  P.m6_slot = P.flow_slot;
  P.m6_upd = P.flow_upd;
  auto unit_of_value = [&](std::int32_t pos) { return unit_of_pos[P.flow_pos[pos]]; };
  for (std::size_t q = 0; q < R; ++q) {
    const std::int32_t u = unit_of_pos[q];
    if (u < 0) continue;
    for (std::int32_t j = 0; j < len(q); ++j) {
      std::int32_t* sl = &P.m6_slot[4 * static_cast<std::size_t>(F(q, 0) + j)];
      for (std::int32_t e = sl[0]; e < sl[1]; ++e)
        for (int h = 0; h < 2; ++h) {
          std::int32_t& x = P.m6_upd[2 * static_cast<std::size_t>(e) + h];
          if (unit_of_value(x) == u) x = static_cast<std::int32_t>(kLocalBit | static_cast<std::uint32_t>(loc_of[x]));
        }
      if (sl[0] < sl[1]) {
        sl[2] = P.m6_upd[2 * static_cast<std::size_t>(sl[0])];
        sl[3] = P.m6_upd[2 * static_cast<std::size_t>(sl[0]) + 1];
      }
    }
  }
  // nodes: units 0..nunits-1, then rows outside units
  std::vector<std::int32_t> node_of_pos(R, -1);
  std::int32_t nn = nunits;
  for (std::size_t q = 0; q < R; ++q) node_of_pos[q] = unit_of_pos[q] >= 0 ? unit_of_pos[q] : nn++;
  // node dependences (unique), intra-unit levels
  std::vector<std::vector<std::int32_t>> deps(static_cast<std::size_t>(nn));
  std::vector<std::int32_t> ulevel(R, 0);
  for (std::size_t q = 0; q < R; ++q) {
    const std::int32_t me = node_of_pos[q];
    std::int32_t lv = 1;
    auto src = [&](std::int32_t pos) {
      const std::int32_t sq = P.flow_pos[pos];
      const std::int32_t sn = node_of_pos[sq];
      if (sn == me) lv = std::max(lv, ulevel[sq] + 1);
      else deps[me].push_back(sn);
    };
    if (kind(q) == kTrsm) src(F(q, 2));
    for (std::int32_t j = 0; j < len(q); ++j) {
      const std::int32_t* sl = &P.flow_slot[4 * static_cast<std::size_t>(F(q, 0) + j)];
      for (std::int32_t e = sl[0]; e < sl[1]; ++e) {
        src(P.flow_upd[2 * static_cast<std::size_t>(e)]);
        src(P.flow_upd[2 * static_cast<std::size_t>(e) + 1]);
      }
    }
    ulevel[q] = lv;
  }
  std::vector<std::int32_t> indeg(static_cast<std::size_t>(nn), 0), level(static_cast<std::size_t>(nn), 1);
  std::vector<std::vector<std::int32_t>> succ(static_cast<std::size_t>(nn));
  for (std::int32_t v = 0; v < nn; ++v) {
    auto& d = deps[v];
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    indeg[v] = static_cast<std::int32_t>(d.size());
    for (std::int32_t x : d) succ[x].push_back(v);
  }
  std::vector<std::int32_t> ready, topo;
  for (std::int32_t v = 0; v < nn; ++v)
    if (indeg[v] == 0) ready.push_back(v);
  while (!ready.empty()) {
    const std::int32_t v = ready.back();
    ready.pop_back();
    topo.push_back(v);
    for (std::int32_t w : succ[v]) {
      level[w] = std::max(level[w], level[v] + 1);
      if (--indeg[w] == 0) ready.push_back(w);
    }
  }
  if (static_cast<std::int32_t>(topo.size()) != nn) throw std::logic_error("units: dependence cycle");
  // first flow position of every node, for a stable order inside a level
  std::vector<std::int32_t> first(static_cast<std::size_t>(nn), std::numeric_limits<std::int32_t>::max());
  for (std::size_t q = 0; q < R; ++q)
    first[node_of_pos[q]] = std::min(first[node_of_pos[q]], static_cast<std::int32_t>(q));
  std::vector<std::int32_t> order(static_cast<std::size_t>(nn));
  for (std::int32_t v = 0; v < nn; ++v) order[v] = v;
  std::stable_sort(order.begin(), order.end(), [&](std::int32_t x, std::int32_t y) {
    return level[x] != level[y] ? level[x] < level[y] : first[x] < first[y];
  });
  std::vector<std::int32_t> pos_of_node(static_cast<std::size_t>(nn));
  for (std::int32_t k = 0; k < nn; ++k) pos_of_node[order[k]] = k;
  // rows: records in node order; units: rows by intra-unit level
  P.m6_row_rec.clear();
  P.m6_row_item.clear();
  P.m6_row_node.clear();
  std::vector<std::vector<std::int32_t>> urows(static_cast<std::size_t>(nunits));
  std::vector<std::int32_t> row_at_node(static_cast<std::size_t>(nn), -1);
  for (std::size_t q = 0; q < R; ++q) {
    if (unit_of_pos[q] >= 0) urows[unit_of_pos[q]].push_back(static_cast<std::int32_t>(q));
    else row_at_node[node_of_pos[q]] = static_cast<std::int32_t>(q);
  }
  P.m6_unit_rec.clear();
  P.m6_urow_rec.clear();
  P.m6_urow_lbase.clear();
  P.m6_urow_item.clear();
  P.m6_ulev.clear();
  std::int64_t smem_max = 0;
  std::int32_t depth_max = 0;
  for (std::int32_t k = 0; k < nn; ++k) {
    const std::int32_t v = order[k];
    if (v >= nunits) {
      const std::size_t q = static_cast<std::size_t>(row_at_node[v]);
      P.m6_row_rec.insert(P.m6_row_rec.end(), &P.flow_rec[q * kFlowWords], &P.flow_rec[q * kFlowWords] + kFlowWords);
      P.m6_row_item.push_back(P.flow_item[q]);
      P.m6_row_node.push_back(k);
      continue;
    }
    auto& rows = urows[v];
    std::stable_sort(rows.begin(), rows.end(), [&](std::int32_t x, std::int32_t y) { return ulevel[x] < ulevel[y]; });
    const auto rb = static_cast<std::int32_t>(P.m6_urow_item.size());
    const auto lb = static_cast<std::int32_t>(P.m6_ulev.size());
    std::int32_t cur = 0;
    for (std::int32_t q : rows) {
      if (ulevel[q] != cur) {
        P.m6_ulev.push_back(static_cast<std::int32_t>(P.m6_urow_item.size()));
        cur = ulevel[q];
      }
      P.m6_urow_rec.insert(P.m6_urow_rec.end(), &P.flow_rec[static_cast<std::size_t>(q) * kFlowWords],
                           &P.flow_rec[static_cast<std::size_t>(q) * kFlowWords] + kFlowWords);
      P.m6_urow_lbase.push_back(lbase[q]);
      P.m6_urow_item.push_back(P.flow_item[q]);
    }
    P.m6_ulev.push_back(static_cast<std::int32_t>(P.m6_urow_item.size()));
    const auto le = static_cast<std::int32_t>(P.m6_ulev.size());
    // {first level slot, end level slot, first row, node position}; level slot
    // l covers rows [ulev[l-1] or rb, ulev[l])
    P.m6_unit_rec.insert(P.m6_unit_rec.end(), {lb, le, rb, k});
    smem_max = std::max(smem_max, ucount[v] * 8);
    depth_max = std::max(depth_max, le - lb);
  }
  P.m6_units = nunits;
  P.m6_smem = smem_max;
  P.stats.unit_count = nunits;
  P.stats.unit_rows = static_cast<std::int64_t>(P.m6_urow_item.size());
  P.stats.unit_depth = level.empty() ? 0 : *std::max_element(level.begin(), level.end());
  P.stats.unit_max_levels = depth_max;
}

}  // namespace

Plan build_plan(const CsrMatrix& u, const std::vector<double>& init_values,
                const RangeList& ranges, bool with_work, const PlanOptions& opt) {
  if (u.nrows != u.ncols) throw std::invalid_argument("factor pattern not square");
  if (static_cast<offset_t>(init_values.size()) != u.nnz())
    throw std::invalid_argument("initial values do not match the pattern");
  Plan P;
  P.n = u.nrows;
  P.nnz = u.nnz();
  auto t0 = std::chrono::steady_clock::now();
  P.blocks = build_block_layout(u, ranges);
  P.stats.block_build_seconds = since(t0);
  t0 = std::chrono::steady_clock::now();
  const BlockLayout& bl = P.blocks;
  const index_t m = bl.m;

  // diagonal entries must lead every row (kernels.hpp:46-48)
  for (index_t i = 0; i < u.nrows; ++i)
    if (u.row_begin(i) == u.row_end(i) || u.col_idx[u.row_begin(i)] != i)
      throw std::invalid_argument("chol_block: missing diagonal entry in row " + std::to_string(i));

  P.cols.assign(u.col_idx.begin(), u.col_idx.end());
  P.values = init_values;

  BlockColumns bc;
  if (with_work) bc = transpose_blocks(u, ranges, bl);

  auto span = [&](offset_t blk, index_t local, std::int32_t& b, std::int32_t& e) {
    b = bl.span_b[bl.span_off[blk] + local];
    e = bl.span_e[bl.span_off[blk] + local];
  };

  std::vector<std::int32_t> last_writer(static_cast<std::size_t>(bl.nblocks()), -1);
  std::vector<std::int32_t>& tr = P.task_rec;
  std::vector<std::int32_t>& ir = P.item_rec;
  std::vector<std::int32_t>& sr = P.src_rec;

  auto new_task = [&](std::int32_t kind, index_t bi, index_t bj,
                      std::initializer_list<offset_t> reads, offset_t writes) -> std::int32_t {
    const auto id = static_cast<std::int32_t>(P.node_kind.size());
    P.node_kind.push_back(kind);
    P.node_i.push_back(bi);
    P.node_j.push_back(bj);
    for (offset_t blk : reads)
      if (last_writer[blk] >= 0) {
        P.edge_from.push_back(last_writer[blk]);
        P.edge_to.push_back(id);
      }
    last_writer[writes] = id;
    ++P.stats.tasks[kind];
    tr.insert(tr.end(), kTaskWords, 0);
    std::int32_t* rec = &tr[static_cast<std::size_t>(id) * kTaskWords];
    rec[0] = kind;
    rec[2] = rec[3] = static_cast<std::int32_t>(ir.size() / kItemWords);
    rec[8] = rec[9] = static_cast<std::int32_t>(sr.size() / kSrcWords);
    rec[10] = static_cast<std::int32_t>(writes);
    // blocks the rows of this task read: multipliers U(r,t) and operands U(r,c)
    const offset_t* rd = reads.begin();
    const offset_t mult = rd[0];
    const offset_t oper = (kind == kTrsm || kind == kGemm) ? rd[1] : rd[0];
    P.task_blk.insert(P.task_blk.end(), {static_cast<std::int32_t>(writes),
                                         static_cast<std::int32_t>(mult),
                                         static_cast<std::int32_t>(oper), 0});
    return id;
  };
  auto add_item = [&](std::int32_t tb, std::int32_t te, std::int32_t local, std::int32_t dpos,
                      std::int64_t src_begin, std::int32_t t) {
    const std::int64_t src_end = static_cast<std::int64_t>(sr.size() / kSrcWords);
    ir.insert(ir.end(), {tb, te, local, dpos, static_cast<std::int32_t>(src_begin),
                         static_cast<std::int32_t>(src_end), 0, t});
    P.stats.max_target_len = std::max(P.stats.max_target_len, te - tb);
    ++P.stats.items;
  };
  auto add_src = [&](std::int32_t r_local, std::int32_t pos_rt, std::int32_t sb, std::int32_t se) {
    sr.insert(sr.end(), {r_local, pos_rt, sb, se});
    ++P.stats.sources;
    P.stats.pairs += se - sb;
  };
  // Per-task finishing pass:
  //  * Chol/Trsm rows depend on earlier rows of the same task. Items are
  //    re-ordered by intra-task level (stable, so ascending t inside a level)
  //    and each source's wait field is rewritten from "row r" to "position of
  //    row r's item", so that warps claiming items in order never wait on a
  //    row that is claimed later and rows of one level run concurrently.
  //  * the CTA width (how many CTAs cooperate on the task) from its size.
  std::vector<std::int32_t> item_of_row, level, order, tmp_items;
  auto close_task = [&](std::int32_t id) {
    std::int32_t* rec = &tr[static_cast<std::size_t>(id) * kTaskWords];
    const std::int32_t ib = rec[2];
    const auto ie = static_cast<std::int32_t>(ir.size() / kItemWords);
    rec[3] = ie;
    rec[9] = static_cast<std::int32_t>(sr.size() / kSrcWords);
    if (sr.size() / kSrcWords > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
      throw std::invalid_argument("plan: source table exceeds 2^31 records");
    const std::int32_t ni = ie - ib;
    double cost = 0.0;
    std::int32_t nlev = ni > 0 ? 1 : 0, widest = ni;
    for (std::int32_t it = ib; it < ie; ++it) {
      const std::int32_t* r = &ir[static_cast<std::size_t>(it) * kItemWords];
      std::int64_t pairs = 0;
      for (std::int32_t s = r[4]; s < r[5]; ++s)
        pairs += sr[static_cast<std::size_t>(s) * kSrcWords + 3] - sr[static_cast<std::size_t>(s) * kSrcWords + 2];
      cost += 2.0 + (r[5] - r[4]) / 8.0 + static_cast<double>(pairs) / 32.0 + (r[1] - r[0]) / 32.0;
    }
    if ((rec[0] == kChol || rec[0] == kTrsm) && ni > 0) {
      const std::int32_t nrows = rec[1];
      item_of_row.assign(static_cast<std::size_t>(nrows), -1);
      for (std::int32_t it = ib; it < ie; ++it)
        item_of_row[ir[static_cast<std::size_t>(it) * kItemWords + 2]] = it - ib;
      level.assign(static_cast<std::size_t>(ni), 0);
      for (std::int32_t k = 0; k < ni; ++k) {  // items ascend in t: sources precede
        const std::int32_t* r = &ir[static_cast<std::size_t>(ib + k) * kItemWords];
        std::int32_t lv = 0;
        for (std::int32_t s = r[4]; s < r[5]; ++s) {
          const std::int32_t dep = item_of_row[sr[static_cast<std::size_t>(s) * kSrcWords]];
          if (dep < 0) throw std::logic_error("plan: source row without an item");
          lv = std::max(lv, level[dep] + 1);
        }
        level[k] = lv;
      }
      order.resize(static_cast<std::size_t>(ni));
      for (std::int32_t k = 0; k < ni; ++k) order[k] = k;
      std::stable_sort(order.begin(), order.end(),
                       [&](std::int32_t x, std::int32_t y) { return level[x] < level[y]; });
      std::vector<std::int32_t> pos(static_cast<std::size_t>(ni));
      for (std::int32_t k = 0; k < ni; ++k) pos[order[k]] = k;
      for (std::int32_t k = 0; k < ni; ++k) {
        const std::int32_t* r = &ir[static_cast<std::size_t>(ib + k) * kItemWords];
        for (std::int32_t s = r[4]; s < r[5]; ++s) {
          std::int32_t& w = sr[static_cast<std::size_t>(s) * kSrcWords];
          w = pos[item_of_row[w]];
        }
      }
      tmp_items.assign(ir.begin() + static_cast<std::ptrdiff_t>(ib) * kItemWords, ir.end());
      for (std::int32_t k = 0; k < ni; ++k)
        std::copy_n(&tmp_items[static_cast<std::size_t>(order[k]) * kItemWords], kItemWords,
                    &ir[static_cast<std::size_t>(ib + k) * kItemWords]);
      std::vector<std::int32_t> per_level;
      for (std::int32_t k = 0; k < ni; ++k) {
        if (level[k] >= static_cast<std::int32_t>(per_level.size())) per_level.resize(level[k] + 1, 0);
        ++per_level[level[k]];
      }
      nlev = static_cast<std::int32_t>(per_level.size());
      widest = *std::max_element(per_level.begin(), per_level.end());
    }
    // CTA width: enough CTAs to give each warp ~kCtaCost/8 steps, never more
    // warps than the widest level offers rows.
    std::int32_t width = static_cast<std::int32_t>(std::ceil(cost / opt.cta_cost));
    width = std::min(width, (widest + 7) / 8);
    // rows of a Chol/Trsm chain hand off through shared memory inside one
    // CTA (~0.3 us) but through global flags across CTAs (~1.4 us): spread
    // such a task only when a level carries more work than one CTA clears
    // in about one hand-off time
    if ((rec[0] == kChol || rec[0] == kTrsm) && cost < opt.dep_wide_cost * nlev) width = 1;
    width = std::max(1, std::min(width, opt.max_width));
    rec[1] = width;
    rec[7] = nlev;
    P.stats.max_width = std::max(P.stats.max_width, width);
    P.stats.helpers += width - 1;
  };

  for (index_t p = 0; p < m; ++p) {
    const offset_t rb = bl.brow_ptr[p], re = bl.brow_ptr[p + 1];
    if (rb == re || bl.bcol_idx[rb] != p)
      throw std::logic_error("factor_by_blocks: diagonal block missing");
    const Range Rp = ranges.ranges[p];

    // genTaskChol (factorize.hpp:177-184)
    {
      const std::int32_t id = new_task(kChol, p, p, {rb}, rb);
      tr[static_cast<std::size_t>(id) * kTaskWords + 1] = Rp.size();
      tr[static_cast<std::size_t>(id) * kTaskWords + 6] = Rp.begin;
      P.stats.max_flag_rows = std::max(P.stats.max_flag_rows, Rp.size());
      if (with_work) {
        // the diagonal block's columns are exactly Rp (full diagonal)
        for (std::int64_t h = bc.ptr[rb]; h < bc.ptr[rb + 1]; ++h) {
          const std::int32_t t = bc.col[h];
          std::int32_t tb, te;
          span(rb, t - Rp.begin, tb, te);
          const std::int64_t s0 = static_cast<std::int64_t>(sr.size() / kSrcWords);
          for (std::int32_t c = bc.cb[h]; c < bc.ce[h]; ++c) {
            const std::int32_t r = bc.csc_row[c];
            if (r == t) continue;  // the diagonal itself
            std::int32_t sb, se;
            span(rb, r - Rp.begin, sb, se);
            add_src(r - Rp.begin, bc.csc_pos[c], bc.csc_pos[c], se);
          }
          add_item(tb, te, t - Rp.begin, tb, s0, t);
        }
      }
      close_task(id);
    }

    // genTaskTrsm (factorize.hpp:186-196)
    for (offset_t qj = rb + 1; qj < re; ++qj) {
      const std::int32_t id = new_task(kTrsm, p, bl.bcol_idx[qj], {rb, qj}, qj);
      tr[static_cast<std::size_t>(id) * kTaskWords + 1] = Rp.size();
      tr[static_cast<std::size_t>(id) * kTaskWords + 6] = Rp.begin;
      if (with_work) {
        for (std::int64_t h = bc.ptr[rb]; h < bc.ptr[rb + 1]; ++h) {
          const std::int32_t t = bc.col[h];
          std::int32_t tb, te;
          span(qj, t - Rp.begin, tb, te);
          if (tb == te) continue;
          const std::int64_t s0 = static_cast<std::int64_t>(sr.size() / kSrcWords);
          for (std::int32_t c = bc.cb[h]; c < bc.ce[h]; ++c) {
            const std::int32_t r = bc.csc_row[c];
            if (r == t) continue;
            std::int32_t sb, se;
            span(qj, r - Rp.begin, sb, se);
            if (sb == se) continue;
            add_src(r - Rp.begin, bc.csc_pos[c], sb, se);
          }
          add_item(tb, te, t - Rp.begin, static_cast<std::int32_t>(u.row_begin(t)), s0, t);
        }
      }
      close_task(id);
    }

    // genTaskHerk / Gemm (factorize.hpp:198-224)
    for (offset_t qi = rb + 1; qi < re; ++qi) {
      const index_t i = bl.bcol_idx[qi];
      for (offset_t qj = qi; qj < re; ++qj) {
        const index_t j = bl.bcol_idx[qj];
        const offset_t target = bl.find(i, j);
        if (target < 0) continue;
        const bool herk = (i == j);
        const std::int32_t id = herk ? new_task(kHerk, j, j, {qj, target}, target)
                                     : new_task(kGemm, i, j, {qi, qj, target}, target);
        if (with_work) {
          const index_t Ri = ranges.ranges[i].begin;
          // target rows t: the non-empty columns of panel block (p, i)
          for (std::int64_t h = bc.ptr[qi]; h < bc.ptr[qi + 1]; ++h) {
            const std::int32_t t = bc.col[h];
            std::int32_t tb, te;
            span(target, t - Ri, tb, te);
            if (tb == te) continue;
            const std::int64_t s0 = static_cast<std::int64_t>(sr.size() / kSrcWords);
            for (std::int32_t c = bc.cb[h]; c < bc.ce[h]; ++c) {
              const std::int32_t r = bc.csc_row[c];
              const std::int32_t pos = bc.csc_pos[c];
              std::int32_t sb, se;
              span(qj, r - Rp.begin, sb, se);
              if (herk) sb = pos;  // Herk: entries c2 >= c1 = t of row r
              if (sb == se) continue;
              add_src(r - Rp.begin, pos, sb, se);  // row in the panel (no wait)
            }
            if (static_cast<std::int64_t>(sr.size() / kSrcWords) == s0) continue;
            add_item(tb, te, -1, -1, s0, t);
          }
          const std::int32_t* rec = &tr[static_cast<std::size_t>(id) * kTaskWords];
          if (static_cast<std::int32_t>(ir.size() / kItemWords) == rec[2]) ++P.stats.empty_tasks;
        }
        close_task(id);
      }
    }
  }

  if (with_work && opt.programs) build_programs(P, opt.threads);
  if (with_work) build_item_deps(P, ranges, opt.hot_fraction);
  if (with_work && opt.programs) build_flow(P, u, opt.flow_merge_rows);
  if (with_work && opt.programs) build_units(P, ranges, opt.unit_min_rows, opt.unit_smem_cap);

  // successors + in-degrees (edge multiplicity preserved)
  const std::size_t T = P.node_kind.size();
  P.indeg.assign(T, 0);
  std::vector<std::int32_t> cnt(T + 1, 0);
  for (std::size_t e = 0; e < P.edge_from.size(); ++e) {
    ++cnt[P.edge_from[e] + 1];
    ++P.indeg[P.edge_to[e]];
  }
  for (std::size_t t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
  P.succ.assign(P.edge_from.size(), 0);
  {
    std::vector<std::int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (std::size_t e = 0; e < P.edge_from.size(); ++e) P.succ[fill[P.edge_from[e]]++] = P.edge_to[e];
  }
  for (std::size_t t = 0; t < T; ++t) {
    tr[t * kTaskWords + 4] = cnt[t];
    tr[t * kTaskWords + 5] = cnt[t + 1];
    if (P.indeg[t] == 0) P.roots.push_back(static_cast<std::int32_t>(t));
  }
  // edge records for the device: {successor, 0, 0, 0} followed by a copy of
  // the successor's task record, so a CTA that readies a successor already
  // holds everything it needs to start it (no dependent load on the hop)
  P.succ_rec.assign(P.succ.size() * kSuccWords, 0);
  for (std::size_t e = 0; e < P.succ.size(); ++e) {
    std::int32_t* r = &P.succ_rec[e * kSuccWords];
    r[0] = P.succ[e];
    std::copy_n(&tr[static_cast<std::size_t>(P.succ[e]) * kTaskWords], kTaskWords, r + 4);
  }
  P.stats.edges = static_cast<std::int64_t>(P.edge_from.size());
  std::vector<std::int32_t> depth(T, 1);
  for (std::size_t e = 0; e < P.edge_from.size(); ++e)  // edges ascend in `to`
    depth[P.edge_to[e]] = std::max(depth[P.edge_to[e]], depth[P.edge_from[e]] + 1);
  for (std::size_t t = 0; t < T; ++t) P.stats.dag_depth = std::max(P.stats.dag_depth, depth[t]);
  P.stats.plan_seconds = since(t0);
  return P;
}

FlowPart build_flow_part(const Plan& P, const std::vector<std::int32_t>& part_of_row, std::int32_t nparts,
                         std::int32_t part) {
  if (P.flow_rec.empty()) throw std::invalid_argument("flow part: the plan has no value-flow tables");
  if (nparts < 1 || nparts > 64 || part < 0 || part >= nparts)
    throw std::invalid_argument("flow part: need 1 <= nparts <= 64 and 0 <= part < nparts");
  if (static_cast<index_t>(part_of_row.size()) != P.n) throw std::invalid_argument("flow part: one owner per row");
  if (P.nnz >= (std::int64_t{1} << kRemoteShift)) throw std::length_error("flow part: U beyond 2^25 entries");
  for (std::int32_t o : part_of_row)
    if (o < 0 || o >= nparts) throw std::invalid_argument("flow part: owner out of range");
  const std::size_t R = P.flow_item.size();
  auto owner_of_pos = [&](std::int32_t pos) {
    const std::int32_t item = P.flow_owner[pos];
    return part_of_row[P.row_rec[static_cast<std::size_t>(item) * kRowWords + 5]];
  };
  // rows of this part that other parts read: they publish at system scope
  std::vector<char> exported(static_cast<std::size_t>(P.n), 0);
  for (std::size_t q = 0; q < R; ++q) {
    const std::int32_t* r = &P.flow_rec[q * kFlowWords];
    if (part_of_row[r[3]] == part) continue;
    const std::int32_t L = r[1] & ((1 << kFlowKindShift) - 1);
    for (std::int32_t j = 0; j < L; ++j) {
      const std::int32_t* sl = &P.flow_slot[4 * static_cast<std::size_t>(r[0] + j)];
      for (std::int32_t e = sl[0]; e < sl[1]; ++e)
        for (int h = 0; h < 2; ++h) {
          const std::int32_t x = P.flow_upd[2 * static_cast<std::size_t>(e) + h];
          if (owner_of_pos(x) == part)
            exported[P.row_rec[static_cast<std::size_t>(P.flow_owner[x]) * kRowWords + 5]] = 1;
        }
    }
  }
  FlowPart F;
  F.slot.assign(4 * static_cast<std::size_t>(P.nnz), 0);
  for (std::size_t q = 0; q < R; ++q) {
    const std::int32_t* r = &P.flow_rec[q * kFlowWords];
    if (part_of_row[r[3]] != part) continue;
    F.rec.insert(F.rec.end(), r, r + kFlowWords);
    if (exported[r[3]]) {  // bit 31 of the length word: publish at system scope
      F.rec[F.rec.size() - 3] = static_cast<std::int32_t>(static_cast<std::uint32_t>(F.rec[F.rec.size() - 3]) | 0x80000000u);
      ++F.exported_rows;
    }
    F.item.push_back(P.flow_item[q]);
    const std::int32_t L = r[1] & ((1 << kFlowKindShift) - 1);
    for (std::int32_t j = 0; j < L; ++j) {
      const std::int32_t* sl = &P.flow_slot[4 * static_cast<std::size_t>(r[0] + j)];
      std::int32_t* o = &F.slot[4 * static_cast<std::size_t>(r[0] + j)];
      o[0] = static_cast<std::int32_t>(F.upd.size() / 2);
      for (std::int32_t e = sl[0]; e < sl[1]; ++e)
        for (int h = 0; h < 2; ++h) {
          std::int32_t x = P.flow_upd[2 * static_cast<std::size_t>(e) + h];
          const std::int32_t ow = owner_of_pos(x);
          if (ow != part) {
            x = static_cast<std::int32_t>(kRemoteBit | (static_cast<std::uint32_t>(ow) << kRemoteShift) |
                                          static_cast<std::uint32_t>(x));
            ++F.remote_operands;
          }
          F.upd.push_back(x);
        }
      o[1] = static_cast<std::int32_t>(F.upd.size() / 2);
      if (o[0] < o[1]) {
        o[2] = F.upd[2 * static_cast<std::size_t>(o[0])];
        o[3] = F.upd[2 * static_cast<std::size_t>(o[0]) + 1];
      }
    }
    // the Trsm divisor U(t,t) belongs to row t: same part
  }
  F.rows = static_cast<std::int64_t>(F.item.size());
  return F;
}

}  // namespace tcb
