// Host flattener of the task-DAG plan: block layout, the reference's task
// DAG in generation order and the task executors' per-task gather work. Built
// on request (tcg_plan_expand): the default value-flow path needs only the
// lean plan (flow_plan.cpp).
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

}  // namespace tcb
