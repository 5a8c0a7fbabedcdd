// Lean host plan of the value-flow factorization (flow_plan.hpp).
#include "flow_plan.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>

namespace tcb {

namespace {

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int host_threads() {
  if (const char* e = std::getenv("TCG_PLAN_THREADS")) return std::max(1, std::atoi(e));
  const unsigned h = std::thread::hardware_concurrency();
  return static_cast<int>(std::clamp(h ? h : 1u, 1u, 32u));
}

// fn(row_begin, row_end) over contiguous row chunks on `threads` threads
template <class F>
void parallel_rows(index_t n, int threads, F&& fn) {
  const int T = std::max(1, std::min<int>(threads, std::max<index_t>(1, n / 4096)));
  if (T == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int k = 0; k < T; ++k) {
    const auto b = static_cast<index_t>(static_cast<std::int64_t>(n) * k / T);
    const auto e = static_cast<index_t>(static_cast<std::int64_t>(n) * (k + 1) / T);
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& th : pool) th.join();
}

// Rows in a topological order of some row DAG, on the host threads: a row
// is handed out once its counter (its unprocessed predecessors) reaches zero.
// body(r, release) processes row r and calls release(s) once for every
// successor s of r. Rows are handed out through a bag of n slots (a taker
// spins on its slot until a producer fills it); the counters' acq_rel
// decrements and the slot's release/acquire order a row's writes before
// every successor's reads. No deadlock: while rows remain, some unprocessed
// row has a zero counter and was put in the bag by whoever released it last.
// (Handing out layers between barriers instead was slower on C3, whose
// layers are narrow: 0.18 -> 0.37 s.)
template <class Body>
void ready_rows(index_t n, int threads, std::vector<std::atomic<std::int32_t>>& count, Body&& body) {
  std::vector<std::atomic<std::int32_t>> slot(static_cast<std::size_t>(n));
  std::atomic<std::int64_t> head{0}, tail{0};
  for (index_t r = 0; r < n; ++r) slot[r].store(-1, std::memory_order_relaxed);
  for (index_t r = 0; r < n; ++r)
    if (count[r].load(std::memory_order_relaxed) == 0) slot[tail.fetch_add(1)].store(r, std::memory_order_relaxed);
  auto release = [&](index_t s) {
    if (count[s].fetch_sub(1, std::memory_order_acq_rel) == 1)
      slot[tail.fetch_add(1, std::memory_order_relaxed)].store(s, std::memory_order_release);
  };
  auto worker = [&] {
    for (;;) {
      const std::int64_t k = head.fetch_add(1, std::memory_order_relaxed);
      if (k >= n) return;
      std::int32_t r;
      unsigned spins = 0;
      while ((r = slot[k].load(std::memory_order_acquire)) < 0)
        if (++spins > 64) std::this_thread::yield();
      body(static_cast<index_t>(r), release);
    }
  };
  const int T = std::max(1, std::min<int>(threads, std::max<index_t>(1, n / 4096)));
  std::vector<std::thread> pool;
  for (int k = 1; k < T; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

// validate_csr (sparse.cpp) over the host threads: the same checks and
// messages, the first failing row reported
void validate_ref(const CsrRef& m, int threads) {
  if (m.n < 0 || m.nnz < 0) throw std::invalid_argument("csr: negative dimension");
  if (!m.row_ptr) throw std::invalid_argument("csr view: null or negative sizes");
  if (m.row_ptr[0] != 0) throw std::invalid_argument("csr: row_ptr[0] != 0");
  if (m.row_ptr[m.n] != m.nnz) throw std::invalid_argument("csr: array length mismatch");
  if (m.nnz > 0 && !m.col_idx) throw std::invalid_argument("csr view: null col_idx");
  std::atomic<index_t> bad{std::numeric_limits<index_t>::max()};
  parallel_rows(m.n, threads, [&](index_t b, index_t e) {
    for (index_t i = b; i < e && i < bad.load(std::memory_order_relaxed); ++i) {
      bool ok = m.row_ptr[i] <= m.row_ptr[i + 1];
      for (offset_t q = m.row_ptr[i]; ok && q < m.row_ptr[i + 1]; ++q)
        ok = m.col_idx[q] >= 0 && m.col_idx[q] < m.n && (q == m.row_ptr[i] || m.col_idx[q] > m.col_idx[q - 1]);
      if (!ok) {
        index_t cur = bad.load();
        while (i < cur && !bad.compare_exchange_weak(cur, i)) {
        }
        return;
      }
    }
  });
  const index_t i = bad.load();
  if (i == std::numeric_limits<index_t>::max()) return;
  if (m.row_ptr[i] > m.row_ptr[i + 1]) throw std::invalid_argument("csr: row_ptr not non-decreasing");
  for (offset_t q = m.row_ptr[i]; q < m.row_ptr[i + 1]; ++q) {
    if (m.col_idx[q] < 0 || m.col_idx[q] >= m.n) throw std::invalid_argument("csr: column index out of range");
    if (q > m.row_ptr[i] && m.col_idx[q] <= m.col_idx[q - 1])
      throw std::invalid_argument("csr: columns not strictly increasing in row " + std::to_string(i));
  }
}

// Block CSR of the reference's 2D layout (block (I,J), I <= J, exists iff U
// has an entry in ranges[I] x ranges[J]; block_layout.hpp:71-72) and the
// task counts of its generation walk (factorize.hpp:177-224): one Chol per
// block row, one Trsm and one Herk per off-diagonal block, one Gemm per pair
// of off-diagonal blocks (i < j) of a block row whose target (i, j) exists.
void count_tasks(const FlowPlan& P, const RangeList& ranges, const std::vector<index_t>& owner,
                 FlowPlanStats& st, int threads) {
  const index_t m = ranges.count();
  const std::int32_t* cols = P.cols.data();
  // block columns of every block row, over contiguous block-row ranges on the
  // host threads (each with its own stamp array), concatenated in order
  const int T = std::max(1, std::min<int>(threads, std::max<index_t>(1, m / 256)));
  std::vector<std::vector<index_t>> part_cols(static_cast<std::size_t>(T));
  std::vector<std::vector<offset_t>> part_len(static_cast<std::size_t>(T));
  {
    std::vector<std::thread> pool;
    for (int k = 0; k < T; ++k)
      pool.emplace_back([&, k] {
        const index_t b0 = static_cast<index_t>(static_cast<std::int64_t>(m) * k / T);
        const index_t b1 = static_cast<index_t>(static_cast<std::int64_t>(m) * (k + 1) / T);
        std::vector<index_t> stamp(static_cast<std::size_t>(m), -1), present;
        auto& out = part_cols[static_cast<std::size_t>(k)];
        auto& len = part_len[static_cast<std::size_t>(k)];
        for (index_t bi = b0; bi < b1; ++bi) {
          present.clear();
          for (index_t i = ranges.ranges[bi].begin; i < ranges.ranges[bi].end; ++i)
            for (std::int32_t q = P.row_ptr[i], qe = P.row_ptr[i + 1]; q < qe;) {
              const index_t bj = owner[cols[q]];
              if (stamp[bj] != bi) {
                stamp[bj] = bi;
                present.push_back(bj);
              }
              // skip the rest of this block's slice of the row
              q = static_cast<std::int32_t>(std::lower_bound(cols + q, cols + qe, ranges.ranges[bj].end) - cols);
            }
          std::sort(present.begin(), present.end());
          out.insert(out.end(), present.begin(), present.end());
          len.push_back(static_cast<offset_t>(present.size()));
        }
      });
    for (auto& th : pool) th.join();
  }
  std::vector<offset_t> bptr(static_cast<std::size_t>(m) + 1, 0);
  std::vector<index_t> bcol;
  {
    index_t bi = 0;
    for (int k = 0; k < T; ++k) {
      bcol.insert(bcol.end(), part_cols[static_cast<std::size_t>(k)].begin(), part_cols[static_cast<std::size_t>(k)].end());
      for (offset_t l : part_len[static_cast<std::size_t>(k)]) {
        bptr[bi + 1] = bptr[bi] + l;
        ++bi;
      }
    }
  }
  const offset_t nb = static_cast<offset_t>(bcol.size());
  // one Gemm per pair of off-diagonal blocks (i < j) of a block row whose target (i, j) exists
  std::atomic<std::int64_t> gemm{0};
  parallel_rows(m, threads, [&](index_t b0, index_t b1) {
    std::int64_t local = 0;
    for (index_t p = b0; p < b1; ++p) {
      // off-diagonal block columns of row p (the diagonal block leads)
      const offset_t b = bptr[p] + 1, e = bptr[p + 1];
      for (offset_t x = b; x < e; ++x) {
        const index_t i = bcol[x];
        const auto re = bcol.begin() + bptr[i + 1];
        auto it = bcol.begin() + bptr[i];
        for (offset_t y = x + 1; y < e; ++y) {  // targets (i, j), j ascending: one forward merge
          it = std::lower_bound(it, re, bcol[y]);
          if (it == re) break;
          if (*it == bcol[y]) ++local;
        }
      }
    }
    gemm.fetch_add(local, std::memory_order_relaxed);
  });
  st.nblock_rows = m;
  st.nblocks = nb;
  st.tasks[0] = m;
  st.tasks[1] = st.tasks[2] = nb - m;
  st.tasks[3] = gemm.load();
}

}  // namespace

int flow_slack_pct(std::int64_t n, std::int64_t nnz, std::int64_t units) {
  if (const char* e = std::getenv("TCG_FLOW_SLACK")) return std::clamp(std::atoi(e), 0, 100);
  // short rows (so short programs: the product-parallel kernel) and more units
  // than that kernel's lower size bound (capi.cpp pick_pp)
  return nnz < 12 * n && units > 400000 ? 100 : 0;
}

CsrMatrix flow_plan_pattern(const FlowPlan& P) {
  CsrMatrix u;
  u.nrows = u.ncols = P.n;
  u.row_ptr.assign(P.row_ptr.begin(), P.row_ptr.end());
  u.col_idx.assign(P.cols.begin(), P.cols.end());
  u.values.assign(P.cols.size(), 1.0);
  return u;
}

FlowPlan build_flow_plan(const CsrRef& a, const CsrRef& u, const RangeList& ranges, bool schedule) {
  const auto t0 = std::chrono::steady_clock::now();
  const int threads = host_threads();
  const bool say = std::getenv("TCG_PLAN_TIMES") != nullptr;
  auto mark = [&](const char* what) {
    if (say) std::fprintf(stderr, "flow plan %-10s %8.3f s\n", what, since(t0));
  };
  validate_ref(a, threads);
  if (a.nnz > 0 && !a.values) throw std::invalid_argument("csr view: values required");
  validate_ref(u, threads);
  if (a.n != u.n) throw std::invalid_argument("a_permuted and pattern sizes differ");
  validate_ranges(ranges, u.n);
  if (u.nnz > std::numeric_limits<std::int32_t>::max())
    throw std::invalid_argument("factor has more than 2^31-1 entries");
  const index_t n = u.n;
  // diagonal entries must lead every row (kernels.hpp:46-48)
  for (index_t i = 0; i < n; ++i)
    if (u.row_ptr[i] == u.row_ptr[i + 1] || u.col_idx[u.row_ptr[i]] != i)
      throw std::invalid_argument("chol_block: missing diagonal entry in row " + std::to_string(i));
  mark("validate");

  FlowPlan P;
  P.n = n;
  P.nnz = u.nnz;
  P.nnz_a = a.nnz;
  P.stats.threads = threads;
  P.cols.resize(static_cast<std::size_t>(u.nnz));
  P.row_ptr.resize(static_cast<std::size_t>(n) + 1);
  P.values.resize(static_cast<std::size_t>(u.nnz));
  P.a_map.resize(static_cast<std::size_t>(u.nnz));
  // initial values (factorize.hpp:71-89) by rows on the host threads: the
  // sorted merge of A's upper row into U's, recording where each slot starts
  // from (the device init's map; 0.0 + a as there). A slot fed twice
  // (duplicate entries in A) has no map and keeps the sum, as the reference.
  const bool mappable = a.nnz <= 0x7fffffffLL;
  std::atomic<bool> dup{!mappable};
  parallel_rows(n, threads, [&](index_t b, index_t e) {
    for (index_t i = b; i < e; ++i) {
      const offset_t ub = u.row_ptr[i], ue = u.row_ptr[i + 1];
      P.row_ptr[i] = static_cast<std::int32_t>(ub);
      for (offset_t t = ub; t < ue; ++t) {
        P.cols[t] = u.col_idx[t];
        P.values[t] = 0.0;
        P.a_map[t] = -1;
      }
      offset_t t = ub;
      for (offset_t q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) {
        const index_t c = a.col_idx[q];
        if (c < i) continue;
        while (t < ue && u.col_idx[t] < c) ++t;
        if (t < ue && u.col_idx[t] == c) {
          P.values[t] += a.values[q];
          if (P.a_map[t] >= 0) dup.store(true, std::memory_order_relaxed);
          P.a_map[t] = static_cast<std::int32_t>(q);
        }
      }
    }
  });
  P.row_ptr[n] = static_cast<std::int32_t>(u.nnz);
  if (dup.load()) P.a_map.clear();  // no device init (host values only)
  mark("init");

  std::vector<index_t> owner(static_cast<std::size_t>(n));
  for (index_t r = 0; r < ranges.count(); ++r)
    for (index_t c = ranges.ranges[r].begin; c < ranges.ranges[r].end; ++c) owner[c] = r;
  // the block layout's task counts on a second thread (FactorStats)
  std::thread blocks([&] {
    const auto tb = std::chrono::steady_clock::now();
    count_tasks(P, ranges, owner, P.stats, threads);
    P.stats.block_build_seconds = since(tb);
  });
  try {
    // units in natural order (row ascending; a row's Chol slice, then its chunks)
    const std::int32_t* cols = P.cols.data();
    // Chol units hold at most chol_max = 32 coordinates (one warp pass); the
    // rest of a longer diagonal-block slice runs as chunks dividing by U(t,t),
    // on other warps, side by side with the Chol unit instead of after it in
    // the same warp. On the critical path a second pass over a 33-64 wide
    // slice cost its whole program after the late operand arrived (C3 trace:
    // 1.8 ms of row tails on a 555-row path). B200: C3 3.25 -> 2.83 ms,
    // elast6 0.96 -> 0.33, s27 1.11 -> 0.94, C4 unchanged; bitwise.
    // With panel > 0 (TCG_FLOW_PANEL) the diagonal-block slice is cut at fixed
    // columns instead (block begin + k * panel): the Chol unit of row t ends
    // at its panel's end, so row t+1 of the same panel finds every operand it
    // takes from row t in t's Chol unit, never in a chunk finishing one hop
    // later. B200, panel 32: elast6 0.357 -> 0.312 ms (depth 350 -> 255), but
    // C3 2.66 -> 2.69 and C4 1.30 -> 1.34 (more units, depth 725 -> 705 only),
    // so it is off by default.
    std::int32_t chol_max = 32, panel = 0;
    if (const char* e = std::getenv("TCG_FLOW_CHOL_MAX")) chol_max = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("TCG_FLOW_PANEL")) panel = std::clamp(std::atoi(e), 0, 32);
    // the units of row t in order: emit(first position, length)
    auto split_row = [&](index_t t, auto&& emit) {
      const std::int32_t rb = P.row_ptr[t], re = P.row_ptr[t + 1];
      if (re - rb <= 32) {  // one warp pass: the whole row
        emit(rb, re - rb);
        return;
      }
      const Range blk = ranges.ranges[owner[t]];
      const auto ds = static_cast<std::int32_t>(std::lower_bound(cols + rb, cols + re, blk.end) - cols);
      if (panel > 0) {
        auto panel_end = [&](index_t c) { return std::min<index_t>(blk.end, blk.begin + panel * ((c - blk.begin) / panel + 1)); };
        for (std::int32_t q = rb; q < ds;) {
          const auto qe = static_cast<std::int32_t>(std::lower_bound(cols + q, cols + ds, panel_end(cols[q])) - cols);
          emit(q, qe - q);
          q = qe;
        }
      } else {
        const std::int32_t ce = std::min(ds, rb + chol_max);
        emit(rb, ce - rb);
        for (std::int32_t c0 = ce; c0 < ds; c0 += 32) emit(c0, std::min(ds - c0, 32));
      }
      for (std::int32_t c0 = ds; c0 < re; c0 += 32) emit(c0, std::min(re - c0, 32));
    };
    std::vector<std::int32_t> ufirst(static_cast<std::size_t>(n) + 1, 0);
    parallel_rows(n, threads, [&](index_t b, index_t e) {
      for (index_t t = b; t < e; ++t) {
        std::int32_t k = 0;
        split_row(t, [&](std::int32_t, std::int32_t) { ++k; });
        ufirst[t + 1] = k;
      }
    });
    for (index_t t = 0; t < n; ++t) ufirst[t + 1] += ufirst[t];
    const std::size_t U = static_cast<std::size_t>(ufirst[n]);
    if (U >= (1u << 31)) throw std::length_error("flow: too many units");
    // per unit: first position, length, row
    std::atomic<bool> miscount{false}, too_long{false};
    P.ufirst.assign(ufirst.begin(), ufirst.end());
    P.u_tb.resize(U);
    P.u_len.resize(U);
    P.u_row.resize(U);
    parallel_rows(n, threads, [&](index_t b, index_t e) {
      for (index_t t = b; t < e; ++t) {
        std::int32_t g = ufirst[t];
        split_row(t, [&](std::int32_t tb, std::int32_t len) {
          P.u_tb[g] = tb;
          P.u_len[g] = len;
          P.u_row[g] = static_cast<std::int32_t>(t);
          if (len >= (1 << 30)) too_long.store(true, std::memory_order_relaxed);
          ++g;
        });
        if (g != ufirst[t + 1]) miscount.store(true, std::memory_order_relaxed);
      }
    });
    if (miscount.load()) throw std::logic_error("flow plan: unit count mismatch");
    if (too_long.load()) throw std::length_error("flow: row slice too long");
    P.stats.units = static_cast<std::int64_t>(U);
    mark("units");
    if (schedule) flow_plan_schedule(P);
    mark("schedule");
  } catch (...) {
    blocks.join();
    throw;
  }
  blocks.join();
  mark("blocks");
  P.stats.plan_seconds = since(t0);
  return P;
}

void flow_plan_schedule(FlowPlan& P) {
  if (P.scheduled) return;
  const index_t n = P.n;
  const int threads = host_threads();
  const std::size_t U = P.u_tb.size();
  const std::int32_t* cols = P.cols.data();
  const std::int32_t* ufirst = P.ufirst.data();
  const std::int32_t* u_tb = P.u_tb.data();
  const std::int32_t* u_len = P.u_len.data();
  const std::int32_t* row_of = P.u_row.data();
  hvec<std::int32_t> u_c0(U), u_c1(U);  // first and last column of every unit
  parallel_rows(static_cast<index_t>(U), threads, [&](index_t b, index_t e) {
    for (index_t g = b; g < e; ++g) {
      u_c0[g] = cols[u_tb[g]];
      u_c1[g] = cols[u_tb[g] + u_len[g] - 1];
    }
  });
  {

    // Dependences of unit g (row t, last column c1(g)): for every source r of
    // t (an entry U(r,t) at position q), the units of row r from the one
    // holding q on, up to the last one starting at a column <= c1(g) (they
    // hold the multiplier and every operand U(r,c) g reads); a chunk also
    // reads U(t,t), its row's Chol unit. Every dependence points to a lower
    // row (or the row's own Chol unit). Levels (longest chain from a source)
    // and heights (longest chain to a sink) are computed row by row, each
    // row pulling from rows that are final: levels in a topological order of
    // the rows (ready once all its sources are done, through U's transposed
    // index), heights in a reverse one (ready once every row it feeds is
    // done); both on the host threads (ready_rows).
    hvec<std::int32_t> level(U), height(U);
    std::int32_t depth = 0;
    // Long rows (C3: 69 entries, three units per row) carry enough work per
    // row for the parallel traversal (C3 0.39 -> 0.22 s of plan on 8 threads);
    // shorter ones (C1, C2, C4-C6) sweep faster on one thread than through
    // any hand-out of their rows (C4: levels and heights 0.14 s on one
    // thread, 0.20 s in parallel).
    if (threads > 1 && P.nnz >= 48 * static_cast<std::int64_t>(n)) {
      std::vector<std::atomic<std::int32_t>> cnt(static_cast<std::size_t>(n));
      for (index_t t = 0; t < n; ++t) cnt[t].store(0, std::memory_order_relaxed);
      parallel_rows(n, threads, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r)
          for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q)
            cnt[cols[q]].fetch_add(1, std::memory_order_relaxed);
      });
      // transposed index: the sources (r, q) of every row t, in any order
      std::vector<std::int64_t> sptr(static_cast<std::size_t>(n) + 1, 0);
      for (index_t t = 0; t < n; ++t) sptr[t + 1] = sptr[t] + cnt[t].load(std::memory_order_relaxed);
      hvec<std::int32_t> src_r(static_cast<std::size_t>(sptr[n])), src_q(static_cast<std::size_t>(sptr[n]));
      {
        std::vector<std::atomic<std::int64_t>> fill(static_cast<std::size_t>(n));
        for (index_t t = 0; t < n; ++t) fill[t].store(sptr[t], std::memory_order_relaxed);
        parallel_rows(n, threads, [&](index_t b, index_t e) {
          for (index_t r = b; r < e; ++r)
            for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q) {
              const std::int64_t k = fill[cols[q]].fetch_add(1, std::memory_order_relaxed);
              src_r[k] = static_cast<std::int32_t>(r);
              src_q[k] = q;
            }
        });
      }
      ready_rows(n, threads, cnt, [&](index_t t, auto&& release) {
        const std::int32_t g0 = ufirst[t], g1 = ufirst[t + 1];
        for (std::int32_t g = g0; g < g1; ++g) level[g] = 1;
        for (std::int64_t k = sptr[t]; k < sptr[t + 1]; ++k) {
          const index_t r = src_r[k];
          const std::int32_t q = src_q[k], vr1 = ufirst[r + 1];
          std::int32_t v = ufirst[r];
          while (v + 1 < vr1 && u_tb[v + 1] <= q) ++v;  // the unit of row r holding q
          std::int32_t lv = level[v];
          for (std::int32_t g = g0; g < g1; ++g) {
            while (v + 1 < vr1 && u_c0[v + 1] <= u_c1[g]) lv = std::max(lv, level[++v]);
            level[g] = std::max(level[g], lv + 1);
          }
        }
        for (std::int32_t g = g0 + 1; g < g1; ++g) level[g] = std::max(level[g], level[g0] + 1);
        for (std::int32_t q = P.row_ptr[t] + 1; q < P.row_ptr[t + 1]; ++q) release(cols[q]);
      });
      for (std::size_t g = 0; g < U; ++g) depth = std::max(depth, level[g]);
      // heights: row r is ready once every row its entries feed is done
      for (index_t r = 0; r < n; ++r) cnt[r].store(P.row_ptr[r + 1] - P.row_ptr[r] - 1, std::memory_order_relaxed);
      ready_rows(n, threads, cnt, [&](index_t r, auto&& release) {
        thread_local std::vector<std::int32_t> vmax;
        const std::int32_t vr0 = ufirst[r], vr1 = ufirst[r + 1];
        for (std::int32_t v = vr0; v < vr1; ++v) height[v] = 1;
        std::int32_t v0 = vr0;
        for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q) {
          while (v0 + 1 < vr1 && u_tb[v0 + 1] <= q) ++v0;
          const index_t t = cols[q];
          const std::int32_t g0 = ufirst[t], g1 = ufirst[t + 1];
          if (vr1 - vr0 == 1) {  // one unit: every dependent of the entry reads it
            std::int32_t hm = 0;
            for (std::int32_t g = g0; g < g1; ++g) hm = std::max(hm, height[g] + 1);
            height[v0] = std::max(height[v0], hm);
            continue;
          }
          vmax.resize(static_cast<std::size_t>(g1 - g0));
          for (std::int32_t g = g0, v = v0; g < g1; ++g) {
            while (v + 1 < vr1 && u_c0[v + 1] <= u_c1[g]) ++v;
            vmax[g - g0] = v;
          }
          // unit v of row r is read by the dependents g with vmax(g) >= v
          std::int32_t hm = 0;
          for (std::int32_t g = g1; g-- > g0;) {
            hm = std::max(hm, height[g] + 1);
            const std::int32_t lo = g > g0 ? vmax[g - 1 - g0] + 1 : v0;
            for (std::int32_t v = lo; v <= vmax[g - g0]; ++v) height[v] = std::max(height[v], hm);
          }
        }
        for (std::int32_t g = vr0 + 1; g < vr1; ++g) height[vr0] = std::max(height[vr0], height[g] + 1);
        for (std::int64_t k = sptr[r]; k < sptr[r + 1]; ++k) release(src_r[k]);
      });
    } else {
      std::vector<std::int32_t> vmax;
      std::fill(level.begin(), level.end(), 1);
      std::fill(height.begin(), height.end(), 1);
      for (index_t r = 0; r < n; ++r) {
        const std::int32_t vr0 = ufirst[r], vr1 = ufirst[r + 1];
        for (std::int32_t g = vr0 + 1; g < vr1; ++g) level[g] = std::max(level[g], level[vr0] + 1);
        for (std::int32_t g = vr0; g < vr1; ++g) depth = std::max(depth, level[g]);
        std::int32_t v0 = vr0;
        for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q) {
          while (v0 + 1 < vr1 && u_tb[v0 + 1] <= q) ++v0;
          const index_t t = cols[q];
          std::int32_t v = v0, lv = level[v0];
          for (std::int32_t g = ufirst[t]; g < ufirst[t + 1]; ++g) {
            while (v + 1 < vr1 && u_c0[v + 1] <= u_c1[g]) lv = std::max(lv, level[++v]);
            level[g] = std::max(level[g], lv + 1);
          }
        }
      }
      for (index_t r = n; r-- > 0;) {
        const std::int32_t vr0 = ufirst[r], vr1 = ufirst[r + 1];
        std::int32_t v0 = vr0;
        for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q) {
          while (v0 + 1 < vr1 && u_tb[v0 + 1] <= q) ++v0;
          const index_t t = cols[q];
          const std::int32_t g0 = ufirst[t], g1 = ufirst[t + 1];
          if (vr1 - vr0 == 1) {  // one unit: every dependent of the entry reads it
            std::int32_t hm = 0;
            for (std::int32_t g = g0; g < g1; ++g) hm = std::max(hm, height[g] + 1);
            height[v0] = std::max(height[v0], hm);
            continue;
          }
          vmax.resize(static_cast<std::size_t>(g1 - g0));
          for (std::int32_t g = g0, v = v0; g < g1; ++g) {
            while (v + 1 < vr1 && u_c0[v + 1] <= u_c1[g]) ++v;
            vmax[g - g0] = v;
          }
          // unit v of row r is read by the dependents g with vmax(g) >= v
          std::int32_t hm = 0;
          for (std::int32_t g = g1; g-- > g0;) {
            hm = std::max(hm, height[g] + 1);
            const std::int32_t lo = g > g0 ? vmax[g - 1 - g0] + 1 : v0;
            for (std::int32_t v = lo; v <= vmax[g - g0]; ++v) height[v] = std::max(height[v], hm);
          }
        }
        for (std::int32_t g = vr0 + 1; g < vr1; ++g) height[vr0] = std::max(height[vr0], height[g] + 1);
      }
    }
    // schedule: level ascending, height descending, unit id ascending (two
    // stable counting sorts, the second key first)
    std::int32_t hmax = 0;
    for (std::int32_t h : height) hmax = std::max(hmax, h);
    hvec<std::int32_t> tmp(U), order(U);
    {
      std::vector<std::int64_t> cnt(static_cast<std::size_t>(hmax) + 2, 0);
      for (std::size_t g = 0; g < U; ++g) ++cnt[static_cast<std::size_t>(hmax - height[g]) + 1];
      for (std::size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
      for (std::size_t g = 0; g < U; ++g)
        tmp[cnt[static_cast<std::size_t>(hmax - height[g])]++] = static_cast<std::int32_t>(g);
    }
    {
      // a unit's place: its level, moved towards its latest level (depth + 1 -
      // height) by flow_slack_pct percent of its slack (a topological key
      // still: both ends grow by at least 1 along a dependence)
      const int pct = flow_slack_pct(n, P.nnz, static_cast<std::int64_t>(U));
      auto place = [&](std::int32_t g) {
        const std::int32_t slack = depth + 1 - height[g] - level[g];
        return level[g] + static_cast<std::int32_t>(static_cast<std::int64_t>(pct) * slack / 100);
      };
      std::vector<std::int64_t> cnt(static_cast<std::size_t>(depth) + 2, 0);
      for (std::size_t g = 0; g < U; ++g) ++cnt[static_cast<std::size_t>(place(static_cast<std::int32_t>(g)))];
      for (std::size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
      for (std::size_t x = 0; x < U; ++x) {
        const std::int32_t g = tmp[x];
        order[cnt[static_cast<std::size_t>(place(g)) - 1]++] = g;
      }
    }
    P.rec.resize(4 * U);
    P.unit.resize(U);
    parallel_rows(static_cast<index_t>(U), threads, [&](index_t b, index_t e) {
      for (index_t q = b; q < e; ++q) {
        const std::int32_t g = order[q];
        const std::int32_t t = row_of[g];
        P.rec[4 * q + 0] = u_tb[g];
        P.rec[4 * q + 1] = u_len[g] | ((g == ufirst[t] ? 0 : 1) << 30);  // Chol unit, else a chunk (Trsm)
        P.rec[4 * q + 2] = P.row_ptr[t];
        P.rec[4 * q + 3] = t;
        P.unit[q] = g;
      }
    });
    P.stats.depth = depth;
    P.scheduled = true;
  }
}

FlowPart build_flow_part(const FlowPlan& P, const std::vector<std::int32_t>& part_of_row, std::int32_t nparts,
                         std::int32_t part) {
  if (nparts < 1 || nparts > 64 || part < 0 || part >= nparts)
    throw std::invalid_argument("flow part: need 1 <= nparts <= 64 and 0 <= part < nparts");
  if (static_cast<index_t>(part_of_row.size()) != P.n) throw std::invalid_argument("flow part: one owner per row");
  if (P.nnz >= (std::int64_t{1} << kRemoteShift)) throw std::length_error("flow part: U beyond 2^25 entries");
  for (std::int32_t o : part_of_row)
    if (o < 0 || o >= nparts) throw std::invalid_argument("flow part: owner out of range");
  // rows of this part that other parts read (sources of their rows)
  FlowPart F;
  std::vector<char> exported(static_cast<std::size_t>(P.n), 0);
  for (index_t r = 0; r < P.n; ++r)
    for (std::int32_t q = P.row_ptr[r] + 1; q < P.row_ptr[r + 1]; ++q) {
      const index_t t = P.cols[q];
      if (part_of_row[r] == part && part_of_row[t] != part) exported[r] = 1;
      if (part_of_row[t] == part && part_of_row[r] != part) ++F.remote_sources;
    }
  const std::size_t U = P.unit.size();
  for (std::size_t q = 0; q < U; ++q) {
    const std::int32_t* r = &P.rec[4 * q];
    if (part_of_row[r[3]] != part) continue;
    F.rec.insert(F.rec.end(), r, r + 4);
    if (exported[r[3]]) {  // bit 31 of the length word: publish at system scope
      F.rec[F.rec.size() - 3] = static_cast<std::int32_t>(static_cast<std::uint32_t>(F.rec[F.rec.size() - 3]) | kRemoteBit);
      ++F.exported_rows;
    }
    F.unit.push_back(P.unit[q]);
  }
  F.rows = static_cast<std::int64_t>(F.unit.size());
  return F;
}

}  // namespace tcb
