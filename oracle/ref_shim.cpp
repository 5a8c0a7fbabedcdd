// extern "C" shim over the UNMODIFIED reference headers — TEST/BASELINE ONLY.
//
// Compiled from /root/reference/proj/include (never copied) into
// oracle/_ref/libtaskchol_ref.so with the reference's canonical flags
// (RelWithDebInfo: -O2 -g, no -march). Used to
//   * pin the plain-C oracle and this repo's host analysis against the
//     reference (tests/golden/make_golden.py), and
//   * time the reference's own CPU path for bench.py --impl reference and
//     the cpu_baseline leg.
// The product path never loads it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "taskchol/factorize.hpp"
#include "taskchol/matrix_market.hpp"
#include "taskchol/pipeline.hpp"
#include "taskchol/symbolic.hpp"
// the reference's own test generators (tests/support), compiled where they
// lie: they pin this repo's grid2d / path / random_spd generators
#include "test_matrices.hpp"
// this repo's seeded generators, compiled into the
// shim so bench.py's reference arm builds its inputs without loading the
// product library
#include "../paper_1601_05871_b200/csrc/host/sparse.hpp"

using namespace taskchol;

namespace {
thread_local std::string g_err;

CsrMatrix make_csr(int32_t n, const int64_t* ptr, const int32_t* col, const double* val) {
  CsrMatrix m;
  m.nrows = m.ncols = n;
  m.row_ptr.assign(ptr, ptr + n + 1);
  m.col_idx.assign(col, col + ptr[n]);
  if (val)
    m.values.assign(val, val + ptr[n]);
  else
    m.values.assign(static_cast<std::size_t>(ptr[n]), 1.0);
  return m;
}

RangeList make_ranges(int32_t m, const int32_t* b) {
  RangeList rl;
  for (int32_t r = 0; r < m; ++r) rl.ranges.push_back({b[r], b[r + 1]});
  return rl;
}

FillPattern make_fp(int32_t n, const int64_t* ptr, const int32_t* col) {
  FillPattern fp;
  fp.pattern = make_csr(n, ptr, col, nullptr);
  return fp;
}
}  // namespace

struct ref_analysis {
  Analysis an;
  std::vector<int32_t> bounds;
};
struct ref_dag {
  std::vector<int32_t> kind, bi, bj, from, to;
};
struct ref_csr {
  CsrMatrix m;
};

extern "C" {

const char* ref_error() { return g_err.c_str(); }

ref_analysis* ref_analyze(int32_t n, const int64_t* ptr, const int32_t* col, const double* val,
                          int32_t level, int32_t treecut, int32_t leaf, int32_t max_depth) {
  try {
    const CsrMatrix a = make_csr(n, ptr, col, val);
    AnalyzeOptions o;
    o.level = level;
    o.treecut = treecut;
    o.leaf_size = leaf;
    o.max_depth = max_depth;
    auto out = std::make_unique<ref_analysis>();
    out->an = analyze(a, o);
    for (const Range& r : out->an.ranges.ranges) {
      if (out->bounds.empty()) out->bounds.push_back(r.begin);
      out->bounds.push_back(r.end);
    }
    if (out->bounds.empty()) out->bounds.push_back(0);
    return out.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_analysis_free(ref_analysis* a) { delete a; }
const int32_t* ref_analysis_perm(const ref_analysis* a) { return a->an.perm.perm.data(); }
int32_t ref_analysis_nranges(const ref_analysis* a) { return a->an.ranges.count(); }
const int32_t* ref_analysis_bounds(const ref_analysis* a) { return a->bounds.data(); }
int64_t ref_analysis_nnz_u(const ref_analysis* a) { return a->an.pattern.pattern.nnz(); }
const int64_t* ref_analysis_u_ptr(const ref_analysis* a) { return a->an.pattern.pattern.row_ptr.data(); }
const int32_t* ref_analysis_u_col(const ref_analysis* a) { return a->an.pattern.pattern.col_idx.data(); }
int64_t ref_analysis_nnz_a(const ref_analysis* a) { return a->an.a_permuted.nnz(); }
const int64_t* ref_analysis_a_ptr(const ref_analysis* a) { return a->an.a_permuted.row_ptr.data(); }
const int32_t* ref_analysis_a_col(const ref_analysis* a) { return a->an.a_permuted.col_idx.data(); }
const double* ref_analysis_a_val(const ref_analysis* a) { return a->an.a_permuted.values.data(); }
double ref_analysis_seconds(const ref_analysis* a, int which) {
  return which == 0 ? a->an.ordering_seconds : a->an.symbolic_seconds;
}

// levelk_pattern_bfs (symbolic.hpp:57-120) for an already-permuted matrix.
int64_t ref_levelk(int32_t n, const int64_t* ptr, const int32_t* col, int32_t k, int64_t* out_ptr,
                   int32_t* out_col, int64_t cap) {
  const FillPattern fp = levelk_pattern_bfs(make_csr(n, ptr, col, nullptr), k);
  const int64_t nnz = fp.pattern.nnz();
  if (out_ptr && out_col && cap >= nnz) {
    std::memcpy(out_ptr, fp.pattern.row_ptr.data(), sizeof(int64_t) * (n + 1));
    std::memcpy(out_col, fp.pattern.col_idx.data(), sizeof(int32_t) * nnz);
  }
  return nnz;
}

// factor_serial (factorize.hpp:94-130). 0 ok, 1 breakdown, 2 other error.
int ref_factor_serial(int32_t n, const int64_t* a_ptr, const int32_t* a_col, const double* a_val,
                      const int64_t* u_ptr, const int32_t* u_col, double* out, double* seconds,
                      int32_t* brow, double* bpiv) {
  try {
    const FactorResult r =
        factor_serial(make_csr(n, a_ptr, a_col, a_val), make_fp(n, u_ptr, u_col));
    std::memcpy(out, r.factor.values.data(), sizeof(double) * r.factor.values.size());
    if (seconds) *seconds = r.stats.numeric_seconds;
    return 0;
  } catch (const BreakdownError& e) {
    if (brow) *brow = e.row();
    if (bpiv) *bpiv = e.pivot();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// factor_by_blocks (factorize.hpp:134-235); workers == 0 -> sequential policy.
int ref_factor_by_blocks(int32_t n, const int64_t* a_ptr, const int32_t* a_col,
                         const double* a_val, const int64_t* u_ptr, const int32_t* u_col,
                         int32_t m, const int32_t* bounds, int32_t workers, double* out,
                         double* seconds, double* block_seconds, int64_t* tasks, int32_t* brow,
                         double* bpiv) {
  try {
    const CsrMatrix a = make_csr(n, a_ptr, a_col, a_val);
    const FillPattern fp = make_fp(n, u_ptr, u_col);
    const RangeList rl = make_ranges(m, bounds);
    if (workers <= 0) {
      TaskPolicy pol = TaskPolicy::sequential();
      const FactorResult r = factor_by_blocks(a, fp, rl, pol);
      if (out) std::memcpy(out, r.factor.values.data(), sizeof(double) * r.factor.values.size());
      if (seconds) *seconds = r.stats.numeric_seconds;
      if (block_seconds) *block_seconds = r.stats.block_build_seconds;
      if (tasks) *tasks = r.stats.total_tasks();
    } else {
      TaskPolicy pol = TaskPolicy::pooled(workers);
      const FactorResult r = factor_by_blocks(a, fp, rl, pol);
      if (out) std::memcpy(out, r.factor.values.data(), sizeof(double) * r.factor.values.size());
      if (seconds) *seconds = r.stats.numeric_seconds;
      if (block_seconds) *block_seconds = r.stats.block_build_seconds;
      if (tasks) *tasks = r.stats.total_tasks();
    }
    return 0;
  } catch (const BreakdownError& e) {
    if (brow) *brow = e.row();
    if (bpiv) *bpiv = e.pivot();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// export_task_dag (factorize.hpp:260-302); labels parsed back to (kind, i, j).
ref_dag* ref_export_dag(int32_t n, const int64_t* u_ptr, const int32_t* u_col, int32_t m,
                        const int32_t* bounds) {
  try {
    const TaskDag dag = export_task_dag(make_fp(n, u_ptr, u_col), make_ranges(m, bounds));
    auto out = std::make_unique<ref_dag>();
    for (const auto& nd : dag.nodes) {
      const std::string& l = nd.label;
      int32_t k = -1;
      if (l.rfind("CHOL", 0) == 0) k = 0;
      else if (l.rfind("TRSM", 0) == 0) k = 1;
      else if (l.rfind("HERK", 0) == 0) k = 2;
      else if (l.rfind("GEMM", 0) == 0) k = 3;
      out->kind.push_back(k);
      out->bi.push_back(nd.block_row);
      out->bj.push_back(nd.block_col);
    }
    for (const auto& e : dag.edges) {
      out->from.push_back(e.first);
      out->to.push_back(e.second);
    }
    return out.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_dag_free(ref_dag* d) { delete d; }
int64_t ref_dag_nnodes(const ref_dag* d) { return static_cast<int64_t>(d->kind.size()); }
int64_t ref_dag_nedges(const ref_dag* d) { return static_cast<int64_t>(d->from.size()); }
const int32_t* ref_dag_kind(const ref_dag* d) { return d->kind.data(); }
const int32_t* ref_dag_bi(const ref_dag* d) { return d->bi.data(); }
const int32_t* ref_dag_bj(const ref_dag* d) { return d->bj.data(); }
const int32_t* ref_dag_from(const ref_dag* d) { return d->from.data(); }
const int32_t* ref_dag_to(const ref_dag* d) { return d->to.data(); }

// build_block_matrix (block_layout.hpp:98-181): block CSR only.
int64_t ref_blocks(int32_t n, const int64_t* u_ptr, const int32_t* u_col, int32_t m,
                   const int32_t* bounds, int64_t* brow_ptr, int32_t* bcol, int64_t cap) {
  CsrMatrix u = make_csr(n, u_ptr, u_col, nullptr);
  const BlockMatrix bm = build_block_matrix(u, make_ranges(m, bounds));
  const int64_t nb = bm.block_count();
  if (brow_ptr && bcol && cap >= nb) {
    std::memcpy(brow_ptr, bm.brow_ptr.data(), sizeof(int64_t) * (m + 1));
    std::memcpy(bcol, bm.bcol_idx.data(), sizeof(int32_t) * nb);
  }
  return nb;
}

// matrix_market.hpp:159-176 (0 ok, 1 error with ref_error()).
int ref_write_mm(int32_t n, const int64_t* ptr, const int32_t* col, const double* val, const char* path) {
  try {
    write_matrix_market(make_csr(n, ptr, col, val), path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The BASELINE.json matrices (same generators and seeds as tch_generate),
// as a reference CsrMatrix; NULL with ref_error() on failure.
ref_csr* ref_generate(const char* kind, int64_t p0, int64_t p1, uint64_t seed) {
  try {
    const std::string k(kind ? kind : "");
    const auto i0 = static_cast<tcb::index_t>(p0);
    tcb::CsrMatrix g;
    if (k == "grid2d") g = tcb::grid_laplacian_2d(i0, static_cast<tcb::index_t>(p1));
    else if (k == "lap7") g = tcb::laplacian_7pt(i0);
    else if (k == "stencil27") g = tcb::stencil27_variable(i0, seed);
    else if (k == "elasticity") g = tcb::elasticity27(i0, seed);
    else if (k == "diffusion") g = tcb::diffusion_7pt_lognormal(i0, seed, static_cast<double>(p1) / 1000.0);
    else throw std::invalid_argument("unknown generator '" + k + "'");
    auto out = std::make_unique<ref_csr>();
    out->m.nrows = out->m.ncols = g.nrows;
    out->m.row_ptr.assign(g.row_ptr.begin(), g.row_ptr.end());
    out->m.col_idx.assign(g.col_idx.begin(), g.col_idx.end());
    out->m.values.assign(g.values.begin(), g.values.end());
    return out.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// The reference's test generators (tests/support/test_matrices.hpp:18-82):
// "grid" (p0 x p1 5-point Laplacian), "path" (p0 vertices), "random_spd"
// (p0 rows, density p1 / 1e6, a freshly seeded std::mt19937).
ref_csr* ref_test_matrix(const char* kind, int64_t p0, int64_t p1, uint64_t seed) {
  try {
    const std::string k(kind ? kind : "");
    auto out = std::make_unique<ref_csr>();
    if (k == "grid") out->m = testing::grid_laplacian(static_cast<index_t>(p0), static_cast<index_t>(p1));
    else if (k == "path") out->m = testing::path_matrix(static_cast<index_t>(p0));
    else if (k == "random_spd") {
      std::mt19937 rng(static_cast<std::uint32_t>(seed));
      out->m = testing::random_spd(static_cast<index_t>(p0), static_cast<double>(p1) / 1e6, rng);
    } else throw std::invalid_argument("unknown reference test matrix '" + k + "'");
    return out.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// matrix_market.hpp:61-157 (NULL with ref_error() on failure).
ref_csr* ref_load_mm(const char* path) {
  try {
    auto out = std::make_unique<ref_csr>();
    out->m = load_matrix_market(path);
    return out.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_csr_free(ref_csr* c) { delete c; }
int32_t ref_csr_n(const ref_csr* c) { return c->m.nrows; }
int64_t ref_csr_nnz(const ref_csr* c) { return c->m.nnz(); }
const int64_t* ref_csr_ptr(const ref_csr* c) { return c->m.row_ptr.data(); }
const int32_t* ref_csr_col(const ref_csr* c) { return c->m.col_idx.data(); }
const double* ref_csr_val(const ref_csr* c) { return c->m.values.data(); }

// ordering.hpp:355-399: range count (bounds written when cap >= count), or -1.
int32_t ref_load_ordering(const char* path, int32_t n, int32_t* perm, int32_t cap, int32_t* bounds) {
  try {
    auto [p, rl] = load_ordering(path, n);
    if (perm) std::memcpy(perm, p.perm.data(), sizeof(int32_t) * static_cast<std::size_t>(n));
    const int32_t cnt = rl.count();
    if (bounds && cap >= cnt) {
      bounds[0] = cnt ? rl.ranges[0].begin : 0;
      for (int32_t k = 0; k < cnt; ++k) bounds[k + 1] = rl.ranges[static_cast<std::size_t>(k)].end;
    }
    return cnt;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
