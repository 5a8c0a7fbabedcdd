// tacho_b200.hpp -- header-only C++ drop-in for the reference's
//
//   FactorResult factor_by_blocks(const CsrMatrix& a_permuted,
//                                 const FillPattern& fp,
//                                 const RangeList& ranges,
//                                 TaskPolicy& policy);
//   (reference proj/include/taskchol/factorize.hpp:134-137)
//
// on top of the C ABI in tacho_b200.h. The function is a template over the
// caller's types, so code holding the reference's taskchol::CsrMatrix /
// FillPattern / RangeList / FactorResult calls it unchanged:
//
//   #include "taskchol/taskchol.hpp"
//   #include "tacho_b200.hpp"
//   taskchol::FactorResult r =
//       tacho_b200::factor_by_blocks_gpu<taskchol::FactorResult>(an.a_permuted, an.pattern,
//                                                                an.ranges);
//
// Semantics follow the reference: the result owns a fresh factor with
// fp.pattern's arrays; a non-positive pivot throws the caller's
// BreakdownError type (template parameter) with (row, pivot); malformed
// inputs throw std::invalid_argument; a missing diagonal block throws
// std::logic_error (factorize.hpp:173-174). stats.numeric_seconds is the
// device time of the factorization, stats.block_build_seconds the host
// flattening, stats.backend "gpu".
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tacho_b200.h"

namespace tacho_b200 {

struct GpuOptions {
  int device = 0;
  int threads_per_cta = 0;  // 0 = default
  int mode = 0;             // 0 auto, 1/2 task DAG, 3 row DAG (tacho_b200.h)
  double timeout_s = 0.0;
};

namespace detail {

template <class Csr>
tcg_csr_view view(const Csr& m, bool values) {
  tcg_csr_view v{};
  v.n = static_cast<int32_t>(m.nrows);
  v.nnz = static_cast<int64_t>(m.col_idx.size());
  v.row_ptr = reinterpret_cast<const int64_t*>(m.row_ptr.data());
  v.col_idx = reinterpret_cast<const int32_t*>(m.col_idx.data());
  v.values = values ? m.values.data() : nullptr;
  static_assert(sizeof(m.row_ptr[0]) == 8 && sizeof(m.col_idx[0]) == 4,
                "CSR index types must be int64 offsets / int32 indices");
  return v;
}

struct PlanGuard {
  tcg_plan* p = nullptr;
  ~PlanGuard() { tcg_plan_free(p); }
};
struct CtxGuard {
  tcg_ctx* c = nullptr;
  ~CtxGuard() { tcg_destroy(c); }
};

[[noreturn]] inline void raise(tcg_status st, const std::string& msg) {
  if (st == TCG_INVALID) {
    if (msg.find("diagonal block missing") != std::string::npos) throw std::logic_error(msg);
    throw std::invalid_argument(msg);
  }
  throw std::runtime_error(msg);
}

}  // namespace detail

// Breakdown is reported through the caller's exception type (the reference's
// taskchol::BreakdownError(row, pivot) for drop-in use).
struct BreakdownError : std::runtime_error {
  BreakdownError(int32_t r, double p)
      : std::runtime_error("factorization breakdown at row " + std::to_string(r) + ": pivot " +
                           std::to_string(p) + " is not positive"),
        row_(r),
        pivot_(p) {}
  int32_t row() const { return row_; }
  double pivot() const { return pivot_; }
  int32_t row_;
  double pivot_;
};

template <class FactorResultT, class BreakdownT = BreakdownError, class Csr, class Fp, class Ranges>
FactorResultT factor_by_blocks_gpu(const Csr& a_permuted, const Fp& fp, const Ranges& ranges,
                                   const GpuOptions& opt = GpuOptions()) {
  std::vector<int32_t> bounds;
  for (const auto& r : ranges.ranges) {
    if (bounds.empty()) bounds.push_back(r.begin);
    bounds.push_back(r.end);
  }
  const tcg_csr_view av = detail::view(a_permuted, true);
  const tcg_csr_view uv = detail::view(fp.pattern, false);
  const auto t0 = std::chrono::steady_clock::now();
  detail::PlanGuard plan;
  tcg_status st = tcg_plan_build(&av, &uv, static_cast<int32_t>(bounds.empty() ? 0 : bounds.size() - 1),
                                 bounds.data(), &plan.p);
  if (st != TCG_OK) detail::raise(st, tcg_plan_error());
  if (opt.mode == 1 || opt.mode == 2) {  // the task executors run the task-DAG plan's tables
    if ((st = tcg_plan_expand(plan.p)) != TCG_OK) detail::raise(st, tcg_plan_error());
  }
  const double plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  tcg_problem prob{};
  tcg_plan_problem(plan.p, &prob);
  tcg_plan_stats ps{};
  tcg_plan_get_stats(plan.p, &ps);

  detail::CtxGuard ctx;
  st = tcg_create(opt.device, &ctx.c);
  if (st != TCG_OK) detail::raise(st, tcg_last_error(nullptr));
  tcg_options o{};
  o.threads_per_cta = opt.threads_per_cta;
  o.mode = opt.mode;
  o.timeout_s = opt.timeout_s;
  if ((st = tcg_set_options(ctx.c, &o)) != TCG_OK) detail::raise(st, tcg_last_error(ctx.c));
  if ((st = tcg_upload(ctx.c, &prob)) != TCG_OK) detail::raise(st, tcg_last_error(ctx.c));
  tcg_stats fs{};
  st = tcg_factor(ctx.c, &fs);
  if (st == TCG_BREAKDOWN) throw BreakdownT(fs.breakdown_row, fs.breakdown_pivot);
  if (st != TCG_OK) detail::raise(st, tcg_last_error(ctx.c));

  FactorResultT res{};
  res.factor = fp.pattern;  // fresh CSR with the pattern's arrays (factorize.hpp:139-140)
  res.factor.values.assign(static_cast<std::size_t>(prob.nnz), 0.0);  // a pattern may carry no values
  if ((st = tcg_download(ctx.c, res.factor.values.data())) != TCG_OK)
    detail::raise(st, tcg_last_error(ctx.c));
  res.stats.block_build_seconds = plan_s;
  res.stats.numeric_seconds = fs.device_ms / 1e3;
  res.stats.chol_tasks = ps.tasks[0];
  res.stats.trsm_tasks = ps.tasks[1];
  res.stats.herk_tasks = ps.tasks[2];
  res.stats.gemm_tasks = ps.tasks[3];
  res.stats.workers = fs.grid_ctas;
  res.stats.backend = "gpu";
  res.stats.nnz_u = prob.nnz;
  return res;
}

}  // namespace tacho_b200
