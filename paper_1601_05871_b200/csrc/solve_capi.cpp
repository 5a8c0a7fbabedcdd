// C ABI of the triangular solves with the factor (include/tacho_b200.h,
// "triangular solves"): the preconditioner apply of IC(k)-preconditioned CG,
// SURVEY.md §8(f) rank 3. The reference has no solve; the order
// of operations is the oracle's (oracle.c orc_trisolve), which the device
// reproduces bit for bit. No exception crosses these functions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tacho_b200.h"
#include "device/solve_api.hpp"

namespace tcb_internal {
bool ctx_factor(tcg_ctx* c, int member, int* device, cudaStream_t* stream, const double** vals,
                std::int64_t* n, std::int64_t* nnz);
}

struct tcg_solve {
  tcg_ctx* ctx = nullptr;
  int device = 0;
  int sm_count = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  std::int32_t n = 0;
  std::int64_t nnz = 0, noff = 0;
  std::int32_t depth_f = 0, depth_b = 0;
  void* arena = nullptr;
  int4* rec = nullptr;   // 2 n positions: forward rows by level, then backward rows by level
  int* idx = nullptr;    // operand rows: forward entries (Uᵀ: per column, ascending row), then backward
  int* fpos = nullptr;   // forward entries' positions in U
  double* fval = nullptr;  // forward entries' values, gathered per apply
  double* b = nullptr;   // staged right-hand side
  double* y = nullptr;
  double* x = nullptr;
  int* error = nullptr;
  unsigned long long* trace = nullptr;  // TCG_SOLVE_TRACE=1: per position {start, operands final, end}
  double timeout_s = 30.0;
  void* a_arena = nullptr;  // the system matrix for tcg_solve_spmv (PᵀAP, CSR)
  long long* a_ptr = nullptr;
  int* a_col = nullptr;
  double* a_val = nullptr;
  double* cg_partial = nullptr;  // per block of the CG update kernels
  int cg_grid = 0;
};

namespace {

#define SOLVE_TRY(s, expr)                                                          \
  do {                                                                              \
    const cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess) {                                                        \
      (s)->err = std::string(#expr) + ": " + cudaGetErrorString(e_);                \
      return TCG_CUDA;                                                              \
    }                                                                               \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Forward (Uᵀ y = b): unknown j gathers U(i,j) y_i over column j, ascending i.
// Backward (U x = y): unknown i gathers U(i,j) x_j along row i, ascending j.
// Order: level, then the longer remaining chain first (the other direction's
// level is this one's height), then row.
struct Tables {
  std::vector<int4> rec;
  std::vector<int> idx, fpos;
  std::int32_t depth_f = 0, depth_b = 0;
};

bool build_tables(const tcg_csr_view* u, Tables& T, std::string& err) {
  const std::int32_t n = u->n;
  const std::int64_t* up = u->row_ptr;
  const std::int32_t* uc = u->col_idx;
  for (std::int32_t i = 0; i < n; ++i) {
    if (up[i] >= up[i + 1] || uc[up[i]] != i) {
      err = "tcg_solve_create: every row of U must start with its diagonal";
      return false;
    }
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q)
      if (uc[q] <= uc[q - 1] || uc[q] >= n) {
        err = "tcg_solve_create: U's columns must ascend within [i, n)";
        return false;
      }
  }
  const std::int64_t noff = up[n] - n;
  // the backward records index a table of 2 * noff entries with int32 offsets
  if (2 * noff > 0x7fffffffLL || up[n] > 0x7fffffffLL) {
    err = "tcg_solve_create: U beyond 2^30 off-diagonal entries";
    return false;
  }
  // transposed index of the strict upper part
  std::vector<std::int64_t> cptr(static_cast<size_t>(n) + 1, 0);
  for (std::int32_t i = 0; i < n; ++i)
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q) ++cptr[uc[q] + 1];
  for (std::int32_t j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
  T.idx.assign(static_cast<size_t>(2 * noff), 0);
  T.fpos.assign(static_cast<size_t>(noff), 0);
  std::vector<std::int64_t> fill(cptr.begin(), cptr.end() - 1);
  for (std::int32_t i = 0; i < n; ++i)  // rows ascending: each column's list ascends in i
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q) {
      const std::int64_t e = fill[uc[q]]++;
      T.idx[static_cast<size_t>(e)] = i;
      T.fpos[static_cast<size_t>(e)] = static_cast<int>(q);
    }
  for (std::int32_t i = 0; i < n; ++i)  // backward: U's own rows after the diagonal
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q) T.idx[static_cast<size_t>(noff + q - (i + 1))] = uc[q];
  // levels: forward over columns (sources i < j), backward over rows (sources j > i)
  std::vector<std::int32_t> lf(static_cast<size_t>(n), 1), lb(static_cast<size_t>(n), 1);
  for (std::int32_t i = 0; i < n; ++i)
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q) lf[uc[q]] = std::max(lf[uc[q]], lf[i] + 1);
  for (std::int32_t i = n - 1; i >= 0; --i)
    for (std::int64_t q = up[i] + 1; q < up[i + 1]; ++q) lb[i] = std::max(lb[i], lb[uc[q]] + 1);
  for (std::int32_t i = 0; i < n; ++i) {
    T.depth_f = std::max(T.depth_f, lf[i]);
    T.depth_b = std::max(T.depth_b, lb[i]);
  }
  std::vector<std::int32_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  T.rec.clear();
  T.rec.reserve(static_cast<size_t>(2 * n));
  std::stable_sort(order.begin(), order.end(), [&](std::int32_t a, std::int32_t b) {
    return lf[a] != lf[b] ? lf[a] < lf[b] : lb[a] > lb[b];
  });
  for (std::int32_t j : order)
    T.rec.push_back(make_int4(static_cast<int>(cptr[j]), static_cast<int>(cptr[j + 1] - cptr[j]),
                              static_cast<int>(up[j]), j));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](std::int32_t a, std::int32_t b) {
    return lb[a] != lb[b] ? lb[a] < lb[b] : lf[a] > lf[b];
  });
  for (std::int32_t i : order) {
    const int len = static_cast<int>(up[i + 1] - up[i] - 1);
    T.rec.push_back(make_int4(static_cast<int>(noff + up[i] - i), static_cast<int>(len | 0x80000000u),
                              static_cast<int>(up[i]), i));
  }
  return true;
}

}  // namespace

extern "C" {

tcg_status tcg_solve_create(tcg_ctx* ctx, const tcg_csr_view* u, tcg_solve** out) {
  if (!out) return TCG_INVALID;
  *out = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(ctx, 0, &device, &stream, &vals, &n, &nnz)) return TCG_INVALID;
  if (!u || u->n != n || u->nnz != nnz || !u->row_ptr || (u->nnz > 0 && !u->col_idx) ||
      u->row_ptr[0] != 0 || u->row_ptr[u->n] != u->nnz)
    return TCG_INVALID;
  auto s = std::make_unique<tcg_solve>();
  s->ctx = ctx;
  s->device = device;
  s->n = u->n;
  s->nnz = u->nnz;
  Tables T;
  if (!build_tables(u, T, s->err)) {
    tcg_solve_destroy(s.release());
    return TCG_INVALID;
  }
  s->noff = static_cast<std::int64_t>(T.fpos.size());
  s->depth_f = T.depth_f;
  s->depth_b = T.depth_b;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev1);
  const size_t nd = sizeof(double) * std::max<std::int64_t>(n, 1);
  const size_t noff1 = static_cast<size_t>(std::max<std::int64_t>(s->noff, 1));
  const size_t o_rec = 0, o_idx = align_up(sizeof(int4) * std::max<size_t>(T.rec.size(), 1), 256);
  const size_t o_fpos = o_idx + align_up(sizeof(int) * 2 * noff1, 256);
  const size_t o_fval = o_fpos + align_up(sizeof(int) * noff1, 256);
  const size_t o_b = o_fval + align_up(sizeof(double) * noff1, 256);
  const size_t o_y = o_b + align_up(nd, 256), o_x = o_y + align_up(nd, 256), o_err = o_x + align_up(nd, 256);
  if (e == cudaSuccess) e = cudaMalloc(&s->arena, o_err + 256);
  if (e != cudaSuccess) {
    tcg_solve_destroy(s.release());
    return TCG_CUDA;
  }
  char* base = static_cast<char*>(s->arena);
  s->rec = reinterpret_cast<int4*>(base + o_rec);
  s->idx = reinterpret_cast<int*>(base + o_idx);
  s->fpos = reinterpret_cast<int*>(base + o_fpos);
  s->fval = reinterpret_cast<double*>(base + o_fval);
  s->b = reinterpret_cast<double*>(base + o_b);
  s->y = reinterpret_cast<double*>(base + o_y);
  s->x = reinterpret_cast<double*>(base + o_x);
  s->error = reinterpret_cast<int*>(base + o_err);
  if (!T.rec.empty()) e = cudaMemcpy(s->rec, T.rec.data(), sizeof(int4) * T.rec.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !T.idx.empty())
    e = cudaMemcpy(s->idx, T.idx.data(), sizeof(int) * T.idx.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !T.fpos.empty())
    e = cudaMemcpy(s->fpos, T.fpos.data(), sizeof(int) * T.fpos.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(s->error, 0, sizeof(int));  // the sticky watchdog flag
  if (e != cudaSuccess) {
    tcg_solve_destroy(s.release());
    return TCG_CUDA;
  }
  *out = s.release();
  return TCG_OK;
}

void tcg_solve_destroy(tcg_solve* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  if (s->arena) cudaFree(s->arena);
  if (s->trace) cudaFree(s->trace);
  if (s->a_arena) cudaFree(s->a_arena);
  if (s->cg_partial) cudaFree(s->cg_partial);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  delete s;
}

const char* tcg_solve_error(const tcg_solve* s) { return s ? s->err.c_str() : "null tcg_solve"; }

namespace {

// Enqueue one apply on the context's stream (no host wait). The watchdog flag
// is sticky: the kernel only sets it; read_and_clear_error() consumes it.
tcg_status enqueue_apply(tcg_solve* s, const double* b_dev, double* x_dev, int32_t which, int* grid_out,
                         cudaStream_t* stream_out) {
  if (!s || which < 1 || which > 3 || (s->n > 0 && (!b_dev || !x_dev))) {
    if (s) s->err = "tcg_solve_apply: which must be 1, 2 or 3 and the vectors non-null";
    return TCG_INVALID;
  }
  int device = 0;
  cudaStream_t stream = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(s->ctx, 0, &device, &stream, &vals, &n, &nnz) || n != s->n || nnz != s->nnz) {
    s->err = "tcg_solve_apply: the context no longer holds this factor's pattern";
    return TCG_INVALID;
  }
  SOLVE_TRY(s, cudaSetDevice(device));
  const size_t nd = sizeof(double) * static_cast<size_t>(s->n);
  int occ = 0;
  SOLVE_TRY(s, tcbdev::solve_occupancy(&occ));
  if (const char* e = std::getenv("TCG_SOLVE_CTAS")) occ = std::max(1, std::min(occ, std::atoi(e)));  // experiments
  const int warps = tcbdev::kSolveThreads / 32;
  tcbdev::SolveParams P{};
  P.pos_begin = which == 2 ? s->n : 0;
  P.pos_end = which == 1 ? s->n : 2 * s->n;
  P.rec = s->rec;
  P.idx = s->idx;
  P.fval = s->fval;
  P.u = vals;
  P.b = b_dev;
  P.y = s->y;
  P.x = s->x;
  P.poll_y = which == 3;
  P.error = s->error;
  P.timeout_ns = static_cast<unsigned long long>(s->timeout_s * 1e9);
  if (!s->trace && std::getenv("TCG_SOLVE_TRACE") && s->n > 0)
    SOLVE_TRY(s, cudaMalloc(&s->trace, sizeof(unsigned long long) * 6 * static_cast<size_t>(s->n)));
  P.trace = s->trace;
  const int npos = P.pos_end - P.pos_begin;
  const int grid = std::max(1, std::min(s->sm_count * std::max(occ, 1), (npos + warps - 1) / warps));
  SOLVE_TRY(s, cudaEventRecord(s->ev0, stream));
  if (s->n > 0) {
    SOLVE_TRY(s, cudaMemsetAsync(s->y, 0xFF, 2 * align_up(nd, 256), stream));  // y and x: the marker
    if (which & 1) SOLVE_TRY(s, tcbdev::launch_solve_gather(vals, s->fpos, s->fval, s->noff, s->sm_count, stream));
    SOLVE_TRY(s, tcbdev::launch_trisolve(P, grid, stream));
    SOLVE_TRY(s, cudaMemcpyAsync(x_dev, which == 1 ? s->y : s->x, nd, cudaMemcpyDeviceToDevice, stream));
  }
  SOLVE_TRY(s, cudaEventRecord(s->ev1, stream));
  *grid_out = grid;
  *stream_out = stream;
  return TCG_OK;
}

// After the stream is idle: report (and clear) a watchdog expiry of any apply since the last check.
tcg_status read_and_clear_error(tcg_solve* s) {
  if (s->n <= 0) return TCG_OK;
  int error = 0;
  SOLVE_TRY(s, cudaMemcpy(&error, s->error, sizeof(int), cudaMemcpyDeviceToHost));
  if (!error) return TCG_OK;
  SOLVE_TRY(s, cudaMemset(s->error, 0, sizeof(int)));
  s->err = "tcg_solve_apply: device watchdog expired";
  return TCG_TIMEOUT;
}

}  // namespace

tcg_status tcg_solve_apply_device(tcg_solve* s, const double* b_dev, double* x_dev, int32_t which,
                                  tcg_solve_stats* st) {
  int grid = 0;
  cudaStream_t stream = nullptr;
  const tcg_status q = enqueue_apply(s, b_dev, x_dev, which, &grid, &stream);
  if (q != TCG_OK) return q;
  SOLVE_TRY(s, cudaEventSynchronize(s->ev1));
  const tcg_status e = read_and_clear_error(s);
  if (st) {
    float ms = 0.f;
    SOLVE_TRY(s, cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    st->device_ms = ms;
    st->depth_forward = s->depth_f;
    st->depth_backward = s->depth_b;
    st->grid_ctas = grid;
    st->kernel_launches = s->n > 0 ? ((which & 1) && s->noff > 0 ? 2 : 1) : 0;
  }
  return e;
}

tcg_status tcg_solve_apply_async(tcg_solve* s, const double* b_dev, double* x_dev, int32_t which) {
  int grid = 0;
  cudaStream_t stream = nullptr;
  return enqueue_apply(s, b_dev, x_dev, which, &grid, &stream);
}

tcg_status tcg_solve_sync(tcg_solve* s) {
  if (!s) return TCG_INVALID;
  int device = 0;
  cudaStream_t stream = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(s->ctx, 0, &device, &stream, &vals, &n, &nnz)) return TCG_INVALID;
  SOLVE_TRY(s, cudaSetDevice(device));
  SOLVE_TRY(s, cudaStreamSynchronize(stream));
  return read_and_clear_error(s);
}

tcg_status tcg_solve_trace(tcg_solve* s, uint64_t* stamps, void* recs) {
  if (!s || !s->trace || !stamps) return TCG_INVALID;
  SOLVE_TRY(s, cudaSetDevice(s->device));
  SOLVE_TRY(s, cudaMemcpy(stamps, s->trace, sizeof(uint64_t) * 6 * static_cast<size_t>(s->n), cudaMemcpyDeviceToHost));
  if (recs) SOLVE_TRY(s, cudaMemcpy(recs, s->rec, sizeof(int4) * 2 * static_cast<size_t>(s->n), cudaMemcpyDeviceToHost));
  return TCG_OK;
}

tcg_status tcg_solve_set_matrix(tcg_solve* s, const tcg_csr_view* a) {
  if (!s || !a || a->n != s->n || a->nnz < 0 || !a->row_ptr || (a->nnz > 0 && (!a->col_idx || !a->values)) ||
      a->row_ptr[0] != 0 || a->row_ptr[a->n] != a->nnz) {
    if (s) s->err = "tcg_solve_set_matrix: the matrix must be n x n CSR with values";
    return TCG_INVALID;
  }
  for (int32_t i = 0; i < a->n; ++i)
    for (int64_t q = a->row_ptr[i]; q < a->row_ptr[i + 1]; ++q)
      if (a->col_idx[q] < 0 || a->col_idx[q] >= a->n) {
        s->err = "tcg_solve_set_matrix: column index out of range";
        return TCG_INVALID;
      }
  SOLVE_TRY(s, cudaSetDevice(s->device));
  if (s->a_arena) {
    SOLVE_TRY(s, cudaDeviceSynchronize());
    SOLVE_TRY(s, cudaFree(s->a_arena));
    s->a_arena = nullptr;
  }
  const size_t np1 = static_cast<size_t>(a->n) + 1, nz = static_cast<size_t>(std::max<int64_t>(a->nnz, 1));
  const size_t o_col = align_up(sizeof(long long) * np1, 256), o_val = o_col + align_up(sizeof(int) * nz, 256);
  SOLVE_TRY(s, cudaMalloc(&s->a_arena, o_val + sizeof(double) * nz));
  char* base = static_cast<char*>(s->a_arena);
  s->a_ptr = reinterpret_cast<long long*>(base);
  s->a_col = reinterpret_cast<int*>(base + o_col);
  s->a_val = reinterpret_cast<double*>(base + o_val);
  SOLVE_TRY(s, cudaMemcpy(s->a_ptr, a->row_ptr, sizeof(long long) * np1, cudaMemcpyHostToDevice));
  if (a->nnz > 0) {
    SOLVE_TRY(s, cudaMemcpy(s->a_col, a->col_idx, sizeof(int) * a->nnz, cudaMemcpyHostToDevice));
    SOLVE_TRY(s, cudaMemcpy(s->a_val, a->values, sizeof(double) * a->nnz, cudaMemcpyHostToDevice));
  }
  return TCG_OK;
}

tcg_status tcg_solve_spmv(tcg_solve* s, const double* x_dev, double* y_dev) {
  if (!s || !s->a_arena || (s->n > 0 && (!x_dev || !y_dev))) {
    if (s) s->err = "tcg_solve_spmv: no matrix set (tcg_solve_set_matrix) or null vectors";
    return TCG_INVALID;
  }
  int device = 0;
  cudaStream_t stream = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(s->ctx, 0, &device, &stream, &vals, &n, &nnz)) return TCG_INVALID;
  SOLVE_TRY(s, cudaSetDevice(device));
  SOLVE_TRY(s, tcbdev::launch_spmv(s->n, s->a_ptr, s->a_col, s->a_val, x_dev, y_dev, s->sm_count, stream));
  return TCG_OK;
}

namespace {

tcg_status cg_prepare(tcg_solve* s, cudaStream_t* stream) {
  int device = 0;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(s->ctx, 0, &device, stream, &vals, &n, &nnz)) return TCG_INVALID;
  SOLVE_TRY(s, cudaSetDevice(device));
  if (!s->cg_partial) {
    SOLVE_TRY(s, tcbdev::cg_grid(s->sm_count, &s->cg_grid));
    SOLVE_TRY(s, cudaMalloc(&s->cg_partial, sizeof(double) * static_cast<size_t>(s->cg_grid)));
  }
  return TCG_OK;
}

}  // namespace

tcg_status tcg_solve_cg_step(tcg_solve* s, double* x, double* r, const double* p, const double* ap, double* state,
                             double* hist, int32_t it) {
  if (!s || !state || !hist || it < 0 || (s->n > 0 && (!x || !r || !p || !ap))) {
    if (s) s->err = "tcg_solve_cg_step: null vectors";
    return TCG_INVALID;
  }
  cudaStream_t st = nullptr;
  const tcg_status ok = cg_prepare(s, &st);
  if (ok != TCG_OK) return ok;
  SOLVE_TRY(s, tcbdev::launch_cg_step(s->n, x, r, p, ap, state, hist, it, s->cg_partial, s->cg_grid, st));
  return TCG_OK;
}

tcg_status tcg_solve_cg_direction(tcg_solve* s, const double* r, const double* z, double* p, double* state) {
  if (!s || !state || (s->n > 0 && (!r || !z || !p))) {
    if (s) s->err = "tcg_solve_cg_direction: null vectors";
    return TCG_INVALID;
  }
  cudaStream_t st = nullptr;
  const tcg_status ok = cg_prepare(s, &st);
  if (ok != TCG_OK) return ok;
  SOLVE_TRY(s, tcbdev::launch_cg_direction(s->n, r, z, p, state, s->cg_partial, s->cg_grid, st));
  return TCG_OK;
}

tcg_status tcg_solve_stream(tcg_solve* s, void** stream) {
  int device = 0;
  cudaStream_t st = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!s || !stream || !tcb_internal::ctx_factor(s->ctx, 0, &device, &st, &vals, &n, &nnz)) return TCG_INVALID;
  *stream = st;
  return TCG_OK;
}

tcg_status tcg_solve_apply(tcg_solve* s, const double* b, double* x, int32_t which, tcg_solve_stats* st) {
  if (!s || (s->n > 0 && (!b || !x))) return TCG_INVALID;
  int device = 0;
  cudaStream_t stream = nullptr;
  const double* vals = nullptr;
  std::int64_t n = 0, nnz = 0;
  if (!tcb_internal::ctx_factor(s->ctx, 0, &device, &stream, &vals, &n, &nnz)) return TCG_INVALID;
  SOLVE_TRY(s, cudaSetDevice(device));
  const size_t nd = sizeof(double) * static_cast<size_t>(s->n);
  if (s->n > 0) SOLVE_TRY(s, cudaMemcpyAsync(s->b, b, nd, cudaMemcpyHostToDevice, stream));
  const tcg_status r = tcg_solve_apply_device(s, s->b, s->b, which, st);
  if (r != TCG_OK) return r;
  if (s->n > 0) {
    SOLVE_TRY(s, cudaMemcpyAsync(x, s->b, nd, cudaMemcpyDeviceToHost, stream));
    SOLVE_TRY(s, cudaStreamSynchronize(stream));
  }
  return TCG_OK;
}

}  // extern "C"
