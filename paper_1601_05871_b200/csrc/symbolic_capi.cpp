// C ABI of the device level-k symbolic phase (include/tacho_b200.h, "level-k
// on the device"): the reference's levelk_pattern_bfs (symbolic.hpp:57-120)
// run by csrc/device/symbolic_kernel.cu. No exception crosses these functions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tacho_b200.h"
#include "device/symbolic_api.hpp"

struct tcg_sym {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  int32_t n = 0;
  int64_t nnz_a = 0, nnz_triu = 0, nnz_u = -1;
  long long* a_ptr = nullptr;  // device copies of PᵀAP's pattern
  int* a_col = nullptr;
  long long* count = nullptr;  // n + 1
  long long* u_ptr = nullptr;  // n + 1
  int* u_col = nullptr;
  int64_t u_cap = 0;
  int* over = nullptr;         // two row lists of n + 1, then their two counts
  int* mark = nullptr;         // slow path scratch
  int* front = nullptr;
  int64_t slow_slots = 0;
  int64_t cap_mark = 0;        // slow_slots * n the scratch was allocated for
  int32_t cap_n = -1;          // capacities of the per-row and per-entry buffers
  int64_t cap_nnz = -1;
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
  long long* soff = nullptr;        // per row: offset of its copy in scratch, or -1
  unsigned long long* cursor = nullptr;
  int* scratch = nullptr;           // rows written by the count pass
  int64_t scratch_cap = 0;          // ints; grown to the last run's need
};

namespace {

#define SYM_TRY(s, expr)                                                            \
  do {                                                                              \
    const cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess) {                                                        \
      (s)->err = std::string(#expr) + ": " + cudaGetErrorString(e_);                \
      return TCG_CUDA;                                                              \
    }                                                                               \
  } while (0)

void free_dev(void*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

template <class T>
void free_dev(T*& p) {
  void* q = p;
  free_dev(q);
  p = nullptr;
}

void free_problem(tcg_sym* s) {
  free_dev(s->a_ptr);
  free_dev(s->a_col);
  free_dev(s->count);
  free_dev(s->u_ptr);
  free_dev(s->u_col);
  free_dev(s->over);
  free_dev(s->mark);
  free_dev(s->front);
  free_dev(s->scan_tmp);
  free_dev(s->soff);
  free_dev(s->cursor);
  free_dev(s->scratch);
  s->scratch_cap = 0;
  s->u_cap = 0;
  s->slow_slots = 0;
  s->cap_mark = 0;
  s->cap_n = -1;
  s->cap_nnz = -1;
  s->scan_bytes = 0;
  s->nnz_u = -1;
}

}  // namespace

extern "C" {

tcg_status tcg_sym_create(int device, tcg_sym** out) {
  if (!out) return TCG_INVALID;
  *out = nullptr;
  auto s = std::make_unique<tcg_sym>();
  s->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev1);
  if (e != cudaSuccess) {
    tcg_sym_destroy(s.release());
    return TCG_CUDA;
  }
  *out = s.release();
  return TCG_OK;
}

void tcg_sym_destroy(tcg_sym* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  free_problem(s);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

const char* tcg_sym_error(const tcg_sym* s) { return s ? s->err.c_str() : "null tcg_sym"; }

tcg_status tcg_sym_upload(tcg_sym* s, const tcg_csr_view* a) {
  if (!s) return TCG_INVALID;
  // input checks of levelk_pattern_bfs (square, symbolic.hpp:58-59) and of a CSR
  if (!a || a->n < 0 || a->nnz < 0 || (a->n > 0 && !a->row_ptr) || (a->nnz > 0 && !a->col_idx)) {
    s->err = "tcg_sym_upload: null or negative sizes";
    return TCG_INVALID;
  }
  if (a->n > 0 && (a->row_ptr[0] != 0 || a->row_ptr[a->n] != a->nnz)) {
    s->err = "tcg_sym_upload: row_ptr must run from 0 to nnz";
    return TCG_INVALID;
  }
  // the checks and count_upper (csr_matrix.hpp:219-225) over row blocks on the host threads
  const int nt = static_cast<int>(std::clamp<int64_t>(a->n / 65536, 1,
                                                      std::max(1u, std::thread::hardware_concurrency())));
  std::vector<int64_t> triu_part(static_cast<size_t>(nt), 0);
  std::vector<int> bad(static_cast<size_t>(nt), 0);  // 1 row_ptr decreases, 2 column out of range
  auto check = [&](int k) {
    const int32_t b = static_cast<int32_t>(static_cast<int64_t>(a->n) * k / nt);
    const int32_t e = static_cast<int32_t>(static_cast<int64_t>(a->n) * (k + 1) / nt);
    int64_t triu = 0;
    for (int32_t i = b; i < e; ++i) {
      if (a->row_ptr[i + 1] < a->row_ptr[i]) {
        bad[static_cast<size_t>(k)] = 1;
        return;
      }
      for (int64_t q = a->row_ptr[i]; q < a->row_ptr[i + 1]; ++q) {
        const int32_t c = a->col_idx[q];
        if (c < 0 || c >= a->n) {
          bad[static_cast<size_t>(k)] = 2;
          return;
        }
        triu += c >= i;
      }
    }
    triu_part[static_cast<size_t>(k)] = triu;
  };
  {
    std::vector<std::thread> pool;
    for (int k = 1; k < nt; ++k) pool.emplace_back(check, k);
    check(0);
    for (auto& th : pool) th.join();
  }
  int64_t triu = 0;
  for (int k = 0; k < nt; ++k) {  // the first failing block's error, as the sequential scan reports
    if (bad[static_cast<size_t>(k)] == 1) {
      s->err = "tcg_sym_upload: row_ptr decreases";
      return TCG_INVALID;
    }
    if (bad[static_cast<size_t>(k)] == 2) {
      s->err = "tcg_sym_upload: column index out of range";
      return TCG_INVALID;
    }
    triu += triu_part[static_cast<size_t>(k)];
  }
  SYM_TRY(s, cudaSetDevice(s->device));
  SYM_TRY(s, cudaStreamSynchronize(s->stream));
  // device buffers are kept when they are large enough (re-uploads of a new
  // matrix of the same or smaller size cost only the copies)
  if (a->n > s->cap_n || a->nnz > s->cap_nnz) {
    free_problem(s);
    const size_t np1 = static_cast<size_t>(a->n) + 1;
    SYM_TRY(s, cudaMalloc(&s->a_ptr, sizeof(long long) * np1));
    SYM_TRY(s, cudaMalloc(&s->a_col, sizeof(int) * std::max<int64_t>(a->nnz, 1)));
    SYM_TRY(s, cudaMalloc(&s->count, sizeof(long long) * np1));
    SYM_TRY(s, cudaMalloc(&s->u_ptr, sizeof(long long) * np1));
    SYM_TRY(s, cudaMalloc(&s->over, sizeof(int) * (2 * np1 + 2)));
    SYM_TRY(s, cudaMalloc(&s->soff, sizeof(long long) * np1));
    SYM_TRY(s, cudaMalloc(&s->cursor, sizeof(unsigned long long)));
    s->cap_n = a->n;
    s->cap_nnz = a->nnz;
  }
  const size_t np1 = static_cast<size_t>(a->n) + 1;
  s->n = a->n;
  s->nnz_a = a->nnz;
  s->nnz_triu = triu;
  s->nnz_u = -1;
  if (s->mark && s->n > 0 && s->slow_slots * s->n > s->cap_mark) {  // slow-path slots are sized per n
    free_dev(s->mark);
    free_dev(s->front);
    s->slow_slots = 0;
  }
  if (a->n > 0) {
    SYM_TRY(s, cudaMemcpyAsync(s->a_ptr, a->row_ptr, sizeof(long long) * np1, cudaMemcpyHostToDevice, s->stream));
    if (a->nnz > 0)
      SYM_TRY(s, cudaMemcpyAsync(s->a_col, a->col_idx, sizeof(int) * a->nnz, cudaMemcpyHostToDevice, s->stream));
  }
  size_t need = 0;
  SYM_TRY(s, tcbdev::sym_scan(s->count, s->u_ptr, s->n, nullptr, &need, s->stream));
  if (!s->scan_tmp || need > s->scan_bytes) {
    free_dev(s->scan_tmp);
    SYM_TRY(s, cudaMalloc(&s->scan_tmp, std::max<size_t>(need, 16)));
    s->scan_bytes = std::max<size_t>(need, 16);
  }
  SYM_TRY(s, cudaStreamSynchronize(s->stream));
  return TCG_OK;
}

tcg_status tcg_sym_levelk(tcg_sym* s, int32_t level, int32_t flags, tcg_sym_stats* st) {
  if (!s || !s->a_ptr) {
    if (s) s->err = "tcg_sym_levelk: nothing uploaded";
    return TCG_INVALID;
  }
  const auto t0 = std::chrono::steady_clock::now();
  SYM_TRY(s, cudaSetDevice(s->device));
  const int n = s->n;
  tcbdev::SymParams P{};
  P.n = n;
  // levels never exceed n (symbolic.hpp:77-78); a negative level searches like 0
  P.kk = std::min<int32_t>(std::max<int32_t>(level, 0), n);
  P.a_ptr = s->a_ptr;
  P.a_col = s->a_col;
  P.count = s->count;
  P.u_ptr = s->u_ptr;
  // row lists: tier 2 (rows that outgrew tier 1), global-memory path; counters
  int* list1 = s->over;
  int* list2 = s->over + (n + 1);
  int* counters = s->over + 2 * (n + 1);  // [tier 2 rows, global-path rows]
  const int warps = tcbdev::kSymThreads / 32;
  int occ1 = 0, occ2 = 0;
  // small searches (level <= 1, sparse rows): tier 1 runs 4 rows per warp, 8 lanes each
  bool tiny = P.kk <= 1 && s->nnz_a <= 10LL * n;
  if (const char* e = std::getenv("TCG_SYM_TINY")) tiny = std::atoi(e) != 0;
  const int hb1 = tiny ? tcbdev::kSymHashTiny : tcbdev::kSymHashSmall;
  SYM_TRY(s, tcbdev::sym_occupancy(hb1, &occ1));
  SYM_TRY(s, tcbdev::sym_occupancy(tcbdev::kSymHashLarge, &occ2));
  const int grid1 = std::max(1, std::min(s->sm_count * std::max(occ1, 1), (n + warps - 1) / warps));
  const int grid2 = std::max(1, s->sm_count * std::max(occ2, 1));
  int launches = 0;
  if (s->scratch_cap == 0) {  // first run: about the pattern of a level-1 fill; then what the last run used
    const int64_t want = 2 * s->nnz_a + n + 1024;
    SYM_TRY(s, cudaMalloc(&s->scratch, sizeof(int) * static_cast<size_t>(want)));
    s->scratch_cap = want;
  }
  P.scratch = s->scratch;
  P.scratch_cap = s->scratch_cap;
  P.cursor = s->cursor;
  P.soff = s->soff;
  SYM_TRY(s, cudaEventRecord(s->ev0, s->stream));
  SYM_TRY(s, cudaMemsetAsync(s->count + n, 0, sizeof(long long), s->stream));
  SYM_TRY(s, cudaMemsetAsync(counters, 0, 2 * sizeof(int), s->stream));
  SYM_TRY(s, cudaMemsetAsync(s->cursor, 0, sizeof(unsigned long long), s->stream));
  SYM_TRY(s, cudaMemsetAsync(s->soff, 0xFF, sizeof(long long) * (static_cast<size_t>(n) + 1), s->stream));
  int cnt[2] = {0, 0};
  if (flags & TCG_SYM_ALL_SLOW) {  // test hook: every row through the global-memory path
    std::vector<int> all(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) all[static_cast<size_t>(i)] = i;
    cnt[1] = n;
    if (n > 0) SYM_TRY(s, cudaMemcpyAsync(list2, all.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s->stream));
    SYM_TRY(s, cudaMemcpyAsync(counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice, s->stream));
    SYM_TRY(s, cudaStreamSynchronize(s->stream));
  } else if (n > 0) {
    tcbdev::SymParams A = P;  // tier 1: every row
    A.over = list1;
    A.nover = counters;
    SYM_TRY(s, tcbdev::launch_levelk_fast(A, 0, hb1, grid1, s->stream));
    tcbdev::SymParams B = P;  // tier 2: the rows tier 1 handed on (count read on the device)
    B.list = list1;
    B.nlist = counters;
    B.over = list2;
    B.nover = counters + 1;
    SYM_TRY(s, tcbdev::launch_levelk_fast(B, 0, tcbdev::kSymHashLarge, grid2, s->stream));
    launches += 2;
    SYM_TRY(s, cudaMemcpyAsync(cnt, counters, sizeof(cnt), cudaMemcpyDeviceToHost, s->stream));
    SYM_TRY(s, cudaStreamSynchronize(s->stream));
  }
  const int nover = cnt[1];
  P.list = list2;
  P.nlist = counters + 1;
  if (nover > 0) {
    // slots of n stamps + 2 n frontier entries, at most ~1 GiB of scratch
    const int64_t per = 12 * static_cast<int64_t>(n);
    const int64_t cap = std::max<int64_t>(warps, (int64_t{1} << 30) / std::max<int64_t>(per, 1));
    const int64_t slots = std::min<int64_t>({static_cast<int64_t>(nover), cap, int64_t{8} * warps * s->sm_count});
    const int64_t want = (slots + warps - 1) / warps * warps;
    if (want > s->slow_slots) {
      free_dev(s->mark);
      free_dev(s->front);
      SYM_TRY(s, cudaMalloc(&s->mark, sizeof(int) * static_cast<size_t>(want) * n));
      SYM_TRY(s, cudaMalloc(&s->front, sizeof(int) * 2 * static_cast<size_t>(want) * n));
      s->slow_slots = want;
      s->cap_mark = want * n;
    }
    SYM_TRY(s, cudaMemsetAsync(s->mark, 0, sizeof(int) * static_cast<size_t>(s->slow_slots) * n, s->stream));
    P.slow_mark = s->mark;
    P.slow_front = s->front;
    SYM_TRY(s, tcbdev::launch_levelk_slow(P, 0, static_cast<int>(want / warps), s->stream));
    ++launches;
  }
  SYM_TRY(s, tcbdev::sym_scan(s->count, s->u_ptr, n, s->scan_tmp, &s->scan_bytes, s->stream));
  ++launches;
  long long nnz_u = 0;
  unsigned long long used = 0;
  SYM_TRY(s, cudaMemcpyAsync(&nnz_u, s->u_ptr + n, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
  SYM_TRY(s, cudaMemcpyAsync(&used, s->cursor, sizeof(used), cudaMemcpyDeviceToHost, s->stream));
  SYM_TRY(s, cudaStreamSynchronize(s->stream));
  // rows that found no room in scratch are searched again below
  const bool short_scratch = static_cast<int64_t>(used) > s->scratch_cap;
  if (nnz_u >= (int64_t{1} << 31)) {
    s->err = "tcg_sym_levelk: the pattern has 2^31 entries or more";
    return TCG_INVALID;
  }
  if (nnz_u > s->u_cap) {
    free_dev(s->u_col);
    SYM_TRY(s, cudaMalloc(&s->u_col, sizeof(int) * std::max<long long>(nnz_u, 1)));
    s->u_cap = nnz_u;
  }
  P.u_col = s->u_col;
  if (n > 0 && !(flags & TCG_SYM_ALL_SLOW)) {
    const bool long_rows = nnz_u > 24LL * n;  // mean row length
    SYM_TRY(s, tcbdev::launch_levelk_copy(P, long_rows ? grid1 : std::max(1, std::min(32 * s->sm_count, (n + 255) / 256)),
                                          long_rows, s->stream));
    ++launches;
  }
  if (n > 0 && !(flags & TCG_SYM_ALL_SLOW) && short_scratch) {
    tcbdev::SymParams A = P;
    A.list = nullptr;
    SYM_TRY(s, tcbdev::launch_levelk_fast(A, 1, hb1, grid1, s->stream));
    ++launches;
    if (cnt[0] > 0) {
      tcbdev::SymParams B = P;
      B.list = list1;
      B.nlist = counters;
      SYM_TRY(s, tcbdev::launch_levelk_fast(B, 1, tcbdev::kSymHashLarge, grid2, s->stream));
      ++launches;
    }
  }
  if (nover > 0) {
    SYM_TRY(s, tcbdev::launch_levelk_slow(P, 1, static_cast<int>(s->slow_slots / warps), s->stream));
    ++launches;
  }
  SYM_TRY(s, cudaEventRecord(s->ev1, s->stream));
  SYM_TRY(s, cudaStreamSynchronize(s->stream));
  s->nnz_u = nnz_u;
  if (short_scratch) {  // the next run fits in one pass
    free_dev(s->scratch);
    s->scratch_cap = 0;
    const int64_t want = static_cast<int64_t>(used) + static_cast<int64_t>(used) / 8 + 1024;
    SYM_TRY(s, cudaMalloc(&s->scratch, sizeof(int) * static_cast<size_t>(want)));
    s->scratch_cap = want;
  }
  if (st) st->single_pass = short_scratch ? 0 : 1;
  if (st) {
    float ms = 0.f;
    SYM_TRY(s, cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    st->device_ms = ms;
    st->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    st->nnz_u = nnz_u;
    st->nnz_triu_input = s->nnz_triu;
    st->slow_rows = nover;
    st->tier2_rows = cnt[0];
    st->kernel_launches = launches;
    st->grid_ctas = grid1;
  }
  return TCG_OK;
}

tcg_status tcg_sym_download(tcg_sym* s, int64_t* row_ptr, int32_t* col_idx) {
  if (!s || s->nnz_u < 0 || !row_ptr || (s->nnz_u > 0 && !col_idx)) {
    if (s) s->err = "tcg_sym_download: no pattern computed, or null output";
    return TCG_INVALID;
  }
  SYM_TRY(s, cudaSetDevice(s->device));
  SYM_TRY(s, cudaMemcpyAsync(row_ptr, s->u_ptr, sizeof(long long) * (static_cast<size_t>(s->n) + 1),
                             cudaMemcpyDeviceToHost, s->stream));
  if (s->nnz_u > 0)
    SYM_TRY(s, cudaMemcpyAsync(col_idx, s->u_col, sizeof(int) * s->nnz_u, cudaMemcpyDeviceToHost, s->stream));
  SYM_TRY(s, cudaStreamSynchronize(s->stream));
  return TCG_OK;
}

int64_t tcg_sym_nnz(const tcg_sym* s) { return s ? s->nnz_u : -1; }

}  // extern "C"
