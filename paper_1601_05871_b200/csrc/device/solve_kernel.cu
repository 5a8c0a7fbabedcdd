// Triangular solves with the factor U on the device (SURVEY.md §8(f) rank 3:
// the preconditioner apply z = (UᵀU)⁻¹ r of an IC(k)-preconditioned CG).
//
// The same value-flow schedule as the factorization (flow_kernel.cu): the
// outputs y (forward, Uᵀ y = b) and x (backward, U x = y) start as a marker
// NaN; one warp per unknown gathers its operands with strong loads and
// re-polls any that still read the marker; the data is its own flag. Rows run
// in a static topological order (forward rows by level, then backward rows by
// level) dealt round-robin to the co-resident warps, so the lowest unfinished
// position only reads final values and the launch cannot deadlock.
//
// Per unknown the products U(i,j)*v_i are formed in parallel by the lanes
// (each rounded on its own) and subtracted in ascending source order by a
// broadcast chain -- the oracle's sequential order (oracle.c orc_trisolve),
// so the solution is bitwise equal to it.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "solve_api.hpp"
#include "sync.cuh"

namespace tcbdev {

namespace {

constexpr unsigned long long kSolveUnset = ~0ull;  // memset 0xFF; a NaN arithmetic never yields
constexpr unsigned long long kCanonNaN = 0x7FFFFFFFFFFFFFFFull;

__device__ __forceinline__ double poll(const double* p, const SolveParams& P, unsigned long long t0) {
  unsigned long long x = ld_relaxed_u64(p);
  if (x == kSolveUnset) {
    unsigned spins = 0;
    do {
      x = ld_relaxed_u64(p);
      if (++spins == 1024u) {
        spins = 0;
        if (ld_relaxed(P.error) || gtimer() - t0 > P.timeout_ns) {
          atomicCAS(P.error, 0, 1);  // abandoned: the host reports TCG_TIMEOUT
          return 0.0;
        }
      }
    } while (x == kSolveUnset);
  }
  return __longlong_as_double(static_cast<long long>(x));
}

}  // namespace

// One unknown per warp; the record, operand indices, values, diagonal and
// right-hand side of the warp's next row are loaded while the current row
// polls (all immutable during the launch), so only the operand hand-off is on
// a row's critical path.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) trisolve_flow(SolveParams P) {
  constexpr int kWarps = THREADS / 32;
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * kWarps;
  const unsigned long long t0 = gtimer();
  struct Row {
    int4 r;
    int i;       // lane's operand index (first 32 entries)
    double v;    // lane's value
    double d;    // diagonal
    double b;    // right-hand side (forward rows, and backward rows without poll_y)
  };
  auto fetch = [&](int q) {
    Row w{};
    if (q >= P.pos_end) return w;
    w.r = __ldg(P.rec + q);
    const bool back = w.r.y < 0;
    const int len = w.r.y & 0x7fffffff;
    if (lane < len) {
      w.i = __ldg(P.idx + w.r.x + lane);
      w.v = back ? __ldg(P.u + w.r.z + 1 + lane) : __ldg(P.fval + w.r.x + lane);
    }
    w.d = __ldg(P.u + w.r.z);
    if (!back || !P.poll_y) w.b = __ldg(P.b + w.r.w);
    return w;
  };
  int q = P.pos_begin + blockIdx.x * kWarps + (threadIdx.x >> 5);
  Row cur = fetch(q);
  for (; q < P.pos_end; q += W) {
    const Row nxt = fetch(q + W);  // in flight while this row polls
    const bool back = cur.r.y < 0;
    const int len = cur.r.y & 0x7fffffff, row = cur.r.w;
    const double* src = back ? P.x : P.y;
    double* dst = back ? P.x : P.y;
    unsigned long long* stamp = P.trace ? P.trace + 3 * static_cast<long long>(q) : nullptr;
    if (stamp && lane == 0) stamp[0] = gtimer();
    double t = (back && P.poll_y) ? poll(P.y + row, P, t0) : cur.b;  // backward: this row's forward result
    // 32 entries per round, one per lane; the next round's entry loads
    // overlap this round's chain. (Issuing several rounds' operand loads
    // together was slower overall on B200: C2-C6 +8-20%, C3 backward -17%.)
    int i = cur.i;
    double v = cur.v;
    for (int c0 = 0; c0 < len; c0 += 32) {
      const int k = c0 + lane;
      double p = 0.0;
      if (k < len) p = __dmul_rn(v, poll(src + i, P, t0));
      // reconverge before the chain: without it the lanes that found their
      // operand final park at the first shuffle while the others spin, and
      // the apply ran 2.7-4x slower on B200 (C2 forward 1.06 -> 0.26 ms)
      __syncwarp();
      if (stamp && c0 == 0 && lane == 0) stamp[1] = gtimer();
      if (k + 32 < len) {
        i = __ldg(P.idx + cur.r.x + k + 32);
        v = back ? __ldg(P.u + cur.r.z + 1 + k + 32) : __ldg(P.fval + cur.r.x + k + 32);
      }
      const int m = min(32, len - c0);
      for (int j = 0; j < m; ++j) t = __dsub_rn(t, __shfl_sync(0xffffffffu, p, j));
    }
    if (stamp && len == 0 && lane == 0) stamp[1] = gtimer();
    if (lane == 0) {
      unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(__ddiv_rn(t, cur.d)));
      if (bits == kSolveUnset) bits = kCanonNaN;
      st_relaxed_u64(dst + row, bits);
      if (stamp) stamp[2] = gtimer();
    }
    cur = nxt;
  }
}

__global__ void solve_gather(const double* __restrict__ u, const int* __restrict__ pos, double* __restrict__ fval,
                             long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
    fval[e] = __ldg(u + __ldg(pos + e));
}

cudaError_t launch_solve_gather(const double* u, const int* pos, double* fval, long long n, int sm_count,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  blocks = blocks > 8LL * sm_count ? 8LL * sm_count : blocks;
  solve_gather<<<static_cast<int>(blocks), 256, 0, st>>>(u, pos, fval, n);
  return cudaGetLastError();
}

// The caller's other operation per CG iteration: y = A x with the system
// matrix. HBM-bound (12 bytes per entry), one thread per row, sums in column
// order; a stencil row is 7-81 entries, so the rows of a warp touch
// neighbouring lines and L2 serves most of the gather of x.
__global__ void spmv_csr(int n, const long long* __restrict__ ptr, const int* __restrict__ col,
                         const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (long long q = __ldg(ptr + i), e = __ldg(ptr + i + 1); q < e; ++q)
      s = __dadd_rn(s, __dmul_rn(__ldg(val + q), __ldg(x + __ldg(col + q))));
    y[i] = s;
  }
}

cudaError_t launch_spmv(int n, const long long* ptr, const int* col, const double* val, const double* x,
                        double* y, int sm_count, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 255) / 256;
  blocks = blocks > 16 * sm_count ? 16 * sm_count : blocks;
  spmv_csr<<<blocks, 256, 0, st>>>(n, ptr, col, val, x, y);
  return cudaGetLastError();
}

// ---- conjugate-gradient vector updates (the caller of the apply) ----------
// Two cooperative kernels per iteration replace a dozen small launches. The
// dots are deterministic: every thread sums its strided elements in order,
// every block reduces its threads in a fixed tree into partial[block], and
// after a grid barrier every block sums the partials in block order -- the
// same bits in every block and in every run. state = {rz, live (1/0), thr}.
namespace {

template <int T>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < T / 32; ++i) s = __dadd_rn(s, red[i]);
  return s;  // valid in thread 0
}

// the sum of the blocks' partials in a fixed order (lane l sums blocks l, l+32,
// ... in order, then a fixed shuffle tree), broadcast to the block
__device__ __forceinline__ double grid_total(const double* partial, double* red) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) s = __dadd_rn(s, __ldcg(partial + b));
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(kFull, s, o));
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const double s = red[0];
  __syncthreads();
  return s;
}

// alpha = rz / (p . ap); x += alpha p and r -= alpha ap where live; ||r|| -> hist[it]; live &= ||r|| > thr
__global__ void __launch_bounds__(256) cg_step(int n, double* x, double* r, const double* p, const double* ap,
                                               double* state, double* hist, int it, double* partial) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[8];
  const int stride = gridDim.x * blockDim.x;
  double d = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) d = __dadd_rn(d, __dmul_rn(p[i], ap[i]));
  d = block_sum<256>(d, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = d;
  __threadfence();
  grid.sync();
  const double pap = grid_total(partial, red);
  const bool live = __ldcg(state + 1) != 0.0;
  const double alpha = __ddiv_rn(__ldcg(state), pap);
  double q = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double ri = r[i];
    if (live) {  // (where, not alpha * live: a frozen step may carry 0/0)
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      ri = __dsub_rn(ri, __dmul_rn(alpha, ap[i]));
      r[i] = ri;
    }
    q = __dadd_rn(q, __dmul_rn(ri, ri));
  }
  q = block_sum<256>(q, red);
  grid.sync();  // every block has read `partial` (pap) before it is reused
  if (threadIdx.x == 0) partial[blockIdx.x] = q;
  __threadfence();
  grid.sync();
  const double nr = __dsqrt_rn(grid_total(partial, red));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hist[it] = nr;
    if (live && nr <= state[2]) state[1] = 0.0;  // a NaN norm stays live
  }
}

// beta = (r . z) / rz; p = p * beta + z; rz = r . z
__global__ void __launch_bounds__(256) cg_direction(int n, const double* r, const double* z, double* p,
                                                    double* state, double* partial) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[8];
  const int stride = gridDim.x * blockDim.x;
  double d = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) d = __dadd_rn(d, __dmul_rn(r[i], z[i]));
  d = block_sum<256>(d, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = d;
  __threadfence();
  grid.sync();
  const double rz_new = grid_total(partial, red);
  const double beta = __ddiv_rn(rz_new, __ldcg(state));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = __dadd_rn(__dmul_rn(p[i], beta), z[i]);
  grid.sync();  // every block has read the old rz
  if (blockIdx.x == 0 && threadIdx.x == 0) state[0] = rz_new;
}

}  // namespace

cudaError_t cg_grid(int sm_count, int* grid) {
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_step, 256, 0);
  int occ2 = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, cg_direction, 256, 0);
  // one block per SM: enough threads for these vectors, and few partials to sum
  *grid = (std::min(occ, occ2) >= 1 ? 1 : 0) * sm_count;
  if (*grid < 1) *grid = 1;
  return e;
}

cudaError_t launch_cg_step(int n, double* x, double* r, const double* p, const double* ap, double* state,
                           double* hist, int it, double* partial, int grid, cudaStream_t st) {
  void* args[] = {&n, &x, &r, const_cast<const double**>(&p), const_cast<const double**>(&ap), &state, &hist, &it,
                  &partial};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&cg_step), grid, 256, args, 0, st);
}

cudaError_t launch_cg_direction(int n, const double* r, const double* z, double* p, double* state, double* partial,
                                int grid, cudaStream_t st) {
  void* args[] = {&n, const_cast<const double**>(&r), const_cast<const double**>(&z), &p, &state, &partial};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&cg_direction), grid, 256, args, 0, st);
}

cudaError_t solve_occupancy(int* ctas_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, trisolve_flow<kSolveThreads>, kSolveThreads,
                                                       0);
}

cudaError_t launch_trisolve(const SolveParams& p, int grid, cudaStream_t st) {
  return launch_resident(reinterpret_cast<const void*>(&trisolve_flow<kSolveThreads>), grid, kSolveThreads, 0, st, p);
}

}  // namespace tcbdev
