// Persistent-scheduler IC(k) Cholesky-by-blocks for sm_100a.
//
// One launch executes the whole task DAG of the reference's factor_by_blocks
// (factorize.hpp:134-235). The host launch list per factorization is
// {prepare, factor}; no per-task host work remains.
//
// Scheduler (replaces TaskPolicy, scheduler.hpp:85-363):
//   * a device ready queue: tasks are appended by whichever thread drops a
//     successor's dependence counter to zero (acq_rel atomics, the device
//     form of complete_locked, scheduler.hpp:232-251); idle CTAs take
//     monotonically increasing tickets and poll their slot;
//   * inline continuation: the first successor a CTA readies is run by that
//     CTA directly, no queue round trip (scheduler.hpp:239-241);
//   * a breakdown latch: the first non-positive pivot wins by CAS and later
//     task bodies are skipped (factorize.hpp:146-167);
//   * a globaltimer watchdog in every spin loop so that a malformed DAG
//     ends the kernel with an error instead of hanging the GPU.
//
// Task bodies (replace kernels.hpp:40-132). A task is executed by one CTA;
// its target rows ("items", host plan.hpp) are claimed by warps in
// ascending row order. Each warp stages the target row's column indices and
// values in shared memory, then streams the (source, entry) pairs of all its
// source rows 32 at a time: every lane loads one entry, forms the product
// with __dmul_rn, locates the column in the staged row by binary search
// (absent columns are the pattern drop) and the products are subtracted with
// __dsub_rn in ascending source order per coordinate (__match_any_sync groups
// lanes hitting the same slot; the lowest lane, i.e. the earliest source,
// goes first). Chol and Trsm rows depend on earlier rows of the same task;
// a per-CTA shared-memory bitmask publishes finished rows. The arithmetic
// sequence per coordinate is exactly the reference's, so the factor is
// bitwise equal to factor_serial (factorize.hpp:94-130): no FMA contraction,
// IEEE division and square root.
#include <cuda_runtime.h>

#include "factor_kernel.cuh"

namespace tcbdev {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_dec_acq_rel(int* p) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ __forceinline__ void raise_error(Ctrl* c, int code) { atomicCAS(&c->error, 0, code); }

// lower_bound over a sorted int array; returns the index of `key` or -1.
template <typename IntPtr>
__device__ __forceinline__ int find_col(IntPtr cols, int len, int key) {
  int lo = 0, n = len;
  while (n > 0) {
    const int half = n >> 1;
    if (cols[lo + half] < key) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return (lo < len && cols[lo] == key) ? lo : -1;
}

// Spin until local row `r` of the running Chol/Trsm task is published.
__device__ __forceinline__ void wait_row(const unsigned* flags, int r, const Params& P,
                                        unsigned long long t0) {
  const volatile unsigned* w = flags + (r >> 5);
  const unsigned bit = 1u << (r & 31);
  unsigned spins = 0;
  while (!(*w & bit)) {
    if (++spins == 4096u) {
      spins = 0;
      if (ld_relaxed(&P.ctrl->error)) return;
      if (gtimer() - t0 > P.timeout_ns) {
        raise_error(P.ctrl, 1);
        return;
      }
    }
  }
}

// Subtract `prod` from tval[slot] for every lane with slot >= 0, lanes with
// equal slots strictly in lane order (lane order == ascending source row).
template <typename ValPtr>
__device__ __forceinline__ void apply_ordered(ValPtr tval, int slot, double prod, int lane) {
  unsigned pend = __ballot_sync(kFull, slot >= 0);
  while (pend) {
    const bool mine = (pend >> lane) & 1u;
    const unsigned peers = __match_any_sync(kFull, mine ? slot : -(lane + 1));
    const bool go = mine && (__ffs(peers) - 1 == lane);
    if (go) tval[slot] = __dsub_rn(tval[slot], prod);
    __syncwarp();
    pend &= ~__ballot_sync(kFull, go);
  }
}

template <int KIND>
__device__ void run_item(const Params& P, int item, int lane, int* scol, double* sval,
                         unsigned* flags, int row_begin, unsigned long long t0) {
  const int4 ia = P.items[2 * item];
  const int4 ib = P.items[2 * item + 1];
  const int tb = ia.x, te = ia.y, local = ia.z, dpos = ia.w;
  const int src_b = ib.x, src_e = ib.y;
  const int L = te - tb;
  const bool staged = L <= P.cap;

  if (staged) {
    for (int k = lane; k < L; k += 32) {
      scol[k] = P.cols[tb + k];
      sval[k] = P.vals[tb + k];
    }
  }
  double diag = 1.0;
  if (KIND == kTrsm) diag = P.vals[dpos];  // final since the Chol task completed
  __syncwarp();
  const int* tcol = staged ? scol : P.cols + tb;
  double* tval = staged ? sval : P.vals + tb;

  for (int s0 = src_b; s0 < src_e; s0 += 32) {
    const int ns = min(32, src_e - s0);
    int4 rec = make_int4(-1, 0, 0, 0);
    if (lane < ns) rec = P.srcs[s0 + lane];
    if (KIND == kChol || KIND == kTrsm) {
      if (lane < ns) wait_row(flags, rec.x, P, t0);
      __syncwarp();
      __threadfence_block();
    }
    const double vrt = (lane < ns) ? P.vals[rec.y] : 0.0;
    const int len = (lane < ns) ? rec.w - rec.z : 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl_own = incl - len;
    for (int q0 = 0; q0 < total; q0 += 32) {
      const int q = q0 + lane;
      int s = 0;
#pragma unroll
      for (int b = 16; b >= 1; b >>= 1) {
        const int v = __shfl_sync(kFull, incl, s + b - 1);
        if (v <= q) s += b;
      }
      const int excl = __shfl_sync(kFull, excl_own, s);
      const int sb = __shfl_sync(kFull, rec.z, s);
      const double v1 = __shfl_sync(kFull, vrt, s);
      int slot = -1;
      double prod = 0.0;
      if (q < total) {
        const int pos = sb + (q - excl);
        const int c = P.cols[pos];
        prod = __dmul_rn(v1, P.vals[pos]);
        slot = find_col(tcol, L, c);
      }
      apply_ordered(tval, slot, prod, lane);
    }
  }

  // finalize: Chol takes the square root and scales the row
  // (kernels.hpp:49-53), Trsm divides by U(t,t) (kernels.hpp:76-78).
  if (KIND == kChol) {
    const double piv = tval[0];
    __syncwarp();
    if (!(piv > 0.0) && lane == 0) {
      if (atomicCAS(&P.ctrl->failed, 0, 1) == 0) {
        P.ctrl->fail_row = row_begin + local;
        P.ctrl->fail_pivot = piv;
      }
    }
    const double d = __dsqrt_rn(piv);
    for (int k = lane; k < L; k += 32) tval[k] = (k == 0) ? d : __ddiv_rn(tval[k], d);
  } else if (KIND == kTrsm) {
    for (int k = lane; k < L; k += 32) tval[k] = __ddiv_rn(tval[k], diag);
  }
  __syncwarp();
  if (staged)
    for (int k = lane; k < L; k += 32) P.vals[tb + k] = sval[k];
  if (KIND == kChol || KIND == kTrsm) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0) atomicOr(flags + (local >> 5), 1u << (local & 31));
  }
  __syncwarp();
}

// Ticket-based pop: returns a ready task id, or -1 once all tasks are done
// (or the run was aborted).
__device__ int pop_task(const Params& P, unsigned long long t0) {
  const int ticket = atomicAdd(&P.ctrl->q_head, 1);
  unsigned spins = 0;
  unsigned ns = 32;
  while (true) {
    if (ticket < P.ntasks) {
      const int v = ld_acquire(P.queue + ticket);
      if (v >= 0) return v;
    }
    if (ld_relaxed(&P.ctrl->done) >= P.ntasks) return -1;
    if (ld_relaxed(&P.ctrl->error)) return -1;
    if (++spins == 256u) {
      spins = 0;
      if (gtimer() - t0 > P.timeout_ns) {
        raise_error(P.ctrl, 1);
        return -1;
      }
    }
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

}  // namespace

template <int THREADS>
__global__ void __launch_bounds__(THREADS) factor_persistent(Params P) {
  constexpr int kWarps = THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* flags = reinterpret_cast<unsigned*>(smem);
  int* wcols = reinterpret_cast<int*>(flags + P.flag_words);
  double* wvals = reinterpret_cast<double*>(wcols + kWarps * P.cap);  // even word count: 8-B aligned
  __shared__ int s_task, s_cont, s_next, s_skip;
  __shared__ int4 s_h0, s_h1;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* scol = wcols + warp * P.cap;
  double* sval = wvals + warp * P.cap;
  const unsigned long long t0 = gtimer();

  if (tid == 0) s_cont = -1;
  __syncthreads();
  while (true) {
    if (tid == 0) {
      int t = s_cont;
      s_cont = -1;
      if (t < 0) t = pop_task(P, t0);
      s_task = t;
      if (t >= 0) {
        s_h0 = P.tasks[2 * t];
        s_h1 = P.tasks[2 * t + 1];
        s_skip = ld_relaxed(&P.ctrl->failed) | ld_relaxed(&P.ctrl->error);
        s_next = 0;
        if (P.trace) P.trace[2 * t] = gtimer();
      }
    }
    __syncthreads();
    const int t = s_task;
    if (t < 0) break;
    const int4 h0 = s_h0, h1 = s_h1;
    const int kind = h0.x, flag_rows = h0.y, item_b = h0.z, item_e = h0.w;
    const int succ_b = h1.x, succ_e = h1.y, row_begin = h1.z;

    if (!s_skip && item_e > item_b) {
      if (kind == kChol || kind == kTrsm) {
        for (int w = tid; w < ((flag_rows + 31) >> 5); w += THREADS) flags[w] = 0u;
        __syncthreads();
      }
      while (true) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&s_next, 1);
        k = __shfl_sync(kFull, k, 0);
        const int item = item_b + k;
        if (item >= item_e) break;
        switch (kind) {
          case kChol: run_item<kChol>(P, item, lane, scol, sval, flags, row_begin, t0); break;
          case kTrsm: run_item<kTrsm>(P, item, lane, scol, sval, flags, row_begin, t0); break;
          case kHerk: run_item<kHerk>(P, item, lane, scol, sval, flags, row_begin, t0); break;
          default: run_item<kGemm>(P, item, lane, scol, sval, flags, row_begin, t0); break;
        }
      }
      if (tid == 0) atomicAdd(&P.ctrl->executed, 1);
    }
    __syncthreads();

    // release successors (acq_rel: publishes this CTA's writes, which the
    // barrier above ordered before this thread, and acquires the other
    // predecessors' writes for the thread that readies the successor)
    for (int k = succ_b + tid; k < succ_e; k += THREADS) {
      const int s = P.succ[k];
      if (atom_dec_acq_rel(P.indeg + s) == 1) {
        if (atomicCAS(&s_cont, -1, s) != -1) {
          const int slot = atomicAdd(&P.ctrl->q_tail, 1);
          st_release(P.queue + slot, s);
        }
      }
    }
    if (tid == 0) {
      if (P.trace) P.trace[2 * t + 1] = gtimer();
      atomicAdd(&P.ctrl->done, 1);
    }
    __syncthreads();
  }
}

__global__ void prepare_kernel(PrepParams Q) {
  const int stride = gridDim.x * blockDim.x;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < Q.ntasks; k += stride) {
    Q.indeg[k] = Q.indeg0[k];
    Q.queue[k] = k < Q.nroots ? Q.roots[k] : -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctrl c = {};
    c.q_tail = Q.nroots;
    c.fail_row = -1;
    *Q.ctrl = c;
  }
}

// ---- host-side launch helpers (declared in device_api.hpp) ----------------

size_t factor_smem_bytes(int threads, int cap, int flag_words) {
  // flag_words and cap are even (host contract), so the double staging
  // area that follows the int words stays 8-byte aligned.
  const size_t warps = static_cast<size_t>(threads / 32);
  return static_cast<size_t>(flag_words) * 4 + warps * static_cast<size_t>(cap) * 12;
}

static const void* kernel_for(int threads) {
  switch (threads) {
    case 128: return reinterpret_cast<const void*>(&factor_persistent<128>);
    case 256: return reinterpret_cast<const void*>(&factor_persistent<256>);
    case 512: return reinterpret_cast<const void*>(&factor_persistent<512>);
    default: return nullptr;
  }
}

cudaError_t factor_occupancy(int threads, size_t smem, int* ctas_per_sm) {
  const void* k = kernel_for(threads);
  if (!k) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, threads, smem);
}

cudaError_t launch_prepare(const PrepParams& q, cudaStream_t st) {
  const int threads = 256;
  int blocks = (q.ntasks + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  prepare_kernel<<<blocks, threads, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_factor(const Params& p, int grid, int threads, size_t smem, cudaStream_t st) {
  switch (threads) {
    case 128: factor_persistent<128><<<grid, 128, smem, st>>>(p); break;
    case 256: factor_persistent<256><<<grid, 256, smem, st>>>(p); break;
    case 512: factor_persistent<512><<<grid, 512, smem, st>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tcbdev
