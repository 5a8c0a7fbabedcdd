// Row-level dataflow execution of the Cholesky-by-blocks DAG (mode 3).
//
// The task DAG of factor_by_blocks (factorize.hpp:169-225) is executed at
// the granularity of its target rows ("items", host plan.hpp): an item runs
// as soon as the rows it reads are final and the previous item writing its
// own (block, row) slice has finished. Those row-level edges are the block
// edges of the generation walk restricted to rows that actually interact
// (plan.cpp build_item_deps), so every coordinate of U still receives its
// updates in ascending source row and the factor is bitwise equal to
// factor_serial (factorize.hpp:94-130). What changes is the critical path:
// a chain of Herk tasks into one separator block is no longer serialised
// unless their rows overlap (C2: 2,046 task levels -> 230 row levels).
//
// Every warp is an independent worker of one persistent kernel:
//   pop a ready row (ticket queue) or take the continuation it readied itself
//   -> apply the row's update program (lane per target slot, host-merged
//      sorted indices, products in source order, __dmul_rn/__dsub_rn)
//   -> Chol: pivot test + sqrt + scale; Trsm: divide by U(t,t)
//   -> publish (fence) and decrement the successors' counters (acq_rel);
//      the first successor reaching zero becomes the warp's continuation,
//      the others are appended to the queue.
#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

__device__ __forceinline__ double row_slot(const RowParams& P, double v, const int4 sr) {
  const int ub = sr.x, ue = sr.y;
  if (ub >= ue) return v;
  const double a0 = P.vals[sr.z], b0 = P.vals[sr.w];
  constexpr int kB = 8;
  int u = ub + 1;
  int2 p[kB];
#pragma unroll
  for (int j = 0; j < kB; ++j) p[j] = (u + j < ue) ? P.upd[u + j] : make_int2(0, 0);
  v = __dsub_rn(v, __dmul_rn(a0, b0));
  while (u < ue) {
    const int n = min(kB, ue - u);
    double a[kB], b[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      a[j] = (j < n) ? P.vals[p[j].x] : 0.0;
      b[j] = (j < n) ? P.vals[p[j].y] : 0.0;
    }
    u += kB;
#pragma unroll
    for (int j = 0; j < kB; ++j) p[j] = (u + j < ue) ? P.upd[u + j] : make_int2(0, 0);
#pragma unroll
    for (int j = 0; j < kB; ++j)
      if (j < n) v = __dsub_rn(v, __dmul_rn(a[j], b[j]));
  }
  return v;
}

template <int KIND>
__device__ __forceinline__ void row_compute(const RowParams& P, int tb, int L, int dpos, int soff,
                                            int t, int lane) {
  double v = 0.0;
  int4 sr = make_int4(0, 0, 0, 0);
  if (lane < L) {
    v = P.vals[tb + lane];
    sr = P.slot_rec[soff + lane];
  }
  double d = 1.0;
  if (KIND == kTrsm) d = P.vals[dpos];
  if (lane < L) v = row_slot(P, v, sr);
  if (KIND == kChol) {
    // kernels.hpp:49-53: pivot test, square root, row scaling
    const double piv = __shfl_sync(kFull, v, 0);
    if (!(piv > 0.0) && lane == 0) {
      if (atomicCAS(&P.ctrl->failed.v, 0, 1) == 0) {
        P.ctrl->fail_row = t;
        P.ctrl->fail_pivot = piv;
      }
    }
    d = __dsqrt_rn(piv);
  }
  auto finish = [&](int k, double x) {
    if (KIND == kChol) return k == 0 ? d : __ddiv_rn(x, d);
    if (KIND == kTrsm) return __ddiv_rn(x, d);  // kernels.hpp:76-78
    return x;
  };
  if (lane < L) P.vals[tb + lane] = finish(lane, v);
  for (int k = lane + 32; k < L; k += 32) {
    const double w = row_slot(P, P.vals[tb + k], P.slot_rec[soff + k]);
    P.vals[tb + k] = finish(k, w);
  }
}

// lane 0 only: next ready row, -1 once every row is done or the run aborted.
// Rows flagged hot by the host (high on the critical path) sit in a
// priority queue that is tried first; the bulk goes through a FIFO. Both
// are ticket queues: a warp holds at most one ticket of each (taking a
// priority ticket only when that queue looks non-empty) and returns
// whichever of its two slots fills first, keeping the other ticket.
__device__ __forceinline__ int pop_row(const RowParams& P, unsigned long long t0, int& ticket,
                                       int& hticket) {
  if (ticket < 0) ticket = atomicAdd(&P.ctrl->q_head.v, 1);
  unsigned spins = 0, ns = 32;
  while (true) {
    if (hticket < 0 && ld_relaxed(&P.ctrl->hi_head.v) < ld_relaxed(&P.ctrl->hi_tail.v))
      hticket = atomicAdd(&P.ctrl->hi_head.v, 1);
    if (hticket >= 0 && hticket < P.nitems) {
      const int v = ld_acquire(P.hiq + hticket);
      if (v >= 0) {
        hticket = -1;
        return v;
      }
    }
    if (ticket < P.nitems) {
      const int v = ld_acquire(P.queue + ticket);
      if (v >= 0) {
        ticket = -1;
        return v;
      }
    }
    if ((spins & 7u) == 0) {
      if (ld_relaxed(&P.ctrl->done.v) >= P.nitems) return -1;
      if (ld_relaxed(&P.ctrl->error.v)) return -1;
    }
    if (++spins == 1024u) {
      spins = 0;
      if (gtimer() - t0 > P.timeout_ns) {
        atomicCAS(&P.ctrl->error.v, 0, 1);
        return -1;
      }
    }
    __nanosleep(ns);
    if (ns < 128) ns <<= 1;
  }
}

}  // namespace

template <int THREADS>
__global__ void __launch_bounds__(THREADS) factor_rows(RowParams P) {
  const int lane = threadIdx.x & 31;
  const unsigned long long t0 = gtimer();
  int cont = -1, pending_done = 0, pending_exec = 0, latched = 0, ticket = -1, hticket = -1;
  while (true) {
    int k = cont;
    cont = -1;
    if (k < 0) {
      // going idle: publish this warp's completions first (termination test);
      // the counters are per-warp sums so no global address is hit per row
      int e = 0;
      if (lane == 0) {
        if (pending_exec) atomicAdd(&P.ctrl->executed.v, pending_exec);
        if (pending_done) atomicAdd(&P.ctrl->done.v, pending_done);
        e = pop_row(P, t0, ticket, hticket);
        latched = ld_relaxed(&P.ctrl->failed.v) | ld_relaxed(&P.ctrl->error.v);
      }
      pending_done = 0;
      pending_exec = 0;
      k = __shfl_sync(kFull, e, 0);
      latched = __shfl_sync(kFull, latched, 0);
      if (k < 0) break;
    }
    __syncwarp();  // lane 0's acquire (pop) or the readying lane's (continuation) covers the warp
    const int4 a = P.rows[2 * k];
    const int4 b = P.rows[2 * k + 1];
    const int tb = a.x, L = a.y - a.x, dpos = a.z, soff = a.w;
    const int kind = b.x, t = b.y, sb = b.z, se = b.w;
    // successor ids stream in while the row is computed
    int s_own = (sb + lane < se) ? P.succ[sb + lane] : -1;
    if (P.trace && lane == 0) P.trace[2 * static_cast<long long>(k)] = gtimer();
    if (!latched) {
      switch (kind) {
        case kChol: row_compute<kChol>(P, tb, L, dpos, soff, t, lane); break;
        case kTrsm: row_compute<kTrsm>(P, tb, L, dpos, soff, t, lane); break;
        default: row_compute<kHerk>(P, tb, L, dpos, soff, t, lane); break;
      }
      ++pending_exec;
    }
    // publish this row, then release its successors. One release fence per
    // row (fence.acq_rel + relaxed decrements form the release pattern), and
    // one acquire fence when some successor became ready (relaxed RMW + fence
    // is the acquire pattern; the same fence releases the queue stores).
    __threadfence();
    __syncwarp();
    if (P.trace && lane == 0) P.trace[2 * static_cast<long long>(k) + 1] = gtimer();  // finished
    int mine = -1;
    for (int j0 = sb; j0 < se; j0 += 32) {
      const int s = (j0 == sb) ? s_own : ((j0 + lane < se) ? P.succ[j0 + lane] : -1);
      const bool ready = (s >= 0) && atom_add_relaxed(P.indeg + (s & ~kRowHotBit), -1) == 1;
      unsigned m = __ballot_sync(kFull, ready);
      if (!m) continue;
      __threadfence();
      __syncwarp();
      if (mine < 0) {  // successor lists are sorted by falling height
        const int leader = __ffs(m) - 1;
        mine = __shfl_sync(kFull, s, leader);
        m &= m - 1;
      }
      const unsigned hot = m & __ballot_sync(kFull, (s & kRowHotBit) != 0);
      const unsigned cold = m & ~hot;
      if (hot) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&P.ctrl->hi_tail.v, __popc(hot));
        base = __shfl_sync(kFull, base, 0);
        if ((hot >> lane) & 1u)
          st_relaxed(P.hiq + base + __popc(hot & ((1u << lane) - 1u)), s & ~kRowHotBit);
      }
      if (cold) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&P.ctrl->q_tail.v, __popc(cold));
        base = __shfl_sync(kFull, base, 0);
        if ((cold >> lane) & 1u)
          st_relaxed(P.queue + base + __popc(cold & ((1u << lane) - 1u)), s & ~kRowHotBit);
      }
    }
    mine &= ~kRowHotBit;
    cont = mine;
    ++pending_done;
  }
}

static const void* row_kernel_for(int threads) {
  switch (threads) {
    case 128: return reinterpret_cast<const void*>(&factor_rows<128>);
    case 256: return reinterpret_cast<const void*>(&factor_rows<256>);
    case 512: return reinterpret_cast<const void*>(&factor_rows<512>);
    default: return nullptr;
  }
}

cudaError_t rows_occupancy(int threads, int* ctas_per_sm) {
  const void* k = row_kernel_for(threads);
  if (!k) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, threads, 0);
}

cudaError_t launch_rows(const RowParams& p, int grid, int threads, cudaStream_t st) {
  switch (threads) {
    case 128: factor_rows<128><<<grid, 128, 0, st>>>(p); break;
    case 256: factor_rows<256><<<grid, 256, 0, st>>>(p); break;
    case 512: factor_rows<512><<<grid, 512, 0, st>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tcbdev
