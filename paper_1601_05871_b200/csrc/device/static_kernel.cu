// Static row schedule (mode 4): the row-level DAG of mode 3 (row_kernel.cu)
// executed without queues or counters.
//
// The host orders the rows by level (longest chain from a root), most
// critical first inside a level; that order is topological, and the rows
// are stored in it ("positions", plan.cpp: 48-byte records with the first
// four predecessor positions inline). Warp w of the W co-resident warps runs
// positions w, w+W, w+2W, ... in order. Before a row it waits for the epoch
// stamps of the rows it depends on (the previous writer of its own slice and
// the last writers of the slices it reads, plan.cpp build_item_deps); after
// the row it publishes its values with one release fence and its own stamp.
// Any unfinished row at the smallest position has all its predecessors at
// smaller positions, so the schedule cannot deadlock while all warps are
// resident (the grid is sized to the occupancy; a watchdog ends the kernel
// otherwise). Per coordinate the products still arrive in ascending source
// row, so the factor is bitwise equal to factor_serial
// (factorize.hpp:94-130).
//
// The hand-off between two dependent rows costs the producer's fence plus
// the consumer's poll; everything immutable (the next position's record and
// its slot records) is loaded while the current row waits and computes, so
// only the predecessor-dependent gathers remain on the critical path.
#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "row_compute.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

__device__ __forceinline__ bool wait_stamp(const int* f, int epoch, const StaticParams& P,
                                           unsigned long long t0) {
  unsigned spins = 0;
  while (ld_relaxed(f) != epoch) {
    if (++spins == 2048u) {
      spins = 0;
      if (ld_relaxed(&P.ctrl->error.v) || gtimer() - t0 > P.timeout_ns) {
        atomicCAS(&P.ctrl->error.v, 0, 1);
        return false;
      }
    }
  }
  return true;
}

}  // namespace

template <int THREADS, int KB>
__global__ void __launch_bounds__(THREADS, 768 / THREADS) factor_static(StaticParams P) {
  constexpr int kWarps = THREADS / 32;
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * kWarps;
  const unsigned long long t0 = gtimer();
  int ran = 0, executed = 0, latched = 0;
  int pos = blockIdx.x * kWarps + (threadIdx.x >> 5);
  // current position's record (a: tb, L, dpos, soff; b: kind, t, npred, pred_off;
  // c: inline predecessor positions) and the lane's first slot record
  int4 a = make_int4(0, 0, 0, 0), b = a, c = a, d = a, sr0 = a;
  if (pos < P.nitems) {
    a = P.pos[4 * pos];
    b = P.pos[4 * pos + 1];
    c = P.pos[4 * pos + 2];
    d = P.pos[4 * pos + 3];
    if (lane < a.y) sr0 = P.slot_rec[a.w + lane];
  }
  while (pos < P.nitems) {
    // prefetch the next position's record
    const int nxt = pos + W;
    int4 na = make_int4(0, 0, 0, 0), nb = na, nc = na, nd = na;
    if (nxt < P.nitems) {
      na = P.pos[4 * nxt];
      nb = P.pos[4 * nxt + 1];
      nc = P.pos[4 * nxt + 2];
      nd = P.pos[4 * nxt + 3];
    }
    const int tb = a.x, L = a.y, dpos = a.z, soff = a.w;
    const int kind = b.x, t = b.y, npred = b.z, poff = b.w;
    // wait for the predecessor rows: lanes 0..3 the inline ones, the others
    // the overflow list (relaxed polls, one acquire fence after)
    bool ok = true;
    if (lane < 4 && lane < npred) {
      const int pp = lane == 0 ? c.x : lane == 1 ? c.y : lane == 2 ? c.z : c.w;
      ok = wait_stamp(P.flag + pp, P.epoch, P, t0);
    }
    for (int j = 4 + lane; j < npred && ok; j += 32)
      ok = wait_stamp(P.flag + P.pos_pred[poff + j - 4], P.epoch, P, t0);
    if (__any_sync(kFull, !ok)) break;
    fence_acquire_gpu();
    __syncwarp();
    if (P.trace && lane == 0) P.trace[2 * static_cast<long long>(d.x)] = gtimer();
    if ((ran & 15) == 0) latched = ld_relaxed(&P.ctrl->failed.v);  // breakdown: skip the rest
    if (!__shfl_sync(kFull, latched, 0)) {
      switch (kind) {
        case kChol: row_compute<kChol, 32, KB>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
        case kTrsm: row_compute<kTrsm, 32, KB>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
        default: row_compute<kHerk, 32, KB>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
      }
      ++executed;
    }
    // publish: fence.acq_rel + relaxed stamp is the release pattern (the
    // fence waits for every outstanding access of the warp, so nothing else
    // is issued between the row's stores and it)
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      if (P.trace) P.trace[2 * static_cast<long long>(d.x) + 1] = gtimer();
      st_relaxed(P.flag + d.x, P.epoch);
    }
    // the next row's slot records are immutable: in flight during its wait
    sr0 = make_int4(0, 0, 0, 0);
    if (nxt < P.nitems && lane < na.y) sr0 = P.slot_rec[na.w + lane];
    ++ran;
    pos = nxt;
    a = na;
    b = nb;
    c = nc;
    d = nd;
  }
  if (lane == 0) {
    if (ran) atomicAdd(&P.ctrl->done.v, ran);
    if (executed) atomicAdd(&P.ctrl->executed.v, executed);
  }
}

// KB: products gathered per batch -- 4 for short slot chains (fewer
// registers, more warps), 8 when slots carry several products (C3/C4)
static const void* static_kernel_for(int threads, int kb) {
#define V(T, K) if (threads == T && kb == K) return reinterpret_cast<const void*>(&factor_static<T, K>);
  V(128, 4) V(128, 8) V(256, 4) V(256, 8) V(512, 4) V(512, 8)
#undef V
  return nullptr;
}

cudaError_t static_occupancy(int threads, int kb, int* ctas_per_sm) {
  const void* k = static_kernel_for(threads, kb);
  if (!k) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, threads, 0);
}

cudaError_t launch_static(const StaticParams& p, int grid, int threads, int kb, cudaStream_t st) {
#define V(T, K)                                        \
  if (threads == T && kb == K) {                       \
    factor_static<T, K><<<grid, T, 0, st>>>(p);        \
    return cudaGetLastError();                         \
  }
  V(128, 4) V(128, 8) V(256, 4) V(256, 8) V(512, 4) V(512, 8)
#undef V
  return cudaErrorInvalidValue;
}

}  // namespace tcbdev
