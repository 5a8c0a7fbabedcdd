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
#include "row_compute.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

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

template <int THREADS, int MINB, bool PROF>
__global__ void __launch_bounds__(THREADS, MINB) factor_rows(RowParams P) {
  const int lane = threadIdx.x & 31;
  const unsigned long long t0 = gtimer();
  int cont = -1, pending_done = 0, pending_exec = 0, latched = 0, ticket = -1, hticket = -1;
  constexpr bool prof = PROF;
  unsigned long long acc[7] = {0, 0, 0, 0, 0, 0, 0}, c0 = 0, c1 = 0;
  while (true) {
    int k = cont;
    cont = -1;
    if (prof) c0 = clock64();
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
      if (prof) {
        acc[5] += 1;
        c1 = clock64();
        acc[0] += c1 - c0;
        c0 = c1;
      }
      if (k < 0) break;
    }
    __syncwarp();  // lane 0's acquire (pop) or the readying lane's (continuation) covers the warp
    const int4 a = P.rows[2 * k];
    const int4 b = P.rows[2 * k + 1];
    const int tb = a.x, L = a.y - a.x, dpos = a.z, soff = a.w;
    const int kind = b.x, t = b.y, sb = b.z, se = b.w;
    // successor ids and the first slot record stream in together
    int s_own = (sb + lane < se) ? P.succ[sb + lane] : -1;
    int4 sr0 = make_int4(0, 0, 0, 0);
    if (lane < L) sr0 = P.slot_rec[soff + lane];
    if (P.trace && lane == 0) P.trace[2 * static_cast<long long>(k)] = gtimer();
    if (!latched) {
      switch (kind) {
        case kChol: row_compute<kChol>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
        case kTrsm: row_compute<kTrsm>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
        default: row_compute<kHerk>(P.slot_rec, P.upd, P.vals, P.ctrl, tb, L, dpos, soff, t, lane, sr0); break;
      }
      ++pending_exec;
    }
    if (prof) {
      __syncwarp();
      c1 = clock64();
      acc[1] += c1 - c0;
      c0 = c1;
    }
    // publish this row, then release its successors. One release fence per
    // row (fence.acq_rel + relaxed decrements form the release pattern), and
    // one acquire fence when some successor became ready (relaxed RMW + fence
    // is the acquire pattern; the same fence releases the queue stores).
    __threadfence();
    __syncwarp();
    if (prof) {
      c1 = clock64();
      acc[2] += c1 - c0;
      c0 = c1;
    }
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
      if (prof) acc[6] += __popc(hot) + __popc(cold);
    }
    mine &= ~kRowHotBit;
    cont = mine;
    ++pending_done;
    if (prof) {
      c1 = clock64();
      acc[3] += c1 - c0;
      acc[4] += 1;
    }
  }
  if (prof && lane == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(&P.ctrl->prof[i], acc[i]);
}

// Variants: block size x register budget (MINB = CTAs per SM the register
// allocation must allow; 0 = compiler's choice) x phase profiling.
#define TCG_ROW_VARIANTS(X) \
  X(128, 0) X(256, 0) X(256, 3) X(256, 4) X(256, 5) X(256, 6) X(512, 0)

static const void* row_kernel_for(int threads, int minb, bool prof) {
#define X(T, M)                                                                       \
  if (threads == T && minb == M)                                                      \
    return prof ? reinterpret_cast<const void*>(&factor_rows<T, M, true>)             \
                : reinterpret_cast<const void*>(&factor_rows<T, M, false>);
  TCG_ROW_VARIANTS(X)
#undef X
  return nullptr;
}

cudaError_t rows_occupancy(int threads, int minb, bool prof, int* ctas_per_sm) {
  const void* k = row_kernel_for(threads, minb, prof);
  if (!k) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, threads, 0);
}

cudaError_t launch_rows(const RowParams& p, int grid, int threads, int minb, cudaStream_t st) {
  const bool prof = p.trace != nullptr;
#define X(T, M)                                                      \
  if (threads == T && minb == M) {                                   \
    if (prof)                                                        \
      factor_rows<T, M, true><<<grid, T, 0, st>>>(p);                \
    else                                                             \
      factor_rows<T, M, false><<<grid, T, 0, st>>>(p);               \
    return cudaGetLastError();                                       \
  }
  TCG_ROW_VARIANTS(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace tcbdev
