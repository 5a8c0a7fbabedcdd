// Pieces shared by the value-flow row kernels (flow_kernel.cu: one warp per
// row; flow_pp_kernel.cu: product-parallel row groups): the gather context
// (polling reads of values that are their own flags) and the drain CTAs of
// the end-to-end call.
#pragma once

#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "sync.cuh"

namespace tcbdev {
namespace {

constexpr unsigned long long kCanonicalNaN = 0x7FFFFFFFFFFFFFFFull;

// Slow path of a gather: the value is not written yet.
// Sleep of BO ns between re-polls (0: none). (An exponential back-off, 32 ns
// doubling up to a cap, was slower everywhere on B200: C3 3.09-3.15 ms
// against 2.78 at a fixed 400 ns, C4 1.48-1.65 against 1.40 at 100; its
// extra registers cost a CTA per SM.)
template <int BO>
__device__ __forceinline__ void poll_pause(unsigned&) {
  if (BO > 0) __nanosleep(BO);
}

// BO: poll back-off (poll_pause)
template <int BO = 0>
__device__ __forceinline__ unsigned long long wait_value(const double* p, Ctrl* ctrl,
                                                      unsigned long long t0,
                                                      unsigned long long tmo) {
  unsigned spins = 0, ns = 32;
  for (;;) {
    const unsigned long long x = ld_relaxed_u64(p);
    if (x != kUnset) return x;
    poll_pause<BO>(ns);
    if (++spins == 1024u) {
      spins = 0;
      if (ld_relaxed(&ctrl->error.v) || gtimer() - t0 > tmo) {
        atomicCAS(&ctrl->error.v, 0, 1);
        return 0ull;  // abandoned: the host reports TCG_TIMEOUT
      }
    }
  }
}

// The same poll at system scope: a value owned by a part on another GPU.
__device__ __forceinline__ unsigned long long wait_value_sys(const double* p, Ctrl* ctrl,
                                                          unsigned long long t0,
                                                          unsigned long long tmo) {
  unsigned spins = 0;
  for (;;) {
    const unsigned long long x = ld_relaxed_sys_u64(p);
    if (x != kUnset) return x;
    if (++spins == 1024u) {
      spins = 0;
      if (ld_relaxed(&ctrl->error.v) || gtimer() - t0 > tmo) {
        atomicCAS(&ctrl->error.v, 0, 1);
        return 0ull;
      }
    }
  }
}

// The gather context. Every load of a factor value is a strong (L2) load: a
// location holds kUnset until its single final value is written, so any
// other bits a load returns are the final value (8-byte aligned accesses do
// not tear). (L1-cached first loads, validated against kUnset, measured no
// better in round 1.)
// `vals`/`a`/`member`: the current row's member of a batch (its value sets
// are nnz apart; the pattern, records and programs are shared).
// OPS: how a negative operand position is read. 0: never happens; 2
// (sharded runs): kRemoteBit | part << 25 | position in that part's U.
// BO: poll back-off in ns (a lane sleeps between re-polls of a value not yet
// written). Long programs keep thousands of lanes polling the few lines the
// critical rows are about to write; sleeping between polls frees the L2
// slices serving them (B200, C3: 4.01 ms without, 2.66 ms at 400 ns, 2.60 at
// 600 ns; C4 1.49 -> 1.30 at 200 ns; short programs lose: C2 0.41 -> 0.42-0.45 ms).
template <int OPS = 0, int BO = 0>
struct Ctx {
  const FlowParams& P;
  unsigned long long t0;
  double* vals;
  const double* a;
  int member;
  __device__ __forceinline__ double settle(const double* p, unsigned long long x) const {
    if (x == kUnset) x = wait_value<BO>(p, P.ctrl, t0, P.timeout_ns);
    return __longlong_as_double(static_cast<long long>(x));
  }
  // the same without a sleep between polls: the whole warp waits for this one value (one sector a poll)
  __device__ __forceinline__ double settle_now(const double* p, unsigned long long x) const {
    if (x == kUnset) x = wait_value<0>(p, P.ctrl, t0, P.timeout_ns);
    return __longlong_as_double(static_cast<long long>(x));
  }
  // sharded runs (P.peers): a negative position names another part's value
  __device__ __forceinline__ const double* remote(int pos) const {
    return P.peers[(pos >> 25) & 63] + (pos & 0x1FFFFFF);
  }
  __device__ __forceinline__ unsigned long long ld(int pos) const {
    if (OPS == 2 && pos < 0) return ld_relaxed_sys_u64(remote(pos));
    return ld_relaxed_u64(vals + pos);
  }
  // An operand of an early product: final long ago as a rule, and a final value
  // is final in any cache (written once), so the SM's L1 may serve it -- the
  // lanes of a row read the same multiplier and neighbouring operands. A copy
  // cached before the value was written reads kUnset and is re-read from L2
  // (product()'s strong re-poll).
  __device__ __forceinline__ unsigned long long ld_early(int pos) const {
    if (OPS == 2 && pos < 0) return ld_relaxed_sys_u64(remote(pos));
    return ld_cached_u64(vals + pos);
  }
  __device__ __forceinline__ unsigned long long ld_strong(int pos) const {
    if (OPS == 2 && pos < 0) return ld_relaxed_sys_u64(remote(pos));
    return ld_relaxed_u64(vals + pos);
  }
  // settle an operand by its (encoded) position
  __device__ __forceinline__ double settle_at(int pos, unsigned long long x) const {
    if (x == kUnset) {
      if (OPS == 2 && pos < 0) x = wait_value_sys(remote(pos), P.ctrl, t0, P.timeout_ns);
      else x = wait_value<BO>(vals + pos, P.ctrl, t0, P.timeout_ns);
    }
    return __longlong_as_double(static_cast<long long>(x));
  }
  // both operands of one product: U(r,t) and U(r,c) come from the same
  // source row r, so when r has just been written both still read kUnset;
  // re-polling them together costs one round trip instead of two
  __device__ __forceinline__ double product(int pa, unsigned long long xa, int pb, unsigned long long xb) const {
    if (OPS != 2 && (xa == kUnset || xb == kUnset)) {
      unsigned spins = 0, ns = 32;
      // re-poll, then sleep only if still unwritten: an operand loaded early
      // (a batch ahead) is often final by the time it is settled, and must not
      // pay a back-off for it
      for (;;) {
        if (xa == kUnset) xa = ld_strong(pa);
        if (xb == kUnset) xb = ld_strong(pb);
        if (xa != kUnset && xb != kUnset) break;
        poll_pause<BO>(ns);
        if (++spins == 1024u) {
          spins = 0;
          if (ld_relaxed(&P.ctrl->error.v) || gtimer() - t0 > P.timeout_ns) {
            atomicCAS(&P.ctrl->error.v, 0, 1);  // abandoned: the host reports TCG_TIMEOUT
            xa = xb = 0ull;
          }
        }
      }
    }
    if (OPS != 2)  // settled by the loop above
      return __dmul_rn(__longlong_as_double(static_cast<long long>(xa)), __longlong_as_double(static_cast<long long>(xb)));
    return __dmul_rn(settle_at(pa, xa), settle_at(pb, xb));
  }
  static constexpr bool kSysPublish = OPS == 2;  // readers on other GPUs
};

// Chunked download (end to end, DRAIN = 2): the unit starting at tb is done
// (the whole group `sync`s before its first lane counts it); the unit that
// completes its chunk tells the host, which then copies the chunk with the
// copy engine while the rest of the rows run. The fence orders the group's
// value stores before the count, the system fence the chunk before the flag.
__device__ __forceinline__ void chunk_count(const FlowParams& P, int tb) {
  const int k = static_cast<int>(static_cast<long long>(tb) * P.nchunks / P.nnz);
  __threadfence();
  if (atomicSub(P.chunk_left + k, 1) == 1) {
    __threadfence_system();
    *reinterpret_cast<volatile int*>(P.chunk_flag + k) = P.chunk_seq;
  }
}
__device__ __forceinline__ void chunk_notify(const FlowParams& P, int tb, int lane) {
  __syncwarp();
  if (lane == 0) chunk_count(P, tb);
}

// Drain (end to end): the warps of the CTAs past P.row_ctas copy U to the
// host while the rows run. A value is final as soon as it no longer reads
// kUnset (it is written once), so a warp copies every group of 64 values
// whose loads all see final values -- 16 bytes per lane, one coalesced
// 512-byte store into the pinned host buffer -- and comes back later for
// groups that are not final yet (a bit per group in P.drain_done; a sweep
// that copies nothing backs off for a microsecond, so its re-reads do not
// crowd the lines the rows are writing). Two groups are checked at once; warp
// d owns a contiguous slice of the 2,048-value batches. Measured on B200
// (end to end, wall): 8-byte accesses per lane in groups of 32 gave C2 0.82,
// C6 5.75 ms; this layout C2 0.82, C6 5.48 ms; four groups in flight C2 0.89
// ms; eight (80 registers, harder re-reads of unfinished lines) C2 1.99 ms.
__device__ void drain_values(const FlowParams& P, int dw, int DW) {
  constexpr int kIn = 2;
  const int lane = threadIdx.x & 31;
  const long long total = P.nnz * P.nbatch;  // a batch's members are contiguous
  const long long nb = (total + 2047) / 2048;
  const long long b0 = nb * dw / DW, b1 = nb * (dw + 1) / DW;
  const unsigned long long t0 = gtimer();
  const bool even = (total & 1) == 0;
  long long low = b0;
  while (low < b1) {
    bool progressed = false;
    for (long long b = low; b < b1; ++b) {
      unsigned done = P.drain_done[b];
      if (done == 0xffffffffu) {
        if (b == low) ++low;
        continue;
      }
      for (int j0 = 0; j0 < 32; j0 += kIn) {
        unsigned long long va[kIn], vb[kIn];
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          const long long x = (b * 32 + j0 + j) * 64 + 2 * lane;
          va[j] = vb[j] = 0ull;
          if ((done >> (j0 + j)) & 1u) continue;
          if (even && x + 1 < total) {
            ld_relaxed_v2_u64(P.vals + x, va[j], vb[j]);
          } else {
            if (x < total) va[j] = ld_relaxed_u64(P.vals + x);
            if (x + 1 < total) vb[j] = ld_relaxed_u64(P.vals + x + 1);
          }
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          if ((done >> (j0 + j)) & 1u) continue;
          if (__ballot_sync(kFull, va[j] != kUnset && vb[j] != kUnset) != kFull) continue;
          const long long x = (b * 32 + j0 + j) * 64 + 2 * lane;
          if (even && x + 1 < total) {
            *reinterpret_cast<double2*>(P.drain_out + x) =
                make_double2(__longlong_as_double(static_cast<long long>(va[j])),
                             __longlong_as_double(static_cast<long long>(vb[j])));
          } else {
            if (x < total) P.drain_out[x] = __longlong_as_double(static_cast<long long>(va[j]));
            if (x + 1 < total) P.drain_out[x + 1] = __longlong_as_double(static_cast<long long>(vb[j]));
          }
          done |= 1u << (j0 + j);
          progressed = true;
        }
      }
      if (lane == 0) P.drain_done[b] = done;
      __syncwarp();
      if (done == 0xffffffffu && b == low) ++low;
    }
    if (!progressed && low < b1) {
      if (ld_relaxed(&P.ctrl->error.v) || gtimer() - t0 > P.timeout_ns) return;
      __nanosleep(1000);
    }
  }
}

}  // namespace
}  // namespace tcbdev
