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
//     CTA directly, no queue round trip (scheduler.hpp:239-241); its task
//     record is fetched by the readying thread while the release finishes;
//   * multi-CTA tasks: a task whose plan width is w > 1 also enqueues w-1
//     helper tickets; every participating CTA claims rows from a per-task
//     global counter and the CTA that finishes the last row releases the
//     successors (the reference runs each task on one thread, SPEC.md:335;
//     here the big diagonal blocks at the top of the ND tree get the GPU);
//   * a breakdown latch: the first non-positive pivot wins by CAS and later
//     task bodies are skipped (factorize.hpp:146-167);
//   * a globaltimer watchdog in every spin loop so that a malformed DAG
//     ends the kernel with an error instead of hanging the GPU.
//
// Task bodies (replace kernels.hpp:40-132). A task's target rows ("items",
// host plan.hpp) are claimed by warps in plan order (ascending row; Chol and
// Trsm rows in intra-block level order). A single-CTA task first stages its
// item and source records in shared memory with one cooperative load. Each
// warp stages its target row's column indices and values in shared memory,
// then streams the (source, entry) pairs of all its source rows 32 at a
// time, the loads of the next 32 pairs in flight while the current ones are
// applied: every lane forms one product with __dmul_rn, locates the column
// in the staged row by binary search (absent columns are the pattern drop)
// and the products are subtracted with __dsub_rn in ascending source order
// per coordinate (__match_any_sync groups lanes hitting the same slot; the
// lowest lane, i.e. the earliest source, goes first). Chol and Trsm rows
// wait for the rows they read: a shared-memory bitmask inside one CTA,
// epoch stamps in global memory across CTAs. The arithmetic sequence per
// coordinate is exactly the reference's, so the factor is bitwise equal to
// factor_serial (factorize.hpp:94-130): no FMA contraction, IEEE division
// and square root.
#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

__device__ __forceinline__ void raise_error(Ctrl* c, int code) { atomicCAS(&c->error.v, 0, code); }

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

__device__ __forceinline__ bool timed_out(const Params& P, unsigned long long t0) {
  if (ld_relaxed(&P.ctrl->error.v)) return true;
  if (gtimer() - t0 > P.timeout_ns) {
    raise_error(P.ctrl, 1);
    return true;
  }
  return false;
}

// Row `dep` (item position in the running task) must be final before use.
template <bool WIDE>
__device__ __forceinline__ void wait_row(const unsigned* flags, const int* gflags, int dep,
                                         const Params& P, unsigned long long t0) {
  unsigned spins = 0;
  if (WIDE) {
    while (ld_acquire(gflags + dep) != P.epoch) {
      if (++spins == 1024u) {
        spins = 0;
        if (timed_out(P, t0)) return;
      }
    }
  } else {
    const volatile unsigned* w = flags + (dep >> 5);
    const unsigned bit = 1u << (dep & 31);
    while (!(*w & bit)) {
      if (++spins == 4096u) {
        spins = 0;
        if (timed_out(P, t0)) return;
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

// Pair q of the current source batch -> (source lane s, entry position p).
__device__ __forceinline__ void locate(int q, int incl, int excl_own, int sb_own, int& s, int& p) {
  s = 0;
#pragma unroll
  for (int b = 16; b >= 1; b >>= 1) {
    const int v = __shfl_sync(kFull, incl, s + b - 1);
    if (v <= q) s += b;
  }
  const int excl = __shfl_sync(kFull, excl_own, s);
  const int sb = __shfl_sync(kFull, sb_own, s);
  p = sb + (q - excl);
}

template <int KIND, bool WIDE>
__device__ __forceinline__ void run_item(const Params& P, const int4 ia, const int4 ib, int item,
                                         int pos, int lane, int* scol, double* sval,
                                         unsigned* flags, int* gflags, const int4* sp, int src_off,
                                         int row_begin, unsigned long long t0) {
  constexpr bool kDeps = (KIND == kChol || KIND == kTrsm);
  const int tb = ia.x, te = ia.y, local = ia.z, dpos = ia.w;
  const int src_b = ib.x, src_e = ib.y;
  const int L = te - tb;
  const bool staged = L <= P.cap;
  unsigned long long* it = P.itrace ? P.itrace + 4 * static_cast<long long>(item) : nullptr;
  if (it && lane == 0) it[0] = gtimer();

  // first source batch and the target staging loads are issued together
  int4 rec = make_int4(-1, 0, 0, 0);
  int ns = min(32, src_e - src_b);
  if (lane < ns) rec = sp[src_b + lane - src_off];
  if (staged) {
    for (int k = lane; k < L; k += 32) {
      scol[k] = P.cols[tb + k];
      sval[k] = P.vals[tb + k];
    }
  }
  double diag = 1.0;
  if (KIND == kTrsm) diag = P.vals[dpos];  // final since the Chol task completed
  const int* tcol = staged ? scol : P.cols + tb;
  double* tval = staged ? sval : P.vals + tb;

  for (int s0 = src_b; s0 < src_e; s0 += 32) {
    if (s0 != src_b) {
      ns = min(32, src_e - s0);
      rec = make_int4(-1, 0, 0, 0);
      if (lane < ns) rec = sp[s0 + lane - src_off];
    }
    if (kDeps) {
      if (lane < ns) wait_row<WIDE>(flags, gflags, rec.x, P, t0);
      __syncwarp();
      if (!WIDE) __threadfence_block();
    }
    if (it && lane == 0 && s0 == src_b) it[1] = gtimer();
    const int len = (lane < ns) ? rec.w - rec.z : 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl_own = incl - len;

    // software pipeline: loads of chunk k+1 are issued before chunk k is applied
    int c = 0;
    double v1 = 0.0, v2 = 0.0;
    {
      int s, p;
      locate(lane, incl, excl_own, rec.z, s, p);
      const int prt = __shfl_sync(kFull, rec.y, s);
      if (lane < total) {
        c = P.cols[p];
        v2 = P.vals[p];
        v1 = P.vals[prt];
      }
    }
    __syncwarp();  // staged target row visible to the whole warp
    for (int q0 = 0; q0 < total; q0 += 32) {
      int cn = 0;
      double v1n = 0.0, v2n = 0.0;
      const int qn = q0 + 32 + lane;
      if (q0 + 32 < total) {
        int s, p;
        locate(qn, incl, excl_own, rec.z, s, p);
        const int prt = __shfl_sync(kFull, rec.y, s);
        if (qn < total) {
          cn = P.cols[p];
          v2n = P.vals[p];
          v1n = P.vals[prt];
        }
      }
      int slot = -1;
      double prod = 0.0;
      if (q0 + lane < total) {
        prod = __dmul_rn(v1, v2);
        slot = find_col(tcol, L, c);
      }
      if (it && q0 == 0 && s0 == src_b) {
        const double w = __shfl_sync(kFull, prod, 0) + __shfl_sync(kFull, (double)slot, 0);
        if (lane == 0) it[2] = gtimer() + (w == 12345.678 ? 1 : 0);
      }
      apply_ordered(tval, slot, prod, lane);
      c = cn;
      v1 = v1n;
      v2 = v2n;
    }
  }
  __syncwarp();

  // finalize: Chol takes the square root and scales the row
  // (kernels.hpp:49-53), Trsm divides by U(t,t) (kernels.hpp:76-78).
  if (KIND == kChol) {
    const double piv = tval[0];
    __syncwarp();
    if (!(piv > 0.0) && lane == 0) {
      if (atomicCAS(&P.ctrl->failed.v, 0, 1) == 0) {
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
  if (kDeps) {
    if (WIDE) {
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release(P.iflag + item, P.epoch);
    } else {
      __syncwarp();
      __threadfence_block();
      if (lane == 0) atomicOr(flags + (pos >> 5), 1u << (pos & 31));
    }
  }
  if (it && lane == 0) it[3] = gtimer();
  __syncwarp();
}

// Update-program mode: the host already merged the sorted indices, so slot
// k of the target row receives exactly the products listed for it, in
// source order. Lane j owns slots j, j+32, ...; each slot is one dependent
// chain v = v - U[m]*U[o]. The slot record carries the first (m, o) so the
// gathers start one load after the record; later pairs are fetched two
// ahead of their use.
__device__ __forceinline__ double apply_slot(const Params& P, double v, const int4 sr) {
  const int ub = sr.x, ue = sr.y;
  if (ub >= ue) return v;
  // the first product's operands are named by the slot record itself
  const double a0 = P.vals[sr.z], b0 = P.vals[sr.w];
  constexpr int kB = 8;  // products gathered per batch
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

template <int KIND, bool WIDE>
__device__ __forceinline__ void run_item_prog(const Params& P, const int4 ia, const int4 ib,
                                              int item, int pos, int lane, unsigned* flags,
                                              int* gflags, const int4* sp, int src_off,
                                              int row_begin, unsigned long long t0) {
  constexpr bool kDeps = (KIND == kChol || KIND == kTrsm);
  const int tb = ia.x, te = ia.y, local = ia.z, dpos = ia.w;
  const int src_b = ib.x, src_e = ib.y, soff = ib.z;
  const int L = te - tb;
  unsigned long long* it = P.itrace ? P.itrace + 4 * static_cast<long long>(item) : nullptr;
  if (it && lane == 0) it[0] = gtimer();

  // prologue: everything of this lane's first slot that does not depend on
  // the rows being waited for
  const int k0 = lane;
  double v = 0.0;
  int4 sr0 = make_int4(0, 0, 0, 0);
  if (k0 < L) {
    v = P.vals[tb + k0];
    sr0 = P.slot_rec[soff + k0];
  }
  double d = 1.0;
  if (KIND == kTrsm) d = P.vals[dpos];  // final since the Chol task completed
  if (kDeps) {
    for (int s0 = src_b; s0 < src_e; s0 += 32) {
      if (s0 + lane < src_e) wait_row<WIDE>(flags, gflags, sp[s0 + lane - src_off].x, P, t0);
    }
    __syncwarp();
    if (!WIDE) __threadfence_block();
  }
  if (it && lane == 0) it[1] = gtimer();
  if (k0 < L) v = apply_slot(P, v, sr0);
  if (it && lane == 0) it[2] = gtimer();
  if (KIND == kChol) {
    // kernels.hpp:49-53: pivot test, square root, row scaling
    const double piv = __shfl_sync(kFull, v, 0);
    if (!(piv > 0.0) && lane == 0) {
      if (atomicCAS(&P.ctrl->failed.v, 0, 1) == 0) {
        P.ctrl->fail_row = row_begin + local;
        P.ctrl->fail_pivot = piv;
      }
    }
    d = __dsqrt_rn(piv);
  }
  auto finish = [&](int k, double x) {
    if (KIND == kChol) return k == 0 ? d : __ddiv_rn(x, d);
    if (KIND == kTrsm) return __ddiv_rn(x, d);
    return x;
  };
  if (k0 < L) P.vals[tb + k0] = finish(k0, v);
  for (int k = k0 + 32; k < L; k += 32) {
    const double w = apply_slot(P, P.vals[tb + k], P.slot_rec[soff + k]);
    P.vals[tb + k] = finish(k, w);
  }
  if (kDeps) {
    if (WIDE) {
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release(P.iflag + item, P.epoch);
    } else {
      __syncwarp();
      __threadfence_block();
      if (lane == 0) atomicOr(flags + (pos >> 5), 1u << (pos & 31));
    }
  }
  if (it && lane == 0) it[3] = gtimer();
  __syncwarp();
}

template <bool WIDE>
__device__ __forceinline__ void dispatch(int kind, const Params& P, const int4 ia, const int4 ib,
                                         int item, int pos, int lane, int* scol, double* sval,
                                         unsigned* flags, int* gflags, const int4* sp, int src_off,
                                         int row_begin, unsigned long long t0) {
  if (P.mode == 2) {
    switch (kind) {
      case kChol: run_item_prog<kChol, WIDE>(P, ia, ib, item, pos, lane, flags, gflags, sp, src_off, row_begin, t0); break;
      case kTrsm: run_item_prog<kTrsm, WIDE>(P, ia, ib, item, pos, lane, flags, gflags, sp, src_off, row_begin, t0); break;
      case kHerk: run_item_prog<kHerk, WIDE>(P, ia, ib, item, pos, lane, flags, gflags, sp, src_off, row_begin, t0); break;
      default: run_item_prog<kGemm, WIDE>(P, ia, ib, item, pos, lane, flags, gflags, sp, src_off, row_begin, t0); break;
    }
    return;
  }
  switch (kind) {
    case kChol: run_item<kChol, WIDE>(P, ia, ib, item, pos, lane, scol, sval, flags, gflags, sp, src_off, row_begin, t0); break;
    case kTrsm: run_item<kTrsm, WIDE>(P, ia, ib, item, pos, lane, scol, sval, flags, gflags, sp, src_off, row_begin, t0); break;
    case kHerk: run_item<kHerk, WIDE>(P, ia, ib, item, pos, lane, scol, sval, flags, gflags, sp, src_off, row_begin, t0); break;
    default: run_item<kGemm, WIDE>(P, ia, ib, item, pos, lane, scol, sval, flags, gflags, sp, src_off, row_begin, t0); break;
  }
}

// Claim items until exhausted; the next item's record is fetched before the
// current one runs. Claims ascend, and an item only waits for items with a
// smaller position, so the claim order is deadlock-free.
template <bool WIDE>
__device__ __forceinline__ int work_items(const Params& P, int kind, int t, int item_b, int nitems,
                                          const int4* ip, const int4* sp, int src_off,
                                          int* s_next, int lane, int* scol, double* sval,
                                          unsigned* flags, int row_begin, unsigned long long t0) {
  int* gflags = P.iflag + item_b;
  auto claim = [&]() {
    int k = 0;
    if (lane == 0) k = WIDE ? atomicAdd(P.claim + t, 1) : atomicAdd(s_next, 1);
    return __shfl_sync(kFull, k, 0);
  };
  int done = 0;
  int k = claim();
  int4 ia = make_int4(0, 0, 0, 0), ib = ia;
  if (k < nitems) {
    ia = ip[2 * k];
    ib = ip[2 * k + 1];
  }
  while (k < nitems) {
    const int k2 = claim();
    int4 ja = make_int4(0, 0, 0, 0), jb = ja;
    if (k2 < nitems) {
      ja = ip[2 * k2];
      jb = ip[2 * k2 + 1];
    }
    dispatch<WIDE>(kind, P, ia, ib, item_b + k, k, lane, scol, sval, flags, gflags, sp, src_off,
                   row_begin, t0);
    ++done;
    k = k2;
    ia = ja;
    ib = jb;
  }
  return done;
}

// Ticket-based pop: returns a queue entry (task id, possibly with the helper
// bit), or -1 once all tasks are done (or the run was aborted).
__device__ __forceinline__ int pop_entry(const Params& P, unsigned long long t0) {
  const int ticket = atomicAdd(&P.ctrl->q_head.v, 1);
  unsigned spins = 0;
  unsigned ns = 32;
  while (true) {
    if (ticket < P.qcap) {
      const int v = ld_acquire(P.queue + ticket);
      if (v >= 0) return v;
    }
    if ((spins & 7u) == 0) {
      if (ld_relaxed(&P.ctrl->done.v) >= P.ntasks) return -1;
      if (ld_relaxed(&P.ctrl->error.v)) return -1;
    }
    if (++spins == 1024u) {
      spins = 0;
      if (gtimer() - t0 > P.timeout_ns) {
        raise_error(P.ctrl, 1);
        return -1;
      }
    }
    __nanosleep(ns);
    if (ns < 128) ns <<= 1;
  }
}

}  // namespace

template <int THREADS>
__global__ void __launch_bounds__(THREADS) factor_persistent(Params P) {
  constexpr int kWarps = THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* flags = reinterpret_cast<unsigned*>(smem);
  int* wcols = reinterpret_cast<int*>(flags + P.flag_words);
  double* wvals = reinterpret_cast<double*>(wcols + kWarps * P.cap);
  int4* s_items = reinterpret_cast<int4*>(wvals + kWarps * P.cap);
  int4* s_srcs = s_items + 2 * P.icap;
  __shared__ int s_entry, s_cont, s_next, s_skip, s_done, s_release, s_pref;
  __shared__ int4 s_h[kTaskInt4];
  constexpr int kPre = 64;  // successor records prefetched per task
  __shared__ int4 s_succ[kPre][4];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* scol = wcols + warp * P.cap;
  double* sval = wvals + warp * P.cap;
  const unsigned long long t0 = gtimer();

  if (tid == 0) {
    s_cont = -1;
    s_pref = 0;
  }
  __syncthreads();
  // breakdown/abort latch as seen at the end of the previous task: reading it
  // there keeps the load off the next task's critical path (a task started
  // just after a breakdown may still run; its values are discarded anyway)
  int latched = 0;
  while (true) {
    if (tid == 0) {
      int e = s_cont;
      s_cont = -1;
      if (e < 0) {
        e = pop_entry(P, t0);
        latched = ld_relaxed(&P.ctrl->failed.v) | ld_relaxed(&P.ctrl->error.v);
      }
      s_entry = e;
      if (e >= 0) {
        const int t = e & ~kHelperBit;
        if (!s_pref) {
          s_h[0] = P.tasks[kTaskInt4 * t];
          s_h[1] = P.tasks[kTaskInt4 * t + 1];
          s_h[2] = P.tasks[kTaskInt4 * t + 2];
        }
        s_skip = latched;
        s_next = 0;
        s_done = 0;
        s_release = 0;
        if (P.trace && !(e & kHelperBit)) P.trace[2 * t] = gtimer();
      }
      s_pref = 0;
    }
    __syncthreads();
    const int e = s_entry;
    if (e < 0) break;
    const bool helper = (e & kHelperBit) != 0;
    const int t = e & ~kHelperBit;
    const int4 h0 = s_h[0], h1 = s_h[1], h2 = s_h[2];
    const int kind = h0.x, width = h0.y, item_b = h0.z, nitems = h0.w - h0.z;
    const int succ_b = h1.x, succ_e = h1.y, row_begin = h1.z;
    const int src_b = h2.x, nsrc = h2.y - h2.x;
    const bool skip = s_skip != 0;
    bool release;
    // successor records (id + task record) stream into shared memory while
    // the task body runs; the releasing thread reads its own copy
    if (tid < kPre && succ_b + tid < succ_e) {
      const int4* g = P.succ + 4 * (succ_b + tid);
#pragma unroll
      for (int w = 0; w < 4; ++w) cp_async16(&s_succ[tid][w], g + w);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }

    if (width > 1 && !(skip && !helper) && nitems > 0) {
      // ---- multi-CTA task -------------------------------------------------
      if (!helper) {
        if (tid == 0) s_next = atomicAdd(&P.ctrl->q_tail.v, width - 1);
        __syncthreads();
        if (tid < width - 1) st_release(P.queue + s_next + tid, t | kHelperBit);
      } else if (tid == 0) {
        atomicAdd(&P.ctrl->helpers_run.v, 1);
      }
      const int mine = work_items<true>(P, kind, t, item_b, nitems, P.items + 2 * item_b, P.srcs, 0,
                                        &s_next, lane, scol, sval, flags, row_begin, t0);
      if (lane == 0 && mine) atomicAdd(&s_done, mine);
      __syncthreads();
      if (tid == 0) {
        const int n = s_done;
        s_release = (n > 0 && atom_add_acq_rel(P.fin + t, n) + n == nitems) ? 1 : 0;
        if (s_release && !skip) atomicAdd(&P.ctrl->executed.v, 1);
      }
      __syncthreads();
      release = s_release != 0;
    } else {
      // ---- single-CTA task ------------------------------------------------
      if (!skip && nitems > 0) {
        const bool deps = (kind == kChol || kind == kTrsm);
        // Herk/Gemm rows of the program mode need no source records and no
        // flags: warps fetch their item records directly, no barrier
        const bool direct = (P.mode == 2 && !deps);
        const bool stage = !direct && nitems <= P.icap && nsrc <= P.scap;
        if (stage) {
          const int4* gi = P.items + 2 * item_b;
          for (int k = tid; k < 2 * nitems; k += THREADS) s_items[k] = gi[k];
          const int4* gs = P.srcs + src_b;
          for (int k = tid; k < nsrc; k += THREADS) s_srcs[k] = gs[k];
        }
        if (deps)
          for (int w = tid; w < ((nitems + 31) >> 5); w += THREADS) flags[w] = 0u;
        if (!direct) __syncthreads();
        work_items<false>(P, kind, t, item_b, nitems, stage ? s_items : P.items + 2 * item_b,
                          stage ? s_srcs : P.srcs, stage ? src_b : 0, &s_next, lane, scol, sval,
                          flags, row_begin, t0);
        if (tid == 0) atomicAdd(&P.ctrl->executed.v, 1);
      }
      __syncthreads();
      release = true;
    }

    if (tid == 0) latched = ld_relaxed(&P.ctrl->failed.v) | ld_relaxed(&P.ctrl->error.v);
    if (release) {
      // release successors (acq_rel: publishes the writes ordered before
      // this thread by the barrier, and acquires the other predecessors'
      // writes for the thread that readies the successor)
      cp_async_wait_all();
      if (tid == 0 && P.trace) P.trace[2 * t + 1] = gtimer();  // finished, before any release
      for (int k = succ_b + tid; k < succ_e; k += THREADS) {
        const bool pre = (k - succ_b) < kPre;
        const int s = pre ? s_succ[k - succ_b][0].x : P.succ[4 * k].x;
        if (atom_add_acq_rel(P.indeg + s, -1) == 1) {
          if (atomicCAS(&s_cont, -1, s) == -1) {
            // continuation: its task record travels with the edge
#pragma unroll
            for (int w = 0; w < kTaskInt4; ++w)
              s_h[w] = pre ? s_succ[k - succ_b][1 + w] : P.succ[4 * k + 1 + w];
            s_pref = 1;
          } else {
            const int slot = atomicAdd(&P.ctrl->q_tail.v, 1);
            st_release(P.queue + slot, s);
          }
        }
      }
      if (tid == 0) atomicAdd(&P.ctrl->done.v, 1);
    } else {
      cp_async_wait_all();  // helper CTAs: retire the prefetch before smem reuse
    }
    __syncthreads();
  }
}

__global__ void prepare_kernel(PrepParams Q) {
  const int stride = gridDim.x * blockDim.x;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < Q.qcap; k += stride) {
    if (k < Q.ntasks) {
      Q.indeg[k] = Q.indeg0[k];
      if (Q.claim) Q.claim[k] = 0;
      if (Q.fin) Q.fin[k] = 0;
    }
    Q.queue[k] = k < Q.nroots ? Q.roots[k] : -1;
    if (Q.queue2) Q.queue2[k] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctrl c = {};
    c.q_tail.v = Q.nroots;
    c.fail_row = -1;
    *Q.ctrl = c;
  }
}

// ---- host-side launch helpers (declared in device_api.hpp) ----------------

size_t factor_smem_bytes(int threads, int cap, int flag_words, int icap, int scap) {
  // flag_words and cap are multiples of 4, so every region stays 16-B aligned.
  const size_t warps = static_cast<size_t>(threads / 32);
  return static_cast<size_t>(flag_words) * 4 + warps * static_cast<size_t>(cap) * 12 +
         static_cast<size_t>(icap) * 32 + static_cast<size_t>(scap) * 16;
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
  int blocks = (q.qcap + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  prepare_kernel<<<blocks, threads, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_factor(const Params& p, int grid, int threads, size_t smem, cudaStream_t st) {
  switch (threads) {
    case 128: return launch_resident(reinterpret_cast<const void*>(&factor_persistent<128>), grid, 128, smem, st, p);
    case 256: return launch_resident(reinterpret_cast<const void*>(&factor_persistent<256>), grid, 256, smem, st, p);
    case 512: return launch_resident(reinterpret_cast<const void*>(&factor_persistent<512>), grid, 512, smem, st, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tcbdev
