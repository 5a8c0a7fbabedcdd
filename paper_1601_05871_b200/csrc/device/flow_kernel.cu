// Value-flow schedule (mode 5, the default executor), one lane per
// coordinate: a static order of the finalising rows without flags, fences or
// any per-row synchronisation. (flow_pp_kernel.cu runs the same schedule with
// a unit's products spread over a group of warps, for short programs.)
//
// Only the finalising rows run (the Chol/Trsm units of flow_plan.cpp, which
// fold every Herk/Gemm product of a slice into the row that finalises it, in
// generation order), so every coordinate of U is written exactly once.
// The prelude snapshots the input values and sets the output to kUnset (a
// NaN payload arithmetic never produces); a row gathers its operands with
// 64-bit strong loads and re-polls any that still read kUnset.
// A value is single-copy atomic, so a reader sees either kUnset or the final
// value: the data is its own flag, and a hand-off between rows costs one
// store reaching L2 plus one load, instead of store + release fence + flag
// store + flag poll + acquire + load.
//
// Warp w of the W co-resident warps runs positions w, w+W, ... The order is
// topological (level, then falling height), so the row at the smallest
// unfinished position only reads values that are final: the schedule cannot
// deadlock while all warps are resident (a cooperative launch; a watchdog
// ends the kernel otherwise). Per coordinate the products arrive in ascending
// source row, so the factor is bitwise equal to factor_serial
// (factorize.hpp:94-130; kernels.hpp:40-132 for one target row).
#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "flow_common.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {


// An input value: the prelude's snapshot, immutable during the launch.
__device__ __forceinline__ double input_ld(const FlowParams&, const double* p) { return __ldg(p); }
__device__ __forceinline__ double input_settle(const FlowParams&, const double*, double x, unsigned long long) {
  return x;
}

// One coordinate: v -= U[m]*U[o] over its merged program, in order. The
// first pair rides in the slot record; the rest are fetched a batch ahead.
// (Issuing the first batch's operand loads before settling the first pair
// measured slower on B200: C2 0.63 -> 0.68 ms.)
template <int KB, class Cx>
__device__ __forceinline__ double flow_slot(const Cx& C, double v, const int4 sr) {
  const int ub = sr.x, ue = sr.y;
  if (ub >= ue) return v;
  TCG_CHECK((ub >= 0 && ue <= C.P.nupd) || C.P.npeers > 1);
  // long programs (KB >= 3): pull the rest of the (m, o) pairs into L2 now, so
  // the batch-ahead loads below hit L2 instead of HBM (C3's programs are
  // 1.5 GB). B200: C3 4.03 -> 3.88, C4 1.474 -> 1.453 ms; with short programs
  // it cost 1-2% (C2, C6), so the KB = 1-2 kernels do not do it.
  if (KB >= 3)
    for (int q = ub + 1 + 2 * KB; q < ue; q += 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(C.P.upd + q));
  const unsigned long long xa0 = C.ld(sr.z), xb0 = C.ld(sr.w);
  int u = ub + 1;
  int2 p[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) p[j] = (u + j < ue) ? __ldg(C.P.upd + u + j) : make_int2(0, 0);
  v = __dsub_rn(v, C.product(sr.z, xa0, sr.w, xb0));
  while (u < ue) {
    const int n = min(KB, ue - u);
    unsigned long long xa[KB], xb[KB];
    int2 c[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      c[j] = p[j];
      TCG_CHECK(j >= n || C.P.npeers > 1 || (c[j].x >= 0 && c[j].x <= c[j].y && c[j].y < C.P.nnz));
      xa[j] = (j < n) ? C.ld(c[j].x) : 0ull;
      xb[j] = (j < n) ? C.ld(c[j].y) : 0ull;
    }
    u += KB;
#pragma unroll
    for (int j = 0; j < KB; ++j) p[j] = (u + j < ue) ? __ldg(C.P.upd + u + j) : make_int2(0, 0);
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < n)
        v = __dsub_rn(v, C.product(c[j].x, xa[j], c[j].y, xb[j]));
  }
  return v;
}

// flow_slot for the first pass of a unit, called by the whole warp (`on`: the
// lane has a coordinate). Every batch but the last runs as in flow_slot, each
// lane on its own. The last batch's operands are loaded as each lane gets
// there, and what is still unwritten then is re-polled by the lanes of the
// unit together, on one clock. The lanes of a critical row mostly wait for the
// same source row, whose values arrive together: polling each on its own
// clock, they saw them up to a sleep plus a round trip apart (C3 trace: 1.7
// us), and the pivot waits for the last; together the unit is done one poll
// after the values are. A round re-polls every operand of the batch that is
// still unwritten (the polls of a warp coalesce now; lane by lane the same
// re-reads made things slower), and the rounds follow each other at the pace
// of the round trip, without a sleep (a warp's coalesced polls are few enough:
// C3 2.17 -> 2.13 ms, C4 1.21 -> 1.17 against sleeping 100-600 ns after a
// round without progress). B200: C3 2.60 -> 2.38 ms, C4 1.30 -> 1.25, then C3
// 2.34 -> 2.19, s27 0.80 -> 0.72 with the whole batch re-polled; bitwise.
template <int KB, class Cx>
__device__ __forceinline__ double flow_slot_conv(const Cx& C, double v, const int4 sr, bool on, unsigned gmask,
                                               int dpos = -1, unsigned long long* xd = nullptr) {
  auto LD = [&](int pos) { return C.ld_early(pos); };
  const int ub = sr.x, ue = on ? sr.y : sr.x;
  int u = ub;
  int2 p[KB];
  if (ub < ue) {
    if (KB >= 3)
      for (int q = ub + 1 + 2 * KB; q < ue; q += 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(C.P.upd + q));
    const unsigned long long xa0 = LD(sr.z), xb0 = LD(sr.w);
    u = ub + 1;
#pragma unroll
    for (int j = 0; j < KB; ++j) p[j] = (u + j < ue) ? __ldg(C.P.upd + u + j) : make_int2(0, 0);
    v = __dsub_rn(v, C.product(sr.z, xa0, sr.w, xb0));
    // the short batch goes first, so that the last one -- the one the warp
    // settles together -- always holds KB products (when there are that many)
    int take = (ue - u) % KB;
    if (take == 0) take = KB;
    while (ue - u > KB) {  // (a batch, and a full one after it)
      unsigned long long xa[KB], xb[KB];
      int2 c[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        c[j] = p[j];
        xa[j] = (j < take) ? LD(c[j].x) : 0ull;
        xb[j] = (j < take) ? LD(c[j].y) : 0ull;
      }
      u += take;
#pragma unroll
      for (int j = 0; j < KB; ++j) p[j] = (u + j < ue) ? __ldg(C.P.upd + u + j) : make_int2(0, 0);
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < take) v = __dsub_rn(v, C.product(c[j].x, xa[j], c[j].y, xb[j]));
      take = KB;
    }
  }
  // the last batch
  const int n = ue - u;  // 0..KB
  unsigned long long xa[KB], xb[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    xa[j] = (j < n) ? LD(p[j].x) : 0ull;
    xb[j] = (j < n) ? LD(p[j].y) : 0ull;
  }
  int j = 0;
  unsigned spins = 0;
  for (;;) {
#pragma unroll
    for (int jj = 0; jj < KB; ++jj)
      if (jj == j && jj < n && xa[jj] != kUnset && xb[jj] != kUnset) {
        v = __dsub_rn(v, __dmul_rn(__longlong_as_double(static_cast<long long>(xa[jj])),
                                   __longlong_as_double(static_cast<long long>(xb[jj]))));
        ++j;
      }
    if (__all_sync(gmask, j >= n)) break;
    // (a chunk looks for its row's pivot in the same rounds, so it need not start waiting for it afterwards)
    if (xd && *xd == kUnset) *xd = C.ld_strong(dpos);
#pragma unroll
    for (int jj = 0; jj < KB; ++jj)
      if (jj >= j && jj < n) {  // every operand of the batch still unwritten, not only the next product's
        if (xa[jj] == kUnset) xa[jj] = C.ld_strong(p[jj].x);
        if (xb[jj] == kUnset) xb[jj] = C.ld_strong(p[jj].y);
      }
    if (++spins == 1024u) {
      spins = 0;
      if (ld_relaxed(&C.P.ctrl->error.v) || gtimer() - C.t0 > C.P.timeout_ns) {
        atomicCAS(&C.P.ctrl->error.v, 0, 1);  // abandoned: the host reports TCG_TIMEOUT
        j = n;
      }
    }
  }
  return v;
}

// One finalising row on a group of G lanes: group lane j owns coordinates
// tb+j, tb+j+G, ... Chol: pivot test (latch), sqrt, scale
// (kernels.hpp:49-53); Trsm: divide by U(t,t) (kernels.hpp:76-78). `a0`/`sr0`:
// the lane's first input value and slot record, prefetched by the caller;
// `gmask` the group's lanes, `lead` its first lane.
template <int KIND, int KB, int G, class Cx>
__device__ __forceinline__ void flow_row(const Cx& C, int tb, int L, int dpos, int t, int gl,
                                         unsigned gmask, int lead, double a0, int4 sr0,
                                         unsigned long long* stamp, bool exported = false,
                                         volatile unsigned long long* piv_slot = nullptr) {
  const FlowParams& P = C.P;
  unsigned long long xd = 0;
  if (KIND == kTrsm) xd = C.ld(dpos);
  double v = 0.0;
  if (G == 32 && !Cx::kSysPublish)  // (sharded parts settle remote operands lane by lane)
    v = flow_slot_conv<KB>(C, gl < L ? a0 : 0.0, sr0, gl < L, gmask, dpos, KIND == kTrsm ? &xd : nullptr);
  else if (gl < L) v = flow_slot<KB>(C, input_settle(P, C.a + tb + gl, a0, C.t0), sr0);
  if (stamp && gl == 0) stamp[1] = gtimer();  // trace: the group's first coordinate is done
  double d;
  if (KIND == kChol) {
    double piv = v;
    if (piv_slot) {
      // The pivot through shared memory: the diagonal's lane publishes as soon
      // as its own program is done, and every other lane divides as soon as
      // its program and the pivot are ready. (A shuffle makes every lane of
      // the unit, and so U(t,t+1) which the next row waits for, wait for the
      // slowest coordinate, whose late operand often sits in the previous
      // row's chunk, one hop later: C3 trace, 1.7 us of a 3.1 us hop.)
      if (gl == 0) {
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
        *piv_slot = b == kUnset ? kCanonicalNaN : b;
      } else {
        unsigned long long b;
        while ((b = *piv_slot) == kUnset) __nanosleep(P.decouple);
        piv = __longlong_as_double(static_cast<long long>(b));
      }
    } else {
      piv = __shfl_sync(gmask, v, lead);
    }
    if (!(piv > 0.0) && gl == 0) {  // first breakdown of the member, and of the launch
      if (atomicCAS(P.m_failed + C.member, 0, 1) == 0) {
        P.m_row[C.member] = t;
        P.m_pivot[C.member] = piv;
      }
      if (atomicCAS(&P.ctrl->failed.v, 0, 1) == 0) {
        P.ctrl->fail_row = t;
        P.ctrl->fail_pivot = piv;
        P.ctrl->fail_member = C.member;
      }
    }
    d = __dsqrt_rn(piv);
  } else {
    // (a chunk's lanes are through with their products: they poll their row's pivot together)
    d = (G == 32 && !Cx::kSysPublish) ? C.settle_now(C.vals + dpos, xd) : C.settle(C.vals + dpos, xd);
  }
  if (stamp) {  // trace: every operand of the first G coordinates is final
    __syncwarp(gmask);
    if (gl == 0) *stamp = gtimer();
  }
  // a result that happens to carry the marker's bits (a NaN payload the
  // arithmetic passed through) is published as the canonical NaN, so no
  // reader mistakes a final value for "not written yet"
  auto finish = [&](int k, double x) {
    const double y = (KIND == kChol && k == 0) ? d : __ddiv_rn(x, d);
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(y));
    return b == kUnset ? kCanonicalNaN : b;
  };
  // sharded runs publish at system scope: readers may sit on other GPUs
  auto publish = [&](int k, unsigned long long y) {
    if (Cx::kSysPublish && exported) st_relaxed_sys_u64(C.vals + tb + k, y);
    else st_relaxed_u64(C.vals + tb + k, y);
  };
  if (gl < L) publish(gl, finish(gl, v));
  for (int k = gl + G; k < L; k += G) {
    const double w = flow_slot<KB>(C, input_settle(P, C.a + tb + k, input_ld(P, C.a + tb + k), C.t0),
                                   __ldg(P.slot + tb + k));
    publish(k, finish(k, w));
  }
}

}  // namespace

// The per-lane value-flow kernel, per-row metadata staged in shared memory: a
// row of a short program is shorter than an L2 round trip, so prefetching its
// record and first slot one row ahead in registers exposed the round trip
// (the loop-carried register copies wait for the loads). Here each warp
// keeps rings in shared memory filled by cp.async (LDGSTS): the record four
// rows ahead, the lanes' first slot records and input values two rows ahead;
// iteration k waits only for the copies issued at iteration k-2.
// (G = 32, static hand-out.)
// EXTRAS = 0: a single matrix without trace stamps (no batch member
// arithmetic, no stamp branches); 1: batches and traces.
template <int THREADS, int KB, int MINB, int REMOTE, int EXTRAS, int DRAIN = 0, int BO = 0>
__global__ void __launch_bounds__(THREADS, (MINB == 3 && THREADS == 256 && KB <= 3 && !EXTRAS) ? 4 : MINB)
    factor_flow_pipe(FlowParams P) {
  constexpr int kWarps = THREADS / 32;
  constexpr int kLenMask = (1 << 30) - 1;
  struct Ring {
    int4 rec[8];
    int4 slot[4][32];
    double in[4][32];
    unsigned long long piv[2];  // Chol pivot of the row (parity k & 1), kUnset until published
  };
  __shared__ Ring rings[kWarps];
  const int lane = threadIdx.x & 31;
  Ring& R = rings[threadIdx.x >> 5];
  if (DRAIN == 1 && static_cast<int>(blockIdx.x) >= P.row_ctas) {
    drain_values(P, (blockIdx.x - P.row_ctas) * kWarps + (threadIdx.x >> 5),
                 (gridDim.x - P.row_ctas) * kWarps);
    return;
  }
  const int W = (DRAIN == 1 ? P.row_ctas : static_cast<int>(gridDim.x)) * kWarps;
  const int w0 = blockIdx.x * kWarps + (threadIdx.x >> 5);
  Ctx<REMOTE ? 2 : 0, BO> C{P, gtimer(), P.vals, P.a, 0};
  int ran = 0, executed = 0, anyfail = 0;
  const int nrows = EXTRAS ? P.nrows * P.nbatch : P.nrows;
  auto member_of = [&](int p, int& q) {
    if (!EXTRAS) {
      q = p;
      return 0;
    }
    q = P.nbatch == 1 ? p : p / P.nbatch;
    return p - q * P.nbatch;
  };
  auto position = [&](int k) { return w0 + k * W; };
  auto fetch_rec = [&](int k) {
    const int p = position(k);
    if (lane == 0 && p < nrows) {
      int q;
      member_of(p, q);
      cp_async16(&R.rec[k & 7], P.rec + q);
    }
  };
  auto fetch_slot = [&](int k) {  // needs R.rec[k & 7] visible
    const int p = position(k);
    if (p >= nrows) return;
    const int4 r = R.rec[k & 7];
    if (lane < (r.y & kLenMask)) {
      int q;
      const long long m = member_of(p, q);
      cp_async16(&R.slot[k & 3][lane], P.slot + r.x + lane);
      cp_async8(&R.in[k & 3][lane], P.a + m * P.nnz + r.x + lane);
    }
  };
  // prologue: records of rows 0..3, then the slots of rows 0 and 1
  if (lane == 0) R.piv[0] = R.piv[1] = kUnset;
  for (int k = 0; k < 4; ++k) fetch_rec(k);
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();
  fetch_slot(0);
  fetch_slot(1);
  cp_async_commit();
  cp_async_wait_all();
  cp_async_commit();  // an empty group: the steady state waits for "all but the newest"
  __syncwarp();
  for (int k = 0; position(k) < nrows; ++k) {
    const int pos = position(k);
    cp_async_wait_group<1>();  // the copies of iteration k-2: slots of row k, record of row k+2
    __syncwarp();
    // every lane is past row k-1: its pivot slot is free for row k+1
    if (lane == 0) R.piv[(k + 1) & 1] = kUnset;
    const int4 a = R.rec[k & 7];
    const int tb = a.x, L = a.y & kLenMask, dpos = a.z, t = a.w;
    TCG_CHECK(tb >= 0 && L > 0 && static_cast<long long>(tb) + L <= P.nnz && dpos >= 0 && dpos <= tb);
    int4 sr0 = make_int4(0, 0, 0, 0);
    double a0 = 0.0;
    if (lane < L) {
      sr0 = R.slot[k & 3][lane];
      a0 = R.in[k & 3][lane];
    }
    fetch_rec(k + 4);
    fetch_slot(k + 2);
    cp_async_commit();
    const bool chol = ((a.y >> 30) & 1) == kChol;
    const bool exported = a.y < 0;
    int q;
    unsigned long long* stamp = nullptr;
    bool traced = false;
    if (EXTRAS) {
      C.member = member_of(pos, q);
      C.vals = P.vals + static_cast<long long>(C.member) * P.nnz;
      C.a = P.a + static_cast<long long>(C.member) * P.nnz;
      traced = P.trace && lane == 0 && C.member == 0;
      stamp = P.trace && C.member == 0 ? P.trace + 4 * static_cast<long long>(P.item[q]) : nullptr;
      if (traced) stamp[0] = gtimer();
    }
    if ((ran & 15) == 0) anyfail = __shfl_sync(kFull, lane == 0 ? ld_relaxed(&P.ctrl->failed.v) : 0, 0);
    int latched = 0;
    if (anyfail) latched = __shfl_sync(kFull, lane == 0 ? ld_relaxed(P.m_failed + C.member) : 0, 0);
    if (!latched) {
      if (chol)
        flow_row<kChol, KB, 32>(C, tb, L, dpos, t, lane, kFull, 0, a0, sr0, stamp ? stamp + 1 : nullptr,
                                exported, P.decouple ? &R.piv[k & 1] : nullptr);
      else
        flow_row<kTrsm, KB, 32>(C, tb, L, dpos, t, lane, kFull, 0, a0, sr0, stamp ? stamp + 1 : nullptr,
                                exported);
      ++executed;
    } else {
      for (int k2 = lane; k2 < L; k2 += 32) {
        unsigned long long x = static_cast<unsigned long long>(__double_as_longlong(__ldg(C.a + tb + k2)));
        if (x == kUnset) x = kCanonicalNaN;
        if (decltype(C)::kSysPublish && exported) st_relaxed_sys_u64(C.vals + tb + k2, x);
        else st_relaxed_u64(C.vals + tb + k2, x);
      }
    }
    if (traced) stamp[3] = gtimer();
    ++ran;
    if (DRAIN == 2) chunk_notify(P, tb, lane);
  }
  cp_async_wait_all();
  if (lane == 0) {
    if (ran) atomicAdd(&P.ctrl->done.v, ran);
    if (executed) atomicAdd(&P.ctrl->executed.v, executed);
  }
}

// Prelude: snapshot the working values, mark the output unwritten, reset
// the status words.
__global__ void flow_prepare(FlowPrepParams Q) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const double unset1 = __longlong_as_double(static_cast<long long>(kUnset));
  if (((reinterpret_cast<unsigned long long>(Q.vals) | reinterpret_cast<unsigned long long>(Q.a) |
        reinterpret_cast<unsigned long long>(Q.out)) & 15ull) != 0) {
    // a batch chunk starting at an odd member of an odd-sized U: 8-byte accesses
    for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < Q.nnz; x += stride) {
      if (Q.a != Q.vals) Q.a[x] = Q.vals[x];
      Q.out[x] = unset1;
    }
    for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < Q.nbatch; x += stride) {
      Q.m_failed[x] = 0;
      Q.m_row[x] = -1;
      Q.m_pivot[x] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      Ctrl c = {};
      c.fail_row = -1;
      c.fail_member = -1;
      *Q.ctrl = c;
    }
    return;
  }
  const long long h = Q.nnz / 2;
  const double2* in2 = reinterpret_cast<const double2*>(Q.vals);
  double2* a2 = reinterpret_cast<double2*>(Q.a);
  double2* o2 = reinterpret_cast<double2*>(Q.out);
  const double unset = __longlong_as_double(static_cast<long long>(kUnset));
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < h; x += stride) {
    if (Q.a != Q.vals) a2[x] = in2[x];  // (the pristine copy serves as input when it is current)
    o2[x] = make_double2(unset, unset);
  }
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < Q.nbatch; x += stride) {
    Q.m_failed[x] = 0;
    Q.m_row[x] = -1;
    Q.m_pivot[x] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (Q.nnz & 1) {
      if (Q.a != Q.vals) Q.a[Q.nnz - 1] = Q.vals[Q.nnz - 1];
      Q.out[Q.nnz - 1] = unset;
    }
    Ctrl c = {};
    c.fail_row = -1;
    c.fail_member = -1;
    *Q.ctrl = c;
  }
}

// init_factor_values on the device: U slot t <- 0.0 + A[map[t]] (the host
// version's `vals[t] += a` from zero, so -0.0 becomes +0.0 exactly as there),
// 0.0 for fill; for every member of a batch; also into the restore copy.
__global__ void init_values(const double* a, const int* map, double* vals, double* vals0, long long nnz,
                            long long nnz_a, int nbatch) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long total = nnz * nbatch;
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < total; x += stride) {
    const long long b = x / nnz, t = x - b * nnz;
    const int m = __ldg(map + t);
    const double v = m >= 0 ? __dadd_rn(0.0, __ldg(a + b * nnz_a + m)) : 0.0;
    vals[x] = v;
    vals0[x] = v;
  }
}

cudaError_t launch_init_values(const double* a, const int* map, double* vals, double* vals0, long long nnz,
                               long long nnz_a, int nbatch, int sm_count, cudaStream_t st) {
  const long long total = nnz * nbatch;
  long long blocks = (total + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 8LL * sm_count ? 8LL * sm_count : blocks);
  init_values<<<static_cast<int>(blocks), 256, 0, st>>>(a, map, vals, vals0, nnz, nnz_a, nbatch);
  return cudaGetLastError();
}

// (threads, KB, CTAs/SM, remote operands, extras, drain, poll back-off ns); the single-matrix
// variants named with 3 CTAs/SM and KB <= 3 are compiled for 4 (64 registers, no spills)
#define TCG_PIPE_VARIANTS(X)                                                                                  \
  X(256, 2, 3, 0, 0, 0, 0) X(256, 3, 3, 0, 0, 0, 0) X(256, 4, 3, 0, 0, 0, 0) X(256, 2, 3, 0, 1, 0, 0)             \
  X(256, 3, 3, 0, 1, 0, 0) X(256, 4, 3, 0, 1, 0, 0) X(256, 2, 3, 1, 1, 0, 0) X(256, 3, 3, 1, 1, 0, 0)             \
  X(256, 4, 3, 1, 1, 0, 0) X(256, 2, 3, 0, 0, 1, 0) X(256, 3, 3, 0, 0, 1, 0) X(256, 4, 3, 0, 0, 1, 0)             \
  X(256, 2, 3, 0, 1, 1, 0) X(256, 3, 3, 0, 1, 1, 0) X(256, 4, 3, 0, 1, 1, 0)                                     \
  X(256, 2, 5, 0, 0, 0, 0) X(256, 2, 5, 0, 0, 1, 0) X(256, 1, 5, 0, 0, 0, 0) X(256, 1, 5, 0, 0, 1, 0)             \
  X(256, 3, 3, 0, 0, 0, 100) X(256, 3, 3, 0, 0, 0, 200) X(256, 3, 3, 0, 0, 0, 400) X(256, 3, 3, 0, 0, 0, 600)   \
  X(256, 3, 3, 0, 0, 0, 1000) X(256, 3, 3, 0, 0, 0, 2400)                                                       \
  X(256, 3, 3, 0, 0, 1, 200) X(256, 3, 3, 0, 1, 0, 200) X(256, 3, 3, 0, 1, 1, 200) X(256, 3, 3, 1, 1, 0, 200)     \
  X(256, 3, 3, 0, 0, 1, 100) X(256, 3, 3, 0, 1, 0, 100) X(256, 3, 3, 0, 1, 1, 100) X(256, 3, 3, 1, 1, 0, 100)     \
  X(256, 3, 3, 0, 0, 2, 100)                                                                                    \
  X(256, 4, 3, 0, 0, 0, 200) X(256, 2, 3, 0, 0, 0, 200) X(256, 2, 3, 0, 1, 0, 200)                              \
  X(256, 3, 3, 0, 0, 1, 600) X(256, 3, 3, 0, 1, 0, 600) X(256, 3, 3, 0, 0, 1, 400) X(256, 3, 3, 0, 1, 0, 400)    \
  X(256, 3, 3, 0, 0, 2, 400)                                                                                    \
  X(256, 3, 3, 0, 0, 2, 600) X(256, 3, 3, 0, 0, 2, 200) X(256, 3, 3, 0, 0, 2, 0) X(256, 2, 3, 0, 0, 2, 0)       \
  X(256, 2, 5, 0, 0, 2, 0) X(256, 1, 5, 0, 0, 2, 0) X(256, 4, 3, 0, 0, 2, 0)

static const void* pipe_kernel_for(int threads, int kb, int minb, int remote, int extras, int drain, int bo) {
#define X(T, K, M, R, E, D, B)                                                                              \
  if (threads == T && kb == K && minb == M && remote == R && extras == E && drain == D && bo == B)          \
    return reinterpret_cast<const void*>(&factor_flow_pipe<T, K, M, R, E, D, B>);
  TCG_PIPE_VARIANTS(X)
#undef X
  return nullptr;
}

// the back-off variant when it exists, else the one without
static int pipe_backoff(int threads, int kb, int minb, int remote, int extras, int drain, int bo) {
  return pipe_kernel_for(threads, kb, minb, remote, extras, drain, bo) ? bo : 0;
}

bool pipe_variant_exists(int threads, int kb, int minb, int remote, int extras, int drain, int bo) {
  return pipe_kernel_for(threads, kb, minb, remote, extras, drain, bo) != nullptr;
}

cudaError_t pipe_occupancy(int threads, int kb, int minb, int remote, int extras, int* ctas_per_sm, int drain,
                           int bo) {
  bo = pipe_backoff(threads, kb, minb, remote, extras, drain, bo);
  const void* k = pipe_kernel_for(threads, kb, minb, remote, extras, drain, bo);
  if (!k) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, threads, 0);
}

cudaError_t launch_flow_pipe(const FlowParams& p, int grid, int threads, int kb, int minb, int remote,
                             int extras, cudaStream_t st, int drain, int bo) {
  bo = pipe_backoff(threads, kb, minb, remote, extras, drain, bo);
#define X(T, K, M, R, E, D, B)                                                                              \
  if (threads == T && kb == K && minb == M && remote == R && extras == E && drain == D && bo == B) {        \
    return launch_resident(reinterpret_cast<const void*>(&factor_flow_pipe<T, K, M, R, E, D, B>), grid, T, 0, \
                           st, p);                                                                          \
  }
  TCG_PIPE_VARIANTS(X)
#undef X
  return cudaErrorInvalidValue;
}

// Chunks of the chunked download: chunk k starts at the first unit start at or
// after k * nnz / nchunks (start[] preset to INT_MAX), and counts its units.
__global__ void flow_chunk_setup(const int4* rec, int nrows, long long nnz, int nchunks, int* start, int* units) {
  const int stride = gridDim.x * blockDim.x;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nrows; q += stride) {
    const int tb = rec[q].x;
    const int k = static_cast<int>(static_cast<long long>(tb) * nchunks / nnz);
    atomicMin(start + k, tb);
    atomicAdd(units + k, 1);
  }
}

cudaError_t launch_chunk_setup(const int4* rec, int nrows, long long nnz, int nchunks, int* start, int* units,
                               int sm_count, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(start, 0x7f, sizeof(int) * nchunks, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(units, 0, sizeof(int) * nchunks, st);
  if (e != cudaSuccess) return e;
  const int blocks = max(1, min((nrows + 255) / 256, 8 * sm_count));
  flow_chunk_setup<<<blocks, 256, 0, st>>>(rec, nrows, nnz, nchunks, start, units);
  return cudaGetLastError();
}

cudaError_t launch_flow_prepare(const FlowPrepParams& q, int sm_count, cudaStream_t st) {
  const long long h = q.nnz / 2;
  long long blocks = (h + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 4LL * sm_count ? 4LL * sm_count : blocks);
  flow_prepare<<<static_cast<int>(blocks), 256, 0, st>>>(q);
  return cudaGetLastError();
}

}  // namespace tcbdev
