// Value flow with product-parallel rows: the same static schedule of
// finalising rows as factor_flow_pipe (flow_kernel.cu), the same data-as-flag
// hand-off, but a row's products are spread over all the threads of its row
// group instead of one lane per coordinate.
//
// A row ("unit": coordinates [tb, tb + L) of U row t) owns the contiguous
// product range [ub[tb], ub[tb + L]) of the device-built programs
// (flow_program.cu), coordinate x's products [ub[x], ub[x + 1]) in ascending
// source row. The group (T = 32 * WPR threads) walks that range in chunks of
// C = T * KP products:
//   phase A  thread i takes products i, i + T, ... of the chunk: it reads the
//            (m, o) pair from shared memory, loads both operands (polling
//            them until they are no longer kUnset), rounds the product
//            U[m] * U[o] on its own and stores it into the chunk's slot in
//            shared memory;
//   phase B  after a group barrier, thread j (coordinate tb + j) subtracts
//            the products of its own range that fall in the chunk, in order.
// So every coordinate still receives v <- v - U(r,t) * U(r,c) for r
// ascending with __dmul_rn / __dsub_rn -- the order of factor_serial
// (factorize.hpp:94-130; kernels.hpp:55-65, :85-89, :104-108, :125-129 per
// target row) -- and the factor stays bitwise equal to it; only the loads
// and the multiplications run in parallel. A row's products cost
// ceil(P / C) round trips instead of its longest program's length (C3: a
// critical row holds up to ~4,000 products, 25 per coordinate on average).
//
// Metadata: the pairs of the first chunk of the group's next rows, the rows'
// records and their coordinates' offsets and inputs arrive by cp.async into
// per-group rings, D rows ahead (the group waits for the copies of D rows
// ago); the later chunks of a long row one chunk ahead. The pairs are read
// once, coalesced, and no per-coordinate slot record is needed (4 bytes of
// offsets per coordinate instead of 16).
//
// Rows with more than T coordinates run in passes of T; the Chol pivot lives
// in pass 0 (kernels.hpp:49-53) and is broadcast to the group.
#include <cuda_runtime.h>

#include "device_api.hpp"
#include "factor_kernel.cuh"
#include "flow_common.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

// Shared memory of one row group (byte offsets).
template <int T, int KP, int NB, int D>
struct PPLayout {
  static constexpr int C = T * KP * NB;     // products per chunk
  static constexpr int RR = 3 * D + 1;      // records: rows k .. k + 3D
  static constexpr int UR = 2 * D + 1;      // coordinate offsets / inputs: rows k .. k + 2D
  static constexpr int FR = D + 1;          // first chunks: rows k .. k + D
  static constexpr int UBW = (T + 1 + 3) & ~3;
  static constexpr int o_prod = 0;                    // double[C]
  static constexpr int o_first = o_prod + 8 * C;      // int2[FR][C]
  static constexpr int o_x = o_first + 8 * C * FR;    // int2[2][C]
  static constexpr int o_in = o_x + 16 * C;           // double[UR][T]
  static constexpr int o_rec = o_in + 8 * T * UR;     // int4[RR]
  static constexpr int o_ub = o_rec + 16 * RR;        // int[UR][UBW]
  static constexpr int o_word = o_ub + 4 * UBW * UR;  // double piv[2]; int flag[2]
  static constexpr int bytes = (o_word + 32 + 127) & ~127;
};

template <int WPR, int KP, int NB, int MINB, int EXTRAS, int DRAIN, int BO, int D>
__global__ void __launch_bounds__(256, MINB) factor_flow_pp(FlowParams P) {
  constexpr int T = 32 * WPR;   // threads per row group
  constexpr int G = 256 / T;    // row groups per CTA
  using Lay = PPLayout<T, KP, NB, D>;
  constexpr int C = Lay::C;
  constexpr int kLenMask = (1 << 30) - 1;
  extern __shared__ __align__(16) unsigned char pp_smem[];
  if (DRAIN == 1 && static_cast<int>(blockIdx.x) >= P.row_ctas) {
    drain_values(P, (blockIdx.x - P.row_ctas) * 8 + (threadIdx.x >> 5), (gridDim.x - P.row_ctas) * 8);
    return;
  }
  const int gi = threadIdx.x / T, j = threadIdx.x % T;
  unsigned char* S = pp_smem + gi * Lay::bytes;
  double* prod = reinterpret_cast<double*>(S + Lay::o_prod);
  int2* first = reinterpret_cast<int2*>(S + Lay::o_first);
  int2* xbuf = reinterpret_cast<int2*>(S + Lay::o_x);
  double* inr = reinterpret_cast<double*>(S + Lay::o_in);
  int4* recr = reinterpret_cast<int4*>(S + Lay::o_rec);
  int* ubr = reinterpret_cast<int*>(S + Lay::o_ub);
  double* pivw = reinterpret_cast<double*>(S + Lay::o_word);
  int* flagw = reinterpret_cast<int*>(S + Lay::o_word + 16);
  const int bar = 1 + gi;
  const int W = (DRAIN == 1 ? P.row_ctas : static_cast<int>(gridDim.x)) * G;
  const int g0 = blockIdx.x * G + gi;
  Ctx<0, BO> Cx{P, gtimer(), P.vals, P.a, 0};
  const int nrows = EXTRAS ? P.nrows * P.nbatch : P.nrows;
  auto split = [&](int p, int& q) -> int {
    if (!EXTRAS) {
      q = p;
      return 0;
    }
    q = P.nbatch == 1 ? p : p / P.nbatch;
    return p - q * P.nbatch;
  };
  auto position = [&](int k) { return g0 + k * W; };
  auto fetch_rec = [&](int k) {
    const int p = position(k);
    if (j == 0 && p < nrows) {
      int q;
      split(p, q);
      cp_async16(recr + k % Lay::RR, P.rec + q);
    }
  };
  auto fetch_coords = [&](int k) {  // needs record k visible
    const int p = position(k);
    if (p >= nrows) return;
    const int4 r = recr[k % Lay::RR];
    const int Lp = min(r.y & kLenMask, T);
    int q;
    const long long m = split(p, q);
    int* u = ubr + (k % Lay::UR) * Lay::UBW;
    if (j <= Lp) cp_async4(u + j, P.ub + r.x + j);
    if (j == 0 && Lp == T) cp_async4(u + T, P.ub + r.x + T);
    if (j < Lp) cp_async8(inr + (k % Lay::UR) * T + j, P.a + m * P.nnz + r.x + j);
  };
  auto fetch_pairs = [&](int2* dst, int c0, int n) {
#pragma unroll
    for (int k = 0; k < KP * NB; ++k) {
      const int i = j + k * T;
      if (i < n) cp_async8(dst + i, P.upd + c0 + i);
    }
  };
  auto fetch_first = [&](int k) {  // needs record k and its offsets visible
    if (position(k) >= nrows) return;
    const int4 r = recr[k % Lay::RR];
    const int Lp = min(r.y & kLenMask, T);
    const int* u = ubr + (k % Lay::UR) * Lay::UBW;
    fetch_pairs(first + (k % Lay::FR) * C, u[0], min(u[Lp] - u[0], C));
  };
  // prologue: records of rows 0 .. 3D-1, then offsets and inputs of rows
  // 0 .. 2D-1, then the first chunks of rows 0 .. D-1
  for (int k = 0; k < 3 * D; ++k) fetch_rec(k);
  cp_async_commit();
  cp_async_wait_all();
  group_sync<T>(bar);
  for (int k = 0; k < 2 * D; ++k) fetch_coords(k);
  cp_async_commit();
  cp_async_wait_all();
  group_sync<T>(bar);
  for (int k = 0; k < D; ++k) fetch_first(k);
  cp_async_commit();
  cp_async_wait_all();

  int ran = 0, executed = 0, anyfail = 0;
  // One chunk [c0, c0 + n) whose pairs are in `pairs` (visible): products
  // into shared memory, barrier, then this thread's coordinate takes the
  // ones of its range [myb, mye) in order.
  // A chunk is large (NB batches of KP products per thread) so that it spans
  // many coordinates: phase B then runs in parallel over them (a chunk
  // covering one coordinate's run would serialise on its dsub chain).
  auto chunk = [&](const int2* pairs, int c0, int n, double& v, int myb, int mye) {
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {
      const int base = b * KP * T;
      if (base >= n) break;
      int2 mo[KP];
      unsigned long long xa[KP], xb[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int i = base + j + k * T;
        if (i < n) {
          mo[k] = pairs[i];
          // both operands lie in one earlier row r: m = U(r,t) <= o = U(r,c) < this row
          TCG_CHECK(mo[k].x >= 0 && mo[k].x <= mo[k].y && mo[k].y < P.nnz);
          xa[k] = Cx.ld(mo[k].x);
          xb[k] = Cx.ld(mo[k].y);
        }
      }
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int i = base + j + k * T;
        if (i < n) prod[i] = Cx.product(mo[k].x, xa[k], mo[k].y, xb[k]);
      }
    }
    group_sync<T>(bar);
    const int lo = max(myb, c0) - c0, hi = min(mye, c0 + n) - c0;
#pragma unroll 4
    for (int i = lo; i < hi; ++i) v = __dsub_rn(v, prod[i]);
  };

  for (int k = 0; position(k) < nrows; ++k) {
    const int pos = position(k);
    // the breakdown decision is one per group: thread 0 reads the latches
    // before the barrier, everyone reads its answer after it
    int q;
    const int member = split(pos, q);
    if (j == 0) {
      if ((ran & 15) == 0) anyfail = ld_relaxed(&P.ctrl->failed.v);
      flagw[k & 1] = anyfail ? ld_relaxed(P.m_failed + member) : 0;
    }
    if (D == 1) cp_async_wait_all();
    else cp_async_wait_group<D - 1>();
    group_sync<T>(bar);
    const int latched = flagw[k & 1];
    const int4 a = recr[k % Lay::RR];
    const int tb = a.x, L = a.y & kLenMask, dpos = a.z, t = a.w;
    const bool chol = ((a.y >> 30) & 1) == kChol;
    const int Lp = min(L, T);
    const int* u = ubr + (k % Lay::UR) * Lay::UBW;
    const int pb = u[0], pe = u[Lp];
    TCG_CHECK(tb >= 0 && L > 0 && static_cast<long long>(tb) + L <= P.nnz && dpos >= 0 && dpos <= tb);
    TCG_CHECK(pb >= 0 && pb <= pe && pe <= P.nupd);
    int myb = 0, mye = 0;
    double v = 0.0;
    if (j < Lp) {
      myb = u[j];
      mye = u[j + 1];
      v = inr[(k % Lay::UR) * T + j];
      TCG_CHECK(pb <= myb && myb <= mye && mye <= pe);
    }
    // the pairs of this row's second chunk, then the rings D rows ahead
    if (pe - pb > C) fetch_pairs(xbuf + C, pb + C, min(pe - pb - C, C));
    cp_async_commit();
    fetch_rec(k + 3 * D);
    fetch_coords(k + 2 * D);
    fetch_first(k + D);
    cp_async_commit();
    if (EXTRAS) {
      Cx.member = member;
      Cx.vals = P.vals + static_cast<long long>(member) * P.nnz;
      Cx.a = P.a + static_cast<long long>(member) * P.nnz;
    }
    ++ran;
    if (latched) {  // the member broke down: its later rows keep their inputs
      for (int x = tb + j; x < tb + L; x += T) {
        unsigned long long y = static_cast<unsigned long long>(__double_as_longlong(__ldg(Cx.a + x)));
        if (y == kUnset) y = kCanonicalNaN;
        st_relaxed_u64(Cx.vals + x, y);
      }
      if (DRAIN == 2) {
        group_sync<T>(bar);
        if (j == 0) chunk_count(P, tb);
      }
      continue;
    }
    ++executed;
    const unsigned long long xd = chol ? 0ull : Cx.ld(dpos);
    // pass 0: the prefetched first chunk, later chunks one ahead in xbuf
    {
      int c = 0;
      for (int c0 = pb; c0 < pe; c0 += C, ++c) {
        const int2* pairs = first + (k % Lay::FR) * C;
        if (c > 0) {
          if (c == 1) cp_async_wait_group<1>();  // the ring copies may still be in flight
          else cp_async_wait_all();
          group_sync<T>(bar);
          pairs = xbuf + (c & 1) * C;
          const int c1 = c0 + C;
          if (c1 < pe) fetch_pairs(xbuf + ((c + 1) & 1) * C, c1, min(pe - c1, C));
          cp_async_commit();
        }
        chunk(pairs, c0, min(C, pe - c0), v, myb, mye);
      }
    }
    // the divisor: Chol sqrt of the pivot (lane 0 of pass 0), Trsm U(t,t)
    double d;
    if (chol) {
      double piv;
      if (T == 32) {
        piv = __shfl_sync(kFull, v, 0);
      } else {
        if (j == 0) pivw[k & 1] = v;
        group_sync<T>(bar);
        piv = pivw[k & 1];
      }
      if (!(piv > 0.0) && j == 0) {  // first breakdown of the member, and of the launch
        if (atomicCAS(P.m_failed + Cx.member, 0, 1) == 0) {
          P.m_row[Cx.member] = t;
          P.m_pivot[Cx.member] = piv;
        }
        if (atomicCAS(&P.ctrl->failed.v, 0, 1) == 0) {
          P.ctrl->fail_row = t;
          P.ctrl->fail_pivot = piv;
          P.ctrl->fail_member = Cx.member;
        }
      }
      d = __dsqrt_rn(piv);
    } else {
      d = Cx.settle(Cx.vals + dpos, xd);
    }
    auto publish = [&](int x, double w, bool diag) {
      const double y = diag ? d : __ddiv_rn(w, d);
      unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(y));
      if (b == kUnset) b = kCanonicalNaN;
      st_relaxed_u64(Cx.vals + x, b);
    };
    if (j < Lp) publish(tb + j, v, chol && j == 0);
    // passes over the coordinates past the first T (long Chol slices)
    for (int cb = tb + T; cb < tb + L; cb += T) {
      const int Lc = min(T, tb + L - cb);
      const int qb = __ldg(P.ub + cb), qe = __ldg(P.ub + cb + Lc);
      double w = 0.0;
      int b0 = 0, b1 = 0;
      if (j < Lc) {
        w = __ldg(Cx.a + cb + j);
        b0 = __ldg(P.ub + cb + j);
        b1 = __ldg(P.ub + cb + j + 1);
      }
      int c = 0;
      for (int c0 = qb; c0 < qe; c0 += C, ++c) {
        cp_async_wait_all();
        group_sync<T>(bar);  // the previous chunk's readers are done with the buffer
        int2* pairs = xbuf + (c & 1) * C;
        fetch_pairs(pairs, c0, min(C, qe - c0));
        cp_async_commit();
        cp_async_wait_all();
        group_sync<T>(bar);
        chunk(pairs, c0, min(C, qe - c0), w, b0, b1);
      }
      if (j < Lc) publish(cb + j, w, false);
    }
    if (DRAIN == 2) {  // chunked download: the unit is done once the whole group has published
      group_sync<T>(bar);
      if (j == 0) chunk_count(P, tb);
    }
  }
  cp_async_wait_all();
  if (j == 0) {
    if (ran) atomicAdd(&P.ctrl->done.v, ran);
    if (executed) atomicAdd(&P.ctrl->executed.v, executed);
  }
}

}  // namespace

// (warps per row group, products per thread and chunk, CTAs/SM, extras, drain, poll back-off ns,
// rows of metadata prefetch)
// Measured on B200 (device ms, one session, against the per-lane kernel
// factor_flow_pipe): (1, 2, 1, 4, ., ., 0, 2) C2 0.395 -> 0.364, C6 1.725 ->
// 1.424, C5 batch of 64 1.816 -> 1.412; (2, 2, 2, 3, ., ., 0, 1) C1 0.044 ->
// 0.040, C5 0.168 -> 0.134. Long programs lose (C3 3.26 -> 7.0, C4 1.41 ->
// 2.95 at best): a critical row waits for about one late product per
// coordinate, and the per-lane kernel has subtracted every earlier product
// by then, while here the whole dsub chain (up to ~200 per diagonal) runs
// after the last product arrives. A poll back-off (50-200 ns) made every
// short-program configuration slower (C6 1.426 -> 1.447-1.455, C2 0.362 ->
// 0.372-0.378 ms). So did 4-byte products ((source index << 16) | in-row
// offset, the row's source positions staged per unit): C6 1.43 -> 1.55, C5
// batch 1.41 -> 1.78 ms, DRAM per C6 launch only 1.21 -> 1.19 GB -- the
// traffic is operand re-reads, not the programs.
#define TCG_PP_VARIANTS(X)                                                                                   \
  X(1, 2, 1, 4, 0, 0, 0, 2) X(1, 2, 1, 4, 0, 1, 0, 2) X(1, 2, 1, 4, 1, 0, 0, 2) X(1, 2, 1, 4, 1, 1, 0, 2)       \
  X(2, 2, 2, 3, 0, 0, 0, 1) X(2, 2, 2, 3, 0, 1, 0, 1) X(2, 2, 2, 3, 1, 0, 0, 1) X(2, 2, 2, 3, 1, 1, 0, 1)       \
  X(2, 1, 4, 4, 0, 0, 0, 1) X(1, 2, 2, 4, 0, 0, 0, 2) X(4, 2, 4, 3, 0, 0, 0, 1) X(4, 4, 4, 2, 0, 0, 0, 1)       \
  X(1, 2, 1, 4, 0, 2, 0, 2) X(2, 2, 2, 3, 0, 2, 0, 1)

template <int WPR, int KP, int NB, int D>
static size_t pp_smem_bytes() {
  return static_cast<size_t>(256 / (32 * WPR)) * PPLayout<32 * WPR, KP, NB, D>::bytes;
}

static const void* pp_kernel_for(int wpr, int kp, int nb, int minb, int extras, int drain, int bo, int d,
                                 size_t* smem) {
#define X(W, K, NBB, M, E, DR, B, DD)                                                                        \
  if (wpr == W && kp == K && nb == NBB && minb == M && extras == E && drain == DR && bo == B && d == DD) {  \
    *smem = pp_smem_bytes<W, K, NBB, DD>();                                                                 \
    return reinterpret_cast<const void*>(&factor_flow_pp<W, K, NBB, M, E, DR, B, DD>);                      \
  }
  TCG_PP_VARIANTS(X)
#undef X
  return nullptr;
}

cudaError_t pp_occupancy(int wpr, int kp, int nb, int minb, int extras, int drain, int bo, int d,
                         int* ctas_per_sm, size_t* smem) {
  const void* k = pp_kernel_for(wpr, kp, nb, minb, extras, drain, bo, d, smem);
  if (!k) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(*smem));
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, 256, *smem);
}

cudaError_t launch_flow_pp(const FlowParams& p, int grid, int wpr, int kp, int nb, int minb, int extras, int drain,
                           int bo, int d, cudaStream_t st) {
  size_t smem = 0;
  const void* k = pp_kernel_for(wpr, kp, nb, minb, extras, drain, bo, d, &smem);
  if (!k) return cudaErrorInvalidValue;
  return launch_resident(k, grid, 256, smem, st, p);
}

}  // namespace tcbdev
