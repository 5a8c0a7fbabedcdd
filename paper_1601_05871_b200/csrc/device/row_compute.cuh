// Row body shared by the row-level executors (modes 3 and 4): apply the
// row's update program and finish it (reference kernels.hpp:40-132 for one
// target row).
#pragma once

#include <cuda_runtime.h>

#include "factor_kernel.cuh"
#include "sync.cuh"

#ifndef TCG_GATHER_BATCH
#define TCG_GATHER_BATCH 4  // products gathered per batch (registers vs memory-level parallelism)
#endif

namespace tcbdev {

// Slot k of the target row: v -= U[m]*U[o] over its products, in source
// order. The first (m, o) is carried by the slot record; later pairs are
// fetched a batch ahead of their use.
template <int kB = TCG_GATHER_BATCH>
__device__ __forceinline__ double row_slot(const int2* __restrict__ upd, const double* vals, double v,
                                           const int4 sr) {
  const int ub = sr.x, ue = sr.y;
  if (ub >= ue) return v;
  const double a0 = vals[sr.z], b0 = vals[sr.w];
  int u = ub + 1;
  int2 p[kB];
#pragma unroll
  for (int j = 0; j < kB; ++j) p[j] = (u + j < ue) ? upd[u + j] : make_int2(0, 0);
  v = __dsub_rn(v, __dmul_rn(a0, b0));
  while (u < ue) {
    const int n = min(kB, ue - u);
    double a[kB], b[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      a[j] = (j < n) ? vals[p[j].x] : 0.0;
      b[j] = (j < n) ? vals[p[j].y] : 0.0;
    }
    u += kB;
#pragma unroll
    for (int j = 0; j < kB; ++j) p[j] = (u + j < ue) ? upd[u + j] : make_int2(0, 0);
#pragma unroll
    for (int j = 0; j < kB; ++j)
      if (j < n) v = __dsub_rn(v, __dmul_rn(a[j], b[j]));
  }
  return v;
}

// Whole row on a group of G lanes (G = 32: a warp): lane j of the group owns
// slots j, j+G, ... `sr0` is the lane's first slot record (prefetched by the
// caller); `gmask` the group's lanes and `lead` the absolute lane holding
// slot 0. Chol: pivot test (latch), sqrt, scale (kernels.hpp:49-53); Trsm:
// divide by U(t,t) (kernels.hpp:76-78).
template <int KIND, int G = 32, int KB = TCG_GATHER_BATCH>
__device__ __forceinline__ void row_compute(const int4* slot_rec, const int2* upd, double* vals,
                                            Ctrl* ctrl, int tb, int L, int dpos, int soff, int t,
                                            int lane, int4 sr0, unsigned gmask = kFull,
                                            int lead = 0) {
  double v = 0.0;
  if (lane < L) v = vals[tb + lane];
  double d = 1.0;
  if (KIND == kTrsm) d = vals[dpos];
  if (lane < L) v = row_slot<KB>(upd, vals, v, sr0);
  if (KIND == kChol) {
    const double piv = __shfl_sync(gmask, v, lead);
    if (!(piv > 0.0) && lane == 0) {
      if (atomicCAS(&ctrl->failed.v, 0, 1) == 0) {
        ctrl->fail_row = t;
        ctrl->fail_pivot = piv;
      }
    }
    d = __dsqrt_rn(piv);
  }
  auto finish = [&](int k, double x) {
    if (KIND == kChol) return k == 0 ? d : __ddiv_rn(x, d);
    if (KIND == kTrsm) return __ddiv_rn(x, d);
    return x;
  };
  if (lane < L) vals[tb + lane] = finish(lane, v);
  for (int k = lane + G; k < L; k += G) {
    const double w = row_slot<KB>(upd, vals, vals[tb + k], slot_rec[soff + k]);
    vals[tb + k] = finish(k, w);
  }
}

}  // namespace tcbdev
