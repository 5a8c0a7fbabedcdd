// Level-k fill pattern of U on the device (the reference's levelk_pattern_bfs,
// symbolic.hpp:57-120). An entry (i, j), j > i, has level <= k exactly when j
// is adjacent to a vertex reachable from i in <= k edges through vertices
// numbered below i (symbolic.hpp:6-9). The per-source searches are
// independent (symbolic.hpp:14-16), so one warp runs one source row:
//
//   frontier F_0 = {i}; for d = 0..k: every neighbour w of F_d is a target
//   when w > i, and joins F_{d+1} when w < i, d < k and w was not seen yet.
//
// This is the reference's search read as sets: its FIFO queue visits a
// vertex first at its shortest distance (largest remaining depth), so the
// later revisits with less depth add nothing; targets are recorded at any
// depth; the interior vertices are expanded while depth remains. The row of U
// is {i} then the targets ascending (symbolic.hpp:97-101).
//
// Fast path (two tiers: 512-slot tables at 7 CTAs/SM, then 2,048-slot tables
// for the rows that outgrow them): the warp's seen-set is an open-addressed
// hash table in shared memory (interior vertices and targets are disjoint key
// ranges, one table) with an insertion list whose depth-d entries are frontier
// d + 1; the adjacency of 32 frontier vertices is
// flattened by a warp prefix sum over their degrees so every lane loads a
// neighbour (7-point stencils have degree 7). A search that outgrows the
// table or the frontier list is handed to the slow path: one warp per row
// with an n-entry stamp array and n-entry frontier lists in global memory, and
// targets emitted by scanning the stamps in (i, n) -- no capacity limit.
//
// One search per row: the count pass also writes the row ({i}, then the
// targets rank-sorted in shared memory) into a scratch array at an offset it
// reserves with an atomic; a device scan turns the lengths into row_ptr and a
// copy kernel moves the rows into place. Rows that find no room in scratch
// (its size adapts to the last run) and the global-memory rows are searched
// again after the scan. All work is integer; the output is bit-exact by
// construction.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "symbolic_api.hpp"

namespace tcbdev {

namespace {

constexpr int kEmpty = -1;
constexpr unsigned kFullMask = 0xffffffffu;

template <int HB, int G = 32>
struct WarpSym {
  static constexpr int kHash = 1 << HB;
  static constexpr int kLoad = kHash * 3 / 4;  // distinct keys beyond this -> next tier
  int tab[kHash];       // seen-set: interior vertices (< i) and targets (> i)
  int ins[kLoad];       // slots in insertion order: depth by depth, so the
                        // interior keys inserted at depth d are frontier d + 1
  long long sb[G];      // adjacency begin of the current G frontier vertices
  int sx[G];            // exclusive prefix of their degrees
  int nfill, ovf;
};

template <int HB>
__device__ __forceinline__ unsigned hash_slot(int key) {
  return (static_cast<unsigned>(key) * 0x9E3779B1u) >> (32 - HB);
}

// true when newly inserted. S.ovf is set exactly when the row has more than
// kLoad distinct keys (the (kLoad+1)-th insert's ticket), so overflow is a
// property of the row, not of the interleaving; the guard at kLoad + 32 (more
// keys than that imply overflow anyway) and the probe bound keep a table that
// keeps filling from spinning.
template <int HB, int G>
__device__ __forceinline__ bool tab_insert(WarpSym<HB, G>& S, int key) {
  using W = WarpSym<HB, G>;
  if (*reinterpret_cast<volatile int*>(&S.nfill) >= W::kLoad + 32) {
    S.ovf = 1;
    return false;
  }
  unsigned h = hash_slot<HB>(key);
  for (int probe = 0; probe < W::kHash; ++probe) {
    const int old = atomicCAS(&S.tab[h], kEmpty, key);
    if (old == kEmpty) {
      const int p = atomicAdd(&S.nfill, 1);
      if (p < W::kLoad) S.ins[p] = static_cast<int>(h);
      else S.ovf = 1;
      return true;
    }
    if (old == key) return false;
    h = (h + 1) & (W::kHash - 1);
  }
  S.ovf = 1;
  return false;
}

// The search from row i in shared memory; the table is empty on entry.
// Returns false on overflow (the table is then cleared whole).
template <int HB, int G>
__device__ bool search_fast(const SymParams& P, WarpSym<HB, G>& S, int i, int lane, unsigned gmask) {
  int lo = 0, hi = 0;  // ins range of the current frontier; depth 0 is {i}
  for (int d = 0; d <= P.kk; ++d) {
    const bool expand = d < P.kk;
    const int ncur = d == 0 ? 1 : hi - lo;
    for (int c0 = 0; c0 < ncur; c0 += G) {
      int v = -1;
      if (c0 + lane < ncur) v = d == 0 ? i : S.tab[S.ins[lo + c0 + lane]];
      if (v > i) v = -1;  // a target: not expanded
      long long b = 0;
      int deg = 0;
      if (v >= 0) {
        b = __ldg(P.a_ptr + v);
        deg = static_cast<int>(__ldg(P.a_ptr + v + 1) - b);
      }
      int incl = deg;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const int y = __shfl_up_sync(gmask, incl, o, G);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(gmask, incl, G - 1, G);
      S.sb[lane] = b;
      S.sx[lane] = incl - deg;
      __syncwarp(gmask);
      for (int e = lane; e < total; e += G) {
        int j = 0;  // last j with sx[j] <= e (a zero degree repeats the prefix; take the last)
#pragma unroll
        for (int step = G / 2; step > 0; step >>= 1)
          if (S.sx[j + step] <= e) j += step;
        const int w = __ldg(P.a_col + S.sb[j] + (e - S.sx[j]));
        if (w > i || (w < i && expand)) tab_insert(S, w);
      }
      __syncwarp(gmask);
    }
    if (S.ovf) {
      for (int s = lane; s < WarpSym<HB, G>::kHash; s += G) S.tab[s] = kEmpty;
      __syncwarp(gmask);
      if (lane == 0) {
        S.nfill = 0;
        S.ovf = 0;
      }
      __syncwarp(gmask);
      return false;
    }
    lo = d == 0 ? 0 : hi;
    hi = S.nfill;
    if (hi == lo) break;
  }
  return true;
}

// Empties the table through the insertion list and moves the targets
// (keys > i) to the front of `ins`; returns their count. Every write of the
// in-place compaction lands at or before the entry being read.
template <int HB, int G>
__device__ int drain_targets(WarpSym<HB, G>& S, int i, int lane, unsigned gmask, int lead) {
  const int nf = S.nfill;
  int base = 0;
  for (int p0 = 0; p0 < nf; p0 += G) {
    const int p = p0 + lane;
    int key = kEmpty;
    if (p < nf) {
      const int slot = S.ins[p];
      key = S.tab[slot];
      S.tab[slot] = kEmpty;
    }
    const bool t = key > i;
    const unsigned bal = (__ballot_sync(gmask, t) >> lead) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
    __syncwarp(gmask);
    if (t) S.ins[base + __popc(bal & ((1u << lane) - 1u))] = key;
    base += __popc(bal);
    __syncwarp(gmask);
  }
  if (lane == 0) S.nfill = 0;
  __syncwarp(gmask);
  return base;
}

}  // namespace

// PASS 0: count[i] = row length, or (the search outgrew this tier's table)
// the row joins the next tier's list; PASS 1: write the row. Warp per row,
// grid-stride over all rows (P.list == nullptr) or over the rows of P.list.
template <int PASS, int HB, int G = 32>
__global__ void __launch_bounds__(kSymThreads) levelk_fast(SymParams P) {
  using W = WarpSym<HB, G>;
  constexpr int kGroups = kSymThreads / G;  // rows in flight per CTA
  extern __shared__ unsigned char smem_raw[];
  W* all = reinterpret_cast<W*>(smem_raw);
  const int lane_w = threadIdx.x & 31;
  const int lane = lane_w & (G - 1), lead = lane_w & ~(G - 1);
  const unsigned gmask = G == 32 ? kFullMask : (((1u << G) - 1u) << lead);
  W& S = all[threadIdx.x / G];
  for (int s = lane; s < W::kHash; s += G) S.tab[s] = kEmpty;
  if (lane == 0) {
    S.nfill = 0;
    S.ovf = 0;
  }
  __syncwarp(gmask);
  const int nw = gridDim.x * kGroups;
  const int nrows = P.list ? *P.nlist : P.n;
  for (int r = blockIdx.x * kGroups + static_cast<int>(threadIdx.x) / G; r < nrows; r += nw) {
    const int i = P.list ? P.list[r] : r;
    if (PASS == 1 && P.soff && P.soff[i] >= 0) continue;  // already written by the count pass
    // overflow is a property of the row, so the fill pass skips exactly the
    // rows the count pass handed on
    const bool ok = search_fast<HB, G>(P, S, i, lane, gmask);
    if (!ok) {
      if (PASS == 0 && lane == 0) {
        P.count[i] = -1;
        P.over[atomicAdd(P.nover, 1)] = i;
      }
      continue;
    }
    const int m = drain_targets<HB, G>(S, i, lane, gmask, lead);
    int* out = nullptr;
    if (PASS == 0) {
      long long off = -1;
      if (P.scratch && lane == 0) {
        off = static_cast<long long>(atomicAdd(P.cursor, static_cast<unsigned long long>(m + 1)));
        if (off + m + 1 > P.scratch_cap) off = -1;
      }
      off = __shfl_sync(gmask, off, lead);
      if (lane == 0) {
        P.count[i] = 1 + m;
        if (P.soff) P.soff[i] = off;
      }
      if (off < 0) continue;
      out = P.scratch + off;
    } else {
      out = P.u_col + P.u_ptr[i];
    }
    // rank sort (keys are distinct)
    if (lane == 0) out[0] = i;
    for (int e = lane; e < m; e += G) {
      const int x = S.ins[e];
      int r = 0;
      for (int q = 0; q < m; ++q) r += S.ins[q] < x;
      out[1 + r] = x;
    }
    __syncwarp(gmask);
  }
}

// Slow path: one warp per overflowing row, stamps and frontiers in global
// memory (slot s owns mark at s * n and two frontier lists at 2 * s * n).
// Stamps are unique per (row, pass) -- row + 1 counting, -(row + 1) filling --
// so the arrays are never cleared between rows.
template <int PASS>
__global__ void __launch_bounds__(kSymThreads) levelk_slow(SymParams P) {
  const int lane = threadIdx.x & 31;
  const long long slot = blockIdx.x * (kSymThreads / 32) + (threadIdx.x >> 5);
  const int nslots = gridDim.x * (kSymThreads / 32);
  const long long n = P.n;
  int* mark = P.slow_mark + slot * n;
  int* fa = P.slow_front + slot * 2 * n;
  int* fb = fa + n;
  const int nrows = *P.nlist;
  for (int o = static_cast<int>(slot); o < nrows; o += nslots) {
    const int i = P.list[o];
    const int stamp = PASS == 0 ? i + 1 : -(i + 1);
    if (lane == 0) fa[0] = i;
    int ncur = 1, ntgt = 0;
    __syncwarp();
    for (int d = 0; d <= P.kk && ncur > 0; ++d) {
      const bool expand = d < P.kk;
      int nnext = 0;
      for (int c = 0; c < ncur; ++c) {  // one frontier vertex at a time, lanes over its row
        const int v = fa[c];
        const long long b = P.a_ptr[v], e = P.a_ptr[v + 1];
        for (long long q0 = b; q0 < e; q0 += 32) {  // whole-warp trips: the counts stay uniform
          const long long q = q0 + lane;
          const int w = q < e ? P.a_col[q] : i;
          bool add_t = false, add_f = false;
          if (w > i || (w < i && expand)) {
            const int old = atomicExch(mark + w, stamp);
            if (old != stamp) {
              add_t = w > i;
              add_f = w < i;
            }
          }
          const unsigned bt = __ballot_sync(kFullMask, add_t);
          const unsigned bf = __ballot_sync(kFullMask, add_f);
          ntgt += __popc(bt);
          if (add_f) fb[nnext + __popc(bf & ((1u << lane) - 1u))] = w;
          nnext += __popc(bf);
        }
      }
      __syncwarp();
      int* t = fa;
      fa = fb;
      fb = t;
      ncur = nnext;
    }
    if (PASS == 0) {
      if (lane == 0) P.count[i] = 1 + ntgt;
      __syncwarp();
      continue;
    }
    int* out = P.u_col + P.u_ptr[i];
    if (lane == 0) out[0] = i;
    int k = 1;
    for (long long w0 = i + 1; w0 < n; w0 += 32) {
      const long long w = w0 + lane;
      const bool t = w < n && mark[w] == stamp;
      const unsigned bal = __ballot_sync(kFullMask, t);
      if (t) out[k + __popc(bal & ((1u << lane) - 1u))] = static_cast<int>(w);
      k += __popc(bal);
    }
    __syncwarp();
  }
}

// Rows the count pass wrote into scratch move into place: one thread per row
// for short rows (a warp per row left most lanes idle: C6, 7.8 entries per
// row, 296 -> ~140 µs), a warp per row for long ones (C3, 69 entries).
__global__ void __launch_bounds__(kSymThreads) levelk_copy_rows(SymParams P) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    const long long off = P.soff[i];
    if (off < 0) continue;
    const long long b = P.u_ptr[i], len = P.u_ptr[i + 1] - b;
    for (long long e = 0; e < len; ++e) P.u_col[b + e] = P.scratch[off + e];
  }
}

__global__ void __launch_bounds__(kSymThreads) levelk_copy_warps(SymParams P) {
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (kSymThreads / 32);
  for (int i = blockIdx.x * (kSymThreads / 32) + (threadIdx.x >> 5); i < P.n; i += nw) {
    const long long off = P.soff[i];
    if (off < 0) continue;
    const long long b = P.u_ptr[i], len = P.u_ptr[i + 1] - b;
    for (long long e = lane; e < len; e += 32) P.u_col[b + e] = P.scratch[off + e];
  }
}

cudaError_t launch_levelk_copy(const SymParams& p, int grid, bool long_rows, cudaStream_t st) {
  if (long_rows) levelk_copy_warps<<<grid, kSymThreads, 0, st>>>(p);
  else levelk_copy_rows<<<grid, kSymThreads, 0, st>>>(p);
  return cudaGetLastError();
}

size_t sym_smem_bytes(int hb) {
  if (hb == kSymHashTiny) return sizeof(WarpSym<kSymHashTiny, 8>) * (kSymThreads / 8);
  return hb == kSymHashSmall ? sizeof(WarpSym<kSymHashSmall>) * (kSymThreads / 32)
                             : sizeof(WarpSym<kSymHashLarge>) * (kSymThreads / 32);
}

template <int PASS, int HB, int G>
static cudaError_t fast_attr() {
  return cudaFuncSetAttribute(levelk_fast<PASS, HB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(sym_smem_bytes(HB)));
}

// hb: kSymHashTiny = 8 lanes per row with 128-slot tables, else a warp per row
cudaError_t sym_occupancy(int hb, int* ctas_per_sm) {
  cudaError_t e = cudaSuccess;
  if (hb == kSymHashTiny) {
    e = fast_attr<0, kSymHashTiny, 8>();
    if (e == cudaSuccess) e = fast_attr<1, kSymHashTiny, 8>();
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, levelk_fast<0, kSymHashTiny, 8>, kSymThreads,
                                                         sym_smem_bytes(hb));
  }
  e = hb == kSymHashSmall ? fast_attr<0, kSymHashSmall, 32>() : fast_attr<0, kSymHashLarge, 32>();
  if (e == cudaSuccess) e = hb == kSymHashSmall ? fast_attr<1, kSymHashSmall, 32>() : fast_attr<1, kSymHashLarge, 32>();
  if (e != cudaSuccess) return e;
  return hb == kSymHashSmall
             ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, levelk_fast<0, kSymHashSmall, 32>,
                                                             kSymThreads, sym_smem_bytes(hb))
             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, levelk_fast<0, kSymHashLarge, 32>,
                                                             kSymThreads, sym_smem_bytes(hb));
}

cudaError_t launch_levelk_fast(const SymParams& p, int pass, int hb, int grid, cudaStream_t st) {
  const size_t sm = sym_smem_bytes(hb);
  if (hb == kSymHashTiny) {
    if (pass == 0) levelk_fast<0, kSymHashTiny, 8><<<grid, kSymThreads, sm, st>>>(p);
    else levelk_fast<1, kSymHashTiny, 8><<<grid, kSymThreads, sm, st>>>(p);
  } else if (hb == kSymHashSmall) {
    if (pass == 0) levelk_fast<0, kSymHashSmall, 32><<<grid, kSymThreads, sm, st>>>(p);
    else levelk_fast<1, kSymHashSmall, 32><<<grid, kSymThreads, sm, st>>>(p);
  } else {
    if (pass == 0) levelk_fast<0, kSymHashLarge, 32><<<grid, kSymThreads, sm, st>>>(p);
    else levelk_fast<1, kSymHashLarge, 32><<<grid, kSymThreads, sm, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_levelk_slow(const SymParams& p, int pass, int grid, cudaStream_t st) {
  if (pass == 0) levelk_slow<0><<<grid, kSymThreads, 0, st>>>(p);
  else levelk_slow<1><<<grid, kSymThreads, 0, st>>>(p);
  return cudaGetLastError();
}

// row_ptr = exclusive scan of the n + 1 counts (count[n] = 0)
cudaError_t sym_scan(const long long* count, long long* u_ptr, int n, void* temp, size_t* temp_bytes,
                     cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, count, u_ptr, n + 1, st);
}

}  // namespace tcbdev
