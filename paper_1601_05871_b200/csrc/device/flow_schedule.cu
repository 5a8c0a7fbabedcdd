// The value-flow schedule built on the device at upload (the host version is
// flow_plan_schedule, csrc/host/flow_plan.cpp; the two are equal record for
// record, tests/test_gpu_parity.py).
//
// Dependences of unit g (row t, last column c1(g)): for every source r of t
// (an entry U(r,t) at position q), the units of row r from the one holding q
// on, up to the last one starting at a column <= c1(g); a chunk also reads its
// row's Chol unit. Every dependence points to a lower row or to the row's own
// Chol unit, so the natural row order is topological and its reverse is for
// the dependents.
//
//   levels   Kahn's algorithm over the rows, frontier by frontier (a grid
//            barrier between frontiers, a warp per row): a row runs once all
//            its sources ran (U's transposed index), and a unit's level is
//            1 + the largest level among its dependences;
//   heights  the same over the reverse dependences: a row runs once every
//            row its entries feed ran, a unit's height is 1 + the largest
//            height among the units that read it;
//   order    a stable radix sort of (level, -height) over the unit ids;
//   records  {tb, L | kind << 30, U(t,t), t} per schedule position.
//
// (Dealing the rows round-robin in natural order to persistent warps that
// poll their sources' levels was 25-100x slower: a round of consecutive rows
// holds whole dependence chains, which then run hop by hop.)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "device_api.hpp"
#include "sync.cuh"

namespace tcbdev {

namespace {

namespace cg = cooperative_groups;

constexpr int kLocal = 8;  // units of a row whose maxima a lane keeps in registers

// One warp computes the levels of row t's units, its sources' levels final.
__device__ void row_levels(const SchedParams& S, int t, int lane) {
  const int g0 = __ldg(S.ufirst + t), g1 = __ldg(S.ufirst + t + 1);
  int m[kLocal];
#pragma unroll
  for (int i = 0; i < kLocal; ++i) m[i] = 0;
  for (int s = __ldg(S.col_ptr + t) + lane; s < __ldg(S.col_ptr + t + 1); s += 32) {
    const int r = __ldg(S.col_src + s), q = __ldg(S.col_pos + s);
    const int vr1 = __ldg(S.ufirst + r + 1);
    int v = __ldg(S.ufirst + r);
    while (v + 1 < vr1 && __ldg(S.u_tb + v + 1) <= q) ++v;  // the unit of row r holding q
    int lv = __ldcg(S.level + v);  // L2: written by other SMs in earlier frontiers
    auto advance = [&](int g) {
      const int c1 = __ldg(S.uc1 + g);
      while (v + 1 < vr1 && __ldg(S.uc0 + v + 1) <= c1) lv = max(lv, __ldcg(S.level + ++v));
    };
#pragma unroll
    for (int i = 0; i < kLocal; ++i)
      if (g0 + i < g1) {
        advance(g0 + i);
        m[i] = max(m[i], lv);
      }
    for (int g = g0 + kLocal; g < g1; ++g) {
      advance(g);
      atomicMax(S.acc + g, lv);
    }
  }
#pragma unroll
  for (int i = 0; i < kLocal; ++i) m[i] = __reduce_max_sync(kFull, m[i]);
  __threadfence();
  __syncwarp();
  if (lane == 0) {
    const int l0 = m[0] + 1;
    S.level[g0] = l0;
    int best = l0;
#pragma unroll
    for (int i = 1; i < kLocal; ++i)
      if (g0 + i < g1) {
        const int l = max(m[i] + 1, l0 + 1);
        S.level[g0 + i] = l;
        best = max(best, l);
      }
    for (int g = g0 + kLocal; g < g1; ++g) {
      const int l = max(atomicAdd(S.acc + g, 0) + 1, l0 + 1);
      S.level[g] = l;
      best = max(best, l);
    }
    atomicMax(S.depth, best);
  }
  __syncwarp();
}

// One warp computes the heights of row r's units, the rows its entries feed final.
__device__ void row_heights(const SchedParams& S, int r, int lane) {
  const int vr0 = __ldg(S.ufirst + r), vr1 = __ldg(S.ufirst + r + 1);
  int m[kLocal];
#pragma unroll
  for (int i = 0; i < kLocal; ++i) m[i] = 0;
  for (int q = __ldg(S.row_ptr + r) + 1 + lane; q < __ldg(S.row_ptr + r + 1); q += 32) {
    int v0 = vr0;
    while (v0 + 1 < vr1 && __ldg(S.u_tb + v0 + 1) <= q) ++v0;
    const int t = __ldg(S.cols + q);
    const int g0 = __ldg(S.ufirst + t), g1 = __ldg(S.ufirst + t + 1);
    // units v0 .. vmax(g) of row r are read by g: their height is at least h(g) + 1
    int v = v0;
    for (int g = g0; g < g1; ++g) {
      const int c1 = __ldg(S.uc1 + g);
      while (v + 1 < vr1 && __ldg(S.uc0 + v + 1) <= c1) ++v;
      const int hg = __ldcg(S.height + g) + 1;
#pragma unroll
      for (int i = 0; i < kLocal; ++i)
        if (vr0 + i >= v0 && vr0 + i <= v) m[i] = max(m[i], hg);
      for (int x = max(v0, vr0 + kLocal); x <= v; ++x) atomicMax(S.acc2 + x, hg);
    }
  }
#pragma unroll
  for (int i = 0; i < kLocal; ++i) m[i] = __reduce_max_sync(kFull, m[i]);
  __threadfence();
  __syncwarp();
  if (lane == 0) {
    int h0 = max(1, m[0]);
#pragma unroll
    for (int i = 1; i < kLocal; ++i)
      if (vr0 + i < vr1) {
        const int h = max(1, m[i]);
        S.height[vr0 + i] = h;
        h0 = max(h0, h + 1);
      }
    for (int v = vr0 + kLocal; v < vr1; ++v) {
      const int h = max(1, atomicAdd(S.acc2 + v, 0));
      S.height[v] = h;
      h0 = max(h0, h + 1);
    }
    S.height[vr0] = h0;
  }
  __syncwarp();
}

__global__ void flow_unit_columns(int nunits, const int* cols, const int* u_tb, const int* u_len, int* uc0, int* uc1) {
  const int stride = gridDim.x * blockDim.x;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nunits; g += stride) {
    uc0[g] = cols[u_tb[g]];
    uc1[g] = cols[u_tb[g] + u_len[g] - 1];
  }
}

// Kahn's algorithm frontier by frontier over the rows, both directions in
// the same rounds: the first half of the warps runs the levels (a row after
// its sources, U's transposed index), the second half the heights (a row
// after the rows its entries feed); a row joins its next frontier once its
// counter of unprocessed predecessors reaches zero, and a grid barrier
// separates the rounds. Frontier k of a direction occupies
// rows[base_k, base_k + fsize[k]) and appends frontier k+1 behind it through
// fsize[k + 1], which nobody reads before the barrier (a single shared tail
// would let a fast thread append before a slow one has read it).
struct Frontier {
  int* cnt;    // n
  int* rows;   // n
  int* fsize;  // n + 1, zeroed
};

__global__ void flow_frontiers(SchedParams S, Frontier up, Frontier down) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int t = gt; t < S.n; t += nt) {
    const int cu = __ldg(S.col_ptr + t + 1) - __ldg(S.col_ptr + t);
    const int cd = __ldg(S.row_ptr + t + 1) - __ldg(S.row_ptr + t) - 1;
    up.cnt[t] = cu;
    down.cnt[t] = cd;
    if (cu == 0) up.rows[atomicAdd(up.fsize, 1)] = t;
    if (cd == 0) down.rows[atomicAdd(down.fsize, 1)] = t;
  }
  __threadfence();
  grid.sync();
  const bool is_up = nw < 2 || gw < nw / 2;  // (one warp: it runs both, up first)
  const int w = is_up ? gw : gw - nw / 2, W = nw < 2 ? 1 : (is_up ? nw / 2 : nw - nw / 2);
  int ubase = 0, dbase = 0;
  for (int k = 0; k <= S.n; ++k) {
    const int usize = __ldcg(up.fsize + k), dsize = __ldcg(down.fsize + k);
    if (usize == 0 && dsize == 0) break;
    const int unext = ubase + usize, dnext = dbase + dsize;
    if (is_up || nw < 2) {
      for (int i = ubase + w; i < unext; i += W) {
        const int t = __ldcg(up.rows + i);
        row_levels(S, t, lane);
        for (int q = __ldg(S.row_ptr + t) + 1 + lane; q < __ldg(S.row_ptr + t + 1); q += 32) {
          const int x = __ldg(S.cols + q);
          if (atomicSub(up.cnt + x, 1) == 1) up.rows[unext + atomicAdd(up.fsize + k + 1, 1)] = x;
        }
      }
    }
    if (!is_up || nw < 2) {
      for (int i = dbase + w; i < dnext; i += W) {
        const int r = __ldcg(down.rows + i);
        row_heights(S, r, lane);
        for (int j = __ldg(S.col_ptr + r) + lane; j < __ldg(S.col_ptr + r + 1); j += 32) {
          const int x = __ldg(S.col_src + j);
          if (atomicSub(down.cnt + x, 1) == 1) down.rows[dnext + atomicAdd(down.fsize + k + 1, 1)] = x;
        }
      }
    }
    __threadfence();
    grid.sync();
    ubase = unext;
    dbase = dnext;
  }
}

// ascending level, descending height; the unit ids as values (a stable sort keeps them ascending)
// (slack_pct: a unit is placed slack_pct % of the way from its earliest level to its latest,
// depth + 1 - height; still a topological key: both ends grow by at least 1 along a dependence)
__global__ void flow_order_keys(int nunits, const int* level, const int* height, const int* depth, int slack_pct,
                                unsigned long long* key, int* id) {
  const int stride = gridDim.x * blockDim.x;
  const int dp = *depth;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nunits; g += stride) {
    const int slack = dp + 1 - height[g] - level[g];
    const int place = level[g] + static_cast<int>(static_cast<long long>(slack_pct) * slack / 100);
    key[g] = (static_cast<unsigned long long>(place) << 32) | static_cast<unsigned>(0x7fffffff - height[g]);
    id[g] = g;
  }
}

__global__ void flow_records(int nunits, const int* order, const int* ufirst, const int* u_tb, const int* u_len,
                             const int* u_row, const int* row_ptr, int4* rec, int* item) {
  const int stride = gridDim.x * blockDim.x;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nunits; q += stride) {
    const int g = order[q], t = u_row[g];
    rec[q] = make_int4(u_tb[g], u_len[g] | ((g == ufirst[t] ? 0 : 1) << 30), row_ptr[t], t);
    item[q] = g;
  }
}

}  // namespace

// Scratch: 6 * nunits ints + 2 * nunits 64-bit keys + the sort's temporary
// storage (temp = nullptr: its size in *temp_bytes). ufirst/u_tb/u_len/u_row
// and the transposed index are device arrays; rec/item are the outputs.
cudaError_t flow_schedule(SchedParams S, const int* u_row, int4* rec, int* item, unsigned long long* keys,
                          unsigned long long* keys_sorted, int* ids, int* order, void* temp, size_t* temp_bytes,
                          int sm_count, cudaStream_t st) {
  if (!temp)
    return cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, keys, keys_sorted, ids, order,
                                           S.nunits > 0 ? S.nunits : 1, 0, 64, st);
  if (S.nunits == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(S.level, 0, sizeof(int) * S.nunits, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.height, 0, sizeof(int) * S.nunits, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.acc, 0, sizeof(int) * S.nunits, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.acc2, 0, sizeof(int) * S.nunits, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.depth, 0, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.error, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  {
    const int blocks = max(1, min((S.nunits + 255) / 256, 8 * sm_count));
    flow_unit_columns<<<blocks, 256, 0, st>>>(S.nunits, S.cols, S.u_tb, S.u_len, S.uc0, S.uc1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // the two frontiers' rows and counters (n ints each) live in the sort's key buffers until the
  // sort, their sizes (n + 1 ints each) in `ids` and `order`
  Frontier up{reinterpret_cast<int*>(keys), reinterpret_cast<int*>(keys) + S.n, ids};
  Frontier down{reinterpret_cast<int*>(keys_sorted), reinterpret_cast<int*>(keys_sorted) + S.n, order};
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, flow_frontiers, 256, 0);
  if (e == cudaSuccess) e = cudaMemsetAsync(up.fsize, 0, sizeof(int) * (S.n + 1), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(down.fsize, 0, sizeof(int) * (S.n + 1), st);
  if (e != cudaSuccess) return e;
  // Long rows (C3: 69 entries) make narrow frontiers of heavy rows: a round is
  // the rows' chains of dependent index loads plus the grid barrier, and one
  // CTA per SM has warps enough while its barrier is the cheapest (B200, C3:
  // 25.6 -> 19.5 ms). Short rows make wide frontiers that want every warp
  // (C6: 7.5 ms at full occupancy, 23.3 at one CTA per SM).
  if (S.nnz >= 48LL * S.n) occ = 1;
  if (const char* ev = std::getenv("TCG_SCHED_CTAS")) occ = max(1, min(occ, std::atoi(ev)));
  void* args[] = {&S, &up, &down};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&flow_frontiers), max(1, occ) * sm_count, 256, args,
                                  0, st);
  if (e != cudaSuccess) return e;
  const int blocks = max(1, min((S.nunits + 255) / 256, 8 * sm_count));
  flow_order_keys<<<blocks, 256, 0, st>>>(S.nunits, S.level, S.height, S.depth, S.slack_pct, keys, ids);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, keys, keys_sorted, ids, order, S.nunits, 0, 64, st);
  if (e != cudaSuccess) return e;
  flow_records<<<blocks, 256, 0, st>>>(S.nunits, order, S.ufirst, S.u_tb, S.u_len, u_row, S.row_ptr, rec, item);
  return cudaGetLastError();
}

}  // namespace tcbdev
