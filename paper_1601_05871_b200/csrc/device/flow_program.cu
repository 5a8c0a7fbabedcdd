// Device-built update programs of the value-flow schedule.
//
// Every coordinate (t, c) of U receives, in ascending source row r, the
// products U(r,t) * U(r,c) over the rows r < t holding both entries -- the
// reference's pattern-restricted merges (kernels.hpp:55-65 chol, :85-89 trsm,
// :104-108 herk, :125-129 gemm) folded per coordinate, the order that makes
// the result bitwise equal to factor_serial (factorize.hpp:94-130). A program
// is the list of (m, o) position pairs of those products; slot[x] =
// {u_b, u_e, m0, o0} with the first pair inline.
//
// One warp per matrix row t (rows handed out by an atomic counter): the
// row's columns are staged in shared memory; for each source r (the
// transposed index, ascending) the lanes walk row r from U(r,t) on, 32
// entries at a time, and binary-search each column among row t's; a hit is
// a product of that coordinate. Sources run one after the other, so the
// fill pass appends each coordinate's products in ascending r. Pass 1
// counts, a device scan turns counts into offsets, pass 2 fills. Integer
// work only: the programs are bit-exact by construction, and equal to the
// host flattener's (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <climits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "factor_kernel.cuh"
#include "sync.cuh"

namespace tcbdev {

namespace {

constexpr int kProgThreads = 256;
constexpr int kProgWarps = kProgThreads / 32;
constexpr int kChunk = 256;  // row-t columns staged per warp and pass

// first index in s[0, n) holding a value >= x (n <= kChunk)
__device__ __forceinline__ int lower_bound_smem(const int* s, int n, int x) {
  int lo = 0, len = n;
  while (len > 0) {
    const int half = len >> 1;
    if (s[lo + half] < x) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

// first position in cols[b, e) holding a value >= x (global, sorted)
__device__ __forceinline__ int lower_bound_global(const int* cols, int b, int e, int x) {
  while (b < e) {
    const int mid = b + ((e - b) >> 1);
    if (__ldg(cols + mid) < x) b = mid + 1;
    else e = mid;
  }
  return b;
}

template <int FILL>
__global__ void __launch_bounds__(kProgThreads) flow_program(ProgParams P) {
  struct Smem {
    int col[kChunk];
    int cnt[kChunk];
    int ub[kChunk];
    int2 first[kChunk];
  };
  __shared__ Smem sm_all[kProgWarps];
  Smem& S = sm_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(P.next_row + FILL, 1);
    t = __shfl_sync(kFull, t, 0);
    if (t >= P.n) break;
    const int rb = __ldg(P.row_ptr + t), re = __ldg(P.row_ptr + t + 1);
    const int sb = __ldg(P.col_ptr + t), se = __ldg(P.col_ptr + t + 1);
    for (int j0 = rb; j0 < re; j0 += kChunk) {
      const int nl = min(kChunk, re - j0);
      for (int k = lane; k < nl; k += 32) {
        S.col[k] = __ldg(P.cols + j0 + k);
        S.cnt[k] = 0;
        if (FILL) {
          S.ub[k] = P.ub[j0 + k];
          S.first[k] = make_int2(0, 0);
        }
      }
      __syncwarp();
      const int cmin = S.col[0], cmax = S.col[nl - 1];
      for (int s = sb; s < se; ++s) {
        const int r = __ldg(P.col_src + s), m = __ldg(P.col_pos + s);
        const int rend = __ldg(P.row_ptr + r + 1);
        // row r's entries from column cmin on (U(r,t) itself for the first chunk)
        const int start = j0 == rb ? m : lower_bound_global(P.cols, m, rend, cmin);
        for (int q0 = start; q0 < rend; q0 += 32) {
          const int q = q0 + lane;
          const int c = q < rend ? __ldg(P.cols + q) : INT_MAX;
          if (c <= cmax) {
            const int j = lower_bound_smem(S.col, nl, c);
            if (S.col[j] == c) {  // (t, c) is in the pattern: a product of coordinate j
              if (FILL) {
                const int k = S.cnt[j];
                const int2 mo = make_int2(m, q);
                P.upd[S.ub[j] + k] = mo;
                if (k == 0) S.first[j] = mo;
              }
              S.cnt[j] += 1;  // one hit per coordinate per source: no race
            }
          }
          if (__any_sync(kFull, c > cmax)) break;  // past the chunk's last column
        }
        __syncwarp();
      }
      for (int k = lane; k < nl; k += 32) {
        if (FILL) {
          const int2 f = S.first[k];
          P.slot[j0 + k] = make_int4(S.ub[k], S.ub[k] + S.cnt[k], f.x, f.y);
        } else {
          P.count[j0 + k] = S.cnt[k];
        }
      }
      __syncwarp();
    }
  }
}

// Transposed index of U's strict upper part: key = column (n for the
// diagonal, which sorts last), value = position; a stable radix sort by key
// leaves every column's entries in ascending row.
__global__ void flow_transpose_keys(int n, const int* row_ptr, const int* cols, int* key, int* pos, int* rowid) {
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
    const int rb = row_ptr[t], re = row_ptr[t + 1];
    for (int q = rb; q < re; ++q) {
      key[q] = q == rb ? n : __ldg(cols + q);
      pos[q] = q;
      rowid[q] = t;
    }
  }
}

// col_ptr[t] = first sorted entry of column t; col_src = the entries' rows
__global__ void flow_transpose_index(int n, int nsrc, const int* key_s, const int* pos_s, const int* rowid,
                                     int* col_ptr, int* col_src) {
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += stride) {
    int lo = 0, hi = nsrc;
    while (lo < hi) {
      const int mid = lo + ((hi - lo) >> 1);
      if (key_s[mid] < t) lo = mid + 1;
      else hi = mid;
    }
    col_ptr[t] = t == n ? nsrc : lo;
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nsrc; k += stride) col_src[k] = rowid[pos_s[k]];
}

// A part of a sharded run: in the programs of the part's coordinates, both
// operands of a product whose source row another part owns (they lie in the
// same row) become kRemoteBit | owner << 25 | position (factor_flow<...,
// REMOTE> reads them from the owner's U through the peer table).
__global__ void flow_program_remote(long long nnz, const int* rowid, const int* owner, int part, int4* slot,
                                    int2* upd) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < nnz; x += stride) {
    if (owner[rowid[x]] != part) continue;
    int4 s = slot[x];
    for (int e = s.x; e < s.y; ++e) {
      const int2 mo = upd[e];
      const int ow = owner[rowid[mo.x]];
      if (ow != part) {
        const int tag = static_cast<int>(0x80000000u | (static_cast<unsigned>(ow) << 25));
        upd[e] = make_int2(tag | mo.x, tag | mo.y);
      }
    }
    if (s.x < s.y) {
      const int2 f = upd[s.x];
      s.z = f.x;
      s.w = f.y;
      slot[x] = s;
    }
  }
}

// total = ub[nnz-1] + count[nnz-1] (64-bit scan), narrowed offsets
__global__ void flow_program_offsets(const long long* ub64, const int* count, int* ub32, long long nnz,
                                     long long* total) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < nnz; x += stride)
    ub32[x] = static_cast<int>(ub64[x]);  // checked against 2^31 by the host before the fill
  if (blockIdx.x == 0 && threadIdx.x == 0) *total = nnz > 0 ? ub64[nnz - 1] + count[nnz - 1] : 0;
}

}  // namespace

cudaError_t flow_program_count(const ProgParams& p, int sm_count, cudaStream_t st) {
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, flow_program<0>, kProgThreads, 0);
  if (e != cudaSuccess) return e;
  flow_program<0><<<max(1, occ) * sm_count, kProgThreads, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t flow_program_fill(const ProgParams& p, int sm_count, cudaStream_t st) {
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, flow_program<1>, kProgThreads, 0);
  if (e != cudaSuccess) return e;
  flow_program<1><<<max(1, occ) * sm_count, kProgThreads, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t flow_program_remote_rewrite(long long nnz, const int* rowid, const int* owner, int part, int4* slot,
                                        int2* upd, int sm_count, cudaStream_t st) {
  long long blocks = (nnz + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 8LL * sm_count ? 8LL * sm_count : blocks);
  flow_program_remote<<<static_cast<int>(blocks), 256, 0, st>>>(nnz, rowid, owner, part, slot, upd);
  return cudaGetLastError();
}

// U's transposed index on the device (scratch: key, pos, rowid, key_s of nnz
// ints; out: pos_s = col_pos (nnz), col_src (nnz - n), col_ptr (n + 1));
// temp = nullptr returns the sort's scratch size
cudaError_t flow_transpose(int n, int nnz, const int* row_ptr, const int* cols, int* key, int* pos, int* rowid,
                           int* key_s, int* pos_s, int* col_ptr, int* col_src, void* temp, size_t* temp_bytes,
                           int sm_count, cudaStream_t st) {
  int bits = 1;
  while ((1LL << bits) <= n) ++bits;
  if (!temp)
    return cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, key, key_s, pos, pos_s, nnz > 0 ? nnz : 1, 0, bits, st);
  const int blocks = max(1, min((n + 255) / 256, 8 * sm_count));
  flow_transpose_keys<<<blocks, 256, 0, st>>>(n, row_ptr, cols, key, pos, rowid);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, key, key_s, pos, pos_s, nnz, 0, bits, st);
  if (e != cudaSuccess) return e;
  const int nsrc = nnz - n;
  const int b2 = max(1, min((max(nsrc, n + 1) + 255) / 256, 8 * sm_count));
  flow_transpose_index<<<b2, 256, 0, st>>>(n, nsrc, key_s, pos_s, rowid, col_ptr, col_src);
  return cudaGetLastError();
}

// exclusive scan of the counts into 64-bit offsets (temp: CUB scratch; call
// with temp = nullptr for its size), then the 32-bit copy and the total
cudaError_t flow_program_scan(const int* count, long long* ub64, int* ub32, long long nnz, long long* total,
                              void* temp, size_t* temp_bytes, int sm_count, cudaStream_t st) {
  if (!temp)
    return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, count, ub64, static_cast<int>(nnz > 0 ? nnz : 1), st);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, count, ub64, static_cast<int>(nnz), st);
  if (e != cudaSuccess) return e;
  long long blocks = (nnz + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 4LL * sm_count ? 4LL * sm_count : blocks);
  flow_program_offsets<<<static_cast<int>(blocks), 256, 0, st>>>(ub64, count, ub32, nnz, total);
  return cudaGetLastError();
}

}  // namespace tcbdev
