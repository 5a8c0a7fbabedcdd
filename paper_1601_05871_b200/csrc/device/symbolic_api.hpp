// Host-callable launch helpers of symbolic_kernel.cu (level-k fill pattern).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace tcbdev {

constexpr int kSymThreads = 256;              // 8 warps, one source row each
constexpr int kSymHashTiny = 7;               // tier 1 for small searches: 8 lanes per row, 128 slots (96 keys)
constexpr int kSymHashSmall = 9;              // tier 1: 512-slot seen-sets (384 keys)
constexpr int kSymHashLarge = 11;             // tier 2: 2,048 slots (1,536 keys); then global memory

struct SymParams {
  int n;
  int kk;                    // min(max(k, 0), n): interior steps
  const long long* a_ptr;    // PᵀAP pattern (row_ptr int64, col_idx int32)
  const int* a_col;
  long long* count;          // n + 1 row lengths (count pass); count[n] = 0
  const long long* u_ptr;    // n + 1 (fill pass)
  int* u_col;                // fill pass
  const int* list;           // rows of this tier (nullptr: all rows)
  const int* nlist;
  int* over;                 // rows this tier hands to the next
  int* nover;
  int* slow_mark;            // slow path: per slot n stamps
  int* slow_front;           // slow path: per slot 2 n frontier entries
  // single pass: the count pass also writes each row ({i} then its targets,
  // sorted) into scratch at a reserved offset; a copy kernel moves the rows
  // into place after the scan. Rows that found no room (-1) are searched again.
  int* scratch;
  long long scratch_cap;
  unsigned long long* cursor;
  long long* soff;           // per row: its offset in scratch, or -1
};

size_t sym_smem_bytes(int hb);
cudaError_t sym_occupancy(int hb, int* ctas_per_sm);
cudaError_t launch_levelk_fast(const SymParams& p, int pass, int hb, int grid, cudaStream_t st);
cudaError_t launch_levelk_slow(const SymParams& p, int pass, int grid, cudaStream_t st);
cudaError_t launch_levelk_copy(const SymParams& p, int grid, bool long_rows, cudaStream_t st);
cudaError_t sym_scan(const long long* count, long long* u_ptr, int n, void* temp, size_t* temp_bytes,
                     cudaStream_t st);

}  // namespace tcbdev
