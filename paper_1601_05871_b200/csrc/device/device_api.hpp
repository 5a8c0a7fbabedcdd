// Host-callable launch helpers of factor_kernel.cu, flow_kernel.cu and flow_program.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "factor_kernel.cuh"

namespace tcbdev {

size_t factor_smem_bytes(int threads, int cap, int flag_words, int icap, int scap);
cudaError_t factor_occupancy(int threads, size_t smem, int* ctas_per_sm);
cudaError_t launch_prepare(const PrepParams& q, cudaStream_t st);
cudaError_t launch_factor(const Params& p, int grid, int threads, size_t smem, cudaStream_t st);



cudaError_t launch_flow_prepare(const FlowPrepParams& q, int sm_count, cudaStream_t st);
// chunked download: chunk starts (first unit start at or after k * nnz / nchunks) and units per chunk
cudaError_t launch_chunk_setup(const int4* rec, int nrows, long long nnz, int nchunks, int* start, int* units,
                               int sm_count, cudaStream_t st);

// whether that exact variant is compiled in (pipe_occupancy / launch_flow_pipe fall back to the
// variant without a back-off when the requested back-off has none)
bool pipe_variant_exists(int threads, int kb, int minb, int remote, int extras, int drain, int backoff_ns);
cudaError_t pipe_occupancy(int threads, int kb, int minb, int remote, int extras, int* ctas_per_sm,
                           int drain = 0, int backoff_ns = 0);
cudaError_t launch_flow_pipe(const FlowParams& p, int grid, int threads, int kb, int minb, int remote,
                             int extras, cudaStream_t st, int drain = 0, int backoff_ns = 0);
// product-parallel rows (flow_pp_kernel.cu): WPR warps per row group, KP products per thread and chunk
cudaError_t pp_occupancy(int wpr, int kp, int nb, int minb, int extras, int drain, int bo, int d,
                         int* ctas_per_sm, size_t* smem);
cudaError_t launch_flow_pp(const FlowParams& p, int grid, int wpr, int kp, int nb, int minb, int extras, int drain,
                           int bo, int d, cudaStream_t st);
cudaError_t launch_init_values(const double* a, const int* map, double* vals, double* vals0, long long nnz,
                               long long nnz_a, int nbatch, int sm_count, cudaStream_t st);

cudaError_t flow_transpose(int n, int nnz, const int* row_ptr, const int* cols, int* key, int* pos, int* rowid,
                           int* key_s, int* pos_s, int* col_ptr, int* col_src, void* temp, size_t* temp_bytes,
                           int sm_count, cudaStream_t st);
// the value-flow schedule on the device (flow_schedule.cu): levels, heights, order, records
cudaError_t flow_schedule(SchedParams S, const int* u_row, int4* rec, int* item, unsigned long long* keys,
                          unsigned long long* keys_sorted, int* ids, int* order, void* temp, size_t* temp_bytes,
                          int sm_count, cudaStream_t st);
cudaError_t flow_program_remote_rewrite(long long nnz, const int* rowid, const int* owner, int part, int4* slot,
                                        int2* upd, int sm_count, cudaStream_t st);
cudaError_t flow_program_count(const ProgParams& p, int sm_count, cudaStream_t st);
cudaError_t flow_program_fill(const ProgParams& p, int sm_count, cudaStream_t st);
cudaError_t flow_program_scan(const int* count, long long* ub64, int* ub32, long long nnz, long long* total,
                              void* temp, size_t* temp_bytes, int sm_count, cudaStream_t st);

}  // namespace tcbdev
