// Host-callable launch helpers of factor_kernel.cu and row_kernel.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "factor_kernel.cuh"

namespace tcbdev {

size_t factor_smem_bytes(int threads, int cap, int flag_words, int icap, int scap);
cudaError_t factor_occupancy(int threads, size_t smem, int* ctas_per_sm);
cudaError_t launch_prepare(const PrepParams& q, cudaStream_t st);
cudaError_t launch_factor(const Params& p, int grid, int threads, size_t smem, cudaStream_t st);

cudaError_t rows_occupancy(int threads, int minb, bool prof, int* ctas_per_sm);
cudaError_t launch_rows(const RowParams& p, int grid, int threads, int minb, cudaStream_t st);

cudaError_t static_occupancy(int threads, int group, int* ctas_per_sm);
cudaError_t launch_static(const StaticParams& p, int grid, int threads, int group, cudaStream_t st);

cudaError_t flow_occupancy(int threads, int kb, int minb, int g, int weak, int dyn, int remote,
                           int* ctas_per_sm);
cudaError_t launch_flow_prepare(const FlowPrepParams& q, int sm_count, cudaStream_t st);
cudaError_t launch_flow(const FlowParams& p, int grid, int threads, int kb, int minb, int g,
                        int weak, int dyn, int remote, cudaStream_t st);

cudaError_t pipe_occupancy(int threads, int kb, int minb, int remote, int extras, int* ctas_per_sm,
                           int drain = 0);
cudaError_t launch_flow_pipe(const FlowParams& p, int grid, int threads, int kb, int minb, int remote,
                             int extras, cudaStream_t st, int drain = 0);
cudaError_t launch_init_values(const double* a, const int* map, double* vals, double* vals0, long long nnz,
                               long long nnz_a, int nbatch, int sm_count, cudaStream_t st);
cudaError_t unit_occupancy(int threads, int kb, int minb, int weak, size_t smem, int* ctas_per_sm);
cudaError_t launch_units(const FlowParams& p, const UnitParams& u, int grid, int threads, int kb, int minb,
                         int weak, size_t smem, cudaStream_t st);

}  // namespace tcbdev
