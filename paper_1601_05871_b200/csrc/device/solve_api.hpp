// Host-callable launch helpers of solve_kernel.cu (triangular solves with U).
#pragma once

#include <cuda_runtime.h>

namespace tcbdev {

constexpr int kSolveThreads = 256;

struct SolveParams {
  int pos_begin, pos_end;      // schedule positions of this launch
  const int4* rec;             // per position {ent_begin, len | backward << 31, diag position, row}
  const int* idx;              // per entry: operand row (forward entries, then backward)
  const double* fval;          // forward entries' values U(i,j), gathered per apply (solve_gather)
  const double* u;             // the factor (backward entries: its own rows, after the diagonal)
  const double* b;             // right-hand side (forward), or the backward input when !poll_y
  double* y;                   // forward output (marker until written)
  double* x;                   // backward output (marker until written)
  int poll_y;                  // backward reads y as the forward rows write it
  int* error;
  unsigned long long timeout_ns;
  unsigned long long* trace;   // optional: per position {start, operands final, end} (globaltimer)
};

cudaError_t solve_occupancy(int* ctas_per_sm);
// y = A x for a CSR matrix (row_ptr int64, col int32, fp64), products summed in
// column order (one thread per row)
cudaError_t launch_spmv(int n, const long long* ptr, const int* col, const double* val, const double* x,
                        double* y, int sm_count, cudaStream_t st);
// fval[e] = u[pos[e]] for the forward entries (the factor in transposed order)
cudaError_t launch_solve_gather(const double* u, const int* pos, double* fval, long long n, int sm_count,
                                cudaStream_t st);
cudaError_t launch_trisolve(const SolveParams& p, int grid, cudaStream_t st);
// conjugate-gradient vector updates (cooperative, deterministic dots); state = {rz, live, thr}
cudaError_t cg_grid(int sm_count, int* grid);
cudaError_t launch_cg_step(int n, double* x, double* r, const double* p, const double* ap, double* state,
                           double* hist, int it, double* partial, int grid, cudaStream_t st);
cudaError_t launch_cg_direction(int n, const double* r, const double* z, double* p, double* state, double* partial,
                                int grid, cudaStream_t st);

}  // namespace tcbdev
