/*
 * CPU oracle for the IC(k) Cholesky-by-blocks hot path — TEST INFRASTRUCTURE.
 *
 * A plain-C restatement of the reference algorithm (arXiv 1601.05871
 * re-implementation `taskchol`, /root/reference/proj/include/taskchol). Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as the checker. The product path never links it.
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref, compiled from the reference headers in the dev container):
 * tests/golden/ JSON files hold reference-generated hashes for every
 * configuration, checked by tests/test_oracle.py.
 */
#ifndef TACHO_ORACLE_H_
#define TACHO_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FNV-style hash used by the survey: h = (h ^ bits(x)) * 1099511628211,
 * h0 = 1469598103934665603, over 64-bit words (ints sign-extended). */
uint64_t orc_hash_f64(const double* x, int64_t n);
uint64_t orc_hash_i32(const int32_t* x, int64_t n);
uint64_t orc_hash_i64(const int64_t* x, int64_t n);

/* factorize.hpp:71-89 */
void orc_init_factor_values(int32_t n, const int64_t* a_ptr, const int32_t* a_col,
                            const double* a_val, const int64_t* u_ptr, const int32_t* u_col,
                            double* u_val);

/* factorize.hpp:94-130. Returns 0, 1 (breakdown; row and pivot set) or 2
 * (missing diagonal). Values are factored in place. */
int orc_factor_serial(int32_t n, const int64_t* u_ptr, const int32_t* u_col, double* u_val,
                      int32_t* row, double* pivot);

/* Static task DAG of factor_by_blocks (factorize.hpp:260-302 over
 * block_layout.hpp:98-181). Pass NULL arrays to query the counts first. */
int orc_export_dag(int32_t n, const int64_t* u_ptr, const int32_t* u_col, int32_t nranges,
                   const int32_t* bounds, int64_t* nnodes, int64_t* nedges, int32_t* kind,
                   int32_t* bi, int32_t* bj, int32_t* efrom, int32_t* eto);

/* Sequential by-blocks execution with the four block kernels restated from
 * kernels.hpp:40-132, tasks run in generation order. Same return codes as
 * orc_factor_serial. */
int orc_factor_by_blocks(int32_t n, const int64_t* u_ptr, const int32_t* u_col, double* u_val,
                         int32_t nranges, const int32_t* bounds, int32_t* row, double* pivot);

/* max over (i,j) in the pattern, i <= j, of |(UᵀU)_ij - A_ij| / max|A|. */
double orc_pattern_residual(int32_t n, const int64_t* a_ptr, const int32_t* a_col,
                            const double* a_val, const int64_t* u_ptr, const int32_t* u_col,
                            const double* u_val);

/* Triangular solves with the factor U (the
 * preconditioner apply; a non-goal of the reference, so this
 * restatement fixes the order): which & 1 -> forward Uᵀ y = b, row-oriented
 * push over U's rows (t_j -= U(i,j) * y_i for i ascending, y_i = t_i / U(i,i));
 * which & 2 -> backward U x = y (x_i = (y_i - sum_j U(i,j) x_j) / U(i,i), j
 * ascending along row i, i descending). `b` and `x` may alias. Returns 0, or 2
 * for a missing/zero diagonal. */
int orc_trisolve(int32_t n, const int64_t* u_ptr, const int32_t* u_col, const double* u_val,
                 const double* b, int32_t which, double* x);

/* Dense level-k DP (symbolic.hpp:124-167); fills a row-major n*n 0/1 mask of
 * the upper pattern. Small n only. */
void orc_levelk_dense(int32_t n, const int64_t* a_ptr, const int32_t* a_col, int32_t k,
                      uint8_t* mask);

#ifdef __cplusplus
}
#endif
#endif
