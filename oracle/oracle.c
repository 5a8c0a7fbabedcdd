/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY) — plain-C restatement of the
 * reference's numeric IC(k) path. See oracle.h for the rules of use.
 * Build flags follow the reference's canonical build: -O2, no -march, and
 * -ffp-contract=off so that `t -= a*b` is never fused.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define H0 1469598103934665603ULL
#define HP 1099511628211ULL

uint64_t orc_hash_f64(const double* x, int64_t n) {
  uint64_t h = H0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t b;
    memcpy(&b, &x[i], 8);
    h = (h ^ b) * HP;
  }
  return h;
}
uint64_t orc_hash_i32(const int32_t* x, int64_t n) {
  uint64_t h = H0;
  for (int64_t i = 0; i < n; ++i) h = (h ^ (uint64_t)(int64_t)x[i]) * HP;
  return h;
}
uint64_t orc_hash_i64(const int64_t* x, int64_t n) {
  uint64_t h = H0;
  for (int64_t i = 0; i < n; ++i) h = (h ^ (uint64_t)x[i]) * HP;
  return h;
}

/* reference factorize.hpp:71-89: zero U, then add triu(A) by a row merge */
void orc_init_factor_values(int32_t n, const int64_t* ap, const int32_t* ac, const double* av,
                            const int64_t* up, const int32_t* uc, double* uv) {
  for (int64_t q = 0; q < up[n]; ++q) uv[q] = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t t = up[i];
    const int64_t te = up[i + 1];
    for (int64_t q = ap[i]; q < ap[i + 1]; ++q) {
      const int32_t c = ac[q];
      if (c < i) continue;
      while (t < te && uc[t] < c) ++t;
      if (t < te && uc[t] == c) uv[t] += av[q];
    }
  }
}

/* reference factorize.hpp:94-130: right-looking scalar IC on the pattern */
int orc_factor_serial(int32_t n, const int64_t* up, const int32_t* uc, double* uv, int32_t* row,
                      double* pivot) {
  for (int32_t r = 0; r < n; ++r) {
    const int64_t rb = up[r], re = up[r + 1];
    if (rb == re || uc[rb] != r) return 2;
    const double piv = uv[rb];
    if (!(piv > 0.0)) {
      if (row) *row = r;
      if (pivot) *pivot = piv;
      return 1;
    }
    const double d = sqrt(piv);
    uv[rb] = d;
    for (int64_t q = rb + 1; q < re; ++q) uv[q] /= d;
    for (int64_t q1 = rb + 1; q1 < re; ++q1) {
      const int32_t c1 = uc[q1];
      const double v1 = uv[q1];
      int64_t t = up[c1];
      const int64_t te = up[c1 + 1];
      for (int64_t q2 = q1; q2 < re; ++q2) {
        const int32_t c2 = uc[q2];
        while (t < te && uc[t] < c2) ++t;
        if (t < te && uc[t] == c2) uv[t] -= v1 * uv[q2];
      }
    }
  }
  return 0;
}

/* ---- 2D block layout (reference block_layout.hpp:98-181) ---------------- */

typedef struct {
  int32_t m;
  int64_t nblk;
  int64_t* brow; /* m + 1 */
  int32_t* bcol; /* nblk */
  int64_t* soff; /* nblk + 1: first (block,row) span slot */
  int64_t* sb;   /* span begin per (block, local row) */
  int64_t* se;
  const int32_t* bounds;
} Blocks;

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static int64_t find_block(const Blocks* B, int32_t i, int32_t j) {
  int64_t lo = B->brow[i], hi = B->brow[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (B->bcol[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return (lo < B->brow[i + 1] && B->bcol[lo] == j) ? lo : -1;
}

static int build_blocks(int32_t n, const int64_t* up, const int32_t* uc, int32_t m,
                        const int32_t* bounds, Blocks* B) {
  memset(B, 0, sizeof(*B));
  if (m < 0 || (m == 0 && n != 0) || (m > 0 && (bounds[0] != 0 || bounds[m] != n))) return 2;
  for (int32_t r = 0; r < m; ++r)
    if (bounds[r + 1] <= bounds[r]) return 2;
  B->m = m;
  B->bounds = bounds;
  int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  for (int32_t r = 0; r < m; ++r)
    for (int32_t c = bounds[r]; c < bounds[r + 1]; ++c) owner[c] = r;
  /* pass 1: block columns present per block row */
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (m + 1));
  for (int32_t r = 0; r < m; ++r) mark[r] = -1;
  int64_t cap = 16, cnt = 0;
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * cap);
  B->brow = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  for (int32_t bi = 0; bi < m; ++bi) {
    const int64_t start = cnt;
    for (int32_t i = bounds[bi]; i < bounds[bi + 1]; ++i)
      for (int64_t q = up[i]; q < up[i + 1]; ++q) {
        const int32_t bj = owner[uc[q]];
        if (mark[bj] == bi) continue;
        mark[bj] = bi;
        if (cnt == cap) {
          cap *= 2;
          cols = (int32_t*)realloc(cols, sizeof(int32_t) * cap);
        }
        cols[cnt++] = bj;
      }
    qsort(cols + start, (size_t)(cnt - start), sizeof(int32_t), cmp_i32);
    B->brow[bi + 1] = cnt;
  }
  B->nblk = cnt;
  B->bcol = cols;
  B->soff = (int64_t*)calloc((size_t)cnt + 1, sizeof(int64_t));
  for (int32_t bi = 0; bi < m; ++bi)
    for (int64_t q = B->brow[bi]; q < B->brow[bi + 1]; ++q)
      B->soff[q + 1] = B->soff[q] + (bounds[bi + 1] - bounds[bi]);
  B->sb = (int64_t*)malloc(sizeof(int64_t) * (B->soff[cnt] + 1));
  B->se = (int64_t*)malloc(sizeof(int64_t) * (B->soff[cnt] + 1));
  /* empty slices are anchored at the row start (block_layout.hpp:167-179) */
  for (int32_t bi = 0; bi < m; ++bi)
    for (int64_t q = B->brow[bi]; q < B->brow[bi + 1]; ++q)
      for (int32_t r = 0; r < bounds[bi + 1] - bounds[bi]; ++r)
        B->sb[B->soff[q] + r] = B->se[B->soff[q] + r] = up[bounds[bi] + r];
  /* pass 2: cut each row at range borders */
  for (int32_t i = 0; i < n; ++i) {
    const int32_t bi = owner[i];
    int64_t q = up[i];
    while (q < up[i + 1]) {
      const int32_t bj = owner[uc[q]];
      const int64_t s = q;
      while (q < up[i + 1] && uc[q] < bounds[bj + 1]) ++q;
      const int64_t blk = find_block(B, bi, bj);
      B->sb[B->soff[blk] + (i - bounds[bi])] = s;
      B->se[B->soff[blk] + (i - bounds[bi])] = q;
    }
  }
  free(owner);
  free(mark);
  return 0;
}

static void free_blocks(Blocks* B) {
  free(B->brow);
  free(B->bcol);
  free(B->soff);
  free(B->sb);
  free(B->se);
}

#define SB(B, blk, r) ((B)->sb[(B)->soff[blk] + (r)])
#define SE(B, blk, r) ((B)->se[(B)->soff[blk] + (r)])

/* reference factorize.hpp:260-302 */
int orc_export_dag(int32_t n, const int64_t* up, const int32_t* uc, int32_t m,
                   const int32_t* bounds, int64_t* nnodes, int64_t* nedges, int32_t* kind,
                   int32_t* bi_out, int32_t* bj_out, int32_t* efrom, int32_t* eto) {
  Blocks B;
  if (build_blocks(n, up, uc, m, bounds, &B)) return 2;
  int32_t* last = (int32_t*)malloc(sizeof(int32_t) * (B.nblk + 1));
  for (int64_t b = 0; b < B.nblk; ++b) last[b] = -1;
  int64_t nn = 0, ne = 0;
#define READ(blk)                                  \
  do {                                             \
    if (last[blk] >= 0) {                          \
      if (efrom) {                                 \
        efrom[ne] = last[blk];                     \
        eto[ne] = (int32_t)nn;                     \
      }                                            \
      ++ne;                                        \
    }                                              \
  } while (0)
#define NODE(k, i, j)  \
  do {                 \
    if (kind) {        \
      kind[nn] = (k);  \
      bi_out[nn] = (i); \
      bj_out[nn] = (j); \
    }                  \
  } while (0)
  for (int32_t p = 0; p < B.m; ++p) {
    const int64_t rb = B.brow[p], re = B.brow[p + 1];
    if (rb == re || B.bcol[rb] != p) {
      free(last);
      free_blocks(&B);
      return 3;
    }
    NODE(0, p, p);
    READ(rb);
    last[rb] = (int32_t)nn++;
    for (int64_t qj = rb + 1; qj < re; ++qj) {
      NODE(1, p, B.bcol[qj]);
      READ(rb);
      READ(qj);
      last[qj] = (int32_t)nn++;
    }
    for (int64_t qi = rb + 1; qi < re; ++qi) {
      const int32_t i = B.bcol[qi];
      for (int64_t qj = qi; qj < re; ++qj) {
        const int32_t j = B.bcol[qj];
        const int64_t tg = find_block(&B, i, j);
        if (tg < 0) continue;
        if (i == j) {
          NODE(2, j, j);
          READ(qj);
          READ(tg);
        } else {
          NODE(3, i, j);
          READ(qi);
          READ(qj);
          READ(tg);
        }
        last[tg] = (int32_t)nn++;
      }
    }
  }
#undef READ
#undef NODE
  *nnodes = nn;
  *nedges = ne;
  free(last);
  free_blocks(&B);
  return 0;
}

/* ---- block kernels (reference kernels.hpp:40-132) ------------------------ */

/* chol_block: kernels.hpp:40-67. blk = (p,p) */
static int k_chol(const Blocks* B, int64_t blk, int32_t p, const int32_t* uc, double* uv,
                  int32_t* row, double* pivot) {
  const int32_t r0 = B->bounds[p], nr = B->bounds[p + 1] - r0;
  for (int32_t r = 0; r < nr; ++r) {
    const int32_t g = r0 + r;
    const int64_t rb = SB(B, blk, r), re = SE(B, blk, r);
    if (rb == re || uc[rb] != g) return 2;
    const double piv = uv[rb];
    if (!(piv > 0.0)) {
      *row = g;
      *pivot = piv;
      return 1;
    }
    const double d = sqrt(piv);
    uv[rb] = d;
    for (int64_t q = rb + 1; q < re; ++q) uv[q] /= d;
    for (int64_t q1 = rb + 1; q1 < re; ++q1) {
      const int32_t c1 = uc[q1];
      const double v1 = uv[q1];
      int64_t t = SB(B, blk, c1 - r0);
      const int64_t te = SE(B, blk, c1 - r0);
      for (int64_t q2 = q1; q2 < re; ++q2) {
        const int32_t c2 = uc[q2];
        while (t < te && uc[t] < c2) ++t;
        if (t < te && uc[t] == c2) uv[t] -= v1 * uv[q2];
      }
    }
  }
  return 0;
}

/* trsm_block: kernels.hpp:72-92. dblk = (p,p), xblk = (p,j) */
static void k_trsm(const Blocks* B, int64_t dblk, int64_t xblk, int32_t p, const int32_t* uc,
                   double* uv) {
  const int32_t r0 = B->bounds[p], nr = B->bounds[p + 1] - r0;
  for (int32_t r = 0; r < nr; ++r) {
    const int64_t db = SB(B, dblk, r), de = SE(B, dblk, r);
    const double d = uv[db];
    const int64_t jb = SB(B, xblk, r), je = SE(B, xblk, r);
    for (int64_t q = jb; q < je; ++q) uv[q] /= d;
    for (int64_t q1 = db + 1; q1 < de; ++q1) {
      const int32_t rr = uc[q1];
      const double v1 = uv[q1];
      int64_t t = SB(B, xblk, rr - r0);
      const int64_t te = SE(B, xblk, rr - r0);
      for (int64_t q2 = jb; q2 < je; ++q2) {
        const int32_t c = uc[q2];
        while (t < te && uc[t] < c) ++t;
        if (t < te && uc[t] == c) uv[t] -= v1 * uv[q2];
      }
    }
  }
}

/* herk_block: kernels.hpp:95-111. pblk = (p,j), tblk = (j,j) */
static void k_herk(const Blocks* B, int64_t pblk, int64_t tblk, int32_t p, int32_t j,
                   const int32_t* uc, double* uv) {
  const int32_t r0 = B->bounds[p], nr = B->bounds[p + 1] - r0, t0 = B->bounds[j];
  for (int32_t r = 0; r < nr; ++r) {
    const int64_t jb = SB(B, pblk, r), je = SE(B, pblk, r);
    for (int64_t q1 = jb; q1 < je; ++q1) {
      const int32_t c1 = uc[q1];
      const double v1 = uv[q1];
      int64_t t = SB(B, tblk, c1 - t0);
      const int64_t te = SE(B, tblk, c1 - t0);
      for (int64_t q2 = q1; q2 < je; ++q2) {
        const int32_t c2 = uc[q2];
        while (t < te && uc[t] < c2) ++t;
        if (t < te && uc[t] == c2) uv[t] -= v1 * uv[q2];
      }
    }
  }
}

/* gemm_block: kernels.hpp:114-132. iblk = (p,i), jblk = (p,j), tblk = (i,j) */
static void k_gemm(const Blocks* B, int64_t iblk, int64_t jblk, int64_t tblk, int32_t p, int32_t i,
                   const int32_t* uc, double* uv) {
  const int32_t r0 = B->bounds[p], nr = B->bounds[p + 1] - r0, t0 = B->bounds[i];
  for (int32_t r = 0; r < nr; ++r) {
    const int64_t ib = SB(B, iblk, r), ie = SE(B, iblk, r);
    const int64_t jb = SB(B, jblk, r), je = SE(B, jblk, r);
    for (int64_t q1 = ib; q1 < ie; ++q1) {
      const int32_t c1 = uc[q1];
      const double v1 = uv[q1];
      int64_t t = SB(B, tblk, c1 - t0);
      const int64_t te = SE(B, tblk, c1 - t0);
      for (int64_t q2 = jb; q2 < je; ++q2) {
        const int32_t c2 = uc[q2];
        while (t < te && uc[t] < c2) ++t;
        if (t < te && uc[t] == c2) uv[t] -= v1 * uv[q2];
      }
    }
  }
}

/* factor_by_blocks (factorize.hpp:134-235) on the sequential policy: every
 * task's dependences precede it in generation order, so tasks run in that
 * order; after a breakdown the remaining tasks are no-ops (:146-167). */
int orc_factor_by_blocks(int32_t n, const int64_t* up, const int32_t* uc, double* uv,
                         int32_t m, const int32_t* bounds, int32_t* row, double* pivot) {
  Blocks B;
  if (build_blocks(n, up, uc, m, bounds, &B)) return 2;
  int failed = 0, rc = 0;
  for (int32_t p = 0; p < B.m && rc != 2 && rc != 3; ++p) {
    const int64_t rb = B.brow[p], re = B.brow[p + 1];
    if (rb == re || B.bcol[rb] != p) {
      rc = 3;
      break;
    }
    if (!failed) {
      const int s = k_chol(&B, rb, p, uc, uv, row, pivot);
      if (s == 2) {
        rc = 2;
        break;
      }
      if (s == 1) failed = 1;
    }
    for (int64_t qj = rb + 1; qj < re; ++qj)
      if (!failed) k_trsm(&B, rb, qj, p, uc, uv);
    for (int64_t qi = rb + 1; qi < re; ++qi) {
      const int32_t i = B.bcol[qi];
      for (int64_t qj = qi; qj < re; ++qj) {
        const int32_t j = B.bcol[qj];
        const int64_t tg = find_block(&B, i, j);
        if (tg < 0 || failed) continue;
        if (i == j) k_herk(&B, qj, tg, p, j, uc, uv);
        else k_gemm(&B, qi, qj, tg, p, i, uc, uv);
      }
    }
  }
  free_blocks(&B);
  if (rc) return rc;
  return failed ? 1 : 0;
}

/* Pattern-restricted residual. (UᵀU)_ij = sum_r U(r,i) U(r,j), r <= i <= j;
 * computed from U's columns (CSC built here), compared with A_ij on the
 * pattern of U. The reference has only a dense version
 * (test_matrices.hpp:128-138); this is its sparse restriction. */
double orc_pattern_residual(int32_t n, const int64_t* ap, const int32_t* ac, const double* av,
                            const int64_t* up, const int32_t* uc, const double* uv) {
  const int64_t nnz = up[n];
  int64_t* cp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* cr = (int32_t*)malloc(sizeof(int32_t) * (nnz + 1));
  double* cv = (double*)malloc(sizeof(double) * (nnz + 1));
  for (int64_t q = 0; q < nnz; ++q) cp[uc[q] + 1]++;
  for (int32_t i = 0; i < n; ++i) cp[i + 1] += cp[i];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  memcpy(fill, cp, sizeof(int64_t) * n);
  for (int32_t r = 0; r < n; ++r)
    for (int64_t q = up[r]; q < up[r + 1]; ++q) {
      const int64_t at = fill[uc[q]]++;
      cr[at] = r;
      cv[at] = uv[q];
    }
  double amax = 0.0;
  for (int64_t q = 0; q < ap[n]; ++q) amax = fmax(amax, fabs(av[q]));
  double worst = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t aq = ap[i];
    for (int64_t q = up[i]; q < up[i + 1]; ++q) {
      const int32_t j = uc[q];
      /* merge column i and column j of U */
      double s = 0.0;
      int64_t x = cp[i], y = cp[j];
      while (x < cp[i + 1] && y < cp[j + 1]) {
        if (cr[x] < cr[y]) ++x;
        else if (cr[x] > cr[y]) ++y;
        else {
          s += cv[x] * cv[y];
          ++x;
          ++y;
        }
      }
      while (aq < ap[i + 1] && ac[aq] < j) ++aq;
      const double a = (aq < ap[i + 1] && ac[aq] == j) ? av[aq] : 0.0;
      worst = fmax(worst, fabs(s - a));
    }
  }
  free(cp);
  free(cr);
  free(cv);
  free(fill);
  return amax > 0.0 ? worst / amax : worst;
}

/* reference symbolic.hpp:124-167 */
void orc_levelk_dense(int32_t n, const int64_t* ap, const int32_t* ac, int32_t k, uint8_t* mask) {
  const int32_t INF = 0x7fffffff / 4;
  int32_t* lev = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * n);
  for (int64_t x = 0; x < (int64_t)n * n; ++x) lev[x] = INF;
  for (int32_t i = 0; i < n; ++i) {
    lev[(int64_t)i * n + i] = 0;
    for (int64_t q = ap[i]; q < ap[i + 1]; ++q) lev[(int64_t)i * n + ac[q]] = 0;
  }
  int32_t* act = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  for (int32_t p = 0; p < n; ++p) {
    int32_t na = 0;
    for (int32_t i = p + 1; i < n; ++i)
      if (lev[(int64_t)p * n + i] < INF) act[na++] = i;
    for (int32_t x = 0; x < na; ++x)
      for (int32_t y = 0; y < na; ++y) {
        const int32_t i = act[x], j = act[y];
        const int32_t v = lev[(int64_t)p * n + i] + lev[(int64_t)p * n + j] + 1;
        if (v < lev[(int64_t)i * n + j]) lev[(int64_t)i * n + j] = v;
      }
  }
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j)
      mask[(int64_t)i * n + j] = (j >= i) && (i == j || lev[(int64_t)i * n + j] <= k);
  free(lev);
  free(act);
}

/* Preconditioner apply (see oracle.h): forward then backward substitution in
 * a fixed sequential order, every product and difference rounded on its own. */
int orc_trisolve(int32_t n, const int64_t* up, const int32_t* uc, const double* uv,
                 const double* b, int32_t which, double* x) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!t) return 3;
  for (int32_t i = 0; i < n; ++i) t[i] = b[i];
  for (int32_t i = 0; i < n; ++i)
    if (up[i] >= up[i + 1] || uc[up[i]] != i || uv[up[i]] == 0.0) {
      free(t);
      return 2;
    }
  if (which & 1) {
    for (int32_t i = 0; i < n; ++i) {
      const double yi = t[i] / uv[up[i]];
      t[i] = yi;
      for (int64_t q = up[i] + 1; q < up[i + 1]; ++q) {
        const double p = uv[q] * yi;
        t[uc[q]] = t[uc[q]] - p;
      }
    }
  }
  if (which & 2) {
    for (int32_t i = n - 1; i >= 0; --i) {
      double s = t[i];
      for (int64_t q = up[i] + 1; q < up[i + 1]; ++q) {
        const double p = uv[q] * t[uc[q]];
        s = s - p;
      }
      t[i] = s / uv[up[i]];
    }
  }
  for (int32_t i = 0; i < n; ++i) x[i] = t[i];
  free(t);
  return 0;
}
