// Seeded synthetic matrices for the BASELINE.json configurations
// plus the small shapes the reference's own tests use
// (reference proj/tests/support/test_matrices.hpp:18-82).
//
// No public matrix suite is involved: BASELINE.json names synthetic stencils
// only, and the paper's SuiteSparse matrices are absent from the container.
#include <cmath>
#include <random>

#include "sparse.hpp"

namespace tcb {

namespace {

struct Entries {
  std::vector<index_t> i, j;
  std::vector<double> v;
  void add(index_t r, index_t c, double x) {
    i.push_back(r);
    j.push_back(c);
    v.push_back(x);
  }
  void sym(index_t r, index_t c, double x) {
    add(r, c, x);
    if (r != c) add(c, r, x);
  }
};

inline index_t lex3(index_t n, index_t x, index_t y, index_t z) { return (x * n + y) * n + z; }

}  // namespace

CsrMatrix grid_laplacian_2d(index_t nx, index_t ny) {
  // vertex (r, c) -> r*ny + c; 4 on the diagonal, -1 to each grid neighbour.
  Entries e;
  for (index_t r = 0; r < nx; ++r)
    for (index_t c = 0; c < ny; ++c) {
      const index_t v = r * ny + c;
      e.add(v, v, 4.0);
      if (c + 1 < ny) e.sym(v, v + 1, -1.0);
      if (r + 1 < nx) e.sym(v, v + ny, -1.0);
    }
  return csr_from_entries(nx * ny, e.i, e.j, e.v);
}

CsrMatrix laplacian_7pt(index_t n) {
  // (x, y, z) -> (x*n + y)*n + z, z fastest; Dirichlet rows keep 6 on the diagonal.
  Entries e;
  for (index_t x = 0; x < n; ++x)
    for (index_t y = 0; y < n; ++y)
      for (index_t z = 0; z < n; ++z) {
        const index_t v = lex3(n, x, y, z);
        e.add(v, v, 6.0);
        if (z + 1 < n) e.sym(v, lex3(n, x, y, z + 1), -1.0);
        if (y + 1 < n) e.sym(v, lex3(n, x, y + 1, z), -1.0);
        if (x + 1 < n) e.sym(v, lex3(n, x + 1, y, z), -1.0);
      }
  return csr_from_entries(n * n * n, e.i, e.j, e.v);
}

CsrMatrix stencil27_variable(index_t n, std::uint64_t seed) {
  // Off-diagonals U(-1,-0.1) drawn for i ascending, offsets (dx,dy,dz) in
  // lexicographic order (dx outermost), neighbour j > i only; symmetrised.
  // Diagonal = sum |offdiag| (accumulated in draw order) + 1e-3.
  const index_t nv = n * n * n;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> draw(-1.0, -0.1);
  std::vector<double> rowsum(nv, 0.0);
  Entries e;
  for (index_t x = 0; x < n; ++x)
    for (index_t y = 0; y < n; ++y)
      for (index_t z = 0; z < n; ++z) {
        const index_t i = lex3(n, x, y, z);
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
              const index_t X = x + dx, Y = y + dy, Z = z + dz;
              if (X < 0 || Y < 0 || Z < 0 || X >= n || Y >= n || Z >= n) continue;
              const index_t j = lex3(n, X, Y, Z);
              if (j <= i) continue;
              const double v = draw(rng);
              e.sym(i, j, v);
              rowsum[i] += std::abs(v);
              rowsum[j] += std::abs(v);
            }
      }
  for (index_t i = 0; i < nv; ++i) e.add(i, i, rowsum[i] + 1e-3);
  return csr_from_entries(nv, e.i, e.j, e.v);
}

CsrMatrix elasticity27(index_t n, std::uint64_t seed) {
  // 3 dofs per node a = (x*n + y)*n + z, row 3a + p. Off-diagonal 3x3 blocks
  // B ~ U[-0.5, 0.5) (row-major) for each 27-neighbour b > a, B_ba = B_abᵀ;
  // |B| accumulated into both rows. Then per node: M ~ U[-0.5,0.5),
  // diagonal block = M·Mᵀ + (rowsum + 1e-2) on the diagonal.
  const index_t nn = n * n * n;
  const index_t nv = 3 * nn;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> draw(-0.5, 0.5);
  std::vector<double> rowsum(nv, 0.0);
  Entries e;
  for (index_t x = 0; x < n; ++x)
    for (index_t y = 0; y < n; ++y)
      for (index_t z = 0; z < n; ++z) {
        const index_t a = lex3(n, x, y, z);
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
              const index_t X = x + dx, Y = y + dy, Z = z + dz;
              if (X < 0 || Y < 0 || Z < 0 || X >= n || Y >= n || Z >= n) continue;
              const index_t b = lex3(n, X, Y, Z);
              if (b <= a) continue;
              double blk[3][3];
              for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) blk[p][q] = draw(rng);
              for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) {
                  e.sym(3 * a + p, 3 * b + q, blk[p][q]);
                  rowsum[3 * a + p] += std::abs(blk[p][q]);
                  rowsum[3 * b + q] += std::abs(blk[p][q]);
                }
            }
      }
  for (index_t a = 0; a < nn; ++a) {
    double m[3][3];
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) m[p][q] = draw(rng);
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) {
        double s = 0.0;
        for (int r = 0; r < 3; ++r) s += m[p][r] * m[q][r];
        if (p == q) s += rowsum[3 * a + p] + 1e-2;
        e.add(3 * a + p, 3 * a + q, s);
      }
  }
  return csr_from_entries(nv, e.i, e.j, e.v);
}

CsrMatrix diffusion_7pt_lognormal(index_t n, std::uint64_t seed, double sigma) {
  // kappa_c = exp(sigma * Z), Z ~ N(0,1) per cell in index order; face
  // coefficient h = 2 k_i k_j / (k_i + k_j) towards +z, +y, +x; A_ij = -h.
  // A_ii = sum of its face h (accumulated in generation order) plus
  // kappa_i per Dirichlet boundary face.
  const index_t nv = n * n * n;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> kappa(nv);
  for (index_t c = 0; c < nv; ++c) kappa[c] = std::exp(sigma * gauss(rng));
  std::vector<double> diag(nv, 0.0);
  std::vector<int> faces(nv, 0);
  Entries e;
  for (index_t x = 0; x < n; ++x)
    for (index_t y = 0; y < n; ++y)
      for (index_t z = 0; z < n; ++z) {
        const index_t i = lex3(n, x, y, z);
        const index_t nb[3] = {z + 1 < n ? lex3(n, x, y, z + 1) : -1,
                               y + 1 < n ? lex3(n, x, y + 1, z) : -1,
                               x + 1 < n ? lex3(n, x + 1, y, z) : -1};
        for (index_t j : nb) {
          if (j < 0) continue;
          const double h = (2.0 * kappa[i] * kappa[j]) / (kappa[i] + kappa[j]);
          e.sym(i, j, -h);
          diag[i] += h;
          diag[j] += h;
          ++faces[i];
          ++faces[j];
        }
      }
  for (index_t i = 0; i < nv; ++i) e.add(i, i, diag[i] + (6 - faces[i]) * kappa[i]);
  return csr_from_entries(nv, e.i, e.j, e.v);
}

CsrMatrix path_matrix(index_t n, double diag) {
  Entries e;
  for (index_t i = 0; i < n; ++i) {
    e.add(i, i, diag);
    if (i + 1 < n) e.sym(i, i + 1, -1.0);
  }
  return csr_from_entries(n, e.i, e.j, e.v);
}

CsrMatrix diagonal_matrix(const std::vector<double>& d) {
  Entries e;
  for (std::size_t i = 0; i < d.size(); ++i) e.add(static_cast<index_t>(i), static_cast<index_t>(i), d[i]);
  return csr_from_entries(static_cast<index_t>(d.size()), e.i, e.j, e.v);
}

CsrMatrix random_spd(index_t n, double density, std::uint32_t seed) {
  // Same draw sequence as the reference test helper random_spd
  // (test_matrices.hpp:63-82) for a freshly seeded std::mt19937.
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> coin(0.0, 1.0);
  std::uniform_real_distribution<double> val(0.1, 1.0);
  std::vector<double> rowsum(n, 0.0);
  Entries e;
  for (index_t i = 0; i < n; ++i)
    for (index_t j = i + 1; j < n; ++j)
      if (coin(rng) < density) {
        const double v = -val(rng);
        e.sym(i, j, v);
        rowsum[i] += std::abs(v);
        rowsum[j] += std::abs(v);
      }
  for (index_t i = 0; i < n; ++i) e.add(i, i, rowsum[i] + 1.0);
  return csr_from_entries(n, e.i, e.j, e.v);
}

}  // namespace tcb
