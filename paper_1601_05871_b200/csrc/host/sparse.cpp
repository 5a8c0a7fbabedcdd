// CSR utilities for the host input side of the IC(k) path.
#include <algorithm>
#include <thread>
#include <numeric>

#include "sparse.hpp"

namespace tcb {

CsrMatrix csr_from_entries(index_t n, const std::vector<index_t>& ti,
                           const std::vector<index_t>& tj,
                           const std::vector<double>& tv) {
  // Counting sort by row (stable in input order), then per-row column sort.
  // Semantics follow reference csr_matrix.hpp:76-122 (duplicates summed).
  const std::size_t ne = ti.size();
  std::vector<offset_t> start(static_cast<std::size_t>(n) + 1, 0);
  for (std::size_t e = 0; e < ne; ++e) {
    if (ti[e] < 0 || ti[e] >= n || tj[e] < 0 || tj[e] >= n)
      throw std::invalid_argument("csr_from_entries: index out of range");
    ++start[ti[e] + 1];
  }
  for (index_t i = 0; i < n; ++i) start[i + 1] += start[i];
  std::vector<offset_t> fill(start.begin(), start.end() - 1);
  std::vector<index_t> c(ne);
  std::vector<double> v(ne);
  for (std::size_t e = 0; e < ne; ++e) {
    const offset_t p = fill[ti[e]]++;
    c[p] = tj[e];
    v[p] = tv[e];
  }
  CsrMatrix m;
  m.nrows = m.ncols = n;
  m.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  m.col_idx.reserve(ne);
  m.values.reserve(ne);
  std::vector<offset_t> idx;
  for (index_t i = 0; i < n; ++i) {
    idx.resize(static_cast<std::size_t>(start[i + 1] - start[i]));
    std::iota(idx.begin(), idx.end(), start[i]);
    std::sort(idx.begin(), idx.end(),
              [&](offset_t x, offset_t y) { return c[x] < c[y]; });
    const std::size_t row0 = m.col_idx.size();
    for (offset_t q : idx) {
      if (m.col_idx.size() > row0 && m.col_idx.back() == c[q]) {
        m.values.back() += v[q];
      } else {
        m.col_idx.push_back(c[q]);
        m.values.push_back(v[q]);
      }
    }
    m.row_ptr[i + 1] = static_cast<offset_t>(m.col_idx.size());
  }
  return m;
}

void validate_csr(const CsrMatrix& m) {
  if (m.nrows < 0 || m.ncols < 0) throw std::invalid_argument("csr: negative dimension");
  if (m.row_ptr.size() != static_cast<std::size_t>(m.nrows) + 1)
    throw std::invalid_argument("csr: row_ptr length mismatch");
  if (m.row_ptr[0] != 0) throw std::invalid_argument("csr: row_ptr[0] != 0");
  if (m.row_ptr.back() != m.nnz() || m.values.size() != m.col_idx.size())
    throw std::invalid_argument("csr: array length mismatch");
  for (index_t i = 0; i < m.nrows; ++i) {
    if (m.row_ptr[i] > m.row_ptr[i + 1])
      throw std::invalid_argument("csr: row_ptr not non-decreasing");
    for (offset_t q = m.row_ptr[i]; q < m.row_ptr[i + 1]; ++q) {
      if (m.col_idx[q] < 0 || m.col_idx[q] >= m.ncols)
        throw std::invalid_argument("csr: column index out of range");
      if (q > m.row_ptr[i] && m.col_idx[q] <= m.col_idx[q - 1])
        throw std::invalid_argument("csr: columns not strictly increasing in row " +
                                    std::to_string(i));
    }
  }
}

void validate_ranges(const RangeList& rl, index_t n) {
  // reference ordering.hpp:43-55
  index_t at = 0;
  for (const Range& r : rl.ranges) {
    if (r.begin != at)
      throw std::invalid_argument("ranges not contiguous at index " + std::to_string(r.begin));
    if (r.end <= r.begin) throw std::invalid_argument("empty or inverted range");
    at = r.end;
  }
  if (at != n) throw std::invalid_argument("ranges do not cover [0, n)");
}

CsrMatrix permute_symmetric(const CsrMatrix& a, const Permutation& p) {
  if (a.nrows != a.ncols) throw std::invalid_argument("permute_symmetric: matrix not square");
  if (static_cast<index_t>(p.perm.size()) != a.nrows)
    throw std::invalid_argument("permute_symmetric: permutation size mismatch");
  const index_t n = a.nrows;
  CsrMatrix b;
  b.nrows = b.ncols = n;
  b.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (index_t i = 0; i < n; ++i) b.row_ptr[p.perm[i] + 1] = a.row_end(i) - a.row_begin(i);
  for (index_t i = 0; i < n; ++i) b.row_ptr[i + 1] += b.row_ptr[i];
  b.col_idx.resize(static_cast<std::size_t>(a.nnz()));
  b.values.resize(static_cast<std::size_t>(a.nnz()));
  // rows are independent: blocks of rows on the host threads
  auto rows = [&](index_t r0, index_t r1) {
    std::vector<std::pair<index_t, double>> row;
    for (index_t r = r0; r < r1; ++r) {
      const index_t src = p.iperm[r];
      row.clear();
      for (offset_t q = a.row_begin(src); q < a.row_end(src); ++q)
        row.emplace_back(p.perm[a.col_idx[q]], a.values[q]);
      std::sort(row.begin(), row.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      offset_t o = b.row_ptr[r];
      for (const auto& e : row) {
        b.col_idx[o] = e.first;
        b.values[o] = e.second;
        ++o;
      }
    }
  };
  const unsigned hc = std::thread::hardware_concurrency();
  const index_t nt = n < 65536 ? 1 : static_cast<index_t>(std::max(1u, std::min(hc, 32u)));
  std::vector<std::thread> pool;
  for (index_t t = 1; t < nt; ++t)
    pool.emplace_back(rows, static_cast<index_t>(static_cast<long long>(n) * t / nt),
                      static_cast<index_t>(static_cast<long long>(n) * (t + 1) / nt));
  rows(0, static_cast<index_t>(n / nt));
  for (auto& th : pool) th.join();
  return b;
}

offset_t count_upper(const CsrMatrix& a) {
  offset_t c = 0;
  for (index_t i = 0; i < a.nrows; ++i)
    for (offset_t q = a.row_begin(i); q < a.row_end(i); ++q) c += a.col_idx[q] >= i;
  return c;
}

std::vector<double> init_factor_values(const CsrMatrix& a, const CsrMatrix& u) {
  // Zero-initialised U slots receive triu(PᵀAP) by a per-row sorted merge
  // (reference factorize.hpp:71-89). `0.0 + a` keeps the sign of zero exactly
  // as the reference does.
  std::vector<double> vals(static_cast<std::size_t>(u.nnz()), 0.0);
  for (index_t i = 0; i < a.nrows; ++i) {
    offset_t t = u.row_begin(i);
    const offset_t te = u.row_end(i);
    for (offset_t q = a.row_begin(i); q < a.row_end(i); ++q) {
      const index_t c = a.col_idx[q];
      if (c < i) continue;
      while (t < te && u.col_idx[t] < c) ++t;
      if (t < te && u.col_idx[t] == c) vals[t] += a.values[q];
    }
  }
  return vals;
}

std::vector<std::int32_t> init_factor_map(const CsrMatrix& a, const CsrMatrix& u) {
  // The same merge as init_factor_values, recording the source instead of
  // adding it: map[t] = position in a.values of the entry U slot t starts
  // from, -1 for fill. A slot fed by two entries (duplicates) has no map.
  std::vector<std::int32_t> map(static_cast<std::size_t>(u.nnz()), -1);
  if (a.nnz() > 0x7fffffffLL) throw std::length_error("init map: A beyond 2^31 entries");
  for (index_t i = 0; i < a.nrows; ++i) {
    offset_t t = u.row_begin(i);
    const offset_t te = u.row_end(i);
    for (offset_t q = a.row_begin(i); q < a.row_end(i); ++q) {
      const index_t c = a.col_idx[q];
      if (c < i) continue;
      while (t < te && u.col_idx[t] < c) ++t;
      if (t < te && u.col_idx[t] == c) {
        if (map[t] >= 0) throw std::invalid_argument("init map: duplicate entry in A");
        map[t] = static_cast<std::int32_t>(q);
      }
    }
  }
  return map;
}

}  // namespace tcb
