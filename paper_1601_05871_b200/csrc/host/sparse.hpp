// Host-side sparse containers for the IC(k) numeric path.
//
// These mirror the reference's input formats field for field so that the
// drop-in (`factor_by_blocks_gpu`) receives exactly what the reference's
// `factor_by_blocks` receives:
//   CsrMatrix    <- taskchol::CsrMatrix   (reference csr_matrix.hpp:16-49)
//   Permutation  <- taskchol::Permutation (reference csr_matrix.hpp:124-156)
//   Range/RangeList <- ordering.hpp:26-41
//   NdNode/NdTree   <- ordering.hpp:57-86
//   FillPattern  <- symbolic.hpp:28-35
// Index type int32, offset type int64, values fp64 (csr_matrix.hpp:16-17).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tcb {

using index_t = std::int32_t;
using offset_t = std::int64_t;

struct CsrMatrix {
  index_t nrows = 0;
  index_t ncols = 0;
  std::vector<offset_t> row_ptr;  // nrows + 1
  std::vector<index_t> col_idx;   // strictly increasing per row
  std::vector<double> values;

  offset_t nnz() const { return static_cast<offset_t>(col_idx.size()); }
  offset_t row_begin(index_t i) const { return row_ptr[i]; }
  offset_t row_end(index_t i) const { return row_ptr[i + 1]; }
};

struct Permutation {
  std::vector<index_t> perm;   // perm[old] = new
  std::vector<index_t> iperm;  // iperm[new] = old
};

struct Range {
  index_t begin = 0;
  index_t end = 0;
  index_t size() const { return end - begin; }
  bool empty() const { return end == begin; }
};

struct RangeList {
  std::vector<Range> ranges;
  index_t count() const { return static_cast<index_t>(ranges.size()); }
};

struct NdNode {
  Range range;                   // own separator (internal) or leaf range
  std::vector<index_t> children; // subtree spans precede the node's range
  index_t depth = 0;
};

struct NdTree {
  std::vector<NdNode> nodes;  // children are stored before their parent
  index_t root = -1;
  index_t span_begin(index_t id) const {
    while (!nodes[id].children.empty()) id = nodes[id].children.front();
    return nodes[id].range.begin;
  }
  index_t span_end(index_t id) const { return nodes[id].range.end; }
};

struct FillPattern {
  CsrMatrix pattern;  // upper factor pattern incl. full diagonal, values 1.0
  index_t level_cap = 0;
  offset_t nnz_triu_input = 0;
};

struct AnalyzeOptions {
  index_t level = 0;
  index_t treecut = 0;
  index_t leaf_size = 64;
  index_t max_depth = 100;
};

struct Analysis {
  Permutation perm;
  NdTree tree;
  RangeList ranges;
  CsrMatrix a_permuted;
  FillPattern pattern;
  double ordering_seconds = 0.0;
  double symbolic_seconds = 0.0;
};

// --- csr utilities (sparse.cpp) --------------------------------------------

// Builds a CSR matrix from (row, col, value) entries given row by row in any
// column order; duplicate coordinates are summed in ascending-column sort order.
CsrMatrix csr_from_entries(index_t n, const std::vector<index_t>& ti,
                           const std::vector<index_t>& tj,
                           const std::vector<double>& tv);
void validate_csr(const CsrMatrix& m);
void validate_ranges(const RangeList& rl, index_t n);
CsrMatrix permute_symmetric(const CsrMatrix& a, const Permutation& p);
offset_t count_upper(const CsrMatrix& a);
// U := pattern with zeros, then triu(PᵀAP) added onto matching slots
// (reference factorize.hpp:71-89).
std::vector<double> init_factor_values(const CsrMatrix& a_permuted,
                                       const CsrMatrix& pattern);
// Per U slot, the position in a_permuted.values init_factor_values draws it
// from (-1: fill); throws std::invalid_argument when a slot has two sources.
std::vector<std::int32_t> init_factor_map(const CsrMatrix& a_permuted, const CsrMatrix& pattern);

// --- analysis (analysis.cpp) -----------------------------------------------
// threads: 0 = all hardware threads (disjoint subtrees in parallel; the
// result is the sequential one whatever the count)
std::pair<Permutation, NdTree> nested_dissection(const CsrMatrix& a,
                                                 index_t leaf_size,
                                                 index_t max_depth, int threads = 1);
RangeList prune_tree(const NdTree& tree, index_t t);
FillPattern levelk_pattern(const CsrMatrix& a_permuted, index_t k,
                           int threads = 0);
Analysis analyze(const CsrMatrix& a, const AnalyzeOptions& opt,
                 int threads = 0);

// --- file formats (io.cpp) --------------------------------------------------
// Matrix Market coordinate files (reference matrix_market.hpp:61-176): real,
// integer or pattern; general or symmetric (mirrored); duplicates summed.
// Errors are std::runtime_error with the reference's messages.
CsrMatrix load_matrix_market(const std::string& path);
void write_matrix_market(const CsrMatrix& m, const std::string& path);
// Ordering file (reference ordering.hpp:355-399): n, n values of perm
// (new index of old), the range count, then "begin end" per range.
std::pair<Permutation, RangeList> load_ordering(const std::string& path, index_t n);
// The pipeline with an imported ordering (reference pipeline.hpp:39-44).
Analysis analyze_with_ordering(const CsrMatrix& a, Permutation perm, RangeList ranges, index_t level,
                               int threads = 0);

// --- generators (generators.cpp) -------------------------------------------
CsrMatrix grid_laplacian_2d(index_t nx, index_t ny);           // C1
CsrMatrix laplacian_7pt(index_t n);                            // C2, C6
CsrMatrix stencil27_variable(index_t n, std::uint64_t seed);   // C3
CsrMatrix elasticity27(index_t n, std::uint64_t seed);         // C4
CsrMatrix diffusion_7pt_lognormal(index_t n, std::uint64_t seed, double sigma);  // C5
CsrMatrix path_matrix(index_t n, double diag);
CsrMatrix diagonal_matrix(const std::vector<double>& d);
CsrMatrix random_spd(index_t n, double density, std::uint32_t seed);

}  // namespace tcb
