// Host analysis that produces the hot path's inputs: nested-dissection
// ordering, range pruning and the level-k fill pattern.
//
// The north star keeps this phase on the host with the reference's
// semantics; because the reference sources cannot ship, this is an
// independent implementation that must reproduce the reference's outputs
// exactly (the DAG is derived from the ranges, so any divergence would break
// DAG parity). Tests pin perm/ranges/pattern hashes against the reference
// (tests/golden, generated from oracle/_ref).
//
//   nested_dissection  <- ordering.hpp:103-314 (BFS level-set bisection from a
//                         pseudo-peripheral vertex, separator = boundary of the
//                         larger half, parts then separator, ascending order)
//   prune_tree         <- ordering.hpp:319-353
//   levelk_pattern     <- symbolic.hpp:57-120 (depth-bounded search through
//                         lower-numbered vertices; here run row-parallel)
//   analyze            <- pipeline.hpp:35-55
#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <thread>

#include "sparse.hpp"

namespace tcb {

namespace {

class Dissector {
 public:
  Dissector(const CsrMatrix& a, index_t leaf, index_t max_depth)
      : a_(a), leaf_(std::max<index_t>(leaf, 1)), max_depth_(max_depth),
        member_(a.nrows, 0), mark_(a.nrows, 0), side_(a.nrows, 0) {
    perm_.perm.assign(a.nrows, -1);
    perm_.iperm.assign(a.nrows, -1);
  }

  std::pair<Permutation, NdTree> run() {
    if (a_.nrows == 0) {
      tree_.nodes.emplace_back();
      tree_.root = 0;
    } else {
      std::vector<index_t> all(a_.nrows);
      for (index_t v = 0; v < a_.nrows; ++v) all[v] = v;
      tree_.root = split(all, 0);
    }
    return {std::move(perm_), std::move(tree_)};
  }

 private:
  // Returns the node id of the subtree ordering `verts` (ascending ids).
  index_t split(const std::vector<index_t>& verts, index_t depth) {
    if (static_cast<index_t>(verts.size()) <= leaf_ || depth >= max_depth_)
      return leaf(verts, depth);

    std::vector<std::vector<index_t>> comps = components(verts);
    if (comps.size() > 1) {
      NdNode nd;
      nd.depth = depth;
      for (auto& c : comps) nd.children.push_back(split(c, depth + 1));
      nd.range = {next_, next_};
      return push(std::move(nd));
    }

    std::vector<index_t> lo, hi, sep;
    if (!bisect(verts, lo, hi, sep) || sep.empty() || (lo.empty() && hi.empty()))
      return leaf(verts, depth);

    NdNode nd;
    nd.depth = depth;
    if (!lo.empty()) nd.children.push_back(split(lo, depth + 1));
    if (!hi.empty()) nd.children.push_back(split(hi, depth + 1));
    nd.range.begin = next_;
    for (index_t v : sep) number(v);
    nd.range.end = next_;
    return push(std::move(nd));
  }

  index_t leaf(const std::vector<index_t>& verts, index_t depth) {
    NdNode nd;
    nd.depth = depth;
    nd.range.begin = next_;
    for (index_t v : verts) number(v);
    nd.range.end = next_;
    return push(std::move(nd));
  }

  void number(index_t v) {
    perm_.perm[v] = next_;
    perm_.iperm[next_] = v;
    ++next_;
  }

  index_t push(NdNode&& nd) {
    tree_.nodes.push_back(std::move(nd));
    return static_cast<index_t>(tree_.nodes.size()) - 1;
  }

  void enter(const std::vector<index_t>& verts) {
    ++member_stamp_;
    for (index_t v : verts) member_[v] = member_stamp_;
  }
  bool inside(index_t v) const { return member_[v] == member_stamp_; }

  // Connected pieces, each sorted, ordered by their smallest vertex.
  std::vector<std::vector<index_t>> components(const std::vector<index_t>& verts) {
    enter(verts);
    ++mark_stamp_;
    std::vector<std::vector<index_t>> out;
    for (index_t s : verts) {
      if (mark_[s] == mark_stamp_) continue;
      std::vector<index_t> piece{s};
      mark_[s] = mark_stamp_;
      for (std::size_t h = 0; h < piece.size(); ++h) {
        const index_t v = piece[h];
        for (offset_t q = a_.row_begin(v); q < a_.row_end(v); ++q) {
          const index_t w = a_.col_idx[q];
          if (w != v && inside(w) && mark_[w] != mark_stamp_) {
            mark_[w] = mark_stamp_;
            piece.push_back(w);
          }
        }
      }
      std::sort(piece.begin(), piece.end());
      out.push_back(std::move(piece));
      // `s` is the smallest unvisited vertex, hence the piece minimum: the
      // pieces come out already ordered by their smallest vertex.
    }
    return out;
  }

  // BFS from `root` over the member set; `order` receives the vertices level
  // by level (each level sorted) and `level_start` the level offsets.
  void levels_from(index_t root, std::vector<index_t>& order,
                   std::vector<std::size_t>& level_start) {
    ++mark_stamp_;
    order.clear();
    level_start.clear();
    order.push_back(root);
    mark_[root] = mark_stamp_;
    std::size_t lb = 0, le = 1;
    level_start.push_back(0);
    while (lb < le) {
      for (std::size_t h = lb; h < le; ++h) {
        const index_t v = order[h];
        for (offset_t q = a_.row_begin(v); q < a_.row_end(v); ++q) {
          const index_t w = a_.col_idx[q];
          if (w != v && inside(w) && mark_[w] != mark_stamp_) {
            mark_[w] = mark_stamp_;
            order.push_back(w);
          }
        }
      }
      std::sort(order.begin() + le, order.end());
      lb = le;
      le = order.size();
      if (lb < le) level_start.push_back(lb);
    }
    level_start.push_back(order.size());
  }

  bool bisect(const std::vector<index_t>& verts, std::vector<index_t>& lo,
              std::vector<index_t>& hi, std::vector<index_t>& sep) {
    enter(verts);
    std::vector<index_t> order;
    std::vector<std::size_t> ls;
    levels_from(verts.front(), order, ls);
    const index_t far = order[ls[ls.size() - 2]];  // smallest vertex of the last level
    levels_from(far, order, ls);
    const index_t nlev = static_cast<index_t>(ls.size()) - 1;
    if (nlev < 2) return false;

    const std::size_t need = (verts.size() + 1) / 2;
    index_t cut = 0;
    std::size_t acc = 0;
    for (index_t l = 0; l + 1 < nlev; ++l) {
      acc += ls[l + 1] - ls[l];
      cut = l;
      if (acc >= need) break;
    }
    const std::size_t split_at = ls[cut + 1];
    for (std::size_t h = 0; h < order.size(); ++h) side_[order[h]] = h < split_at ? 1 : 2;
    lo.assign(order.begin(), order.begin() + split_at);
    hi.assign(order.begin() + split_at, order.end());

    const bool lo_big = lo.size() >= hi.size();
    std::vector<index_t>& big = lo_big ? lo : hi;
    const unsigned char other = lo_big ? 2 : 1;
    std::vector<index_t> keep;
    keep.reserve(big.size());
    for (index_t v : big) {
      bool touches = false;
      for (offset_t q = a_.row_begin(v); q < a_.row_end(v) && !touches; ++q) {
        const index_t w = a_.col_idx[q];
        touches = (w != v && inside(w) && side_[w] == other);
      }
      (touches ? sep : keep).push_back(v);
    }
    big.swap(keep);
    std::sort(lo.begin(), lo.end());
    std::sort(hi.begin(), hi.end());
    // sep inherits level order from `big`; restore ascending order
    std::sort(sep.begin(), sep.end());
    return true;
  }

  const CsrMatrix& a_;
  index_t leaf_, max_depth_;
  std::vector<index_t> member_, mark_;
  std::vector<unsigned char> side_;
  index_t member_stamp_ = 0, mark_stamp_ = 0, next_ = 0;
  Permutation perm_;
  NdTree tree_;
};

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int pick_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

}  // namespace

std::pair<Permutation, NdTree> nested_dissection(const CsrMatrix& a, index_t leaf_size,
                                                 index_t max_depth) {
  if (a.nrows != a.ncols) throw std::invalid_argument("nested_dissection: matrix not square");
  return Dissector(a, leaf_size, max_depth).run();
}

RangeList prune_tree(const NdTree& tree, index_t t) {
  RangeList out;
  if (tree.root < 0) return out;
  const std::size_t nn = tree.nodes.size();
  std::vector<index_t> height(nn, 0);
  for (std::size_t id = 0; id < nn; ++id)  // children precede parents
    for (index_t c : tree.nodes[id].children)
      height[id] = std::max<index_t>(height[id], height[c] + 1);

  std::function<void(index_t)> emit = [&](index_t id) {
    const NdNode& nd = tree.nodes[id];
    if (height[id] <= t) {
      const Range whole{tree.span_begin(id), tree.span_end(id)};
      if (!whole.empty()) out.ranges.push_back(whole);
      return;
    }
    for (index_t c : nd.children) emit(c);
    if (!nd.range.empty()) out.ranges.push_back(nd.range);
  };
  emit(tree.root);
  return out;
}

FillPattern levelk_pattern(const CsrMatrix& a, index_t k, int threads) {
  if (a.nrows != a.ncols) throw std::invalid_argument("levelk_pattern: matrix not square");
  const index_t n = a.nrows;
  // An entry (i, j), j > i, belongs to level <= k iff j is adjacent to a
  // vertex reachable from i in <= k steps through vertices numbered below i.
  const index_t kk = std::min<index_t>(std::max<index_t>(k, 0), n);
  FillPattern fp;
  fp.level_cap = k;
  fp.nnz_triu_input = count_upper(a);
  std::vector<std::vector<index_t>> rows(n);

  const int nt = std::max(1, std::min(pick_threads(threads), n > 0 ? n / 256 + 1 : 1));
  std::atomic<index_t> cursor{0};
  auto worker = [&]() {
    std::vector<index_t> seen(n, -1), hit(n, -1);
    std::vector<index_t> frontier, next_frontier, targets;
    constexpr index_t kChunk = 256;
    while (true) {
      const index_t c0 = cursor.fetch_add(kChunk);
      if (c0 >= n) break;
      const index_t c1 = std::min<index_t>(n, c0 + kChunk);
      for (index_t i = c0; i < c1; ++i) {
        targets.clear();
        frontier.assign(1, i);
        seen[i] = i;
        for (index_t d = 0; d <= kk && !frontier.empty(); ++d) {
          next_frontier.clear();
          for (index_t v : frontier) {
            for (offset_t q = a.row_begin(v); q < a.row_end(v); ++q) {
              const index_t w = a.col_idx[q];
              if (w > i) {
                if (hit[w] != i) {
                  hit[w] = i;
                  targets.push_back(w);
                }
              } else if (w < i && d < kk && seen[w] != i) {
                seen[w] = i;
                next_frontier.push_back(w);
              }
            }
          }
          frontier.swap(next_frontier);
        }
        std::sort(targets.begin(), targets.end());
        std::vector<index_t>& row = rows[i];
        row.reserve(targets.size() + 1);
        row.push_back(i);
        row.insert(row.end(), targets.begin(), targets.end());
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();

  CsrMatrix& u = fp.pattern;
  u.nrows = u.ncols = n;
  u.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (index_t i = 0; i < n; ++i) u.row_ptr[i + 1] = u.row_ptr[i] + static_cast<offset_t>(rows[i].size());
  u.col_idx.reserve(static_cast<std::size_t>(u.row_ptr[n]));
  for (index_t i = 0; i < n; ++i) {
    u.col_idx.insert(u.col_idx.end(), rows[i].begin(), rows[i].end());
    std::vector<index_t>().swap(rows[i]);
  }
  u.values.assign(u.col_idx.size(), 1.0);
  return fp;
}

Analysis analyze(const CsrMatrix& a, const AnalyzeOptions& opt, int threads) {
  Analysis out;
  auto t0 = std::chrono::steady_clock::now();
  auto nd = nested_dissection(a, opt.leaf_size, opt.max_depth);
  out.perm = std::move(nd.first);
  out.tree = std::move(nd.second);
  out.ranges = prune_tree(out.tree, opt.treecut);
  out.a_permuted = permute_symmetric(a, out.perm);
  out.ordering_seconds = since(t0);
  t0 = std::chrono::steady_clock::now();
  out.pattern = levelk_pattern(out.a_permuted, opt.level, threads);
  out.symbolic_seconds = since(t0);
  return out;
}

}  // namespace tcb
