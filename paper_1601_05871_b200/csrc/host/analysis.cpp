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

// The recursion of the reference's nested_dissection, with disjoint subtrees
// run on separate host threads near the top of the tree. A subtree's numbers
// are known before it is dissected (the lower part first, then the upper,
// then the separator: ordering.hpp:239-300), so each subtree numbers its
// vertices from its own base; its tree nodes are built in a private list and
// appended in the sequential post-order, so perm, iperm and the tree are the
// sequential ones whatever the thread count.
class Dissector {
 public:
  Dissector(const CsrMatrix& a, index_t leaf, index_t max_depth, int threads)
      : a_(a), leaf_(std::max<index_t>(leaf, 1)), max_depth_(max_depth) {
    perm_.perm.assign(a.nrows, -1);
    perm_.iperm.assign(a.nrows, -1);
    // spawn below the first levels while threads remain (2^d subtrees at depth d)
    int d = 0;
    while ((1 << d) < threads && d < 12) ++d;
    par_depth_ = threads > 1 ? d : 0;
  }

  std::pair<Permutation, NdTree> run() {
    NdTree tree;
    if (a_.nrows == 0) {
      tree.nodes.emplace_back();
      tree.root = 0;
    } else {
      std::vector<index_t> all(a_.nrows);
      for (index_t v = 0; v < a_.nrows; ++v) all[v] = v;
      Scratch S(a_.nrows);
      tree.root = split(all, 0, 0, S, tree.nodes);
    }
    return {std::move(perm_), std::move(tree)};
  }

 private:
  // per-thread marks; stamps only grow, so a thread's stale marks never match
  struct Scratch {
    explicit Scratch(index_t n) : member(n, 0), mark(n, 0), side(n, 0) {}
    std::vector<index_t> member, mark;
    std::vector<unsigned char> side;
    index_t member_stamp = 0, mark_stamp = 0;
    void enter(const std::vector<index_t>& verts) {
      ++member_stamp;
      for (index_t v : verts) member[v] = member_stamp;
    }
    bool inside(index_t v) const { return member[v] == member_stamp; }
  };

  // Dissects `verts` (ascending ids), numbering them from `base`; appends the
  // subtree's nodes to `out` in post-order and returns the root's index there.
  index_t split(const std::vector<index_t>& verts, index_t depth, index_t base, Scratch& S,
                std::vector<NdNode>& out) {
    if (static_cast<index_t>(verts.size()) <= leaf_ || depth >= max_depth_)
      return leaf(verts, depth, base, out);

    std::vector<std::vector<index_t>> comps = components(verts, S);
    if (comps.size() > 1) {
      NdNode nd;
      nd.depth = depth;
      std::vector<index_t> bases(comps.size());
      index_t at = base;
      for (std::size_t c = 0; c < comps.size(); ++c) {
        bases[c] = at;
        at += static_cast<index_t>(comps[c].size());
      }
      children(comps, depth + 1, bases, S, out, nd);
      nd.range = {at, at};
      return push(out, std::move(nd));
    }

    std::vector<index_t> lo, hi, sep;
    if (!bisect(verts, lo, hi, sep, S) || sep.empty() || (lo.empty() && hi.empty()))
      return leaf(verts, depth, base, out);

    NdNode nd;
    nd.depth = depth;
    const index_t lo_n = static_cast<index_t>(lo.size()), hi_n = static_cast<index_t>(hi.size());
    std::vector<std::vector<index_t>> parts;
    std::vector<index_t> bases;
    if (!lo.empty()) {
      parts.push_back(std::move(lo));
      bases.push_back(base);
    }
    if (!hi.empty()) {
      parts.push_back(std::move(hi));
      bases.push_back(base + lo_n);
    }
    children(parts, depth + 1, bases, S, out, nd);
    nd.range.begin = base + lo_n + hi_n;
    index_t next = nd.range.begin;
    for (index_t v : sep) number(v, next);
    nd.range.end = next;
    return push(out, std::move(nd));
  }

  // the child subtrees in order; near the top, all but the last on new threads
  void children(const std::vector<std::vector<index_t>>& parts, index_t depth,
                const std::vector<index_t>& bases, Scratch& S, std::vector<NdNode>& out, NdNode& nd) {
    const std::size_t np = parts.size();
    if (depth > par_depth_ || np < 2) {
      for (std::size_t c = 0; c < np; ++c) nd.children.push_back(split(parts[c], depth, bases[c], S, out));
      return;
    }
    std::vector<std::vector<NdNode>> sub(np);
    std::vector<index_t> roots(np, -1);
    std::vector<std::thread> pool;
    for (std::size_t c = 0; c + 1 < np; ++c)
      pool.emplace_back([&, c] {
        Scratch own(a_.nrows);
        roots[c] = split(parts[c], depth, bases[c], own, sub[c]);
      });
    roots[np - 1] = split(parts[np - 1], depth, bases[np - 1], S, sub[np - 1]);
    for (auto& t : pool) t.join();
    for (std::size_t c = 0; c < np; ++c) {  // append in order, child indices shifted
      const index_t shift = static_cast<index_t>(out.size());
      for (NdNode& x : sub[c]) {
        for (index_t& ch : x.children) ch += shift;
        out.push_back(std::move(x));
      }
      nd.children.push_back(roots[c] + shift);
    }
  }

  index_t leaf(const std::vector<index_t>& verts, index_t depth, index_t base, std::vector<NdNode>& out) {
    NdNode nd;
    nd.depth = depth;
    nd.range.begin = base;
    index_t next = base;
    for (index_t v : verts) number(v, next);
    nd.range.end = next;
    return push(out, std::move(nd));
  }

  // subtrees write disjoint positions of the shared permutation
  void number(index_t v, index_t& next) {
    perm_.perm[v] = next;
    perm_.iperm[next] = v;
    ++next;
  }

  static index_t push(std::vector<NdNode>& out, NdNode&& nd) {
    out.push_back(std::move(nd));
    return static_cast<index_t>(out.size()) - 1;
  }

  // Connected pieces, each sorted, ordered by their smallest vertex.
  std::vector<std::vector<index_t>> components(const std::vector<index_t>& verts, Scratch& S) {
    S.enter(verts);
    ++S.mark_stamp;
    std::vector<std::vector<index_t>> out;
    for (index_t s : verts) {
      if (S.mark[s] == S.mark_stamp) continue;
      std::vector<index_t> piece{s};
      S.mark[s] = S.mark_stamp;
      for (std::size_t h = 0; h < piece.size(); ++h) {
        const index_t v = piece[h];
        for (offset_t q = a_.row_begin(v); q < a_.row_end(v); ++q) {
          const index_t w = a_.col_idx[q];
          if (w != v && S.inside(w) && S.mark[w] != S.mark_stamp) {
            S.mark[w] = S.mark_stamp;
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
  void levels_from(index_t root, std::vector<index_t>& order, std::vector<std::size_t>& level_start,
                   Scratch& S) {
    ++S.mark_stamp;
    order.clear();
    level_start.clear();
    order.push_back(root);
    S.mark[root] = S.mark_stamp;
    std::size_t lb = 0, le = 1;
    level_start.push_back(0);
    while (lb < le) {
      for (std::size_t h = lb; h < le; ++h) {
        const index_t v = order[h];
        for (offset_t q = a_.row_begin(v); q < a_.row_end(v); ++q) {
          const index_t w = a_.col_idx[q];
          if (w != v && S.inside(w) && S.mark[w] != S.mark_stamp) {
            S.mark[w] = S.mark_stamp;
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

  bool bisect(const std::vector<index_t>& verts, std::vector<index_t>& lo, std::vector<index_t>& hi,
              std::vector<index_t>& sep, Scratch& S) {
    S.enter(verts);
    std::vector<index_t> order;
    std::vector<std::size_t> ls;
    levels_from(verts.front(), order, ls, S);
    const index_t far = order[ls[ls.size() - 2]];  // smallest vertex of the last level
    levels_from(far, order, ls, S);
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
    for (std::size_t h = 0; h < order.size(); ++h) S.side[order[h]] = h < split_at ? 1 : 2;
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
        touches = (w != v && S.inside(w) && S.side[w] == other);
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
  index_t par_depth_ = 0;
  Permutation perm_;
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
                                                 index_t max_depth, int threads) {
  if (a.nrows != a.ncols) throw std::invalid_argument("nested_dissection: matrix not square");
  // small graphs stay on one thread (a thread's scratch is three n-arrays)
  const int nt = a.nrows < 4096 ? 1 : pick_threads(threads);
  return Dissector(a, leaf_size, max_depth, nt).run();
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
  auto nd = nested_dissection(a, opt.leaf_size, opt.max_depth, threads);
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
