// Host symbolic phase: pattern validation, block-graph orderings, clique-completion
// symbolic factorization, elimination tree and levels.
//
// PAPER.md:29 (§II): the auxiliary matrix "is LDL^T factorized via a very fast symbolic
// factorization step [on the] attributed clique graph of the block-wise sparse matrix".
// Reading L14: the attributed clique graph is the block graph with vertex
// weight s_k; eliminating block k turns its current neighbours struct(k) into a clique.
// Reading L8: block elimination order AUTO = lower-flop of ND and weighted minimum degree.
#include "analyze.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <queue>

namespace ddaux {

namespace {

struct Bitset {
  int words = 0;
  std::vector<uint64_t> d;
  void init(int n) { words = (n + 63) / 64; d.assign((size_t)words, 0); }
  void set(int i) { d[i >> 6] |= 1ull << (i & 63); }
  void clr(int i) { d[i >> 6] &= ~(1ull << (i & 63)); }
  bool get(int i) const { return (d[i >> 6] >> (i & 63)) & 1; }
};

// adjacency bitsets (one row per vertex)
struct BitGraph {
  int n = 0, words = 0;
  std::vector<uint64_t> m;
  void init(const Graph& g) {
    n = g.n;
    words = (n + 63) / 64;
    m.assign((size_t)n * words, 0);
    for (int v = 0; v < n; ++v)
      for (int u : g.adj[v]) m[(size_t)v * words + (u >> 6)] |= 1ull << (u & 63);
  }
  uint64_t* row(int v) { return &m[(size_t)v * words]; }
};

template <class F>
inline void for_bits(const uint64_t* a, const uint64_t* notmask, int words, F f) {
  for (int w = 0; w < words; ++w) {
    uint64_t x = a[w] & ~notmask[w];
    while (x) {
      int b = __builtin_ctzll(x);
      f(w * 64 + b);
      x &= x - 1;
    }
  }
}

}  // namespace

std::string validate_pattern(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx) {
  if (nblk <= 0) return "nblk must be > 0";
  if (nblk > (1 << 24)) return "nblk too large";
  for (int64_t j = 0; j < nblk; ++j)
    if (blk_size[j] <= 0) return "block size must be > 0 (block " + std::to_string(j) + ")";
  if (colptr[0] != 0) return "colptr[0] must be 0";
  for (int64_t j = 0; j < nblk; ++j) {
    int64_t b = colptr[j], e = colptr[j + 1];
    if (e <= b) return "missing diagonal block in column " + std::to_string(j);
    if (rowidx[b] != j) return "diagonal block must be present and first in column " + std::to_string(j);
    for (int64_t p = b; p < e; ++p) {
      if (rowidx[p] < 0 || rowidx[p] >= nblk) return "row index out of range in column " + std::to_string(j);
      if (rowidx[p] < j) return "upper-triangle entry in column " + std::to_string(j);
      if (p > b && rowidx[p] <= rowidx[p - 1]) return "unsorted or duplicate row in column " + std::to_string(j);
    }
  }
  return "";
}

Graph graph_from_pattern(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx) {
  Graph g;
  g.n = (int)nblk;
  g.adj.assign(g.n, {});
  g.w.assign(blk_size, blk_size + nblk);
  for (int j = 0; j < g.n; ++j)
    for (int64_t p = colptr[j] + 1; p < colptr[j + 1]; ++p) {
      int i = rowidx[p];
      g.adj[i].push_back(j);
      g.adj[j].push_back(i);
    }
  for (auto& a : g.adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  return g;
}

// ----------------------------------------------------------------------------- symbolic
Symbolic symbolic_from_order(const Graph& g, const std::vector<int>& order) {
  Symbolic S;
  const int n = g.n;
  S.nblk = n;
  S.order = order;
  S.pos.assign(n, -1);
  for (int t = 0; t < n; ++t) S.pos[order[t]] = t;
  BitGraph B;
  B.init(g);
  Bitset elim;
  elim.init(n);
  S.st.assign(n, {});
  std::vector<int> nb;
  for (int t = 0; t < n; ++t) {
    int k = order[t];
    nb.clear();
    for_bits(B.row(k), elim.d.data(), B.words, [&](int u) { nb.push_back(u); });
    // clique completion: every pair of the current neighbours becomes adjacent
    for (int a : nb) {
      uint64_t* ra = B.row(a);
      const uint64_t* rk = B.row(k);
      for (int w = 0; w < B.words; ++w) ra[w] |= rk[w] & ~elim.d[w];
      ra[a >> 6] &= ~(1ull << (a & 63));
    }
    elim.set(k);
    auto& st = S.st[t];
    st.reserve(nb.size());
    double s = (double)g.w[k], r = 0;
    for (int u : nb) {
      st.push_back(S.pos[u]);
      r += (double)g.w[u];
    }
    std::sort(st.begin(), st.end());
    S.nnz_struct += (int64_t)st.size();
    S.flops_factor += s * s * s / 3.0 + r * s * s + r * r * s;
    S.flops_solve += 2.0 * (s * s + 2.0 * r * s);
  }
  S.parent.assign(n, -1);
  S.level.assign(n, 0);
  for (int t = 0; t < n; ++t)
    if (!S.st[t].empty()) S.parent[t] = S.st[t][0];
  for (int t = 0; t < n; ++t)
    if (S.parent[t] >= 0) S.level[S.parent[t]] = std::max(S.level[S.parent[t]], S.level[t] + 1);
  S.nlevels = 0;
  for (int t = 0; t < n; ++t) S.nlevels = std::max(S.nlevels, S.level[t] + 1);
  S.level_nodes.assign(S.nlevels, {});
  for (int t = 0; t < n; ++t) S.level_nodes[S.level[t]].push_back(t);
  return S;
}

double order_flops(const Graph& g, const std::vector<int>& order) {
  const int n = g.n;
  BitGraph B;
  B.init(g);
  Bitset elim;
  elim.init(n);
  double fl = 0;
  std::vector<int> nb;
  for (int t = 0; t < n; ++t) {
    int k = order[t];
    nb.clear();
    for_bits(B.row(k), elim.d.data(), B.words, [&](int u) { nb.push_back(u); });
    double s = (double)g.w[k], r = 0;
    for (int a : nb) {
      uint64_t* ra = B.row(a);
      const uint64_t* rk = B.row(k);
      for (int w = 0; w < B.words; ++w) ra[w] |= rk[w] & ~elim.d[w];
      ra[a >> 6] &= ~(1ull << (a & 63));
      r += (double)g.w[a];
    }
    elim.set(k);
    fl += s * s * s / 3.0 + r * s * s + r * r * s;
  }
  return fl;
}

// ----------------------------------------------------------------------------- min degree
std::vector<int> order_mindeg(const Graph& g) {
  const int n = g.n;
  BitGraph B;
  B.init(g);
  Bitset elim;
  elim.init(n);
  std::vector<int64_t> deg(n, 0);
  for (int v = 0; v < n; ++v)
    for (int u : g.adj[v]) deg[v] += g.w[u];
  std::vector<int> order;
  order.reserve(n);
  std::vector<int> nb;
  for (int step = 0; step < n; ++step) {
    int best = -1;
    for (int v = 0; v < n; ++v)
      if (!elim.get(v) && (best < 0 || deg[v] < deg[best])) best = v;  // ties -> lowest id
    int k = best;
    nb.clear();
    for_bits(B.row(k), elim.d.data(), B.words, [&](int u) { nb.push_back(u); });
    elim.set(k);
    for (int a : nb) {
      uint64_t* ra = B.row(a);
      const uint64_t* rk = B.row(k);
      for (int w = 0; w < B.words; ++w) ra[w] |= rk[w] & ~elim.d[w];
      ra[a >> 6] &= ~(1ull << (a & 63));
      int64_t d = 0;
      for_bits(ra, elim.d.data(), B.words, [&](int u) { d += g.w[u]; });
      deg[a] = d;
    }
    order.push_back(k);
  }
  return order;
}

// ----------------------------------------------------------------------------- nested dissection
namespace {

struct Sub {  // induced subgraph with local ids
  std::vector<int> glob;                 // local -> global
  std::vector<std::vector<int>> adj;     // local adjacency
  std::vector<int64_t> w;
};

Sub induced(const Graph& g, const std::vector<int>& V, std::vector<int>& loc /* size g.n, -1 */) {
  Sub s;
  s.glob = V;
  for (size_t i = 0; i < V.size(); ++i) loc[V[i]] = (int)i;
  s.adj.assign(V.size(), {});
  s.w.resize(V.size());
  for (size_t i = 0; i < V.size(); ++i) {
    s.w[i] = g.w[V[i]];
    for (int u : g.adj[V[i]])
      if (loc[u] >= 0) s.adj[i].push_back(loc[u]);
  }
  for (int v : V) loc[v] = -1;
  return s;
}

Graph as_graph(const Sub& s) {
  Graph g;
  g.n = (int)s.glob.size();
  g.adj = s.adj;
  g.w = s.w;
  return g;
}

std::vector<int> bfs_levels(const Sub& s, int root, int& nlev) {
  std::vector<int> lev(s.glob.size(), -1);
  std::queue<int> q;
  q.push(root);
  lev[root] = 0;
  nlev = 1;
  while (!q.empty()) {
    int v = q.front();
    q.pop();
    for (int u : s.adj[v])
      if (lev[u] < 0) {
        lev[u] = lev[v] + 1;
        nlev = std::max(nlev, lev[u] + 1);
        q.push(u);
      }
  }
  return lev;
}

std::vector<std::vector<int>> components(const Sub& s) {
  int m = (int)s.glob.size();
  std::vector<int> c(m, -1);
  std::vector<std::vector<int>> out;
  for (int v = 0; v < m; ++v) {
    if (c[v] >= 0) continue;
    out.push_back({});
    std::vector<int> stk{v};
    c[v] = (int)out.size() - 1;
    while (!stk.empty()) {
      int x = stk.back();
      stk.pop_back();
      out.back().push_back(x);
      for (int u : s.adj[x])
        if (c[u] < 0) {
          c[u] = c[v];
          stk.push_back(u);
        }
    }
  }
  return out;
}

// score of a vertex separator: w(S) scaled by imbalance (== w(S) when perfectly balanced)
double sep_score(int64_t wS, int64_t wA, int64_t wB) {
  if (wA <= 0 || wB <= 0) return 1e300;
  double W = (double)(wA + wB);
  return (double)wS * W * W / (4.0 * (double)wA * (double)wB);
}

// Vertex-separator FM refinement with locking and rollback to the best state.
void refine_fm(const Sub& s, std::vector<int>& side, double maxfrac) {
  const int m = (int)s.glob.size();
  auto weights = [&](int64_t& wA, int64_t& wB, int64_t& wS) {
    wA = wB = wS = 0;
    for (int v = 0; v < m; ++v) (side[v] == 0 ? wA : side[v] == 1 ? wB : wS) += s.w[v];
  };
  for (int pass = 0; pass < 8; ++pass) {
    int64_t wA, wB, wS;
    weights(wA, wB, wS);
    double best = sep_score(wS, wA, wB);
    std::vector<int> best_side = side;
    std::vector<char> locked(m, 0);
    bool improved = false;
    for (int mv = 0; mv < m; ++mv) {
      // best admissible move of a separator vertex into A or B
      int bv = -1, bx = -1;
      double bsc = 1e300;
      int64_t tot = wA + wB + wS;
      for (int v = 0; v < m; ++v) {
        if (side[v] != 2 || locked[v]) continue;
        for (int X = 0; X < 2; ++X) {
          int Y = 1 - X;
          int64_t moved = 0;
          for (int u : s.adj[v])
            if (side[u] == Y) moved += s.w[u];
          int64_t nX = (X == 0 ? wA : wB) + s.w[v], nY = (Y == 0 ? wA : wB) - moved;
          int64_t nS = wS - s.w[v] + moved;
          if ((double)std::max(nX, nY) > maxfrac * (double)(tot)) continue;
          double sc = sep_score(nS, X == 0 ? nX : nY, X == 0 ? nY : nX);
          if (sc < bsc) {
            bsc = sc;
            bv = v;
            bx = X;
          }
        }
      }
      if (bv < 0) break;
      int Y = 1 - bx;
      side[bv] = bx;
      locked[bv] = 1;
      for (int u : s.adj[bv])
        if (side[u] == Y) {
          side[u] = 2;
          locked[u] = 1;
        }
      weights(wA, wB, wS);
      double sc = sep_score(wS, wA, wB);
      if (sc < best - 1e-9) {
        best = sc;
        best_side = side;
        improved = true;
      }
    }
    side = best_side;
    if (!improved) break;
  }
}

// Returns side[] (0 = A, 1 = B, 2 = S) for a connected subgraph, or empty if no useful split.
std::vector<int> find_separator(const Sub& s, double maxfrac) {
  const int m = (int)s.glob.size();
  std::vector<int> roots;
  // pseudo-peripheral roots from a few seeds
  int seeds[4] = {0, m / 3, (2 * m) / 3, m - 1};
  for (int sd : seeds) {
    int r = sd, nl;
    for (int it = 0; it < 4; ++it) {
      auto lev = bfs_levels(s, r, nl);
      int far = r;
      for (int v = 0; v < m; ++v)
        if (lev[v] == nl - 1 && (s.adj[v].size() < s.adj[far].size() || lev[far] != nl - 1)) far = v;
      if (far == r) break;
      r = far;
    }
    roots.push_back(r);
    roots.push_back(sd);
  }
  std::sort(roots.begin(), roots.end());
  roots.erase(std::unique(roots.begin(), roots.end()), roots.end());
  double best = 1e300;
  std::vector<int> best_side;
  for (int r : roots) {
    int nl;
    auto lev = bfs_levels(s, r, nl);
    if (nl < 3) continue;
    std::vector<int64_t> lw(nl, 0);
    for (int v = 0; v < m; ++v) lw[lev[v]] += s.w[v];
    std::vector<int64_t> pre(nl + 1, 0);
    for (int l = 0; l < nl; ++l) pre[l + 1] = pre[l] + lw[l];
    for (int l = 1; l < nl - 1; ++l) {
      int64_t wA = pre[l], wS = lw[l], wB = pre[nl] - pre[l + 1];
      double sc = sep_score(wS, wA, wB);
      std::vector<int> side(m);
      for (int v = 0; v < m; ++v) side[v] = lev[v] < l ? 0 : (lev[v] == l ? 2 : 1);
      refine_fm(s, side, maxfrac);
      int64_t a = 0, b = 0, c = 0;
      for (int v = 0; v < m; ++v) (side[v] == 0 ? a : side[v] == 1 ? b : c) += s.w[v];
      sc = sep_score(c, a, b);
      if (sc < best) {
        best = sc;
        best_side = side;
      }
    }
  }
  return best_side;
}

void nd_rec(const Graph& g, const std::vector<int>& V, int leaf, double maxfrac, std::vector<int>& loc,
            std::vector<int>& out) {
  if (V.empty()) return;
  Sub s = induced(g, V, loc);
  auto comps = components(s);
  if (comps.size() > 1) {
    for (auto& c : comps) {
      std::vector<int> W;
      for (int x : c) W.push_back(s.glob[x]);
      std::sort(W.begin(), W.end());
      nd_rec(g, W, leaf, maxfrac, loc, out);
    }
    return;
  }
  auto md_local = [&]() {
    Graph lg = as_graph(s);
    for (int x : order_mindeg(lg)) out.push_back(s.glob[x]);
  };
  if ((int)V.size() <= leaf) {
    md_local();
    return;
  }
  auto side = find_separator(s, maxfrac);
  if (side.empty()) {
    md_local();
    return;
  }
  std::vector<int> A, B, S;
  for (int v = 0; v < (int)V.size(); ++v) (side[v] == 0 ? A : side[v] == 1 ? B : S).push_back(s.glob[v]);
  if (A.empty() || B.empty()) {
    md_local();
    return;
  }
  nd_rec(g, A, leaf, maxfrac, loc, out);
  nd_rec(g, B, leaf, maxfrac, loc, out);
  // separator last, ordered by minimum degree on its induced subgraph
  Sub ss = induced(g, S, loc);
  Graph sg = as_graph(ss);
  for (int x : order_mindeg(sg)) out.push_back(ss.glob[x]);
}

}  // namespace

std::vector<int> order_nd(const Graph& g) {
  std::vector<int> V(g.n);
  std::iota(V.begin(), V.end(), 0);
  std::vector<int> loc(g.n, -1);
  std::vector<int> best;
  double bestf = 1e300;
  const int leaves[] = {2, 6};
  const double fracs[] = {0.6, 0.7};
  for (int leaf : leaves)
    for (double fr : fracs) {
      std::vector<int> out;
      out.reserve(g.n);
      nd_rec(g, V, leaf, fr, loc, out);
      double f = order_flops(g, out);
      if (f < bestf) {
        bestf = f;
        best = out;
      }
    }
  return best;
}

}  // namespace ddaux
