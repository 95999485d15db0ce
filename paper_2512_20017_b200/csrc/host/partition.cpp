// Native multilevel k-way graph partitioner of the offline point placement
// (PAPER.md:590-612): one run of the reference scheme of
// /root/reference/pkg/src/splatsched/partition.py:104-434, reproduced
// decision for decision so the labels are identical to the reference's.
//
//   coarsening   heavy-edge matching, vertices in index order, ties among
//                equally heavy free neighbours broken by Generator.integers
//                (partition.py:133-186); stop at <= 30 * parts vertices or
//                when a level shrinks by < 5 %
//   initial      greedy growth of parts 0..k-2 from random seeds, most
//                connected free vertex next, leftovers to part k-1
//                (partition.py:189-223)
//   refinement   forced rebalance (move minimising (-gain, target weight,
//                v, t)), then repeated best single-vertex moves: the
//                largest strictly positive cut gain (first in (v, t) order),
//                else a zero-gain move that strictly lowers the sum of
//                squared part weights (partition.py:248-327)
//
// The random draws are numpy's: PCG64 (XSL-RR 128/64) stepping the state the
// caller extracted from np.random.default_rng(SeedSequence([seed, run])),
// with Generator.integers(n) = Lemire's bounded 32-bit method over
// next_uint32 (which halves one 64-bit output).  All weights are integers
// (or multiples of 0.5) held in doubles, so every sum is exact and the
// arithmetic cannot diverge from numpy's.  Where the reference rescans all
// vertices per step (O(n) per grown vertex, O(n k) per refinement move; it
// needs 129 s at 10k groups), this port keeps max
// trees keyed exactly like numpy's argmax (largest value, lowest index) and
// updates only the entries a step changes: O((deg + 1) k log n) per move.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "../../../include/splat_host.h"

namespace {

using u128 = unsigned __int128;

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t u32;
  uint64_t next64() {
    const u128 mult = (static_cast<u128>(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
    const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32;
    }
    const uint64_t n = next64();
    has32 = true;
    u32 = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n & 0xffffffffu);
  }
  // Generator.integers(n), n >= 1 (random_bounded_uint64_fill, Lemire, unmasked)
  int64_t integers(int64_t n) {
    const uint64_t rng = static_cast<uint64_t>(n - 1);
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFULL) return static_cast<int64_t>(next32());
    if (rng < 0xFFFFFFFFULL) {
      const uint32_t r32 = static_cast<uint32_t>(rng), excl = r32 + 1u;
      uint64_t m = static_cast<uint64_t>(next32()) * excl;
      uint32_t left = static_cast<uint32_t>(m);
      if (left < excl) {
        const uint32_t thr = (UINT32_MAX - r32) % excl;
        while (left < thr) {
          m = static_cast<uint64_t>(next32()) * excl;
          left = static_cast<uint32_t>(m);
        }
      }
      return static_cast<int64_t>(m >> 32);
    }
    // 64-bit Lemire (graphs beyond 4G vertices only)
    const uint64_t excl = rng + 1;
    u128 m = static_cast<u128>(next64()) * excl;
    uint64_t left = static_cast<uint64_t>(m);
    if (left < excl) {
      const uint64_t thr = (UINT64_MAX - rng) % excl;
      while (left < thr) {
        m = static_cast<u128>(next64()) * excl;
        left = static_cast<uint64_t>(m);
      }
    }
    return static_cast<int64_t>(m >> 64);
  }
};

// Max over positions with ties to the lowest index (= numpy argmax order);
// absent entries hold -inf.  O(log n) update, O(1) query of the root.
struct MaxTree {
  int64_t size = 1;
  std::vector<double> val;
  std::vector<int64_t> idx;
  void init(int64_t n) {
    size = 1;
    while (size < std::max<int64_t>(n, 1)) size <<= 1;
    val.assign(2 * size, -std::numeric_limits<double>::infinity());
    idx.assign(2 * size, INT64_MAX);
    for (int64_t i = 0; i < size; ++i) idx[size + i] = i;
    for (int64_t i = size - 1; i >= 1; --i) pull(i);
  }
  void pull(int64_t i) {
    const int64_t a = 2 * i, b = 2 * i + 1;
    if (val[b] > val[a] || (val[b] == val[a] && idx[b] < idx[a])) {
      val[i] = val[b];
      idx[i] = idx[b];
    } else {
      val[i] = val[a];
      idx[i] = idx[a];
    }
  }
  void set(int64_t pos, double v) {
    int64_t i = size + pos;
    val[i] = v;
    for (i >>= 1; i >= 1; i >>= 1) pull(i);
  }
  double top() const { return val[1]; }
  int64_t arg() const { return idx[1]; }
  // max over positions [0, end): (value, index), ties to the lowest index
  void prefix(int64_t end, double& v, int64_t& id) const {
    v = -std::numeric_limits<double>::infinity();
    id = INT64_MAX;
    int64_t lo = size, hi = size + end;
    auto take = [&](int64_t i) {
      if (val[i] > v || (val[i] == v && idx[i] < id)) {
        v = val[i];
        id = idx[i];
      }
    };
    while (lo < hi) {
      if (lo & 1) take(lo++);
      if (hi & 1) take(--hi);
      lo >>= 1;
      hi >>= 1;
    }
  }
};

// Counts of free vertices for "the r-th free vertex in index order".
struct CountTree {
  int64_t size = 1;
  std::vector<int64_t> cnt;
  void init(int64_t n) {
    size = 1;
    while (size < std::max<int64_t>(n, 1)) size <<= 1;
    cnt.assign(2 * size, 0);
    for (int64_t i = 0; i < n; ++i) cnt[size + i] = 1;
    for (int64_t i = size - 1; i >= 1; --i) cnt[i] = cnt[2 * i] + cnt[2 * i + 1];
  }
  void clear(int64_t pos) {
    for (int64_t i = size + pos; i >= 1; i >>= 1) --cnt[i];
  }
  int64_t total() const { return cnt[1]; }
  int64_t kth(int64_t r) const {  // 0-based
    int64_t i = 1;
    while (i < size) {
      if (r < cnt[2 * i]) i = 2 * i;
      else {
        r -= cnt[2 * i];
        i = 2 * i + 1;
      }
    }
    return i - size;
  }
};

// Undirected weighted graph: edge list (eu < ev not required) + CSR
// adjacency with neighbours ascending (WeightedGraph, partition.py:104-131).
struct Graph {
  int64_t n = 0;
  std::vector<double> bal;
  std::vector<int64_t> eu, ev;
  std::vector<double> ew;
  std::vector<int64_t> ptr, adj;
  std::vector<double> adj_w;

  void build_adjacency() {
    const int64_t m = static_cast<int64_t>(eu.size());
    std::vector<int64_t> deg(n, 0);
    for (int64_t e = 0; e < m; ++e) {
      ++deg[eu[e]];
      ++deg[ev[e]];
    }
    ptr.assign(n + 1, 0);
    for (int64_t v = 0; v < n; ++v) ptr[v + 1] = ptr[v] + deg[v];
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    adj.resize(2 * m);
    adj_w.resize(2 * m);
    for (int64_t e = 0; e < m; ++e) {
      adj[fill[eu[e]]] = ev[e];
      adj_w[fill[eu[e]]++] = ew[e];
      adj[fill[ev[e]]] = eu[e];
      adj_w[fill[ev[e]]++] = ew[e];
    }
    std::vector<std::pair<int64_t, double>> tmp;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t a = ptr[v], b = ptr[v + 1];
      tmp.clear();
      for (int64_t i = a; i < b; ++i) tmp.emplace_back(adj[i], adj_w[i]);
      std::stable_sort(tmp.begin(), tmp.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (int64_t i = a; i < b; ++i) {
        adj[i] = tmp[i - a].first;
        adj_w[i] = tmp[i - a].second;
      }
    }
  }
};

class Multilevel {
 public:
  Multilevel(int k, double eps, Pcg64 rng) : k_(k), eps_(eps), rng_(rng) {}

  std::vector<int64_t> run(const Graph& g) {
    double total = 0.0;
    for (double b : g.bal) total += b;
    const double cap = (1.0 + eps_) * total / k_;
    std::vector<Graph> stack;
    std::vector<std::vector<int64_t>> maps;
    stack.push_back(g);
    while (stack.back().n > 30 * static_cast<int64_t>(k_)) {
      Graph next;
      std::vector<int64_t> cid;
      if (!contract(stack.back(), cap, next, cid)) break;
      const int64_t prev_n = stack.back().n;
      stack.push_back(std::move(next));
      maps.push_back(std::move(cid));
      if (prev_n - stack.back().n < std::max<int64_t>(1, prev_n / 20)) break;
    }
    const bool dbg = getenv("BS_PART_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "levels=%zu coarsest n=%ld\n", stack.size(), (long)stack.back().n);
    std::vector<int64_t> lab = grow(stack.back());
    refine(stack.back(), lab, cap);
    for (int64_t level = static_cast<int64_t>(maps.size()) - 1; level >= 0; --level) {
      const auto& m = maps[level];
      std::vector<int64_t> fine(stack[level].n);
      for (int64_t v = 0; v < stack[level].n; ++v) fine[v] = lab[m[v]];
      lab.swap(fine);
      refine(stack[level], lab, cap);
    }
    return lab;
  }

 private:
  int k_;
  double eps_;
  Pcg64 rng_;

  // heavy-edge matching + contraction (partition.py:133-186)
  bool contract(const Graph& g, double cap, Graph& out, std::vector<int64_t>& cid) {
    std::vector<int64_t> mate(g.n, -1), pool;
    bool any = false;
    for (int64_t v = 0; v < g.n; ++v) {
      if (mate[v] != -1) continue;
      double heavy = -std::numeric_limits<double>::infinity();
      bool ok_any = false;
      for (int64_t i = g.ptr[v]; i < g.ptr[v + 1]; ++i) {
        const int64_t u = g.adj[i];
        if (mate[u] != -1 || u == v || g.bal[v] + g.bal[u] > cap) continue;
        ok_any = true;
        heavy = std::max(heavy, g.adj_w[i]);
      }
      if (!ok_any) continue;
      pool.clear();
      for (int64_t i = g.ptr[v]; i < g.ptr[v + 1]; ++i) {
        const int64_t u = g.adj[i];
        if (mate[u] != -1 || u == v || g.bal[v] + g.bal[u] > cap) continue;
        if (g.adj_w[i] == heavy) pool.push_back(u);
      }
      const int64_t u = pool.size() > 1 ? pool[rng_.integers(static_cast<int64_t>(pool.size()))] : pool[0];
      mate[v] = u;
      mate[u] = v;
      any = true;
    }
    if (!any) return false;
    cid.assign(g.n, -1);
    int64_t nxt = 0;
    for (int64_t v = 0; v < g.n; ++v) {
      if (cid[v] == -1) {
        cid[v] = nxt;
        if (mate[v] != -1) cid[mate[v]] = nxt;
        ++nxt;
      }
    }
    out.n = nxt;
    out.bal.assign(nxt, 0.0);
    for (int64_t v = 0; v < g.n; ++v) out.bal[cid[v]] += g.bal[v];
    struct E {
      int64_t key, lo, hi;
      double w;
    };
    std::vector<E> es;
    es.reserve(g.eu.size());
    for (size_t e = 0; e < g.eu.size(); ++e) {
      const int64_t a = cid[g.eu[e]], b = cid[g.ev[e]];
      if (a == b) continue;
      const int64_t lo = std::min(a, b), hi = std::max(a, b);
      es.push_back({lo * nxt + hi, lo, hi, g.ew[e]});
    }
    std::stable_sort(es.begin(), es.end(), [](const E& x, const E& y) { return x.key < y.key; });
    out.eu.clear();
    out.ev.clear();
    out.ew.clear();
    for (size_t i = 0; i < es.size(); ++i) {
      if (i == 0 || es[i].key != es[i - 1].key) {
        out.eu.push_back(es[i].lo);
        out.ev.push_back(es[i].hi);
        out.ew.push_back(es[i].w);
      } else {
        out.ew.back() += es[i].w;
      }
    }
    out.build_adjacency();
    return true;
  }

  // greedy graph growing (partition.py:189-223).  The free vertices live in
  // a count tree (random seed = the r-th free one) and a max tree of their
  // link weights (next = first free vertex of maximal link).
  std::vector<int64_t> grow(const Graph& g) {
    const int k = k_;
    std::vector<int64_t> lab(g.n, -1);
    int64_t left = g.n;
    double total = 0.0;
    for (double b : g.bal) total += b;
    const double goal = total / k;
    std::vector<double> link(g.n, 0.0);
    CountTree freec;
    freec.init(g.n);
    MaxTree lt;
    lt.init(g.n);
    for (int part = 0; part < k - 1; ++part) {
      if (left <= k - part - 1) break;
      int64_t cur = freec.kth(rng_.integers(freec.total()));
      // link[:] = 0 for every vertex; the tree holds the free ones
      std::fill(link.begin(), link.end(), 0.0);
      for (int64_t v = 0; v < g.n; ++v) lt.val[lt.size + v] = lab[v] == -1 ? 0.0 : -std::numeric_limits<double>::infinity();
      for (int64_t i = lt.size - 1; i >= 1; --i) lt.pull(i);
      double mass = 0.0;
      while (true) {
        lab[cur] = part;
        --left;
        mass += g.bal[cur];
        freec.clear(cur);
        lt.set(cur, -std::numeric_limits<double>::infinity());
        for (int64_t i = g.ptr[cur]; i < g.ptr[cur + 1]; ++i) {
          const int64_t u = g.adj[i];
          if (lab[u] == -1) {
            link[u] += g.adj_w[i];
            lt.set(u, link[u]);
          }
        }
        if (mass >= goal || left <= k - part - 1) break;
        if (lt.top() > 0.0) cur = lt.arg();
        else cur = freec.kth(rng_.integers(freec.total()));
      }
    }
    for (auto& l : lab)
      if (l == -1) l = k - 1;
    return lab;
  }

  void move(const Graph& g, std::vector<double>& aff, std::vector<int64_t>& lab, int64_t v, int64_t dst) {
    const int64_t src = lab[v];
    for (int64_t i = g.ptr[v]; i < g.ptr[v + 1]; ++i) {
      aff[g.adj[i] * k_ + src] -= g.adj_w[i];
      aff[g.adj[i] * k_ + dst] += g.adj_w[i];
    }
    lab[v] = dst;
  }

  // partition.py:248-275
  void force_balance(const Graph& g, std::vector<int64_t>& lab, double cap, std::vector<double>& aff,
                     std::vector<double>& pw) {
    const int k = k_;
    int64_t budget = 10 * g.n + 10;
    while (budget > 0) {
      int64_t heavy = -1;
      for (int p = 0; p < k; ++p)
        if (pw[p] > cap && (heavy < 0 || pw[p] > pw[heavy])) heavy = p;
      if (heavy < 0) return;
      --budget;
      bool found = false, any_cand = false;
      double b_ng = 0.0, b_pw = 0.0;
      int64_t b_v = -1, b_t = -1;
      for (int64_t v = 0; v < g.n; ++v) {
        if (lab[v] != heavy || !(g.bal[v] > 0.0)) continue;
        any_cand = true;
        for (int t = 0; t < k; ++t) {
          if (t == heavy) continue;
          const double room = cap - (pw[t] + g.bal[v]);
          if (room < 0.0) continue;
          const double ng = -(aff[v * k + t] - aff[v * k + heavy]);
          bool better = !found;
          if (found) {
            if (ng != b_ng) better = ng < b_ng;
            else if (pw[t] != b_pw) better = pw[t] < b_pw;
            else if (v != b_v) better = v < b_v;
            else better = t < b_t;
          }
          if (better) {
            found = true;
            b_ng = ng;
            b_pw = pw[t];
            b_v = v;
            b_t = t;
          }
        }
      }
      if (!any_cand || !found) return;
      pw[heavy] -= g.bal[b_v];
      pw[b_t] += g.bal[b_v];
      move(g, aff, lab, b_v, b_t);
    }
  }

  // partition.py:277-327.  Gains live in one max tree per target part over
  // the vertices in balance order, so the vertices a target can take
  // (pw[t] + bal[v] <= cap) are a prefix; each tree answers "largest gain,
  // lowest vertex" for its prefix, and the best over targets (ties to the
  // lowest (v, t)) is the reference's argmax over the feasible gain matrix.
  // A move updates the k leaves of the moved vertex and of its neighbours.
  void refine(const Graph& g, std::vector<int64_t>& lab, double cap) {
    const int k = k_;
    const int64_t n = g.n, limit = 100 * n + 100;
    std::vector<double> aff(static_cast<size_t>(n) * k, 0.0), pw(k, 0.0);
    for (size_t e = 0; e < g.eu.size(); ++e) {
      aff[g.eu[e] * k + lab[g.ev[e]]] += g.ew[e];
      aff[g.ev[e] * k + lab[g.eu[e]]] += g.ew[e];
    }
    for (int64_t v = 0; v < n; ++v) pw[lab[v]] += g.bal[v];
    force_balance(g, lab, cap, aff, pw);
    const double ninf = -std::numeric_limits<double>::infinity();
    std::vector<int64_t> by_bal(n), pos(n);
    std::iota(by_bal.begin(), by_bal.end(), 0);
    std::stable_sort(by_bal.begin(), by_bal.end(), [&](int64_t a, int64_t b) { return g.bal[a] < g.bal[b]; });
    for (int64_t i = 0; i < n; ++i) pos[by_bal[i]] = i;
    std::vector<MaxTree> tree(k);
    for (int t = 0; t < k; ++t) {
      tree[t].init(n);
      for (int64_t v = 0; v < n; ++v) {
        tree[t].idx[tree[t].size + pos[v]] = v;
        tree[t].val[tree[t].size + pos[v]] = t == lab[v] ? ninf : aff[v * k + t] - aff[v * k + lab[v]];
      }
      for (int64_t i = tree[t].size - 1; i >= 1; --i) tree[t].pull(i);
    }
    // zmask[v]: targets t != lab[v] with gain(v, t) == 0 (zero-gain candidates)
    std::vector<uint32_t> zmask(n, 0u);
    auto update = [&](int64_t v) {
      const double own = aff[v * k + lab[v]];
      uint32_t z = 0u;
      for (int t = 0; t < k; ++t) {
        const double gain = t == lab[v] ? ninf : aff[v * k + t] - own;
        if (gain == 0.0) z |= 1u << t;
        tree[t].set(pos[v], gain);
      }
      zmask[v] = z;
    };
    for (int64_t v = 0; v < n; ++v) {
      const double own = aff[v * k + lab[v]];
      for (int t = 0; t < k; ++t)
        if (t != lab[v] && aff[v * k + t] - own == 0.0) zmask[v] |= 1u << t;
    }

    auto feasible_end = [&](int t) {  // vertices (in balance order) part t can take
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (pw[t] + g.bal[by_bal[mid]] <= cap) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    int64_t it = 0, zero_moves = 0;
    for (; it < limit; ++it) {
      double top = ninf;
      int64_t mv = INT64_MAX;
      int mt = -1;
      for (int t = 0; t < k; ++t) {
        double v;
        int64_t id;
        tree[t].prefix(feasible_end(t), v, id);
        if (v == ninf) continue;
        if (v > top || (v == top && id < mv)) {
          top = v;
          mv = id;
          mt = t;
        }
      }
      if (top < 0.0 || mt < 0) break;
      if (!(top > 0.0)) {
        ++zero_moves;
        // zero-gain move lowering sum(pw^2) the most (first strict minimum in
        // (v, t) order)
        double best = 0.0;
        mv = -1;
        mt = -1;
        for (int64_t v = 0; v < n; ++v) {
          uint32_t z = zmask[v];
          const double w = g.bal[v];
          if (z == 0u || w == 0.0) continue;
          for (; z; z &= z - 1) {
            const int t = __builtin_ctz(z);
            if (!(pw[t] + w <= cap)) continue;
            const double delta = 2.0 * w * (pw[t] - pw[lab[v]] + w);
            if (delta < best - 1e-12) {
              best = delta;
              mv = v;
              mt = t;
            }
          }
        }
        if (mv < 0) break;
      }
      pw[lab[mv]] -= g.bal[mv];
      pw[mt] += g.bal[mv];
      move(g, aff, lab, mv, mt);
      update(mv);
      for (int64_t i = g.ptr[mv]; i < g.ptr[mv + 1]; ++i) update(g.adj[i]);
    }
    if (getenv("BS_PART_DEBUG")) fprintf(stderr, "refine n=%ld moves=%ld zero=%ld\n", (long)n, (long)it, (long)zero_moves);
  }
};

}  // namespace

extern "C" int32_t bs_partition_multilevel(int64_t n, const double* balance, int64_t n_edges, const int64_t* eu,
                                           const int64_t* ev, const double* ew, int32_t parts, double eps,
                                           const uint64_t* pcg_state, int64_t* labels) {
  if (n < 1 || parts < 2 || !balance || !labels || !pcg_state || n_edges < 0 || (n_edges > 0 && (!eu || !ev || !ew)))
    return BS_HOST_ERR_PARAMETER;
  Graph g;
  g.n = n;
  g.bal.assign(balance, balance + n);
  g.eu.assign(eu, eu + n_edges);
  g.ev.assign(ev, ev + n_edges);
  g.ew.assign(ew, ew + n_edges);
  for (int64_t e = 0; e < n_edges; ++e)
    if (g.eu[e] < 0 || g.eu[e] >= n || g.ev[e] < 0 || g.ev[e] >= n) return BS_HOST_ERR_PARAMETER;
  g.build_adjacency();
  Pcg64 rng;
  rng.state = (static_cast<u128>(pcg_state[0]) << 64) | pcg_state[1];
  rng.inc = (static_cast<u128>(pcg_state[2]) << 64) | pcg_state[3];
  rng.has32 = pcg_state[4] != 0;
  rng.u32 = static_cast<uint32_t>(pcg_state[5]);
  Multilevel ml(parts, eps, rng);
  const std::vector<int64_t> lab = ml.run(g);
  std::memcpy(labels, lab.data(), sizeof(int64_t) * n);
  return BS_HOST_OK;
}
