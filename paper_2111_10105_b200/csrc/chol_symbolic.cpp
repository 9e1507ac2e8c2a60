// Host analysis + CPU reference numerics for the supernodal Cholesky of
// M = L^T L + S^T S (see chol.h).  The fill-reducing ordering is nested
// dissection by BFS level sets on M's graph (a single level of M's graph is
// a vertex separator of M), the same scheme the oracle uses for its sparse
// LDL^T restatement of SimplicialLDLT.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <functional>
#include <thread>
#include <mutex>
#include <map>

#include "chol.h"
#include "par.h"

namespace dmcg {

namespace {

struct Graph {
  uint32_t n;
  const uint32_t* rp;
  const uint32_t* ci;
};

// Nested dissection on M's graph.  Each sub-problem is a contiguous range
// of one index array, partitioned in place (parts A | B | separator S);
// two BFS per split: from any vertex to the farthest one (pseudo-
// peripheral), then the level structure from there.  A BFS marks a vertex
// visited by moving it to a fresh part id (one random read per edge, no
// per-vertex level array) and its queue, which holds the vertices level by
// level, is the new order of the range: A = the levels before the
// separator, S = the separator levels, B = the levels after it are
// contiguous pieces of the queue.  Leaves of <= 48 vertices keep their
// order.  Because every range is partitioned in place as A | B | S, the
// final index array IS the elimination order (old indices; A's order, then
// B's, then S).  The two halves of the upper dissection levels run on
// separate threads: they touch disjoint ranges, and the only cross-range
// read (part_ of a neighbour) compares against an id the other range never
// holds.
class NestedDissection {
 public:
  // wide: g is the 1-ring graph G of a matrix whose pattern is G^2 (M = L^T L
  // + S^T S); two consecutive BFS levels of G separate G^2 (every 2-path
  // between the levels before and after them passes through one of the two),
  // at a third of the edge visits of BFS on G^2.
  explicit NestedDissection(const Graph& g, bool wide = false)
      : g_(g), wide_(wide), part_(g.n, 0), queue_(g.n), idx_(g.n), lstart_(2 * (size_t)g.n + 2) {}

  std::vector<uint32_t> run() {
    for (uint32_t i = 0; i < g_.n; ++i) idx_[i] = i;
    process(0, g_.n, 0, 0);
    return std::move(idx_);
  }

  // The splits of ranges of >= kSplitRecord vertices, (b << 32 | e) ->
  // (end of A, end of B): in the final order, A | B | S of a range.  Rows of
  // A reference only A (B, S come later or are not adjacent), so the
  // elimination tree of A and of B can be built concurrently.
  static constexpr uint32_t kSplitRecord = 8192;
  std::map<uint64_t, std::pair<uint32_t, uint32_t>> splits;

 private:
  static constexpr int kParDepth = 4;      // up to 2^4 concurrent ranges
  static constexpr uint32_t kParMin = 4096;  // smallest half worth a thread
  const Graph g_;
  const bool wide_;
  // ranges of <= leaf_ vertices are not dissected further (one leaf front each)
  const uint32_t leaf_ = [] {
    const char* e = std::getenv("DMCG_ND_LEAF");
    return e ? (uint32_t)std::max(49, std::atoi(e)) : 48u;
  }();
  std::vector<int32_t> part_;
  std::vector<uint32_t> queue_, idx_;
  std::vector<uint32_t> lstart_;  // level starts of the last BFS of a range, at [2 b + level]
  std::atomic<int32_t> next_id_{1};
  std::mutex split_mu_;

  int32_t part(uint32_t v) const { return __atomic_load_n(&part_[v], __ATOMIC_RELAXED); }
  void set_part(uint32_t v, int32_t id) { __atomic_store_n(&part_[v], id, __ATOMIC_RELAXED); }

  void process(uint32_t b0, uint32_t e0, int32_t id0, int depth0) {
    struct Task {
      uint32_t b, e;
      int32_t id;
      int depth;
    };
    std::vector<Task> st;
    st.push_back({b0, e0, id0, depth0});
    while (!st.empty()) {
      const Task t = st.back();
      st.pop_back();
      if (t.e - t.b <= leaf_) continue;
      uint32_t na, ns;
      int32_t ia, ib;
      if (split(t.b, t.e, t.id, &na, &ns, &ia, &ib) == 0) continue;  // no useful split
      const uint32_t e_a = t.b + na, e_b = t.e - ns;
      if (t.e - t.b >= kSplitRecord) {
        std::lock_guard<std::mutex> lk(split_mu_);
        splits[((uint64_t)t.b << 32) | t.e] = {e_a, e_b};
      }
      if (t.depth < kParDepth && na >= kParMin && e_b - e_a >= kParMin) {
        std::thread th([this, t, e_a, ia] { process(t.b, e_a, ia, t.depth + 1); });
        process(e_a, e_b, ib, t.depth + 1);
        th.join();
        continue;
      }
      st.push_back({e_a, e_b, ib, t.depth + 1});
      st.push_back({t.b, e_a, ia, t.depth + 1});
    }
  }

  // BFS over the vertices of part `from`, moving every reached vertex to part
  // `to`; queue = range-local buffer, lstart[l] = queue position where level l
  // begins (lstart[levels] = reached).  Returns the number of levels.
  uint32_t bfs(uint32_t root, int32_t from, int32_t to, uint32_t* queue, uint32_t* lstart,
               uint32_t* reached) {
    uint32_t head = 0, tail = 0, levels = 0;
    queue[tail++] = root;
    set_part(root, to);
    while (head < tail) {
      lstart[levels++] = head;
      for (const uint32_t lend = tail; head < lend; ++head) {
        const uint32_t v = queue[head];
        for (uint32_t p = g_.rp[v]; p < g_.rp[v + 1]; ++p) {
          const uint32_t w = g_.ci[p];
          if (part(w) == from) {
            set_part(w, to);
            queue[tail++] = w;
          }
        }
      }
    }
    lstart[levels] = tail;
    *reached = tail;
    return levels;
  }

  // Partitions idx_[b, e) (all of part `id`) into A | B | S; *ia / *ib = the
  // part ids of A and B afterwards.  Returns 0 if no split is made (the range
  // keeps one id, returned in *ia); a disconnected range becomes A = reached
  // component, B = rest, S empty.
  int split(uint32_t b, uint32_t e, int32_t id, uint32_t* na, uint32_t* ns, int32_t* ia,
            int32_t* ib) {
    const uint32_t cnt = e - b;
    uint32_t* queue = queue_.data() + b;
    uint32_t* lstart = lstart_.data() + 2 * (size_t)b;  // <= cnt + 1 entries of the range's 2 cnt
    const int32_t t1 = next_id_.fetch_add(4), t2 = t1 + 1, t3 = t1 + 2, t4 = t1 + 3;
    uint32_t reached;
    uint32_t levels = bfs(idx_[b], id, t1, queue, lstart, &reached);
    if (reached < cnt) {
      // A = the reached component (now part t1) in BFS order, B = the rest (still `id`)
      uint32_t z = reached;
      for (uint32_t q = b; q < e; ++q) {
        const uint32_t v = idx_[q];
        if (part(v) == id) queue[z++] = v;
      }
      std::copy(queue, queue + cnt, idx_.begin() + b);
      *na = reached;
      *ns = 0;
      *ia = t1;
      *ib = id;
      return 1;
    }
    const uint32_t root = queue[cnt - 1];
    levels = bfs(root, t1, t2, queue, lstart, &reached);
    const uint32_t maxlev = levels - 1;
    const uint32_t wsep = wide_ ? 2u : 1u;  // separator levels
    *ia = t2;
    if (maxlev < 1 + wsep) {
      std::copy(queue, queue + cnt, idx_.begin() + b);
      return 0;
    }
    // separator = the level where the running count first exceeds half
    uint32_t sep = 1;
    for (uint32_t l = 0; l <= maxlev; ++l)
      if (lstart[l + 1] > cnt / 2) {
        sep = l;
        break;
      }
    if (sep == 0) sep = 1;
    if (sep + wsep > maxlev) sep = maxlev - wsep;
    const uint32_t sep_hi = sep + wsep - 1;  // separator = levels [sep, sep_hi]
    const uint32_t a_end = lstart[sep], s_end = lstart[sep_hi + 1];
    // new order: A = queue[0, a_end) | B = queue[s_end, cnt) | S = queue[a_end, s_end)
    uint32_t* dst = idx_.data() + b;
    std::copy(queue, queue + a_end, dst);
    std::copy(queue + s_end, queue + cnt, dst + a_end);
    std::copy(queue + a_end, queue + s_end, dst + a_end + (cnt - s_end));
    for (uint32_t q = s_end; q < cnt; ++q) set_part(queue[q], t3);
    for (uint32_t q = a_end; q < s_end; ++q) set_part(queue[q], t4);
    *ib = t3;
    *na = a_end;
    *ns = s_end - a_end;
    return 2;
  }
};

}  // namespace

void chol_order_graph(uint32_t n, const std::vector<uint32_t>& g_rp,
                      const std::vector<uint32_t>& g_ci, CholOrdering* out) {
  NestedDissection nd(Graph{n, g_rp.data(), g_ci.data()}, true);
  out->perm0 = nd.run();
  out->splits = std::move(nd.splits);
}

void chol_analyze(uint32_t n, const std::vector<uint32_t>& rp, const std::vector<uint32_t>& ci,
                  const std::vector<float>& val, CholPlan* P, const std::vector<uint32_t>* g_rp,
                  const std::vector<uint32_t>* g_ci, CholOrdering* pre) {
  CholPlan& p = *P;
  p = CholPlan();
  p.n = n;
  static const bool timing = std::getenv("DMCG_TIMING") != nullptr;
  auto clk = [] { return std::chrono::steady_clock::now(); };
  auto t_prev = clk();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t = clk();
    std::fprintf(stderr, "  chol_analyze %-12s %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_prev).count());
    t_prev = t;
  };
  // (1) ordering
  // the ordering runs on the 1-ring graph when the caller has it (M's pattern
  // is its square), else on M's own graph
  static const bool m_graph = std::getenv("DMCG_ND_MGRAPH") != nullptr;
  const bool wide = g_rp && g_ci && g_rp->size() == (size_t)n + 1 && !m_graph;
  CholOrdering own;
  if (!pre || pre->perm0.size() != n) {
    Graph g = wide ? Graph{n, g_rp->data(), g_ci->data()} : Graph{n, rp.data(), ci.data()};
    NestedDissection nd(g, wide);
    own.perm0 = nd.run();
    own.splits = std::move(nd.splits);
    pre = &own;
  }
  std::vector<uint32_t>& perm0 = pre->perm0;
  const auto& nd_splits = pre->splits;
  lap("ordering");
  std::vector<uint32_t> iperm0(n);
  for (uint32_t k = 0; k < n; ++k) iperm0[perm0[k]] = k;
  // strictly lower pattern of P M P^T (row k: columns r < k), built in
  // parallel so the sequential etree pass below streams contiguous rows
  std::vector<uint32_t> lp((size_t)n + 1, 0), li;
  {
    parallel_for(n, 2048, [&](uint32_t k0, uint32_t k1, uint32_t) {
      for (uint32_t k = k0; k < k1; ++k) {
        const uint32_t ko = perm0[k];
        uint32_t c = 0;
        for (uint32_t q = rp[ko]; q < rp[ko + 1]; ++q) c += iperm0[ci[q]] < k;
        lp[k + 1] = c;
      }
    });
    for (uint32_t k = 0; k < n; ++k) lp[k + 1] += lp[k];
    li.resize(lp[n]);
    parallel_for(n, 2048, [&](uint32_t k0, uint32_t k1, uint32_t) {
      for (uint32_t k = k0; k < k1; ++k) {
        const uint32_t ko = perm0[k];
        uint32_t o = lp[k];
        for (uint32_t q = rp[ko]; q < rp[ko + 1]; ++q) {
          const uint32_t r = iperm0[ci[q]];
          if (r < k) li[o++] = r;
        }
      }
    });
  }
  lap("lower pattern");
  // (2) elimination tree (Liu, path compression) of P M P^T; the two parts
  // of every recorded dissection split are independent (rows of A touch only
  // A), so their trees are built concurrently, the separator's rows after
  std::vector<int32_t> par(n, -1), anc(n, -1);
  auto liu = [&](uint32_t k0, uint32_t k1) {
    for (uint32_t k = k0; k < k1; ++k) {
      for (uint32_t q = lp[k]; q < lp[k + 1]; ++q) {
        int32_t r = (int32_t)li[q];
        while (anc[r] != -1 && anc[r] != (int32_t)k) {
          const int32_t nx = anc[r];
          anc[r] = (int32_t)k;
          r = nx;
        }
        if (anc[r] == -1) {
          anc[r] = (int32_t)k;
          par[r] = (int32_t)k;
        }
      }
    }
  };
  std::function<void(uint32_t, uint32_t, int)> etree = [&](uint32_t b, uint32_t e, int depth) {
    const auto it = nd_splits.find(((uint64_t)b << 32) | e);
    if (it == nd_splits.end()) {
      liu(b, e);
      return;
    }
    const uint32_t ea = it->second.first, eb = it->second.second;
    if (depth < 4) {
      std::thread th([&, b, ea, depth] { etree(b, ea, depth + 1); });
      etree(ea, eb, depth + 1);
      th.join();
    } else {
      etree(b, ea, depth + 1);
      etree(ea, eb, depth + 1);
    }
    liu(eb, e);
  };
  etree(0, n, 0);
  lap("etree");
  // (3) postorder (iterative DFS, children in increasing order)
  std::vector<int32_t> head(n, -1), nxt(n, -1);
  for (int32_t j = (int32_t)n - 1; j >= 0; --j)
    if (par[j] != -1) {
      nxt[j] = head[par[j]];
      head[par[j]] = j;
    }
  std::vector<uint32_t> post;
  post.reserve(n);
  std::vector<int32_t> stack;
  for (uint32_t r = 0; r < n; ++r) {
    if (par[r] != -1) continue;
    stack.push_back((int32_t)r);
    while (!stack.empty()) {
      const int32_t t = stack.back();
      const int32_t c = head[t];
      if (c == -1) {
        stack.pop_back();
        post.push_back((uint32_t)t);
      } else {
        head[t] = nxt[c];
        stack.push_back(c);
      }
    }
  }
  p.perm.resize(n);
  p.iperm.resize(n);
  std::vector<uint32_t> ipost(n);
  for (uint32_t j = 0; j < n; ++j) ipost[post[j]] = j;
  for (uint32_t j = 0; j < n; ++j) p.perm[j] = perm0[post[j]];
  for (uint32_t j = 0; j < n; ++j) p.iperm[p.perm[j]] = j;
  std::vector<int32_t> parent(n, -1);
  for (uint32_t j = 0; j < n; ++j) {
    const int32_t q = par[post[j]];
    parent[j] = q == -1 ? -1 : (int32_t)ipost[q];
  }
  lap("postorder");
  // upper pattern + values in the final numbering: column j holds the rows
  // i >= j (diagonal first is not required), used by the column counts,
  // the front structures and the scatter list
  std::vector<uint32_t> up((size_t)n + 1, 0), ui;
  std::vector<float> uv;
  {
    parallel_for(n, 2048, [&](uint32_t j0, uint32_t j1, uint32_t) {
      for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t jo = p.perm[j];
        uint32_t c = 0;
        for (uint32_t q = rp[jo]; q < rp[jo + 1]; ++q) c += p.iperm[ci[q]] >= j;
        up[j + 1] = c;
      }
    });
    for (uint32_t j = 0; j < n; ++j) up[j + 1] += up[j];
    ui.resize(up[n]);
    uv.resize(up[n]);
    parallel_for(n, 2048, [&](uint32_t j0, uint32_t j1, uint32_t) {
      for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t jo = p.perm[j];
        uint32_t o = up[j];
        for (uint32_t q = rp[jo]; q < rp[jo + 1]; ++q) {
          const uint32_t i = p.iperm[ci[q]];
          if (i >= j) {
            ui[o] = i;
            uv[o++] = val[q];
          }
        }
      }
    });
  }
  lap("upper pattern");
  // (4) column counts (Gilbert, Ng & Peyton 1994: row-subtree leaves and
  // least common ancestors, near O(nnz(M))).  The matrix is already in
  // postorder, so the postorder of the tree is the identity.
  std::vector<uint32_t> colcnt(n, 0);
  {
    std::vector<int32_t> delta(n, 0), first(n, -1), maxfirst(n, -1), prevleaf(n, -1), anc(n);
    for (uint32_t k = 0; k < n; ++k) {
      delta[k] = first[k] == -1 ? 1 : 0;  // k is a leaf of the etree
      for (int32_t j = (int32_t)k; j != -1 && first[j] == -1; j = parent[j]) first[j] = (int32_t)k;
    }
    for (uint32_t i = 0; i < n; ++i) anc[i] = (int32_t)i;
    for (uint32_t j = 0; j < n; ++j) {
      if (parent[j] != -1) delta[parent[j]]--;
      for (uint32_t q = up[j]; q < up[j + 1]; ++q) {
        const uint32_t i = ui[q];
        // is j a leaf of the row subtree of i?
        if (i <= j || first[j] <= maxfirst[i]) continue;
        maxfirst[i] = first[j];
        const int32_t jprev = prevleaf[i];
        prevleaf[i] = (int32_t)j;
        delta[j]++;
        if (jprev == -1) continue;  // first leaf: lca is the subtree root i
        int32_t lca = jprev;
        while (lca != anc[lca]) lca = anc[lca];
        for (int32_t s2 = jprev; s2 != lca;) {  // path compression
          const int32_t nx = anc[s2];
          anc[s2] = lca;
          s2 = nx;
        }
        delta[lca]--;
      }
      if (parent[j] != -1) anc[j] = parent[j];
    }
    for (uint32_t j = 0; j < n; ++j)
      if (parent[j] != -1) delta[parent[j]] += delta[j];
    for (uint32_t j = 0; j < n; ++j) colcnt[j] = (uint32_t)delta[j];
    static const bool check = std::getenv("DMCG_CHECK_SYMBOLIC") != nullptr;
    if (check) {  // row-subtree traversal (Davis, LDL symbolic)
      std::vector<uint32_t> cc(n, 1);
      std::vector<int32_t> flag(n, -1);
      for (uint32_t k = 0; k < n; ++k) {
        flag[k] = (int32_t)k;
        const uint32_t ko = p.perm[k];
        for (uint32_t q = rp[ko]; q < rp[ko + 1]; ++q) {
          uint32_t i = p.iperm[ci[q]];
          if (i >= k) continue;
          for (; flag[i] != (int32_t)k; i = (uint32_t)parent[i]) {
            cc[i]++;
            flag[i] = (int32_t)k;
          }
        }
      }
      if (cc != colcnt) {
        std::fprintf(stderr, "dmcg: column-count mismatch\n");
        std::abort();
      }
    }
  }
  lap("colcounts");
  // (5) fundamental supernodes
  std::vector<uint32_t> nchild(n, 0);
  for (uint32_t j = 0; j < n; ++j)
    if (parent[j] != -1) nchild[parent[j]]++;
  std::vector<uint32_t> sfirst;  // first column of each fundamental supernode
  for (uint32_t j = 0; j < n; ++j) {
    const bool cont = j > 0 && parent[j - 1] == (int32_t)j && nchild[j] == 1 &&
                      colcnt[j - 1] == colcnt[j] + 1;
    if (!cont) sfirst.push_back(j);
  }
  sfirst.push_back(n);
  uint32_t ns = (uint32_t)sfirst.size() - 1;
  std::vector<uint32_t> sup_of(n);
  for (uint32_t s = 0; s < ns; ++s)
    for (uint32_t j = sfirst[s]; j < sfirst[s + 1]; ++j) sup_of[j] = s;
  // (6) relaxed amalgamation: merge a supernode into its parent when it is
  // the parent's last child (contiguous columns) and the merged front stays
  // dense enough.  Stats per supernode: width, m (rows incl. own columns),
  // true nonzeros (from colcnt), stored lower-triangle entries.
  std::vector<int32_t> spar(ns, -1);
  std::vector<uint64_t> nz_true(ns, 0);
  std::vector<uint32_t> sw(ns), sm(ns), sf(ns);
  for (uint32_t s = 0; s < ns; ++s) {
    const uint32_t last = sfirst[s + 1] - 1;
    spar[s] = parent[last] == -1 ? -1 : (int32_t)sup_of[parent[last]];
    sw[s] = sfirst[s + 1] - sfirst[s];
    sm[s] = colcnt[sfirst[s]];
    sf[s] = sfirst[s];
    for (uint32_t j = sfirst[s]; j < sfirst[s + 1]; ++j) nz_true[s] += colcnt[j];
  }
  auto stored = [](uint64_t w, uint64_t m) { return w * m - w * (w - 1) / 2; };
  std::vector<int32_t> merged_into(ns, -1);
  for (uint32_t c = 0; c < ns; ++c) {  // supernodes are in postorder
    const int32_t pp = spar[c];
    if (pp < 0) continue;
    if (sf[c] + sw[c] != sf[pp]) continue;  // not contiguous (not the last child)
    const uint64_t w = (uint64_t)sw[c] + sw[pp];
    const uint64_t m = (uint64_t)sw[c] + sm[pp];
    const uint64_t st = stored(w, m);
    const uint64_t nzt = nz_true[c] + nz_true[pp];
    const double zf = 1.0 - (double)nzt / (double)st;
    const bool ok = w <= 4 || (w <= 16 && zf <= 0.8) || (w <= 48 && zf <= 0.1) || zf <= 0.05;
    if (!ok || w > 1024) continue;
    // merge c into pp
    sf[pp] = sf[c];
    sw[pp] = (uint32_t)w;
    sm[pp] = (uint32_t)m;
    nz_true[pp] = st;  // merged front is now stored densely
    merged_into[c] = pp;
  }
  // collect surviving supernodes in column order
  p.first.clear();
  std::vector<uint32_t> old_to_new(ns, UINT32_MAX);
  for (uint32_t s = 0; s < ns; ++s)
    if (merged_into[s] == -1) {
      old_to_new[s] = (uint32_t)p.first.size();
      p.first.push_back(sf[s]);
    }
  p.nsup = (uint32_t)p.first.size();
  p.first.push_back(n);
  // sort by first column (postorder keeps them sorted already; enforce)
  {
    std::vector<uint32_t> chk(p.first.begin(), p.first.end() - 1);
    if (!std::is_sorted(chk.begin(), chk.end())) {
      std::sort(p.first.begin(), p.first.end() - 1);
    }
  }
  const uint32_t NS = p.nsup;
  std::vector<uint32_t> col_sup(n);
  for (uint32_t s = 0; s < NS; ++s)
    for (uint32_t j = p.first[s]; j < p.first[s + 1]; ++j) col_sup[j] = s;
  lap("supernodes");
  // (7) supernodal tree (parent = supernode of the etree parent of the last
  // column), children, levels; then the row structures, one tree level at a
  // time with the supernodes of a level in parallel (a structure needs only
  // its own columns of M and its children's structures).
  p.parent.assign(NS, -1);
  std::vector<std::vector<uint32_t>> kids(NS);
  for (uint32_t s = 0; s < NS; ++s) {
    const int32_t pc = parent[p.first[s + 1] - 1];
    if (pc >= 0) {
      p.parent[s] = (int32_t)col_sup[pc];
      kids[p.parent[s]].push_back(s);
    }
  }
  p.child_ptr.assign(NS + 1, 0);
  p.child_idx.clear();
  for (uint32_t s = 0; s < NS; ++s) {
    p.child_idx.insert(p.child_idx.end(), kids[s].begin(), kids[s].end());
    p.child_ptr[s + 1] = (uint32_t)p.child_idx.size();
  }
  std::vector<uint32_t> lev(NS, 0);
  uint32_t maxlev = 0;
  for (uint32_t s = 0; s < NS; ++s) {
    for (uint32_t c : kids[s]) lev[s] = std::max(lev[s], lev[c] + 1);
    maxlev = std::max(maxlev, lev[s]);
  }
  p.nlevels = NS ? maxlev + 1 : 0;
  p.level_ptr.assign(p.nlevels + 1, 0);
  for (uint32_t s = 0; s < NS; ++s) p.level_ptr[lev[s] + 1]++;
  for (uint32_t l = 0; l < p.nlevels; ++l) p.level_ptr[l + 1] += p.level_ptr[l];
  p.level_sup.assign(NS, 0);
  {
    std::vector<uint32_t> fill(p.level_ptr.begin(), p.level_ptr.end() - 1);
    for (uint32_t s = 0; s < NS; ++s) p.level_sup[fill[lev[s]]++] = s;
  }
  {
    std::vector<std::vector<uint32_t>> str(NS);
    std::vector<std::vector<int32_t>> marks(16);
    for (uint32_t l = 0; l < p.nlevels; ++l) {
      const uint32_t l0 = p.level_ptr[l], cnt = p.level_ptr[l + 1] - l0;
      parallel_for(cnt, 16, [&](uint32_t q0, uint32_t q1, uint32_t c) {
        std::vector<int32_t>& mark = marks[c];
        if (mark.empty()) mark.assign(n, -1);
        for (uint32_t t = q0; t < q1; ++t) {
          const uint32_t s = p.level_sup[l0 + t];
          const uint32_t f0 = p.first[s], f1 = p.first[s + 1];
          std::vector<uint32_t>& rows = str[s];
          for (uint32_t j = f0; j < f1; ++j) {
            rows.push_back(j);
            mark[j] = (int32_t)s;
          }
          for (uint32_t j = f0; j < f1; ++j)
            for (uint32_t q = up[j]; q < up[j + 1]; ++q) {
              const uint32_t i = ui[q];
              if (i >= f1 && mark[i] != (int32_t)s) {
                mark[i] = (int32_t)s;
                rows.push_back(i);
              }
            }
          for (uint32_t ch : kids[s]) {
            const std::vector<uint32_t>& cr = str[ch];
            for (size_t q = p.first[ch + 1] - p.first[ch]; q < cr.size(); ++q) {
              const uint32_t i = cr[q];
              if (i >= f1 && mark[i] != (int32_t)s) {
                mark[i] = (int32_t)s;
                rows.push_back(i);
              }
            }
          }
          std::sort(rows.begin() + (f1 - f0), rows.end());
        }
      });
    }
    p.str_ptr.assign(NS + 1, 0);
    for (uint32_t s = 0; s < NS; ++s) p.str_ptr[s + 1] = p.str_ptr[s] + str[s].size();
    p.str_idx.resize(p.str_ptr[NS]);
    parallel_for(NS, 64, [&](uint32_t s0, uint32_t s1, uint32_t) {
      for (uint32_t s = s0; s < s1; ++s)
        std::copy(str[s].begin(), str[s].end(), p.str_idx.begin() + p.str_ptr[s]);
    });
    static const bool check = std::getenv("DMCG_CHECK_SYMBOLIC") != nullptr;
    if (check)  // the tree from the etree matches the structures' first off-diagonal rows
      for (uint32_t s = 0; s < NS; ++s) {
        const uint32_t w = p.first[s + 1] - p.first[s];
        const int32_t ps = str[s].size() > w ? (int32_t)col_sup[str[s][w]] : -1;
        if (ps != p.parent[s]) {
          std::fprintf(stderr, "dmcg: supernodal parent mismatch at %u\n", s);
          std::abort();
        }
      }
  }
  lap("structure");
  // offsets and statistics
  p.front_off.assign(NS + 1, 0);
  p.inv_off.assign(NS + 1, 0);
  p.rhs_off.assign(NS + 1, 0);
  p.op_off.assign(NS + 1, 0);
  p.nnz_l = 0;
  p.flops_factor = 0;
  p.flops_solve_per_rhs = 0;
  for (uint32_t s = 0; s < NS; ++s) {
    const uint64_t w = p.w(s), m = p.m(s);
    p.front_off[s + 1] = p.front_off[s] + m * m;
    p.inv_off[s + 1] = p.inv_off[s] + w * w;
    p.rhs_off[s + 1] = p.rhs_off[s] + m;
    p.op_off[s + 1] = p.op_off[s] + m * w;
    p.nnz_l += w * m - w * (w - 1) / 2;
    p.max_front = std::max<uint32_t>(p.max_front, (uint32_t)m);
    p.max_width = std::max<uint32_t>(p.max_width, (uint32_t)w);
    // partial Cholesky: sum over pivots t of (m-t)^2 ; L11 inverse w^3/3
    for (uint64_t t = 0; t < w; ++t) p.flops_factor += (double)(m - t) * (m - t);
    p.flops_factor += (double)w * w * w / 3.0;
    // one solve = forward [L11^{-1}; -L21 L11^{-1}] r (m x w) + backward (w x m)
    p.flops_solve_per_rhs += 4.0 * (double)m * w;
  }
  lap("levels+stats");
  // (8) extend-add maps: child update rows -> parent local rows
  p.rel_ptr.assign(NS + 1, 0);
  for (uint32_t c = 0; c < NS; ++c)
    p.rel_ptr[c + 1] = p.rel_ptr[c] + (p.parent[c] >= 0 ? p.m(c) - p.w(c) : 0);
  p.rel_idx.resize(p.rel_ptr[NS]);
  parallel_for(NS, 64, [&](uint32_t c0, uint32_t c1, uint32_t) {
    for (uint32_t c = c0; c < c1; ++c) {
      const int32_t ps = p.parent[c];
      if (ps < 0) continue;
      const uint32_t* pb = &p.str_idx[p.str_ptr[ps]];
      const uint32_t pm = p.m((uint32_t)ps);
      uint64_t o = p.rel_ptr[c];
      const uint32_t* it = pb;
      for (uint64_t q = p.str_ptr[c] + p.w(c); q < p.str_ptr[c + 1]; ++q) {
        it = std::lower_bound(it, pb + pm, p.str_idx[q]);  // rows are sorted
        p.rel_idx[o++] = (uint32_t)(it - pb);
      }
    }
  });
  // (9) scatter list of M into the fronts (lower part, column-major local):
  // on the pool from a helper thread, under the serial pull-list pass below
  std::thread scatter_thread([&] {
    p.a_ptr.assign(NS + 1, 0);
    for (uint32_t s = 0; s < NS; ++s) p.a_ptr[s + 1] = up[p.first[s + 1]];
    p.a_pos.resize(p.a_ptr[NS]);
    p.a_val.resize(p.a_ptr[NS]);
    parallel_for(NS, 64, [&](uint32_t s0, uint32_t s1, uint32_t) {
      std::vector<int32_t> loc(n, -1);
      for (uint32_t s = s0; s < s1; ++s) {
        const uint32_t m = p.m(s), f0 = p.first[s], f1 = p.first[s + 1];
        for (uint32_t t = 0; t < m; ++t) loc[p.str_idx[p.str_ptr[s] + t]] = (int32_t)t;
        for (uint32_t j = f0; j < f1; ++j)
          for (uint32_t q = up[j]; q < up[j + 1]; ++q) {
            p.a_pos[q] = (j - f0) * m + (uint32_t)loc[ui[q]];
            p.a_val[q] = uv[q];
          }
        for (uint32_t t = 0; t < m; ++t) loc[p.str_idx[p.str_ptr[s] + t]] = -1;
      }
    });
  });
  // pull lists (see chol.h): count per parent row, then fill child by child
  {
    const uint64_t R = p.rhs_off[NS];
    p.pull_ptr.assign(R + 1, 0);
    for (uint32_t c = 0; c < NS; ++c) {
      const int32_t ps = p.parent[c];
      if (ps < 0) continue;
      for (uint64_t q = p.rel_ptr[c]; q < p.rel_ptr[c + 1]; ++q)
        p.pull_ptr[p.rhs_off[ps] + p.rel_idx[q] + 1]++;
    }
    for (uint64_t g = 0; g < R; ++g) p.pull_ptr[g + 1] += p.pull_ptr[g];
    p.pull_src.resize(p.pull_ptr[R]);
    std::vector<uint32_t> fill(p.pull_ptr.begin(), p.pull_ptr.end() - 1);
    for (uint32_t s = 0; s < NS; ++s)
      for (uint32_t q = p.child_ptr[s]; q < p.child_ptr[s + 1]; ++q) {
        const uint32_t c = p.child_idx[q];
        const uint32_t wc = p.w(c);
        for (uint64_t e = p.rel_ptr[c]; e < p.rel_ptr[c + 1]; ++e) {
          const uint64_t g = p.rhs_off[s] + p.rel_idx[e];
          p.pull_src[fill[g]++] = (uint32_t)(p.rhs_off[c] + wc + (e - p.rel_ptr[c]));
        }
      }
  }
  scatter_thread.join();
  lap("rel maps+scatter");
}

// ---------------------------------------------------------------------------
// CPU reference numerics (same data flow as the GPU kernels)
// ---------------------------------------------------------------------------
bool chol_factor_cpu(const CholPlan& p, std::vector<double>* Fv, std::vector<double>* Iv) {
  std::vector<double>& F = *Fv;
  std::vector<double>& Linv = *Iv;
  F.assign(p.front_off[p.nsup], 0.0);
  Linv.assign(p.inv_off[p.nsup], 0.0);
  for (uint32_t l = 0; l < p.nlevels; ++l) {
    for (uint32_t q = p.level_ptr[l]; q < p.level_ptr[l + 1]; ++q) {
      const uint32_t s = p.level_sup[q];
      const uint32_t m = p.m(s), w = p.w(s);
      double* A = &F[p.front_off[s]];
      for (uint64_t e = p.a_ptr[s]; e < p.a_ptr[s + 1]; ++e) A[p.a_pos[e]] += p.a_val[e];
      for (uint32_t t = p.child_ptr[s]; t < p.child_ptr[s + 1]; ++t) {
        const uint32_t c = p.child_idx[t];
        const uint32_t mc = p.m(c), wc = p.w(c), uc = mc - wc;
        const double* C = &F[p.front_off[c]];
        const uint32_t* rel = &p.rel_idx[p.rel_ptr[c]];
        for (uint32_t b = 0; b < uc; ++b)
          for (uint32_t a = b; a < uc; ++a)
            A[(size_t)rel[b] * m + rel[a]] += C[(size_t)(wc + b) * mc + (wc + a)];
      }
      for (uint32_t j = 0; j < w; ++j) {
        const double d = A[(size_t)j * m + j];
        if (!(d > 0.0)) return false;
        const double r = std::sqrt(d);
        A[(size_t)j * m + j] = r;
        for (uint32_t i = j + 1; i < m; ++i) A[(size_t)j * m + i] /= r;
        for (uint32_t c = j + 1; c < m; ++c) {
          const double lc = A[(size_t)j * m + c];
          for (uint32_t i = c; i < m; ++i) A[(size_t)c * m + i] -= A[(size_t)j * m + i] * lc;
        }
      }
      // L11^{-1} by forward substitution on the identity
      double* V = &Linv[p.inv_off[s]];
      for (uint32_t c = 0; c < w; ++c) {
        for (uint32_t i = 0; i < w; ++i) {
          double sacc = (i == c) ? 1.0 : 0.0;
          for (uint32_t k = c; k < i; ++k) sacc -= A[(size_t)k * m + i] * V[(size_t)c * w + k];
          V[(size_t)c * w + i] = i < c ? 0.0 : sacc / A[(size_t)i * m + i];
        }
      }
    }
  }
  return true;
}

void chol_solve_cpu(const CholPlan& p, const std::vector<double>& F,
                    const std::vector<double>& Linv, uint32_t W, const double* b, double* x) {
  const uint32_t n = p.n;
  std::vector<double> R(p.rhs_off[p.nsup] * W, 0.0), y((size_t)n * W), xp((size_t)n * W);
  // forward: L y = P b
  for (uint32_t l = 0; l < p.nlevels; ++l)
    for (uint32_t q = p.level_ptr[l]; q < p.level_ptr[l + 1]; ++q) {
      const uint32_t s = p.level_sup[q];
      const uint32_t m = p.m(s), w = p.w(s), f0 = p.first[s];
      double* Rs = &R[p.rhs_off[s] * W];
      for (uint32_t j = 0; j < w; ++j)
        for (uint32_t c = 0; c < W; ++c) Rs[(size_t)j * W + c] = b[(size_t)p.perm[f0 + j] * W + c];
      for (uint32_t t = p.child_ptr[s]; t < p.child_ptr[s + 1]; ++t) {
        const uint32_t ch = p.child_idx[t];
        const uint32_t wc = p.w(ch), uc = p.m(ch) - wc;
        const double* Rc = &R[(p.rhs_off[ch] + wc) * W];
        const uint32_t* rel = &p.rel_idx[p.rel_ptr[ch]];
        for (uint32_t a = 0; a < uc; ++a)
          for (uint32_t c = 0; c < W; ++c) Rs[(size_t)rel[a] * W + c] += Rc[(size_t)a * W + c];
      }
      const double* A = &F[p.front_off[s]];
      const double* V = &Linv[p.inv_off[s]];
      std::vector<double> ys((size_t)w * W, 0.0);
      for (uint32_t i = 0; i < w; ++i)
        for (uint32_t k = 0; k <= i; ++k)
          for (uint32_t c = 0; c < W; ++c) ys[(size_t)i * W + c] += V[(size_t)k * w + i] * Rs[(size_t)k * W + c];
      for (uint32_t i = w; i < m; ++i)
        for (uint32_t k = 0; k < w; ++k)
          for (uint32_t c = 0; c < W; ++c) Rs[(size_t)i * W + c] -= A[(size_t)k * m + i] * ys[(size_t)k * W + c];
      for (uint32_t i = 0; i < w; ++i)
        for (uint32_t c = 0; c < W; ++c) y[(size_t)(f0 + i) * W + c] = ys[(size_t)i * W + c];
    }
  // backward: L^T xp = y
  for (int32_t l = (int32_t)p.nlevels - 1; l >= 0; --l)
    for (uint32_t q = p.level_ptr[l]; q < p.level_ptr[l + 1]; ++q) {
      const uint32_t s = p.level_sup[q];
      const uint32_t m = p.m(s), w = p.w(s), f0 = p.first[s];
      const double* A = &F[p.front_off[s]];
      const double* V = &Linv[p.inv_off[s]];
      const uint32_t* str = &p.str_idx[p.str_ptr[s]];
      std::vector<double> t((size_t)w * W);
      for (uint32_t i = 0; i < w; ++i)
        for (uint32_t c = 0; c < W; ++c) t[(size_t)i * W + c] = y[(size_t)(f0 + i) * W + c];
      for (uint32_t i = 0; i < w; ++i)
        for (uint32_t r = w; r < m; ++r)
          for (uint32_t c = 0; c < W; ++c)
            t[(size_t)i * W + c] -= A[(size_t)i * m + r] * xp[(size_t)str[r] * W + c];
      for (uint32_t i = 0; i < w; ++i)
        for (uint32_t c = 0; c < W; ++c) {
          double sacc = 0.0;
          for (uint32_t k = i; k < w; ++k) sacc += V[(size_t)i * w + k] * t[(size_t)k * W + c];
          xp[(size_t)(f0 + i) * W + c] = sacc;
        }
    }
  for (uint32_t j = 0; j < n; ++j)
    for (uint32_t c = 0; c < W; ++c) x[(size_t)p.perm[j] * W + c] = xp[(size_t)j * W + c];
}

}  // namespace dmcg
