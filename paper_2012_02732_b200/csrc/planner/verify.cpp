// Exhaustive sync-optimality verifiers (the reference's `streamweave.oracle`
// API, /root/reference/pkg/src/streamweave/oracle.py:25-315), used by
// compare_modes(with_oracle=True) (compare.py:85-91) and the CLI `verify`.
//
// Independent of the production pipeline, as in the reference: safety is a
// forward path DP over the topological order (not the closure pair cover),
// assignments are raw set partitions in restricted-growth order, and the
// minimum plan is an exact set cover over per-edge cover masks.  Size guards
// return SW_TOO_LARGE with the reference's texts.
#include <algorithm>
#include <string>
#include <vector>

#include "planner.h"

namespace sw {

static const int64_t kMaxEnumNodes = 10;   // oracle.py:25
static const int64_t kMaxPlanEdges = 20;   // oracle.py:26
static const int64_t kMaxVerifyNodes = 7;  // oracle.py:27

namespace {

// Dense tables of one graph: topo order (ranks), predecessor ranks per rank,
// and a plan-edge membership test over ranks.
struct Walk {
  const Graph* g;
  std::vector<std::vector<int64_t>> pred;  // rank -> predecessor ranks

  explicit Walk(const Graph& gg) : g(&gg) {
    pred.assign(gg.sorted_ids.size(), {});
    for (auto& e : gg.redge) pred[e.second].push_back(e.first);
  }

  // oracle.py:46-66 — is there a u..v path crossing an edge of `plan` (a
  // rank-pair membership matrix)?  synced[w] once some path u..w crosses one.
  bool synced_path(int64_t ru, int64_t rv, const std::vector<char>& plan, std::vector<char>& arrived,
                   std::vector<char>& synced) const {
    const int64_t n = (int64_t)pred.size();
    std::fill(arrived.begin(), arrived.end(), 0);
    std::fill(synced.begin(), synced.end(), 0);
    arrived[ru] = 1;
    bool walking = false;
    for (int64_t w : g->topo_ranks) {
      if (w == ru) {
        walking = true;
        continue;
      }
      if (!walking) continue;
      for (int64_t x : pred[w]) {
        if (!arrived[x]) continue;
        arrived[w] = 1;
        if (synced[x] || plan[(size_t)(x * n + w)]) synced[w] = 1;
      }
      if (w == rv) return synced[rv] != 0;
    }
    return false;
  }
};

int stream_lookup(const Assign& f, int64_t id, int64_t* out) {
  auto it = f.map.find(id);
  if (it == f.map.end()) return fail(SW_KEY_ERROR, std::to_string(id));
  *out = it->second;
  return SW_OK;
}

// oracle.py:30-43
int path_safe(const Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan, bool* out) {
  const int64_t n = (int64_t)g.sorted_ids.size();
  std::vector<char> pm((size_t)(n * n), 0);
  for (auto& e : plan) {
    auto a = g.rank.find(e.first), b = g.rank.find(e.second);
    if (a != g.rank.end() && b != g.rank.end()) pm[(size_t)(a->second * n + b->second)] = 1;
  }
  Walk w(g);
  std::vector<char> arrived(n), synced(n);
  for (size_t k = 0; k < g.edges.size(); ++k) {
    int64_t su, sv;
    int rc = stream_lookup(f, g.edges[k].first, &su);
    if (rc) return rc;
    rc = stream_lookup(f, g.edges[k].second, &sv);
    if (rc) return rc;
    if (su == sv) continue;
    if (!w.synced_path(g.redge[k].first, g.redge[k].second, pm, arrived, synced)) {
      *out = false;
      return SW_OK;
    }
  }
  *out = true;
  return SW_OK;
}

// oracle.py:71-88 — cover[i] bit j: a plan holding edge i alone syncs edge j.
std::vector<uint32_t> cover_masks(const Graph& g) {
  const int64_t n = (int64_t)g.sorted_ids.size();
  const size_t m = g.edges.size();
  Walk w(g);
  std::vector<char> pm((size_t)(n * n), 0), arrived(n), synced(n);
  std::vector<uint32_t> cover(m, 0);
  for (size_t i = 0; i < m; ++i) {
    size_t cell = (size_t)(g.redge[i].first * n + g.redge[i].second);
    pm[cell] = 1;
    for (size_t j = 0; j < m; ++j)
      if (w.synced_path(g.redge[j].first, g.redge[j].second, pm, arrived, synced)) cover[i] |= 1u << j;
    pm[cell] = 0;
  }
  return cover;
}

// Exact minimum number of masks whose union is `need`, or `bound` if no
// cover smaller than bound exists (bound < 0: none).  Branch and bound: the
// uncovered bit with the fewest covering masks branches first.
int64_t min_cover(uint32_t need, const std::vector<uint32_t>& cover, int64_t bound) {
  if (need == 0) return 0;
  std::vector<uint32_t> useful;
  for (uint32_t c : cover)
    if (c & need) useful.push_back(c & need);
  std::sort(useful.begin(), useful.end());
  useful.erase(std::unique(useful.begin(), useful.end()), useful.end());
  std::vector<uint32_t> kept;  // drop masks contained in another
  for (uint32_t c : useful) {
    bool dominated = false;
    for (uint32_t d : useful)
      if (d != c && (c & ~d) == 0) {
        dominated = true;
        break;
      }
    if (!dominated) kept.push_back(c);
  }
  int64_t best = 0;
  for (uint32_t unc = need; unc;) {  // greedy upper bound
    uint32_t pick = 0;
    int pc = 0;
    for (uint32_t c : kept)
      if (__builtin_popcount(c & unc) > pc) pc = __builtin_popcount(c & unc), pick = c;
    if (!pick) {  // cannot cover: impossible for a DAG (edge i covers itself)
      best = 64;
      break;
    }
    unc &= ~pick;
    ++best;
  }
  if (bound >= 0) best = std::min(best, bound);
  int max_pc = 0;
  for (uint32_t c : kept) max_pc = std::max(max_pc, __builtin_popcount(c));
  struct Rec {
    const std::vector<uint32_t>& kept;
    int max_pc;
    int64_t& best;
    void go(uint32_t unc, int64_t size) {
      if (!unc) {
        best = std::min(best, size);
        return;
      }
      int64_t lb = (__builtin_popcount(unc) + max_pc - 1) / max_pc;
      if (size + lb >= best) return;
      uint32_t bit = 0;
      int fewest = 1 << 30;
      for (uint32_t m = unc; m; m &= m - 1) {
        uint32_t low = m & (~m + 1);
        int k = 0;
        for (uint32_t c : kept) k += (c & low) != 0;
        if (k < fewest) fewest = k, bit = low;
      }
      for (uint32_t c : kept)
        if (c & bit) go(unc & ~c, size + 1);
    }
  } rec{kept, max_pc, best};
  rec.go(need, 0);
  return best;
}

int need_mask(const Graph& g, const Assign& f, uint32_t* out) {
  uint32_t m = 0;
  for (size_t j = 0; j < g.edges.size(); ++j) {
    int64_t su, sv;
    int rc = stream_lookup(f, g.edges[j].first, &su);
    if (rc) return rc;
    rc = stream_lookup(f, g.edges[j].second, &sv);
    if (rc) return rc;
    if (su != sv) m |= 1u << j;
  }
  *out = m;
  return SW_OK;
}

int edge_cap(const Graph& g) {
  if ((int64_t)g.edges.size() > kMaxPlanEdges)
    return fail(SW_TOO_LARGE, std::to_string(g.edges.size()) + " edges exceeds the " +
                                  std::to_string(kMaxPlanEdges) + "-edge plan search cap");
  return SW_OK;
}

// oracle.py:172-220 — every set partition of the topological order in
// restricted-growth order; keep those whose blocks are chains (every pair
// ordered).  labels[a] = per-topo-position block label of candidate a.
int64_t enumerate_parts(const Graph& g, std::vector<std::vector<int64_t>>* labels) {
  const int64_t n = (int64_t)g.topo_ranks.size();
  int64_t checked = 0;
  if (n == 0) {
    labels->push_back({});
    return 1;
  }
  std::vector<int64_t> a(n, 0), mx(n, 0);
  auto ordered = [&](int64_t i, int64_t j) {
    int64_t u = g.topo_ranks[i], v = g.topo_ranks[j];
    return g.reaches(u, v) || g.reaches(v, u);
  };
  for (;;) {
    ++checked;
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i)
      for (int64_t j = i + 1; j < n; ++j)
        if (a[i] == a[j] && !ordered(i, j)) {
          ok = false;
          break;
        }
    if (ok) labels->push_back(a);
    int64_t i = n - 1;
    while (i > 0 && a[i] == mx[i - 1] + 1) --i;
    if (i == 0) break;
    ++a[i];
    mx[i] = std::max(mx[i - 1], a[i]);
    for (int64_t j = i + 1; j < n; ++j) {
      a[j] = 0;
      mx[j] = mx[i];
    }
  }
  return checked;
}

Assign assign_of(const Graph& g, const std::vector<int64_t>& lab) {
  std::vector<std::pair<int64_t, int64_t>> v;
  for (size_t i = 0; i < lab.size(); ++i) v.push_back({g.sorted_ids[g.topo_ranks[i]], lab[i]});
  return Assign::from_pairs(v);
}

}  // namespace

// verify_optimal (f == nullptr) / verify_given: oracle.py:271-315.
int verify(Graph& g, const Assign* f_given, const std::vector<std::pair<int64_t, int64_t>>& plan_given,
           int64_t out[5]) {
  if (g.n > kMaxVerifyNodes)
    return fail(SW_TOO_LARGE, std::to_string(g.n) + " nodes exceeds the " + std::to_string(kMaxVerifyNodes) +
                                  "-node verification cap");
  std::vector<std::pair<int64_t, int64_t>> f_algo, plan, meg;
  int rc;
  if (!f_given) {
    Graph ga = g;
    rc = assign_streams(ga, &f_algo, &plan, &meg);
    if (rc) return rc;
  } else {
    plan = plan_given;
  }
  rc = prepare(g, false, true);
  if (rc) return rc;
  std::vector<std::vector<int64_t>> cands;
  int64_t checked = enumerate_parts(g, &cands);
  int64_t best = -1;
  if (!cands.empty()) {
    rc = edge_cap(g);
    if (rc) return rc;
    auto cover = cover_masks(g);
    for (auto& lab : cands) {
      uint32_t need;
      rc = need_mask(g, assign_of(g, lab), &need);
      if (rc) return rc;
      best = min_cover(need, cover, best);
    }
  }
  bool safe = false;
  Assign fa = f_given ? *f_given : Assign::from_pairs(f_algo);
  rc = path_safe(g, fa, plan, &safe);
  if (rc) return rc;
  int64_t algo = (int64_t)plan.size(), omin = best < 0 ? 0 : best;
  out[0] = (algo == omin) && safe;
  out[1] = algo;
  out[2] = omin;
  out[3] = checked;
  out[4] = safe;
  return SW_OK;
}

int oracle_plan_is_safe(Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan,
                        bool* out) {
  int rc = prepare(g, false, false);
  if (rc) return rc;
  return path_safe(g, f, plan, out);
}

int min_syncs_brute(Graph& g, const Assign& f, int64_t bound, int64_t* out) {
  int rc = edge_cap(g);
  if (rc) return rc;
  rc = prepare(g, false, false);
  if (rc) return rc;
  auto cover = cover_masks(g);
  uint32_t need;
  rc = need_mask(g, f, &need);
  if (rc) return rc;
  *out = min_cover(need, cover, bound);
  return SW_OK;
}

int enumerate_assignments(Graph& g, int64_t cap, int64_t* out_order, int64_t* out_streams, int64_t* out_count) {
  if (g.n > kMaxEnumNodes)
    return fail(SW_TOO_LARGE, std::to_string(g.n) + " nodes exceeds the " + std::to_string(kMaxEnumNodes) +
                                  "-node enumeration cap");
  int rc = prepare(g, false, true);
  if (rc) return rc;
  std::vector<std::vector<int64_t>> cands;
  enumerate_parts(g, &cands);
  const int64_t n = (int64_t)g.topo_ranks.size();
  for (int64_t i = 0; i < n; ++i) out_order[i] = g.sorted_ids[g.topo_ranks[i]];
  for (int64_t a = 0; a < (int64_t)cands.size() && a < cap; ++a)
    for (int64_t i = 0; i < n; ++i) out_streams[a * n + i] = cands[a][i];
  *out_count = (int64_t)cands.size();
  return SW_OK;
}

}  // namespace sw
