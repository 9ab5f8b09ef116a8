// Native planning path of the AoT engine — bit-exact with the reference
// `streamweave` package (/root/reference/pkg/src/streamweave/{graph,assign,
// schedule}.py).  Every routine cites the reference lines whose behaviour it
// reproduces; the algorithms are restated for dense integer ranks and 64-bit
// bitsets instead of Python dicts and big ints.
//
// Determinism contract: node order and edge order as given,
// id ranks = ascending id order, min-heap Kahn topological order, Kuhn's scan
// pinned (left ascending, adjacency ascending, one `seen` set per top-level
// augment), canonical stream labels by first use along topo order.
#include "planner.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <queue>
#include <set>
#include <sstream>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

namespace sw {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static const char* kArrow = "\xe2\x86\x92";  // U+2192 '→'

static std::string edge_str(int64_t u, int64_t v) {
  return std::to_string(u) + kArrow + std::to_string(v);
}

// ---------------------------------------------------------------------------
// Graph loading
// ---------------------------------------------------------------------------

Graph Graph::from_view(const sw_graph_view* v) {
  Graph g;
  g.n = v->n_nodes;
  g.ids.assign(v->ids, v->ids + g.n);
  g.dur.resize(g.n);
  g.dem.resize(g.n);
  for (int64_t i = 0; i < g.n; ++i) {
    g.dur[i] = v->durations ? v->durations[i] : 1;
    g.dem[i] = v->demands ? v->demands[i] : 1;
  }
  g.mem_start.assign(g.n + 1, 0);
  if (v->mem_start) {
    for (int64_t i = 0; i <= g.n; ++i) g.mem_start[i] = v->mem_start[i];
    int64_t m = g.mem_start[g.n];
    g.mem_kind.assign(v->mem_kind, v->mem_kind + m);
    g.mem_arg.assign(v->mem_arg, v->mem_arg + m);
  }
  g.edges.resize(v->n_edges);
  for (int64_t i = 0; i < v->n_edges; ++i) g.edges[i] = {v->edges[2 * i], v->edges[2 * i + 1]};
  return g;
}

// Dense view: ranks by ascending id, successor lists in edge order
// (graph.py:89-99 builds adjacency by appending in edge order).
int Graph::index(std::string* missing_key) {
  sorted_ids = ids;
  std::sort(sorted_ids.begin(), sorted_ids.end());
  sorted_ids.erase(std::unique(sorted_ids.begin(), sorted_ids.end()), sorted_ids.end());
  rank.clear();
  rank.reserve(sorted_ids.size() * 2);
  for (size_t i = 0; i < sorted_ids.size(); ++i) rank[sorted_ids[i]] = (int64_t)i;
  const int64_t N = (int64_t)sorted_ids.size();
  first_pos.assign(N, -1);
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = rank[ids[i]];
    if (first_pos[r] < 0) first_pos[r] = i;
  }
  succ.assign(N, {});
  pred.assign(N, {});
  redge.resize(edges.size());
  for (size_t k = 0; k < edges.size(); ++k) {
    auto iu = rank.find(edges[k].first);
    auto iv = rank.find(edges[k].second);
    if (iu == rank.end() || iv == rank.end()) {
      if (missing_key)
        *missing_key = std::to_string(iu == rank.end() ? edges[k].first : edges[k].second);
      return SW_KEY_ERROR;
    }
    redge[k] = {iu->second, iv->second};
    succ[iu->second].push_back(iv->second);
    pred[iv->second].push_back(iu->second);
  }
  return SW_OK;
}

// graph.py:166-197 — iterative three-colour DFS, roots ascending, successors
// in edge order; witness = path from the re-entered node back to itself.
bool Graph::find_cycle(std::vector<int64_t>* witness) const {
  const int64_t N = (int64_t)sorted_ids.size();
  std::vector<uint8_t> color(N, 0);
  std::vector<int64_t> parent(N, -1);
  std::vector<std::pair<int64_t, size_t>> stack;
  for (int64_t root = 0; root < N; ++root) {
    if (color[root]) continue;
    stack.clear();
    stack.push_back({root, 0});
    color[root] = 1;
    while (!stack.empty()) {
      int64_t node = stack.back().first;
      size_t i = stack.back().second;
      if (i < succ[node].size()) {
        stack.back().second = i + 1;
        int64_t nxt = succ[node][i];
        if (color[nxt] == 1) {
          std::vector<int64_t> path{node};
          int64_t cur = node;
          while (cur != nxt) {
            cur = parent[cur];
            path.push_back(cur);
          }
          std::reverse(path.begin(), path.end());
          path.push_back(nxt);
          witness->clear();
          for (int64_t r : path) witness->push_back(sorted_ids[r]);
          return true;
        }
        if (color[nxt] == 0) {
          color[nxt] = 1;
          parent[nxt] = node;
          stack.push_back({nxt, 0});
        }
      } else {
        color[node] = 2;
        stack.pop_back();
      }
    }
  }
  return false;
}

static std::string cycle_str(const std::vector<int64_t>& c) {
  std::string s;
  for (size_t i = 0; i < c.size(); ++i) {
    if (i) s += kArrow;
    s += std::to_string(c[i]);
  }
  return s;
}

// graph.py:200-219 — Kahn with a min-heap of ready ids (rank order == id order).
int Graph::topo(std::vector<int64_t>* order_ranks) const {
  const int64_t N = (int64_t)sorted_ids.size();
  std::vector<int64_t> indeg(N, 0);
  for (auto& e : redge) indeg[e.second]++;
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> ready;
  for (int64_t r = 0; r < N; ++r)
    if (indeg[r] == 0) ready.push(r);
  order_ranks->clear();
  order_ranks->reserve(N);
  while (!ready.empty()) {
    int64_t u = ready.top();
    ready.pop();
    order_ranks->push_back(u);
    for (int64_t v : succ[u])
      if (--indeg[v] == 0) ready.push(v);
  }
  // The reference compares against len(g.nodes) (which counts duplicates).
  if ((int64_t)order_ranks->size() != n) {
    std::vector<int64_t> w;
    if (!find_cycle(&w)) w.clear();
    return fail(SW_CYCLE_DETECTED, cycle_str(w));
  }
  return SW_OK;
}

// graph.py:251-261 — rows[rank u] = OR over succ v of (rows[v] | bit v),
// filled in reverse topological order.
int Graph::closure(const std::vector<int64_t>& order_ranks) {
  const int64_t N = (int64_t)sorted_ids.size();
  words = (N + 63) / 64;
  reach.assign((size_t)(N * words), 0ull);
  for (auto it = order_ranks.rbegin(); it != order_ranks.rend(); ++it) {
    int64_t u = *it;
    uint64_t* ru = &reach[(size_t)(u * words)];
    for (int64_t v : succ[u]) {
      const uint64_t* rv = &reach[(size_t)(v * words)];
      for (int64_t k = 0; k < words; ++k) ru[k] |= rv[k];
      ru[v >> 6] |= 1ull << (v & 63);
    }
  }
  return SW_OK;
}

// graph.py:111-154 — validation order: per node (dup id, then mem), per edge
// (self loop, dangling), duplicate edge, cycle.
int validate(const Graph& g) {
  std::unordered_set<int64_t> seen;
  for (int64_t i = 0; i < g.n; ++i) {
    int64_t id = g.ids[i];
    if (seen.count(id)) return fail(SW_DUPLICATE_NODE_ID, "node id " + std::to_string(id) + " declared twice");
    seen.insert(id);
    int64_t b = g.mem_start[i], e = g.mem_start[i + 1];
    std::unordered_set<int64_t> freed;
    for (int64_t k = b; k < e; ++k) {
      int64_t local = k - b;
      std::string where = "node " + std::to_string(id) + " mem[" + std::to_string(local) + "]";
      if (g.mem_kind[k] == SW_MEM_ALLOC) {
        if (g.mem_arg[k] <= 0) return fail(SW_VALUE_ERROR, where + ": alloc size must be positive");
      } else if (g.mem_kind[k] == SW_MEM_FREE) {
        int64_t ref = g.mem_arg[k];
        if (!(0 <= ref && ref < local) || g.mem_kind[b + ref] != SW_MEM_ALLOC)
          return fail(SW_FREE_BEFORE_ALLOC,
                      where + " frees index " + std::to_string(ref) + ", not an earlier alloc");
        if (freed.count(ref))
          return fail(SW_DOUBLE_FREE, where + " frees index " + std::to_string(ref) + " again");
        freed.insert(ref);
      } else {
        return fail(SW_VALUE_ERROR, where + ": unknown kind '" + std::to_string(g.mem_kind[k]) + "'");
      }
    }
  }
  for (auto& e : g.edges) {
    if (e.first == e.second) return fail(SW_SELF_LOOP, "edge " + edge_str(e.first, e.second));
    if (!seen.count(e.first) || !seen.count(e.second))
      return fail(SW_DANGLING_EDGE, "edge " + edge_str(e.first, e.second) + " references an undeclared node");
  }
  std::set<std::pair<int64_t, int64_t>> es;
  for (auto& e : g.edges) {
    if (es.count(e)) return fail(SW_DUPLICATE_EDGE, "edge " + edge_str(e.first, e.second) + " declared twice");
    es.insert(e);
  }
  // every endpoint is declared now, so the dense index cannot fail
  Graph t = g;
  t.index(nullptr);
  std::vector<int64_t> w;
  if (t.find_cycle(&w)) return fail(SW_CYCLE_DETECTED, cycle_str(w));
  return SW_OK;
}

// Prepare a graph: (optionally) validate, then index + topo (+ closure).
int prepare(Graph& g, bool do_validate, bool need_closure) {
  if (do_validate) {
    int rc = validate(g);
    if (rc != SW_OK) return rc;
  }
  std::string key;
  if (g.index(&key) != SW_OK) return fail(SW_KEY_ERROR, key);
  int rc = g.topo(&g.topo_ranks);
  if (rc != SW_OK) return rc;
  if (need_closure) g.closure(g.topo_ranks);
  return SW_OK;
}

// graph.py:275-288 — keep (u,v) iff no other direct successor w of u reaches v.
std::vector<std::pair<int64_t, int64_t>> meg_edges(const Graph& g) {
  std::vector<std::pair<int64_t, int64_t>> kept;
  for (size_t k = 0; k < g.edges.size(); ++k) {
    int64_t u = g.redge[k].first, v = g.redge[k].second;
    bool bypass = false;
    for (int64_t w : g.succ[u]) {
      if (w != v && g.reaches(w, v)) {
        bypass = true;
        break;
      }
    }
    if (!bypass) kept.push_back(g.edges[k]);
  }
  std::sort(kept.begin(), kept.end());
  return kept;
}

// assign.py:82-102 — Kuhn's augmenting paths with the pinned scan order.
// The recursion is unrolled onto an explicit stack; the visit order of
// (x, y) pairs is identical to the recursive formulation.
std::vector<std::pair<int64_t, int64_t>> kuhn(int64_t left, int64_t right,
                                              const std::vector<std::pair<int64_t, int64_t>>& bedges) {
  std::vector<std::vector<int64_t>> adj(left);
  std::vector<std::pair<int64_t, int64_t>> sorted_edges = bedges;
  std::sort(sorted_edges.begin(), sorted_edges.end());
  for (auto& e : sorted_edges) adj[e.first].push_back(e.second);
  int64_t ny = right;
  for (auto& e : sorted_edges) ny = std::max(ny, e.second + 1);
  std::vector<int64_t> owner(ny, -1);
  std::vector<int64_t> stamp(ny, -1);
  struct Frame {
    int64_t x;
    size_t next;
  };
  std::vector<Frame> st;
  for (int64_t x0 = 0; x0 < left; ++x0) {
    st.clear();
    st.push_back({x0, 0});
    bool found = false;
    while (!st.empty()) {
      if (found) {
        Frame f = st.back();
        owner[adj[f.x][f.next - 1]] = f.x;
        st.pop_back();
        continue;
      }
      Frame& f = st.back();
      if (f.next == adj[f.x].size()) {
        st.pop_back();
        continue;
      }
      int64_t y = adj[f.x][f.next++];
      if (stamp[y] == x0) continue;
      stamp[y] = x0;
      if (owner[y] < 0) {
        found = true;
        continue;
      }
      int64_t nx = owner[y];
      st.push_back({nx, 0});
    }
  }
  std::vector<std::pair<int64_t, int64_t>> pairs;
  for (int64_t y = 0; y < ny; ++y)
    if (owner[y] >= 0) pairs.push_back({owner[y], y});
  std::sort(pairs.begin(), pairs.end());
  return pairs;
}

// assign.py:105-117
int check_matching(const std::vector<std::pair<int64_t, int64_t>>& bedges,
                   const std::vector<std::pair<int64_t, int64_t>>& pairs) {
  std::set<std::pair<int64_t, int64_t>> es(bedges.begin(), bedges.end());
  std::unordered_set<int64_t> xs, ys;
  for (auto& p : pairs) {
    std::string ps = "(" + std::to_string(p.first) + "," + std::to_string(p.second) + ")";
    if (!es.count(p)) return fail(SW_INVALID_MATCHING, "pair " + ps + " is not a bipartite edge");
    if (xs.count(p.first)) return fail(SW_INVALID_MATCHING, "left vertex " + std::to_string(p.first) + " matched twice");
    if (ys.count(p.second)) return fail(SW_INVALID_MATCHING, "right vertex " + std::to_string(p.second) + " matched twice");
    xs.insert(p.first);
    ys.insert(p.second);
  }
  return SW_OK;
}

// assign.py:154-162 — label groups by first use along the canonical topo order.
// group_of is indexed by rank; result: (id, stream) in topo order.
std::vector<std::pair<int64_t, int64_t>> canonical(const Graph& g, const std::vector<int64_t>& group_of) {
  std::unordered_map<int64_t, int64_t> label;
  std::vector<std::pair<int64_t, int64_t>> out;
  out.reserve(g.topo_ranks.size());
  for (int64_t r : g.topo_ranks) {
    int64_t grp = group_of[r];
    auto it = label.find(grp);
    int64_t s;
    if (it == label.end()) {
      s = (int64_t)label.size();
      label.emplace(grp, s);
    } else {
      s = it->second;
    }
    out.push_back({g.sorted_ids[r], s});
  }
  return out;
}

// assign.py:138-151 — union matched pairs, then canonical labels.
std::vector<std::pair<int64_t, int64_t>> partition(const Graph& g, const std::vector<std::pair<int64_t, int64_t>>& pairs) {
  const int64_t N = (int64_t)g.sorted_ids.size();
  std::vector<int64_t> parent(N);
  for (int64_t i = 0; i < N; ++i) parent[i] = i;
  auto find = [&](int64_t x) {
    int64_t r = x;
    while (parent[r] != r) r = parent[r];
    while (parent[x] != r) {
      int64_t nx = parent[x];
      parent[x] = r;
      x = nx;
    }
    return r;
  };
  for (auto& p : pairs) {
    int64_t a = find(p.first), b = find(p.second);
    if (a != b) parent[b] = a;
  }
  std::vector<int64_t> grp(N);
  for (int64_t i = 0; i < N; ++i) grp[i] = find(i);
  return canonical(g, grp);
}

// assign.py:165-179 — every stream must be a chain of the reachability order.
// Equivalent O(V) form: members sorted by topo position, consecutive members
// must be ordered (pairwise order is then implied by transitivity).
int is_max_concurrent(const Graph& g, const Assign& f, bool* out) {
  std::vector<int64_t> topo_pos(g.sorted_ids.size());
  for (size_t i = 0; i < g.topo_ranks.size(); ++i) topo_pos[g.topo_ranks[i]] = (int64_t)i;
  std::map<int64_t, std::vector<int64_t>> by_stream;
  std::vector<int64_t> order_of_streams;
  for (auto& p : f.items) {
    auto it = by_stream.find(p.second);
    if (it == by_stream.end()) order_of_streams.push_back(p.second);
    by_stream[p.second].push_back(p.first);
  }
  for (int64_t s : order_of_streams) {
    auto& mem = by_stream[s];
    if (mem.size() < 2) continue;
    std::vector<std::pair<int64_t, int64_t>> ranked;
    for (int64_t id : mem) {
      auto it = g.rank.find(id);
      if (it == g.rank.end()) return fail(SW_KEY_ERROR, std::to_string(id));
      ranked.push_back({topo_pos[it->second], it->second});
    }
    std::sort(ranked.begin(), ranked.end());
    for (size_t i = 1; i < ranked.size(); ++i) {
      if (ranked[i].second == ranked[i - 1].second) continue;
      if (!g.reaches(ranked[i - 1].second, ranked[i].second)) {
        *out = false;
        return SW_OK;
      }
    }
  }
  *out = true;
  return SW_OK;
}

// assign.py:182-209
int min_sync_plan(const Graph& g, const std::vector<std::pair<int64_t, int64_t>>& meg, const Assign& f,
                  std::vector<std::pair<int64_t, int64_t>>* plan) {
  for (int64_t id : g.ids)
    if (!f.map.count(id)) return fail(SW_UNKNOWN_STREAM, "task " + std::to_string(id) + " has no stream");
  bool ok = false;
  int rc = is_max_concurrent(g, f, &ok);
  if (rc) return rc;
  if (!ok)
    return fail(SW_NOT_MAX_CONCURRENT,
                "two order-independent tasks share a stream; the unique-parent rule does not apply");
  std::unordered_map<int64_t, int64_t> parent_seen;
  std::set<std::pair<int64_t, int64_t>> dropped;
  for (auto& e : meg) {
    auto su = f.map.find(e.first), sv = f.map.find(e.second);
    if (su == f.map.end()) return fail(SW_KEY_ERROR, std::to_string(e.first));
    if (sv == f.map.end()) return fail(SW_KEY_ERROR, std::to_string(e.second));
    if (su->second == sv->second) {
      auto it = parent_seen.find(e.second);
      if (it != parent_seen.end())
        return fail(SW_NOT_MAX_CONCURRENT, "task " + std::to_string(e.second) + " has two same-stream parents " +
                                               std::to_string(it->second) + " and " + std::to_string(e.first));
      parent_seen[e.second] = e.first;
      dropped.insert(e);
    }
  }
  plan->clear();
  for (auto& e : meg)
    if (!dropped.count(e)) plan->push_back(e);
  return SW_OK;
}

// assign.py:212-230 — every cross-stream edge (u,v) needs a plan edge (a,b)
// that is itself a graph edge with u →* a and b →* v (reflexive).
int plan_is_safe(const Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan, bool* out) {
  std::set<std::pair<int64_t, int64_t>> es(g.edges.begin(), g.edges.end());
  std::vector<std::pair<int64_t, int64_t>> covers;  // as ranks
  for (auto& e : plan)
    if (es.count(e)) covers.push_back({g.rank.at(e.first), g.rank.at(e.second)});
  for (size_t k = 0; k < g.edges.size(); ++k) {
    auto su = f.map.find(g.edges[k].first), sv = f.map.find(g.edges[k].second);
    if (su == f.map.end()) return fail(SW_KEY_ERROR, std::to_string(g.edges[k].first));
    if (sv == f.map.end()) return fail(SW_KEY_ERROR, std::to_string(g.edges[k].second));
    if (su->second == sv->second) continue;
    int64_t u = g.redge[k].first, v = g.redge[k].second;
    bool covered = false;
    for (auto& c : covers) {
      bool ua = (u == c.first) || g.reaches(u, c.first);
      if (!ua) continue;
      if (c.second == v || g.reaches(c.second, v)) {
        covered = true;
        break;
      }
    }
    if (!covered) {
      *out = false;
      return SW_OK;
    }
  }
  *out = true;
  return SW_OK;
}

// assign.py:233-240
int assign_streams(Graph& g, std::vector<std::pair<int64_t, int64_t>>* stream_of,
                   std::vector<std::pair<int64_t, int64_t>>* plan, std::vector<std::pair<int64_t, int64_t>>* meg) {
  int rc = prepare(g, true, true);
  if (rc) return rc;
  *meg = meg_edges(g);
  std::vector<std::pair<int64_t, int64_t>> bedges;
  bedges.reserve(meg->size());
  for (auto& e : *meg) bedges.push_back({g.rank[e.first], g.rank[e.second]});
  std::sort(bedges.begin(), bedges.end());
  int64_t N = (int64_t)g.sorted_ids.size();
  auto pairs = kuhn(N, N, bedges);
  rc = check_matching(bedges, pairs);
  if (rc) return rc;
  *stream_of = partition(g, pairs);
  Assign f = Assign::from_pairs(*stream_of);
  return min_sync_plan(g, *meg, f, plan);
}

// assign.py:243-270
int fold_streams(const Graph& g, const Assign& f, int64_t max_streams, std::vector<std::pair<int64_t, int64_t>>* out) {
  if (max_streams < 1) return fail(SW_VALUE_ERROR, "max_streams must be >= 1");
  int64_t ns = -1;
  for (auto& p : f.items) ns = std::max(ns, p.second);
  ns += 1;
  if (ns <= max_streams) {
    *out = f.items;
    return SW_OK;
  }
  std::unordered_map<int64_t, int64_t> dur;
  for (int64_t i = 0; i < g.n; ++i) dur.emplace(g.ids[i], g.dur[i]);
  std::vector<int64_t> work(ns, 0);
  for (auto& p : f.items) {
    auto it = dur.find(p.first);
    if (it == dur.end()) return fail(SW_KEY_ERROR, std::to_string(p.first));
    if (p.second < 0 || p.second >= ns) return fail(SW_KEY_ERROR, std::to_string(p.second));
    work[p.second] += it->second;
  }
  std::vector<int64_t> by_load(ns);
  for (int64_t s = 0; s < ns; ++s) by_load[s] = s;
  std::sort(by_load.begin(), by_load.end(), [&](int64_t a, int64_t b) {
    if (work[a] != work[b]) return work[a] > work[b];
    return a < b;
  });
  std::vector<int64_t> keep(by_load.begin(), by_load.begin() + max_streams);
  std::sort(keep.begin(), keep.end());
  std::vector<int64_t> rest(by_load.begin() + max_streams, by_load.end());
  std::sort(rest.begin(), rest.end(), [&](int64_t a, int64_t b) {
    if (work[a] != work[b]) return work[a] < work[b];
    return a < b;
  });
  std::vector<int64_t> target(ns);
  for (int64_t s : keep) target[s] = s;
  for (size_t i = 0; i < rest.size(); ++i) target[rest[i]] = keep[i % keep.size()];
  std::vector<int64_t> grp(g.sorted_ids.size(), -1);
  for (auto& p : f.items) {
    auto it = g.rank.find(p.first);
    if (it != g.rank.end()) grp[it->second] = target[p.second];
  }
  for (int64_t r = 0; r < (int64_t)grp.size(); ++r)
    if (grp[r] < 0) return fail(SW_KEY_ERROR, std::to_string(g.sorted_ids[r]));
  *out = canonical(g, grp);
  return SW_OK;
}

// schedule.py:118-155 — first fit over a linear trace.
int reserve_arena(int64_t n, const int64_t* keys, const int32_t* kinds, const int64_t* sizes, int64_t* out_offset,
                  int64_t* total_out, int64_t* bad) {
  std::map<int64_t, std::pair<int64_t, int64_t>> live;   // key -> (offset, size)
  std::multiset<std::pair<int64_t, int64_t>> live_sorted;  // sorted (offset, size)
  std::unordered_set<int64_t> placed;
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t key = keys[i];
    if (kinds[i] == SW_MEM_ALLOC) {
      if (placed.count(key)) {
        *bad = i;
        return fail(SW_VALUE_ERROR, "allocated twice");
      }
      int64_t size = sizes[i];
      int64_t off = 0;
      for (auto& blk : live_sorted) {
        if (off + size <= blk.first) break;
        off = std::max(off, blk.first + blk.second);
      }
      live[key] = {off, size};
      live_sorted.insert({off, size});
      placed.insert(key);
      out_offset[i] = off;
      total = std::max(total, off + size);
    } else if (kinds[i] == SW_MEM_FREE) {
      if (!placed.count(key)) {
        *bad = i;
        return fail(SW_FREE_BEFORE_ALLOC, "before its alloc");
      }
      auto it = live.find(key);
      if (it == live.end()) {
        *bad = i;
        return fail(SW_DOUBLE_FREE, "freed twice");
      }
      live_sorted.erase(live_sorted.find(it->second));
      live.erase(it);
    } else {
      *bad = i;
      return fail(SW_VALUE_ERROR, "unknown mem event kind");
    }
  }
  *total_out = total;
  return SW_OK;
}

// schedule.py:53-115
int pre_run(Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan, sw_schedule_out* out) {
  int rc = g.index(nullptr);
  if (rc) return fail(SW_KEY_ERROR, g_last_error);
  for (int64_t id : g.ids)
    if (!f.map.count(id)) return fail(SW_UNKNOWN_STREAM, "task " + std::to_string(id) + " has no stream");
  int64_t ns = -1;
  std::set<int64_t> used;
  for (auto& p : f.items) {
    ns = std::max(ns, p.second);
    used.insert(p.second);
  }
  ns += 1;
  bool dense = (int64_t)used.size() == ns && (used.empty() || (*used.begin() == 0 && *used.rbegin() == ns - 1));
  if (!dense) {
    std::string s = "[";
    bool first = true;
    for (int64_t u : used) {
      if (!first) s += ", ";
      s += std::to_string(u);
      first = false;
    }
    s += "]";
    return fail(SW_UNKNOWN_STREAM, "stream ids are not dense from 0: " + s);
  }
  std::set<std::pair<int64_t, int64_t>> es(g.edges.begin(), g.edges.end());
  for (auto& e : plan)
    if (!es.count(e)) return fail(SW_UNSAFE_PLAN, "sync edge " + edge_str(e.first, e.second) + " is not a graph edge");
  rc = g.topo(&g.topo_ranks);
  if (rc) return rc;
  g.closure(g.topo_ranks);
  bool safe = false;
  rc = plan_is_safe(g, f, plan, &safe);
  if (rc) return rc;
  if (!safe) return fail(SW_UNSAFE_PLAN, "plan leaves a cross-stream dependency uncovered");

  // event id = index in sorted(plan); duplicates keep the last index (dict semantics)
  std::vector<std::pair<int64_t, int64_t>> sp = plan;
  std::sort(sp.begin(), sp.end());
  std::map<std::pair<int64_t, int64_t>, int64_t> event_of;
  for (size_t i = 0; i < sp.size(); ++i) event_of[sp[i]] = (int64_t)i;
  const int64_t N = (int64_t)g.sorted_ids.size();
  std::vector<std::vector<int64_t>> waits(N), records(N);
  for (auto& e : sp) {
    int64_t ev = event_of[e];
    records[g.rank[e.first]].push_back(ev);
    waits[g.rank[e.second]].push_back(ev);
  }
  std::vector<std::vector<std::pair<int32_t, int64_t>>> fifo(ns);
  int64_t n_ops = 0;
  auto emit = [&](int64_t s, int32_t kind, int64_t arg) {
    fifo[s].push_back({kind, arg});
    out->order[n_ops++] = s;
  };
  // mem trace: keys (node, idx) → integer key = global mem index of the alloc
  std::vector<int64_t> tkeys, tsizes, tnode, tidx;
  std::vector<int32_t> tkinds;
  int64_t wpos = 0;
  out->task_args_start[0] = 0;
  for (int64_t r : g.topo_ranks) {
    int64_t v = g.sorted_ids[r];
    int64_t s = f.map.at(v);
    for (int64_t ev : waits[r]) emit(s, SW_OP_WAIT, ev);
    emit(s, SW_OP_LAUNCH, v);
    for (int64_t ev : records[r]) emit(s, SW_OP_RECORD, ev);
    int64_t pos = g.first_pos[r];  // g.node(v): first node with that id
    int64_t b = g.mem_start[pos], e = g.mem_start[pos + 1];
    for (int64_t k = b; k < e; ++k) {
      int64_t local = k - b;
      if (g.mem_kind[k] == SW_MEM_ALLOC) {
        tkeys.push_back(k);
        tidx.push_back(local);
      } else {
        tkeys.push_back(b + g.mem_arg[k]);
        tidx.push_back(g.mem_arg[k]);
      }
      tkinds.push_back(g.mem_kind[k]);
      tsizes.push_back(g.mem_kind[k] == SW_MEM_ALLOC ? g.mem_arg[k] : 0);
      tnode.push_back(v);
    }
    out->walk[wpos++] = v;
  }
  std::vector<int64_t> offs(tkeys.size(), -1);
  int64_t total = 0, bad = -1;
  rc = reserve_arena((int64_t)tkeys.size(), tkeys.data(), tkinds.data(), tsizes.data(), offs.data(), &total, &bad);
  if (rc) {
    std::string key = "(" + std::to_string(tnode[bad]) + ", " + std::to_string(tidx[bad]) + ")";
    if (rc == SW_FREE_BEFORE_ALLOC) return fail(rc, "free of " + key + " before its alloc");
    if (rc == SW_DOUBLE_FREE) return fail(rc, "block " + key + " freed twice");
    return fail(rc, "block " + key + " allocated twice");
  }
  int64_t nb = 0;
  std::unordered_map<int64_t, int64_t> off_of_key;
  for (size_t i = 0; i < tkeys.size(); ++i) {
    if (tkinds[i] != SW_MEM_ALLOC) continue;
    out->block_node[nb] = tnode[i];
    out->block_index[nb] = tidx[i];
    out->block_offset[nb] = offs[i];
    out->block_size[nb] = tsizes[i];
    off_of_key[tkeys[i]] = offs[i];
    ++nb;
  }
  int64_t ta = 0;
  for (int64_t w = 0; w < wpos; ++w) {
    int64_t r = g.rank[out->walk[w]];
    int64_t pos = g.first_pos[r];
    for (int64_t k = g.mem_start[pos]; k < g.mem_start[pos + 1]; ++k)
      if (g.mem_kind[k] == SW_MEM_ALLOC) out->task_args[ta++] = off_of_key[k];
    out->task_args_start[w + 1] = ta;
  }
  int64_t p = 0;
  for (int64_t s = 0; s < ns; ++s) {
    out->stream_len[s] = (int64_t)fifo[s].size();
    for (auto& op : fifo[s]) {
      out->op_kind[p] = op.first;
      out->op_arg[p] = op.second;
      ++p;
    }
  }
  out->n_streams = ns;
  out->n_ops = n_ops;
  out->event_count = (int64_t)event_of.size();
  out->arena_total = total;
  out->n_blocks = nb;
  return SW_OK;
}

// graph.py:291-301
int critical_path(Graph& g, int64_t* out) {
  int rc = prepare(g, false, false);
  if (rc) return rc;
  if (g.n == 0) {
    *out = 0;
    return SW_OK;
  }
  const int64_t N = (int64_t)g.sorted_ids.size();
  std::vector<int64_t> dur(N, 0), best(N, 0);
  // durations(): dict comprehension keeps the LAST duplicate
  for (int64_t i = 0; i < g.n; ++i) dur[g.rank[g.ids[i]]] = g.dur[i];
  int64_t m = 0;
  bool any = false;
  for (int64_t v : g.topo_ranks) {
    int64_t inc = 0;
    for (int64_t p : g.pred[v]) inc = std::max(inc, best[p]);
    best[v] = inc + dur[v];
    m = any ? std::max(m, best[v]) : best[v];
    any = true;
  }
  *out = m;
  return SW_OK;
}

}  // namespace sw
