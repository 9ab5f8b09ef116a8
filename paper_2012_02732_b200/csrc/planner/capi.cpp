// extern "C" boundary of the planner (include/streamweave_b200.h, group 1).
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "planner.h"

namespace sw {
int simulate(const Graph& g, int64_t n_streams, const int64_t* stream_len, const int32_t* op_kind,
             const int64_t* op_arg, int64_t n_order, const int64_t* order, const sw_sim_config* cfg,
             int64_t* makespan, int64_t* active, std::unordered_map<int64_t, std::pair<int64_t, int64_t>>* intervals,
             std::vector<std::pair<int64_t, int64_t>>* fire_log);
}

using sw::Assign;
using sw::Graph;
using Pairs = std::vector<std::pair<int64_t, int64_t>>;

static Pairs pairs_of(int64_t n, const int64_t* flat) {
  Pairs p(n);
  for (int64_t i = 0; i < n; ++i) p[i] = {flat[2 * i], flat[2 * i + 1]};
  return p;
}
static void write_pairs(const Pairs& p, int64_t* out, int64_t* n) {
  for (size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].first;
    out[2 * i + 1] = p[i].second;
  }
  *n = (int64_t)p.size();
}
static void write_assign(const Pairs& p, int64_t* ids, int64_t* streams) {
  for (size_t i = 0; i < p.size(); ++i) {
    ids[i] = p[i].first;
    streams[i] = p[i].second;
  }
}

#define SW_TRY(...)                                        \
  try {                                                    \
    __VA_ARGS__                                                 \
  } catch (const std::exception& ex) {                     \
    return sw::fail(SW_VALUE_ERROR, ex.what());            \
  } catch (...) {                                          \
    return sw::fail(SW_VALUE_ERROR, "unknown C++ error");  \
  }

extern "C" {

const char* sw_last_error(void) { return sw::g_last_error.c_str(); }
const char* sw_version(void) { return "paper_2012_02732_b200 0.1.0 (sm_100a)"; }

int sw_plan_validate(const sw_graph_view* v) {
  SW_TRY(Graph g = Graph::from_view(v); return sw::validate(g);)
}

int sw_plan_topological_order(const sw_graph_view* v, int64_t* out) {
  SW_TRY(Graph g = Graph::from_view(v); int rc = sw::prepare(g, false, false); if (rc) return rc;
         for (size_t i = 0; i < g.topo_ranks.size(); ++i) out[i] = g.sorted_ids[g.topo_ranks[i]];
         return SW_OK;)
}

int sw_plan_transitive_closure(const sw_graph_view* v, uint64_t* out_rows) {
  SW_TRY(Graph g = Graph::from_view(v); int rc = sw::prepare(g, false, true); if (rc) return rc;
         std::copy(g.reach.begin(), g.reach.end(), out_rows); return SW_OK;)
}

int sw_plan_minimum_equivalent_graph(const sw_graph_view* v, int64_t* out_edges, int64_t* out_n) {
  SW_TRY(Graph g = Graph::from_view(v); int rc = sw::prepare(g, false, true); if (rc) return rc;
         write_pairs(sw::meg_edges(g), out_edges, out_n); return SW_OK;)
}

int sw_plan_critical_path_time(const sw_graph_view* v, int64_t* out_time) {
  SW_TRY(Graph g = Graph::from_view(v); return sw::critical_path(g, out_time);)
}

int sw_plan_maximum_matching(int64_t left, int64_t right, int64_t n_edges, const int64_t* edges,
                             int64_t* out_pairs, int64_t* out_n) {
  SW_TRY(Pairs e = pairs_of(n_edges, edges);
         for (auto& p : e) if (p.first < 0 || p.first >= left) return sw::fail(SW_VALUE_ERROR, "left vertex out of range");
         write_pairs(sw::kuhn(left, right, e), out_pairs, out_n); return SW_OK;)
}

int sw_plan_assignment_from_matching(const sw_graph_view* base, int64_t n_meg, const int64_t* meg_edges,
                                     int64_t n_pairs, const int64_t* pairs, int64_t* out_ids,
                                     int64_t* out_streams) {
  SW_TRY(Graph g = Graph::from_view(base); int rc = sw::prepare(g, false, false); if (rc) return rc;
         Pairs meg = pairs_of(n_meg, meg_edges); Pairs bed; for (auto& e : meg) {
           auto iu = g.rank.find(e.first), iv = g.rank.find(e.second);
           if (iu == g.rank.end()) return sw::fail(SW_KEY_ERROR, std::to_string(e.first));
           if (iv == g.rank.end()) return sw::fail(SW_KEY_ERROR, std::to_string(e.second));
           bed.push_back({iu->second, iv->second});
         } std::sort(bed.begin(), bed.end());
         Pairs m = pairs_of(n_pairs, pairs); rc = sw::check_matching(bed, m); if (rc) return rc;
         write_assign(sw::partition(g, m), out_ids, out_streams); return SW_OK;)
}

int sw_plan_is_max_concurrent(const sw_graph_view* v, const sw_assignment_view* f, int32_t* out_bool) {
  SW_TRY(Graph g = Graph::from_view(v); int rc = sw::prepare(g, false, true); if (rc) return rc;
         bool ok = false; rc = sw::is_max_concurrent(g, Assign::from_view(f), &ok); if (rc) return rc;
         *out_bool = ok ? 1 : 0; return SW_OK;)
}

int sw_plan_min_sync_plan(const sw_graph_view* base, int64_t n_meg, const int64_t* meg_edges,
                          const sw_assignment_view* f, int64_t* out_plan, int64_t* out_n) {
  SW_TRY(Graph g = Graph::from_view(base); Assign a = Assign::from_view(f);
         for (int64_t id : g.ids) if (!a.map.count(id))
           return sw::fail(SW_UNKNOWN_STREAM, "task " + std::to_string(id) + " has no stream");
         int rc = sw::prepare(g, false, true); if (rc) return rc;
         Pairs plan; rc = sw::min_sync_plan(g, pairs_of(n_meg, meg_edges), a, &plan); if (rc) return rc;
         write_pairs(plan, out_plan, out_n); return SW_OK;)
}

int sw_plan_plan_is_safe(const sw_graph_view* v, const sw_assignment_view* f, int64_t n_plan,
                         const int64_t* plan, int32_t* out_bool) {
  SW_TRY(Graph g = Graph::from_view(v); int rc = sw::prepare(g, false, true); if (rc) return rc;
         bool ok = false; rc = sw::plan_is_safe(g, Assign::from_view(f), pairs_of(n_plan, plan), &ok);
         if (rc) return rc; *out_bool = ok ? 1 : 0; return SW_OK;)
}

int sw_plan_assign_streams(const sw_graph_view* v, int64_t* out_ids, int64_t* out_streams, int64_t* out_sync,
                           int64_t* out_n_sync, int64_t* out_meg, int64_t* out_n_meg) {
  SW_TRY(Graph g = Graph::from_view(v); Pairs f, plan, meg; int rc = sw::assign_streams(g, &f, &plan, &meg);
         if (rc) return rc; write_assign(f, out_ids, out_streams); write_pairs(plan, out_sync, out_n_sync);
         write_pairs(meg, out_meg, out_n_meg); return SW_OK;)
}

int sw_plan_verify(const sw_graph_view* v, const sw_assignment_view* f, int64_t n_plan, const int64_t* plan,
                   int64_t* out5) {
  SW_TRY(Graph g = Graph::from_view(v); if (!f) return sw::verify(g, nullptr, Pairs(), out5);
         Assign a = Assign::from_view(f); return sw::verify(g, &a, pairs_of(n_plan, plan), out5);)
}

int sw_plan_oracle_plan_is_safe(const sw_graph_view* v, const sw_assignment_view* f, int64_t n_plan,
                                const int64_t* plan, int32_t* out_bool) {
  SW_TRY(Graph g = Graph::from_view(v); bool ok = false;
         int rc = sw::oracle_plan_is_safe(g, Assign::from_view(f), pairs_of(n_plan, plan), &ok);
         if (rc) return rc; *out_bool = ok ? 1 : 0; return SW_OK;)
}

int sw_plan_min_syncs_brute(const sw_graph_view* v, const sw_assignment_view* f, int64_t bound, int64_t* out) {
  SW_TRY(Graph g = Graph::from_view(v); return sw::min_syncs_brute(g, Assign::from_view(f), bound, out);)
}

int sw_plan_enumerate_assignments(const sw_graph_view* v, int64_t cap, int64_t* out_order, int64_t* out_streams,
                                  int64_t* out_count) {
  SW_TRY(Graph g = Graph::from_view(v); return sw::enumerate_assignments(g, cap, out_order, out_streams, out_count);)
}

int sw_plan_fold_streams(const sw_graph_view* v, const sw_assignment_view* f, int64_t max_streams,
                         int64_t* out_ids, int64_t* out_streams) {
  SW_TRY(Graph g = Graph::from_view(v);
         if (max_streams < 1) return sw::fail(SW_VALUE_ERROR, "max_streams must be >= 1");
         int rc = sw::prepare(g, false, false); if (rc) return rc;
         Pairs out; rc = sw::fold_streams(g, Assign::from_view(f), max_streams, &out); if (rc) return rc;
         write_assign(out, out_ids, out_streams); return SW_OK;)
}

int sw_plan_pre_run(const sw_graph_view* v, const sw_assignment_view* f, int64_t n_plan, const int64_t* plan,
                    sw_schedule_out* out) {
  SW_TRY(Graph g = Graph::from_view(v); return sw::pre_run(g, Assign::from_view(f), pairs_of(n_plan, plan), out);)
}

int sw_plan_reserve_arena(int64_t n_events, const int64_t* keys, const int32_t* kinds, const int64_t* sizes,
                          int64_t* out_offset, int64_t* out_total, int64_t* out_bad_event) {
  SW_TRY(*out_bad_event = -1;
         return sw::reserve_arena(n_events, keys, kinds, sizes, out_offset, out_total, out_bad_event);)
}

int sw_plan_simulate(const sw_graph_view* v, int64_t n_streams, const int64_t* stream_len, const int32_t* op_kind,
                     const int64_t* op_arg, int64_t n_order, const int64_t* order, const sw_sim_config* cfg,
                     int64_t* out_makespan, int64_t* out_active, int64_t* out_start, int64_t* out_end,
                     int64_t* out_events, int64_t* out_n_events) {
  SW_TRY(Graph g = Graph::from_view(v);
         std::unordered_map<int64_t, std::pair<int64_t, int64_t>> iv; Pairs log;
         int rc = sw::simulate(g, n_streams, stream_len, op_kind, op_arg, n_order, order, cfg, out_makespan,
                               out_active, &iv, &log);
         if (rc) return rc;
         for (int64_t i = 0; i < g.n; ++i) {
           auto it = iv.find(g.ids[i]);
           out_start[i] = it == iv.end() ? -1 : it->second.first;
           out_end[i] = it == iv.end() ? -1 : it->second.second;
         } write_pairs(log, out_events, out_n_events); return SW_OK;)
}

}  // extern "C"
