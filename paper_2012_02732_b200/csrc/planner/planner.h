// Internal interface of the native planner (see planner.cpp, capi.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <map>

#include "../../../include/streamweave_b200.h"

namespace sw {

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);

struct Graph {
  int64_t n = 0;  // nodes as given (duplicates allowed until validated)
  std::vector<int64_t> ids, dur, dem;
  std::vector<int64_t> mem_start, mem_arg;
  std::vector<int32_t> mem_kind;
  std::vector<std::pair<int64_t, int64_t>> edges;  // ids, given order

  // dense index (after index())
  std::vector<int64_t> sorted_ids;               // rank -> id
  std::unordered_map<int64_t, int64_t> rank;     // id -> rank
  std::vector<int64_t> first_pos;                // rank -> first position in ids
  std::vector<std::vector<int64_t>> succ, pred;  // ranks, edge order
  std::vector<std::pair<int64_t, int64_t>> redge;
  std::vector<int64_t> topo_ranks;
  int64_t words = 0;
  std::vector<uint64_t> reach;

  static Graph from_view(const sw_graph_view* v);
  int index(std::string* missing_key);
  bool find_cycle(std::vector<int64_t>* witness) const;
  int topo(std::vector<int64_t>* order_ranks) const;
  int closure(const std::vector<int64_t>& order_ranks);
  bool reaches(int64_t ru, int64_t rv) const {
    return (reach[(size_t)(ru * words + (rv >> 6))] >> (rv & 63)) & 1ull;
  }
};

// Assignment lookup helper (dict semantics of StreamAssignment.stream_of).
struct Assign {
  std::vector<std::pair<int64_t, int64_t>> items;  // insertion order
  std::unordered_map<int64_t, int64_t> map;
  static Assign from_view(const sw_assignment_view* f) {
    Assign a;
    for (int64_t i = 0; i < f->n; ++i) {
      auto it = a.map.find(f->ids[i]);
      if (it == a.map.end()) {
        a.map.emplace(f->ids[i], f->streams[i]);
        a.items.push_back({f->ids[i], f->streams[i]});
      } else {
        it->second = f->streams[i];
        for (auto& p : a.items)
          if (p.first == f->ids[i]) p.second = f->streams[i];
      }
    }
    return a;
  }
  static Assign from_pairs(const std::vector<std::pair<int64_t, int64_t>>& v) {
    Assign a;
    a.items = v;
    for (auto& p : v) a.map[p.first] = p.second;
    return a;
  }
};

int validate(const Graph& g);
int prepare(Graph& g, bool do_validate, bool need_closure);
std::vector<std::pair<int64_t, int64_t>> meg_edges(const Graph& g);
std::vector<std::pair<int64_t, int64_t>> kuhn(int64_t left, int64_t right,
                                              const std::vector<std::pair<int64_t, int64_t>>& bedges);
int check_matching(const std::vector<std::pair<int64_t, int64_t>>& bedges,
                   const std::vector<std::pair<int64_t, int64_t>>& pairs);
std::vector<std::pair<int64_t, int64_t>> partition(const Graph& g,
                                                   const std::vector<std::pair<int64_t, int64_t>>& pairs);
int assign_streams(Graph& g, std::vector<std::pair<int64_t, int64_t>>* stream_of,
                   std::vector<std::pair<int64_t, int64_t>>* plan, std::vector<std::pair<int64_t, int64_t>>* meg);
int reserve_arena(int64_t n, const int64_t* keys, const int32_t* kinds, const int64_t* sizes, int64_t* out_offset,
                  int64_t* total_out, int64_t* bad);
int critical_path(Graph& g, int64_t* out);
int is_max_concurrent(const Graph& g, const Assign& f, bool* out);
int min_sync_plan(const Graph& g, const std::vector<std::pair<int64_t, int64_t>>& meg, const Assign& f,
                  std::vector<std::pair<int64_t, int64_t>>* plan);
int plan_is_safe(const Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan, bool* out);
int fold_streams(const Graph& g, const Assign& f, int64_t max_streams, std::vector<std::pair<int64_t, int64_t>>* out);
int pre_run(Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan, sw_schedule_out* out);
std::vector<std::pair<int64_t, int64_t>> canonical(const Graph& g, const std::vector<int64_t>& group_of);
// verify.cpp (oracle.py exhaustive verifiers)
int verify(Graph& g, const Assign* f_given, const std::vector<std::pair<int64_t, int64_t>>& plan_given,
           int64_t out[5]);
int oracle_plan_is_safe(Graph& g, const Assign& f, const std::vector<std::pair<int64_t, int64_t>>& plan,
                        bool* out);
int min_syncs_brute(Graph& g, const Assign& f, int64_t bound, int64_t* out);
int enumerate_assignments(Graph& g, int64_t cap, int64_t* out_order, int64_t* out_streams, int64_t* out_count);

}  // namespace sw
