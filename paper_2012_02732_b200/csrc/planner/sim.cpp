// Integer-time multi-stream device simulator — native restatement of the
// reference's semantic model (sim.py:64-234).  It is not the executor (the
// CUDA graph is); it is kept so the drop-in API still answers simulate /
// run_framework_mode / compare_modes, and so measured kernel durations can be
// fed back into the reference's replay semantics.
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "planner.h"

namespace sw {

namespace {
struct QOp {
  int32_t kind;
  int64_t arg;
  int64_t visible;
};
}  // namespace

int simulate(const Graph& g, int64_t n_streams, const int64_t* stream_len, const int32_t* op_kind,
             const int64_t* op_arg, int64_t n_order, const int64_t* order, const sw_sim_config* cfg,
             int64_t* makespan, int64_t* active, std::unordered_map<int64_t, std::pair<int64_t, int64_t>>* intervals,
             std::vector<std::pair<int64_t, int64_t>>* fire_log) {
  // sim.py:84-101 — schedule must launch known tasks; capacity admission.
  std::unordered_map<int64_t, int64_t> duration, demand;
  std::unordered_map<int64_t, std::vector<int64_t>> preds;
  for (int64_t i = 0; i < g.n; ++i) {
    duration[g.ids[i]] = g.dur[i];
    demand[g.ids[i]] = g.dem[i];
    preds[g.ids[i]];
  }
  std::vector<int64_t> sbase(n_streams + 1, 0);
  for (int64_t s = 0; s < n_streams; ++s) sbase[s + 1] = sbase[s] + stream_len[s];
  for (int64_t k = 0; k < sbase[n_streams]; ++k)
    if (op_kind[k] == SW_OP_LAUNCH && !duration.count(op_arg[k]))
      return fail(SW_GRAPH_ERROR, "schedule launches unknown task " + std::to_string(op_arg[k]));
  for (auto& e : g.edges) {
    auto it = preds.find(e.second);
    if (it == preds.end()) return fail(SW_KEY_ERROR, std::to_string(e.second));
    it->second.push_back(e.first);
  }
  const bool bounded = cfg->capacity > 0;
  if (bounded)
    for (int64_t i = 0; i < g.n; ++i)
      if (g.dem[i] > cfg->capacity)
        return fail(SW_CAPACITY_EXCEEDED, "task " + std::to_string(g.ids[i]) + " demands " +
                                              std::to_string(g.dem[i]) + " of capacity " +
                                              std::to_string(cfg->capacity));

  // replay_order (schedule.py:158-165)
  std::vector<std::pair<int64_t, int64_t>> flat;  // (stream, global op index)
  std::vector<int64_t> cursor(n_streams, 0);
  for (int64_t i = 0; i < n_order; ++i) {
    int64_t s = order[i];
    if (s < 0 || s >= n_streams || cursor[s] >= stream_len[s])
      return fail(SW_VALUE_ERROR, "capture order does not match the stream FIFOs");
    flat.push_back({s, sbase[s] + cursor[s]});
    cursor[s]++;
  }
  const bool gated = cfg->framework_mode != 0;
  const int64_t cost = gated ? cfg->overhead_framework : cfg->overhead_replay;

  std::vector<std::vector<QOp>> queues(n_streams);
  std::vector<size_t> qpos(n_streams, 0);
  std::vector<int64_t> free_at(n_streams, 0);
  std::unordered_map<int64_t, int64_t> fired;
  std::vector<std::pair<int64_t, int64_t>> running;  // (end, demand), only end > now kept
  int64_t host = 0;
  size_t sub = 0;

  auto pump = [&]() -> bool {  // sim.py:118-134
    bool changed = false;
    while (sub < flat.size()) {
      int64_t s = flat[sub].first, k = flat[sub].second;
      int64_t begin = host;
      if (gated && op_kind[k] == SW_OP_LAUNCH) {
        auto& ps = preds[op_arg[k]];
        bool all = true;
        for (int64_t p : ps)
          if (!intervals->count(p)) {
            all = false;
            break;
          }
        if (!all) break;
        for (int64_t p : ps) begin = std::max(begin, (*intervals)[p].second);
      }
      int64_t visible = begin + cost;
      queues[s].push_back({op_kind[k], op_arg[k], visible});
      host = visible;
      ++sub;
      changed = true;
    }
    return changed;
  };
  auto available = [&](int64_t now) {  // sim.py:136-138
    int64_t used = 0;
    for (auto& r : running)
      if (r.first > now) used += r.second;
    return cfg->capacity - used;
  };
  auto wave = [&](int64_t now) -> bool {  // sim.py:140-171
    bool changed = false;
    for (int64_t s = 0; s < n_streams; ++s) {
      while (qpos[s] < queues[s].size()) {
        const QOp& op = queues[s][qpos[s]];
        int64_t ready = std::max(op.visible, free_at[s]);
        if (op.kind == SW_OP_WAIT) {
          auto it = fired.find(op.arg);
          if (it == fired.end()) break;
          ready = std::max(ready, it->second);
          if (ready > now) break;
          free_at[s] = ready;
        } else if (op.kind == SW_OP_RECORD) {
          if (ready > now) break;
          fired[op.arg] = ready;
          fire_log->push_back({op.arg, ready});
          free_at[s] = ready;
        } else {
          if (ready > now) break;
          int64_t d = demand[op.arg];
          if (bounded && d > available(now)) break;
          int64_t end = now + duration[op.arg];
          (*intervals)[op.arg] = {now, end};
          running.push_back({end, d});
          free_at[s] = end;
        }
        ++qpos[s];
        changed = true;
      }
    }
    return changed;
  };
  auto drained = [&]() {
    if (sub != flat.size()) return false;
    for (int64_t s = 0; s < n_streams; ++s)
      if (qpos[s] != queues[s].size()) return false;
    return true;
  };
  auto next_candidate = [&](int64_t now, int64_t* best) -> bool {  // sim.py:178-195
    bool have = false;
    for (int64_t s = 0; s < n_streams; ++s) {
      if (qpos[s] == queues[s].size()) continue;
      const QOp& op = queues[s][qpos[s]];
      int64_t ready = std::max(op.visible, free_at[s]);
      if (op.kind == SW_OP_WAIT) {
        auto it = fired.find(op.arg);
        if (it == fired.end()) continue;
        ready = std::max(ready, it->second);
      }
      if (ready > now && (!have || ready < *best)) {
        *best = ready;
        have = true;
      }
    }
    for (auto& r : running)
      if (r.first > now && (!have || r.first < *best)) {
        *best = r.first;
        have = true;
      }
    return have;
  };

  pump();
  int64_t now = 0;
  while (true) {  // sim.py:197-209
    while (true) {
      if (wave(now)) continue;
      if (pump()) continue;
      break;
    }
    if (drained()) break;
    int64_t nxt = 0;
    if (!next_candidate(now, &nxt))
      return fail(SW_DEADLOCK_DETECTED, "no progress possible at t=" + std::to_string(now) + " with ops still pending");
    now = nxt;
    // entries that ended at or before `now` can never count again
    running.erase(std::remove_if(running.begin(), running.end(),
                                 [&](const std::pair<int64_t, int64_t>& r) { return r.first <= now; }),
                  running.end());
  }

  // sim.py:211-234 — makespan and union measure of busy intervals
  int64_t ms = 0;
  std::vector<std::pair<int64_t, int64_t>> spans;
  for (auto& kv : *intervals) {
    ms = std::max(ms, kv.second.second);
    if (kv.second.second > kv.second.first) spans.push_back(kv.second);
  }
  std::sort(spans.begin(), spans.end());
  int64_t total = 0, cs = 0, ce = 0;
  bool open = false;
  for (auto& sp : spans) {
    if (!open || sp.first > ce) {
      if (open) total += ce - cs;
      cs = sp.first;
      ce = sp.second;
      open = true;
    } else if (sp.second > ce) {
      ce = sp.second;
    }
  }
  if (open) total += ce - cs;
  std::sort(fire_log->begin(), fire_log->end());
  *makespan = ms;
  *active = total;
  return SW_OK;
}

}  // namespace sw
