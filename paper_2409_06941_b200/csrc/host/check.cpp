// replay_check (reference engine.hpp:100-104): re-derives
// every module invariant from a finished RunTrace alone.
#include <algorithm>
#include <map>
#include <set>
#include <tuple>

#include "io.hpp"

namespace freeride {

std::vector<std::string> replay_check(const RunTrace& tr) {
  std::vector<std::string> v;
  auto bad = [&](const std::string& s) {
    if (v.size() < 200) v.push_back(s);
  };
  const PipelineConfig& pc = tr.config.pipeline;
  const int p = pc.num_stages, m = pc.num_micro_batches, E = pc.num_epochs;
  auto op_name = [](const OpEvent& o) {
    return std::string(o.kind == OpKind::FP ? "F" : "B") + std::to_string(o.micro_batch) + "@s" +
           std::to_string(o.stage) + "e" + std::to_string(o.epoch);
  };

  // 1. ops: each (stage, kind, mb, epoch) exactly once, with its duration
  // (measured traces: durations are what the GPU took, and only the stages
  // that ran are in the trace)
  std::map<std::tuple<int, int, int, int>, const OpEvent*> at;
  std::set<int> present;
  Tick last_end = 0;
  for (const OpEvent& o : tr.ops) {
    const auto key = std::make_tuple(o.stage, static_cast<int>(o.kind), o.micro_batch, o.epoch);
    if (o.stage < 0 || o.stage >= p || o.micro_batch < 1 || o.micro_batch > m || o.epoch < 0 || o.epoch >= E) {
      bad("op " + op_name(o) + " outside the pipeline");
      continue;
    }
    if (!at.emplace(key, &o).second) bad("op " + op_name(o) + " appears twice");
    present.insert(o.stage);
    if (o.end < o.start) bad("op " + op_name(o) + " ends before it starts");
    const Tick want = o.kind == OpKind::FP ? pc.fp_ticks(o.stage) : pc.bp_ticks(o.stage);
    if (!tr.measured && o.end - o.start != want)
      bad("op " + op_name(o) + " lasts " + std::to_string(o.end - o.start) + " ticks, configured " +
          std::to_string(want));
    last_end = std::max(last_end, o.end);
  }
  const long long stages_run = tr.measured ? static_cast<long long>(present.size()) : p;
  if (static_cast<long long>(at.size()) != 2LL * stages_run * m * E)
    bad("trace has " + std::to_string(at.size()) + " distinct ops, expected " +
        std::to_string(2LL * stages_run * m * E));
  if (tr.makespan != last_end)
    bad("makespan " + std::to_string(tr.makespan) + " != last op end " + std::to_string(last_end));

  // 2. dependency soundness (pipeline.cpp:111-132): same-stage issue chain
  // across epochs, FP(s-1)->FP(s), BP(s+1)->BP(s), FP(s)->BP(s)
  auto get = [&](int s, OpKind k, int mb, int e) -> const OpEvent* {
    auto it = at.find(std::make_tuple(s, static_cast<int>(k), mb, e));
    return it == at.end() ? nullptr : it->second;
  };
  auto after = [&](const OpEvent& o, const OpEvent* d, const char* what) {
    if (d && o.start < d->end)
      bad("op " + op_name(o) + " starts at " + std::to_string(o.start) + " before its " + what + " " +
          op_name(*d) + " ends at " + std::to_string(d->end));
  };
  for (int s = 0; s < p; ++s) {
    const auto order = stage_issue_order(s, p, m);
    const OpEvent* prev = nullptr;
    for (int e = 0; e < E; ++e)
      for (const auto& [k, mb] : order) {
        const OpEvent* o = get(s, k, mb, e);
        if (!o) continue;
        after(*o, prev, "stage predecessor");
        if (k == OpKind::FP && s > 0) after(*o, get(s - 1, OpKind::FP, mb, e), "input");
        if (k == OpKind::BP && s < p - 1) after(*o, get(s + 1, OpKind::BP, mb, e), "gradient");
        if (k == OpKind::BP) after(*o, get(s, OpKind::FP, mb, e), "forward");
        prev = o;
      }
  }

  // 3. GPU exclusivity: a stage's ops and its worker's side-task activities
  // never overlap (simulated traces; on the GPU a step's tail past its bubble
  // co-runs with the next op -- the harness reports it as overrun)
  std::vector<std::vector<std::tuple<Tick, Tick, std::string>>> busy(static_cast<std::size_t>(p));
  for (const OpEvent& o : tr.ops)
    if (o.stage >= 0 && o.stage < p) busy[o.stage].emplace_back(o.start, o.end, "op " + op_name(o));
  for (const ActivityRecord& a : tr.activities) {
    if (a.worker < 0 || a.worker >= p) {
      bad("activity of " + a.task + " on unknown worker " + std::to_string(a.worker));
      continue;
    }
    if (a.end < a.start) bad("activity of " + a.task + " ends before it starts");
    busy[a.worker].emplace_back(a.start, a.end, "activity of " + a.task);
  }
  for (int s = 0; s < p && !tr.measured; ++s) {
    auto& b = busy[s];
    std::stable_sort(b.begin(), b.end());
    for (std::size_t k = 1; k < b.size(); ++k)
      if (std::get<0>(b[k]) < std::get<1>(b[k - 1]))
        bad("GPU " + std::to_string(s) + ": " + std::get<2>(b[k]) + " at " + std::to_string(std::get<0>(b[k])) +
            " overlaps " + std::get<2>(b[k - 1]) + " until " + std::to_string(std::get<1>(b[k - 1])));
  }

  // 4. transition legality per task (task.cpp:38-87), in trace order
  std::map<std::string, std::vector<const TransitionRecord*>> by_task;
  for (const TransitionRecord& t : tr.transitions) by_task[t.task].push_back(&t);
  // state at tick x after the transitions recorded up to x; `before_init`:
  // leave out an InitSideTask landing at x (a zero-length Init activity
  // starts and ends on the tick its transition lands)
  auto state_at = [&](const std::string& task, Tick x, bool before_init) {
    SideTaskState st = SideTaskState::Submitted;
    for (const TransitionRecord* t : by_task[task]) {
      if (t->t > x) break;
      if (before_init && t->t == x && t->kind == TransitionKind::InitSideTask) break;
      if (transition_legal(st, t->kind)) st = transition_target(st, t->kind);
    }
    return st;
  };
  for (const auto& [task, ts] : by_task) {
    SideTaskState st = SideTaskState::Submitted;
    Tick prev = 0;
    for (const TransitionRecord* t : ts) {
      if (t->t < prev) bad("task " + task + ": transitions out of time order at " + std::to_string(t->t));
      prev = t->t;
      if (!transition_legal(st, t->kind)) {
        bad("task " + task + ": illegal transition " + to_string(t->kind) + " from " + to_string(st) +
            " at " + std::to_string(t->t));
        break;
      }
      st = transition_target(st, t->kind);
    }
  }

  // 5. activities only in the state that allows them: Init while CREATED
  // (InitSideTask lands at its end), Check / Step / Kernel while RUNNING
  std::map<std::string, const SideTaskSpec*> spec;
  for (const SideTaskSpec& s : tr.config.tasks) spec[s.id] = &s;
  std::map<std::string, std::int64_t> counted;
  for (const ActivityRecord& a : tr.activities) {
    // measured: the host-clock transition stamps and the device-event
    // activity times agree to within the trace's tolerance
    const Tick at_t = tr.measured ? std::min(a.start + tr.tolerance, a.start + (a.end - a.start) / 2) : a.start;
    const SideTaskState st = state_at(a.task, at_t, a.kind == ActivityKind::Init);
    const bool ok = a.kind == ActivityKind::Init ? st == SideTaskState::Created : st == SideTaskState::Running;
    if (!ok)
      bad("task " + a.task + ": activity at " + std::to_string(a.start) + " while " + to_string(st));
    auto sp = spec.find(a.task);
    if (sp == spec.end()) {
      bad("activity of unknown task " + a.task);
      continue;
    }
    const ActivityKind unit =
        sp->second->interface_kind == TaskInterface::Imperative ? ActivityKind::Kernel : ActivityKind::Step;
    if (a.kind == unit && !a.clipped) ++counted[a.task];
  }

  // 6. submissions, placement (Alg. 1's strict memory filter), dispositions
  std::map<std::string, const TaskProfile*> prof;
  for (const TaskProfile& t : tr.profiles) prof[t.task_id] = &t;
  for (const AssignRecord& a : tr.assigns) {
    auto it = prof.find(a.task);
    if (a.worker < 0 || a.worker >= p) {
      bad("task " + a.task + " assigned to unknown worker " + std::to_string(a.worker));
    } else if (it != prof.end() && !(pc.available_memory(a.worker) > it->second->est_memory)) {
      bad("task " + a.task + " placed on worker " + std::to_string(a.worker) + " without memory for it");
    }
  }
  std::set<std::string> disposed;
  for (const DispositionRecord& d : tr.dispositions) {
    if (!disposed.insert(d.task).second) bad("task " + d.task + " has two dispositions");
    if (spec.find(d.task) == spec.end()) bad("disposition of unknown task " + d.task);
    if (d.steps_completed != counted[d.task])
      bad("task " + d.task + ": " + std::to_string(d.steps_completed) + " steps reported, " +
          std::to_string(counted[d.task]) + " completed in the trace");
  }
  for (const AssignRecord& s : tr.submits)  // every submitted task ends with one
    if (!disposed.count(s.task)) bad("task " + s.task + " was submitted but has no disposition");
  for (const KillRecord& k : tr.kills) {
    const Disposition want = k.reason == KillReason::Oom ? Disposition::KilledOom
                             : k.reason == KillReason::PauseTimeout ? Disposition::KilledPauseTimeout
                                                                    : Disposition::KilledInitTimeout;
    bool found = false;
    for (const DispositionRecord& d : tr.dispositions)
      if (d.task == k.task) found = d.disposition == want;
    if (!found) bad("kill of " + k.task + " without the matching disposition");
  }

  // 7. bubbles are idle time of their stage, and the breakdown conserves them
  for (const Bubble& b : tr.bubbles) {
    if (b.stage < 0 || b.stage >= p || b.duration < 0) {
      bad("malformed bubble");
      continue;
    }
    for (const OpEvent& o : tr.ops)
      if (o.stage == b.stage && o.start < b.end() && b.start < o.end)
        bad("bubble on stage " + std::to_string(b.stage) + " at " + std::to_string(b.start) + " overlaps op " +
            op_name(o));
  }
  const std::vector<StageBreakdown> bd = bubble_breakdown(breakdown_input(tr));
  std::vector<Tick> per(static_cast<std::size_t>(p), 0);
  for (const Bubble& b : tr.bubbles)
    if (b.stage >= 0 && b.stage < p) per[b.stage] += b.duration;
  for (const StageBreakdown& s : bd)
    if (s.stage >= 0 && s.stage < p && s.total() != per[s.stage])
      bad("stage " + std::to_string(s.stage) + ": breakdown sums to " + std::to_string(s.total()) +
          " ticks, bubbles to " + std::to_string(per[s.stage]));
  return v;
}

}  // namespace freeride
