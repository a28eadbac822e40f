// The simulated dispatch engine (reference: engine.hpp:94-98, declared but
// never implemented; semantics SPEC.md:466-517 and SURVEY.md Appendix B,
// ambiguities fixed in DESIGN.md §6).  Produces the step-dispatch order --
// transitions, RPCs and activities -- for a bubble trace, the parity object
// of the bubble-harvesting path.
//
// Mechanics: an agenda of "interesting" ticks (op ends, activity ends, RPC
// landings, limit timers, submissions, leak-OOM crossings); at each one the
// tick phases run in order
//   P1 completions (ops, then side-task activities, by worker)
//   P2 dependency readiness, epoch completion, bubble signals
//   P3 manager events: BubbleEnded < TaskSubmitted < BubbleStarted
//   P4 RPC landings (issue order)       P5 limit timers, leak OOM
//   P6 GPU scheduling per worker: a ready op first, else the current task's
//      Init / Check -> gate -> Step (iterative) / Kernel (imperative)
// Ops on a stage are chained, so each stage has at most one ready op: the
// next in its issue order.  oracle/engine_oracle.py restates the same rules
// by stepping every tick and scanning all state; traces must be identical.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>

#include "freeride.hpp"

namespace freeride {

namespace {

enum class Act { None, Op, Side };

struct GpuSlot {
  Act what = Act::None;
  std::int64_t op = -1;        // Act::Op
  int task = -1;               // Act::Side
  ActivityKind kind = ActivityKind::Step;
  Tick start = 0, end = 0;
};

struct Task {
  SideTaskSpec spec;
  TaskProfile prof;
  SideTaskRuntime rt;
  int worker = -1;
  bool initializing = false, want_init = false, pause_pending = false, gate_closed = false;
  Tick bubble_end = 0;
  Tick busy = 0;
  Tick check_done = -1;
  std::uint64_t rng = 0;
  double limit = 0.0;
  bool submitted = false;
  std::optional<Disposition> disp;
};

struct Rpc {
  Tick land;
  std::int64_t seq;
  TransitionKind kind;
  int task;
  Tick bubble_end;
};

struct Timer {
  Tick due;
  std::int64_t seq;
  KillReason kind;  // PauseTimeout or InitTimeout
  int task;
  Tick issued;
};

struct ProfBubble {
  int stage;
  int prev_k, prev_mb;  // -1: leading
  int next_k, next_mb;  // -1: trailing
  Tick duration;
  BubbleType btype;
};

class Engine {
 public:
  Engine(const ExperimentConfig& c, bool with_tasks, std::uint64_t seed)
      : cfg_(c.pipeline), rt_(c.runtime), lim_(c.limits), seed_(seed), with_(with_tasks) {
    cfg_.validate();
    p_ = cfg_.num_stages;
    m_ = cfg_.num_micro_batches;
    E_ = cfg_.num_epochs;
    per_epoch_ = 2LL * p_ * m_;
    n_ = per_epoch_ * E_;
    if (with_) {
      for (std::size_t i = 0; i < c.tasks.size(); ++i) {
        Task t;
        t.spec = c.tasks[i];
        t.spec.validate("tasks[" + std::to_string(i) + "]");
        tasks_.push_back(t);
      }
    }
    build();
  }

  RunTrace run() {
    std::vector<int> subs(tasks_.size());
    for (std::size_t i = 0; i < tasks_.size(); ++i) subs[i] = static_cast<int>(i);
    std::stable_sort(subs.begin(), subs.end(), [&](int a, int b) {
      return tasks_[a].spec.submit_time < tasks_[b].spec.submit_time;
    });
    for (int i : subs) agenda_.insert(tasks_[i].spec.submit_time);
    sub_order_ = subs;
    agenda_.insert(0);
    while (!agenda_.empty()) {
      const Tick t = *agenda_.begin();
      agenda_.erase(agenda_.begin());
      if (tick(t)) break;
    }
    finish_run();
    return std::move(out_);
  }

 private:
  // ------------------------------------------------------------- setup
  std::int64_t id(std::int64_t e, int s, int k, int mb) const {
    return ((e * p_ + s) * 2 + k) * m_ + (mb - 1);
  }

  void build() {
    PipelineConfig one = cfg_;
    one.num_epochs = 1;
    const ScheduleTrace pt = build_schedule(one);
    for (const LinkedBubble& lb : extract_bubbles_linked(pt)) {
      ProfBubble b{lb.bubble.stage, -1, -1, -1, -1, lb.bubble.duration, lb.bubble.btype};
      if (lb.prev_op >= 0) {
        const OpEvent& o = pt.ops[static_cast<std::size_t>(lb.prev_op)];
        b.prev_k = static_cast<int>(o.kind);
        b.prev_mb = o.micro_batch;
      }
      if (lb.next_op >= 0) {
        const OpEvent& o = pt.ops[static_cast<std::size_t>(lb.next_op)];
        b.next_k = static_cast<int>(o.kind);
        b.next_mb = o.micro_batch;
      }
      pb_.push_back(b);
    }
    order_.resize(static_cast<std::size_t>(p_));
    for (int s = 0; s < p_; ++s) order_[s] = stage_issue_order(s, p_, m_);
    // successors and dependency counts (same edges as build_schedule)
    succ_.assign(static_cast<std::size_t>(n_), {});
    left_.assign(static_cast<std::size_t>(n_), 0);
    for (std::int64_t e = 0; e < E_; ++e)
      for (int s = 0; s < p_; ++s)
        for (int i = 0; i < 2 * m_; ++i) {
          const auto [k, mb] = order_[s][i];
          const std::int64_t v = id(e, s, static_cast<int>(k), mb);
          auto dep = [&](std::int64_t u) {
            succ_[static_cast<std::size_t>(u)].push_back(v);
            left_[static_cast<std::size_t>(v)]++;
          };
          if (i > 0) dep(id(e, s, static_cast<int>(order_[s][i - 1].first), order_[s][i - 1].second));
          else if (e > 0) dep(id(e - 1, s, static_cast<int>(order_[s].back().first), order_[s].back().second));
          if (k == OpKind::FP && s > 0) dep(id(e, s - 1, 0, mb));
          if (k == OpKind::BP) {
            if (s < p_ - 1) dep(id(e, s + 1, 1, mb));
            dep(id(e, s, 0, mb));
          }
        }
    start_.assign(static_cast<std::size_t>(n_), -1);
    end_.assign(static_cast<std::size_t>(n_), -1);
    ready_.assign(static_cast<std::size_t>(n_), -1);
    cursor_.assign(static_cast<std::size_t>(p_), 0);
    epoch_left_.assign(static_cast<std::size_t>(E_), per_epoch_);
    gpu_.assign(static_cast<std::size_t>(p_), GpuSlot{});
    held_.assign(static_cast<std::size_t>(p_), std::nullopt);
    workers_.resize(static_cast<std::size_t>(p_));
    for (int s = 0; s < p_; ++s) {
      workers_[s].worker_id = s;
      workers_[s].gpu_mem = cfg_.available_memory(s);
    }
    // bubble triggers: op id -> bubble keys; key = (e * |pb| + j)
    start_on_end_.assign(static_cast<std::size_t>(n_), {});
    end_on_ready_.assign(static_cast<std::size_t>(n_), {});
    for (std::int64_t e = 0; e < E_; ++e)
      for (std::size_t j = 0; j < pb_.size(); ++j) {
        const ProfBubble& b = pb_[j];
        const std::int64_t key = e * static_cast<std::int64_t>(pb_.size()) + static_cast<std::int64_t>(j);
        if (b.prev_k >= 0) start_on_end_[static_cast<std::size_t>(id(e, b.stage, b.prev_k, b.prev_mb))].push_back(key);
        if (b.next_k >= 0) end_on_ready_[static_cast<std::size_t>(id(e, b.stage, b.next_k, b.next_mb))].push_back(key);
      }
    open_.assign(static_cast<std::size_t>(E_) * pb_.size(), -1);
  }

  // ------------------------------------------------------------- helpers
  TaskView view(const std::string& tid) const {
    const Task& t = tasks_[static_cast<std::size_t>(index_.at(tid))];
    return TaskView{t.rt.state, t.initializing};
  }

  void transition(Task& t, TransitionKind k, Tick now) {
    apply_transition(t.rt, k, now);
    out_.transitions.push_back(TransitionRecord{now, t.spec.id, k, t.worker});
  }

  void finish_task(Task& t, Disposition d) {
    t.disp = d;
    WorkerState& w = workers_[static_cast<std::size_t>(t.worker)];
    if (w.current_task && *w.current_task == t.spec.id) w.current_task.reset();
  }

  void kill(int ti, Tick now, KillReason why) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    GpuSlot& g = gpu_[static_cast<std::size_t>(t.worker)];
    if (g.what == Act::Side && g.task == ti) {
      out_.activities.push_back(ActivityRecord{g.start, now, t.spec.id, t.worker, g.kind, true});
      g = GpuSlot{};
    }
    if (t.rt.state != SideTaskState::Stopped) transition(t, TransitionKind::StopSideTask, now);
    t.initializing = t.want_init = t.pause_pending = false;
    out_.kills.push_back(KillRecord{now, t.spec.id, t.worker, why});
    finish_task(t, why == KillReason::Oom ? Disposition::KilledOom
                  : why == KillReason::PauseTimeout ? Disposition::KilledPauseTimeout
                                                    : Disposition::KilledInitTimeout);
  }

  Tick draw(Task& t) { return jittered_step_ticks(t.spec.per_step_duration, rt_.step_jitter, t.rng); }

  double est(const Task& t) const {
    return rt_.gate_estimate == GateEstimate::Max ? t.prof.max_per_step_duration.value_or(0.0)
                                                  : t.prof.est_per_step_duration.value_or(0.0);
  }

  double leak_alloc(const Task& t, Tick busy) const {
    return t.spec.memory_demand +
           t.spec.misbehavior.leak_rate_gib_per_s * ticks_to_seconds(busy, cfg_.tick_seconds);
  }

  void land(TransitionKind k, int ti, Tick bend, Tick now) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    if (t.rt.state == SideTaskState::Stopped) return;
    if (k == TransitionKind::InitSideTask) {
      if (t.rt.state == SideTaskState::Created && !t.initializing) {
        t.initializing = true;
        t.want_init = true;
      }
    } else if (k == TransitionKind::StartSideTask) {
      if (t.rt.state == SideTaskState::Paused) {
        transition(t, TransitionKind::StartSideTask, now);
        t.bubble_end = bend;
        t.gate_closed = false;
      }
    } else if (k == TransitionKind::PauseSideTask) {
      if (t.rt.state == SideTaskState::Running && t.spec.misbehavior.kind != MisbehaviorKind::IgnoresPause) {
        const GpuSlot& g = gpu_[static_cast<std::size_t>(t.worker)];
        if (g.what == Act::Side && g.task == ti)
          t.pause_pending = true;  // lands when the in-flight activity ends
        else
          pause_now(ti, now);
      }
    }
  }

  void pause_now(int ti, Tick now) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    transition(t, TransitionKind::PauseSideTask, now);
    t.pause_pending = false;
    auto& h = held_[static_cast<std::size_t>(t.worker)];
    if (h) {
      const Bubble b = *h;
      h.reset();
      bubble_started(t.worker, b, now);
    }
  }

  void issue(TransitionKind k, int ti, Tick now, Tick bend = 0) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    out_.rpcs.push_back(RpcRecord{now, t.spec.id, k, t.worker});
    if (rt_.rpc_latency == 0) {
      land(k, ti, bend, now);
    } else {
      rpcs_.push_back(Rpc{now + rt_.rpc_latency, ++seq_, k, ti, bend});
      agenda_.insert(now + rt_.rpc_latency);
    }
  }

  bool pause_pending_on(int w) const {
    const WorkerState& ws = workers_[static_cast<std::size_t>(w)];
    if (!ws.current_task) return false;
    return tasks_[static_cast<std::size_t>(index_.at(*ws.current_task))].pause_pending;
  }

  void bubble_started(int w, const Bubble& b, Tick now) {
    if (pause_pending_on(w)) {  // deferred until the pause lands
      held_[static_cast<std::size_t>(w)] = b;
      return;
    }
    const auto lookup = [this](const std::string& tid) { return view(tid); };
    for (const ManagerAction& a : on_bubble_started(workers_[static_cast<std::size_t>(w)], b, lookup)) {
      const int ti = index_.at(a.task_id);
      if (a.kind == ManagerActionKind::IssueInit) issue(TransitionKind::InitSideTask, ti, now);
      else if (a.kind == ManagerActionKind::IssueStart) issue(TransitionKind::StartSideTask, ti, now, b.start + b.duration);
    }
  }

  void bubble_ended(int w, Tick now) {
    held_[static_cast<std::size_t>(w)].reset();
    const auto lookup = [this](const std::string& tid) { return view(tid); };
    for (const ManagerAction& a : on_bubble_ended(workers_[static_cast<std::size_t>(w)], now, lookup)) {
      const int ti = index_.at(a.task_id);
      if (a.kind == ManagerActionKind::IssuePause) {
        issue(TransitionKind::PauseSideTask, ti, now);
        timers_.push_back(Timer{now + lim_.grace_period, ++seq_, KillReason::PauseTimeout, ti, now});
        agenda_.insert(now + lim_.grace_period);
      } else if (a.kind == ManagerActionKind::ArmInitGuard) {
        timers_.push_back(Timer{now + lim_.grace_period, ++seq_, KillReason::InitTimeout, ti, now});
        agenda_.insert(now + lim_.grace_period);
      }
    }
  }

  void start_side(int s, int ti, ActivityKind k, Tick now, Tick d) {
    GpuSlot& g = gpu_[static_cast<std::size_t>(s)];
    g = GpuSlot{Act::Side, -1, ti, k, now, now + d};
    agenda_.insert(now + d);
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    if ((k == ActivityKind::Step || k == ActivityKind::Kernel) &&
        t.spec.misbehavior.kind == MisbehaviorKind::MemoryLeak && d > 1) {
      // first tick strictly inside the activity whose allocation exceeds the
      // limit (the allocation is monotone in the tick: binary search)
      Tick lo = now + 1, hi = now + d - 1, hit = -1;
      while (lo <= hi) {
        const Tick mid = lo + (hi - lo) / 2;
        if (check_memory(leak_alloc(t, t.busy + mid - now), t.limit) == MemCheck::OomKill) {
          hit = mid;
          hi = mid - 1;
        } else {
          lo = mid + 1;
        }
      }
      if (hit >= 0) {
        leaks_.push_back({hit, ti, now});
        agenda_.insert(hit);
      }
    }
  }

  void complete_init(int ti, Tick now) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    t.initializing = false;
    transition(t, TransitionKind::InitSideTask, now);
    if (check_memory(t.rt.memory_allocated, t.limit) == MemCheck::OomKill) kill(ti, now, KillReason::Oom);
  }

  // ------------------------------------------------------------- one tick
  bool tick(Tick now) {
    // P1a: ops ending now
    for (int s = 0; s < p_; ++s) {
      GpuSlot& g = gpu_[static_cast<std::size_t>(s)];
      if (g.what == Act::Op && g.end == now) {
        ended_now_.push_back(g.op);
        end_[static_cast<std::size_t>(g.op)] = now;
        ++done_;
        g = GpuSlot{};
      }
    }
    const bool last = done_ == n_;
    if (last) makespan_ = now;
    // P1b: side-task activities ending now
    for (int s = 0; s < p_; ++s) {
      GpuSlot g = gpu_[static_cast<std::size_t>(s)];
      if (g.what != Act::Side || g.end != now) continue;
      gpu_[static_cast<std::size_t>(s)] = GpuSlot{};
      Task& t = tasks_[static_cast<std::size_t>(g.task)];
      out_.activities.push_back(ActivityRecord{g.start, now, t.spec.id, s, g.kind, false});
      if (g.kind == ActivityKind::Init) {
        complete_init(g.task, now);
      } else if (g.kind == ActivityKind::Step || g.kind == ActivityKind::Kernel) {
        t.busy += now - g.start;
        t.rt.steps_completed++;
        if (t.spec.total_steps && t.rt.steps_completed >= *t.spec.total_steps) {
          transition(t, TransitionKind::StopSideTask, now);
          t.pause_pending = false;
          finish_task(t, Disposition::Completed);
        } else if (t.pause_pending) {
          pause_now(g.task, now);
        }
      } else if (g.kind == ActivityKind::Check) {
        if (t.pause_pending) pause_now(g.task, now);
        else t.check_done = now;
      }
    }
    // P2: readiness, epoch completion, bubble signals
    std::vector<std::int64_t> starts, ends;
    if (now == 0) {
      for (std::size_t j = 0; j < pb_.size(); ++j)
        if (pb_[j].prev_k < 0) starts.push_back(static_cast<std::int64_t>(j));
      for (int s = 0; s < p_; ++s) try_ready(id(0, s, static_cast<int>(order_[s][0].first), order_[s][0].second), now, ends);
    }
    for (std::int64_t u : ended_now_) {
      for (std::int64_t key : start_on_end_[static_cast<std::size_t>(u)]) starts.push_back(key);
      const std::int64_t e = u / per_epoch_;
      if (--epoch_left_[static_cast<std::size_t>(e)] == 0) {
        for (std::size_t j = 0; j < pb_.size(); ++j) {
          const std::int64_t key = e * static_cast<std::int64_t>(pb_.size()) + static_cast<std::int64_t>(j);
          if (pb_[j].next_k < 0) ends.push_back(key);
          if (pb_[j].prev_k < 0 && e + 1 < E_) starts.push_back(key + static_cast<std::int64_t>(pb_.size()));
        }
      }
      for (std::int64_t v : succ_[static_cast<std::size_t>(u)])
        if (--left_[static_cast<std::size_t>(v)] == 0) try_ready(v, now, ends);
    }
    ended_now_.clear();
    std::set<std::int64_t> st(starts.begin(), starts.end()), en(ends.begin(), ends.end());
    std::vector<std::int64_t> fire_end, fire_start;
    for (std::int64_t key : en) {
      if (st.count(key)) continue;  // zero-length on the delayed timeline: no signals
      Tick& o = open_[static_cast<std::size_t>(key)];
      if (o < 0) continue;
      const ProfBubble& b = pb_[static_cast<std::size_t>(key % static_cast<std::int64_t>(pb_.size()))];
      out_.bubbles.push_back(Bubble{b.stage, static_cast<int>(key / static_cast<std::int64_t>(pb_.size())), o,
                                    now - o, cfg_.available_memory(b.stage), b.btype});
      o = -1;
      fire_end.push_back(key);
    }
    for (std::int64_t key : st) {
      if (en.count(key)) continue;
      open_[static_cast<std::size_t>(key)] = now;
      fire_start.push_back(key);
    }
    if (last) return true;
    // P3: BubbleEnded < TaskSubmitted < BubbleStarted (by worker, epoch, index)
    const auto by_worker = [this](std::int64_t a, std::int64_t b) {
      const auto P = static_cast<std::int64_t>(pb_.size());
      const int sa = pb_[static_cast<std::size_t>(a % P)].stage, sb = pb_[static_cast<std::size_t>(b % P)].stage;
      return std::make_tuple(sa, a / P, a % P) < std::make_tuple(sb, b / P, b % P);
    };
    if (with_) {
      std::sort(fire_end.begin(), fire_end.end(), by_worker);
      for (std::int64_t key : fire_end)
        bubble_ended(pb_[static_cast<std::size_t>(key % static_cast<std::int64_t>(pb_.size()))].stage, now);
      while (next_sub_ < sub_order_.size() &&
             tasks_[static_cast<std::size_t>(sub_order_[next_sub_])].spec.submit_time == now)
        submit(sub_order_[next_sub_++], now);
      std::sort(fire_start.begin(), fire_start.end(), by_worker);
      for (std::int64_t key : fire_start) {
        const auto P = static_cast<std::int64_t>(pb_.size());
        const ProfBubble& b = pb_[static_cast<std::size_t>(key % P)];
        bubble_started(b.stage, Bubble{b.stage, static_cast<int>(key / P), now, b.duration,
                                       cfg_.available_memory(b.stage), b.btype}, now);
      }
      // P4: RPC landings in issue order
      std::vector<Rpc> due;
      for (auto it = rpcs_.begin(); it != rpcs_.end();) {
        if (it->land == now) {
          due.push_back(*it);
          it = rpcs_.erase(it);
        } else {
          ++it;
        }
      }
      std::sort(due.begin(), due.end(), [](const Rpc& a, const Rpc& b) { return a.seq < b.seq; });
      for (const Rpc& r : due) land(r.kind, r.task, r.bubble_end, now);
      // P5: limit timers in arming order, then leak-OOM crossings by worker
      std::vector<Timer> tdue;
      for (auto it = timers_.begin(); it != timers_.end();) {
        if (it->due == now) {
          tdue.push_back(*it);
          it = timers_.erase(it);
        } else {
          ++it;
        }
      }
      std::sort(tdue.begin(), tdue.end(), [](const Timer& a, const Timer& b) { return a.seq < b.seq; });
      for (const Timer& x : tdue) {
        Task& t = tasks_[static_cast<std::size_t>(x.task)];
        if (t.rt.state == SideTaskState::Stopped) continue;
        if (x.kind == KillReason::PauseTimeout) {
          if (framework_enforce(t.rt.last_paused, x.issued, now, lim_.grace_period) == Enforce::Kill)
            kill(x.task, now, KillReason::PauseTimeout);
        } else if (t.initializing) {
          kill(x.task, now, KillReason::InitTimeout);
        }
      }
      for (int s = 0; s < p_; ++s) {
        const GpuSlot& g = gpu_[static_cast<std::size_t>(s)];
        if (g.what != Act::Side) continue;
        for (const auto& lk : leaks_)
          if (lk.at == now && lk.task == g.task && lk.act_start == g.start) {
            kill(g.task, now, KillReason::Oom);
            break;
          }
      }
    }
    // P6: GPU scheduling per worker
    for (int s = 0; s < p_; ++s) {
      if (gpu_[static_cast<std::size_t>(s)].what != Act::None) continue;
      const std::int64_t v = next_ready(s);
      if (v >= 0) {
        start_[static_cast<std::size_t>(v)] = now;
        const int k = static_cast<int>((v / m_) % 2);
        const Tick d = k == 0 ? cfg_.fp_ticks(s) : cfg_.bp_ticks(s);
        gpu_[static_cast<std::size_t>(s)] = GpuSlot{Act::Op, v, -1, ActivityKind::Step, now, now + d};
        agenda_.insert(now + d);
        cursor_[static_cast<std::size_t>(s)]++;
        continue;
      }
      if (!with_) continue;
      const WorkerState& ws = workers_[static_cast<std::size_t>(s)];
      if (!ws.current_task) continue;
      const int ti = index_.at(*ws.current_task);
      Task& t = tasks_[static_cast<std::size_t>(ti)];
      if (t.rt.state == SideTaskState::Stopped) continue;
      if (t.want_init) {
        t.want_init = false;
        if (t.spec.init_duration == 0) {
          out_.activities.push_back(ActivityRecord{now, now, t.spec.id, s, ActivityKind::Init, false});
          complete_init(ti, now);
        } else {
          start_side(s, ti, ActivityKind::Init, now, t.spec.init_duration);
        }
        continue;
      }
      if (t.rt.state != SideTaskState::Running || t.pause_pending || t.gate_closed) continue;
      if (t.spec.interface_kind == TaskInterface::Imperative) {
        start_side(s, ti, ActivityKind::Kernel, now, draw(t));
        continue;
      }
      if (t.check_done != now && rt_.check_overhead > 0) {
        start_side(s, ti, ActivityKind::Check, now, rt_.check_overhead);
        continue;
      }
      t.check_done = -1;
      const IterativeDecision d = iterative_run(t.rt, t.bubble_end, now, est(t), cfg_.tick_seconds, 0);
      if (!d.run) {
        t.gate_closed = true;  // yield until the next transition
        continue;
      }
      start_side(s, ti, ActivityKind::Step, now, draw(t));
    }
    return false;
  }

  void try_ready(std::int64_t v, Tick now, std::vector<std::int64_t>& ends) {
    if (left_[static_cast<std::size_t>(v)] != 0 || ready_[static_cast<std::size_t>(v)] >= 0) return;
    ready_[static_cast<std::size_t>(v)] = now;
    for (std::int64_t key : end_on_ready_[static_cast<std::size_t>(v)]) ends.push_back(key);
  }

  // the stage's next op in issue order, if its dependencies are met
  std::int64_t next_ready(int s) const {
    const std::int64_t c = cursor_[static_cast<std::size_t>(s)];
    if (c >= 2LL * m_ * E_) return -1;
    const std::int64_t e = c / (2 * m_);
    const auto [k, mb] = order_[s][static_cast<std::size_t>(c % (2 * m_))];
    const std::int64_t v = id(e, s, static_cast<int>(k), mb);
    return ready_[static_cast<std::size_t>(v)] >= 0 ? v : -1;
  }

  void submit(int ti, Tick now) {
    Task& t = tasks_[static_cast<std::size_t>(ti)];
    ProfileOptions po;
    po.n_steps = rt_.profile_steps;
    po.step_jitter = rt_.step_jitter;
    po.tick_seconds = cfg_.tick_seconds;
    t.prof = profile_task(t.spec, po, seed_);
    t.rng = stream_seed(seed_, t.spec.id, "run");
    t.limit = t.spec.memory_limit ? *t.spec.memory_limit : t.prof.est_memory + lim_.memory_headroom;
    t.rt.spec = t.spec;
    t.submitted = true;
    index_[t.spec.id] = ti;
    out_.profiles.push_back(t.prof);
    out_.submits.push_back(AssignRecord{now, t.spec.id, -1});
    const SubmitOutcome o = submit_task(t.prof, workers_);
    if (o.assigned) {
      t.worker = o.worker_id;
      out_.assigns.push_back(AssignRecord{now, t.spec.id, o.worker_id});
      transition(t, TransitionKind::CreateSideTask, now);
    } else {
      out_.rejects.push_back(AssignRecord{now, t.spec.id, -1});
      t.disp = Disposition::Rejected;
    }
  }

  void finish_run() {
    for (int s = 0; s < p_; ++s) {
      const GpuSlot& g = gpu_[static_cast<std::size_t>(s)];
      if (g.what == Act::Side)
        out_.activities.push_back(ActivityRecord{g.start, makespan_, tasks_[static_cast<std::size_t>(g.task)].spec.id,
                                                 s, g.kind, true});
    }
    out_.ops.resize(static_cast<std::size_t>(n_));
    for (std::int64_t v = 0; v < n_; ++v) {
      OpEvent& o = out_.ops[static_cast<std::size_t>(v)];
      o.micro_batch = static_cast<int>(v % m_) + 1;
      o.kind = static_cast<OpKind>((v / m_) % 2);
      o.stage = static_cast<int>((v / (2LL * m_)) % p_);
      o.epoch = static_cast<int>(v / per_epoch_);
      o.start = start_[static_cast<std::size_t>(v)];
      o.end = end_[static_cast<std::size_t>(v)];
    }
    std::sort(out_.ops.begin(), out_.ops.end(), [](const OpEvent& a, const OpEvent& b) {
      return std::tie(a.start, a.stage, a.end, a.micro_batch) < std::tie(b.start, b.stage, b.end, b.micro_batch);
    });
    for (int ti : sub_order_) {
      const Task& t = tasks_[static_cast<std::size_t>(ti)];
      if (!t.submitted) continue;
      DispositionRecord d;
      d.task = t.spec.id;
      d.disposition = t.disp.value_or(Disposition::Active);
      d.steps_completed = t.rt.steps_completed;
      if (t.worker >= 0) d.worker = t.worker;
      out_.dispositions.push_back(d);
    }
    out_.makespan = makespan_;
  }

  struct Leak {
    Tick at;
    int task;
    Tick act_start;
  };

  PipelineConfig cfg_;
  RuntimeOptions rt_;
  LimitConfig lim_;
  std::uint64_t seed_;
  bool with_;
  int p_ = 0, m_ = 0;
  std::int64_t E_ = 0, per_epoch_ = 0, n_ = 0, done_ = 0;
  std::vector<ProfBubble> pb_;
  std::vector<std::vector<std::pair<OpKind, int>>> order_;
  std::vector<std::vector<std::int64_t>> succ_, start_on_end_, end_on_ready_;
  std::vector<int> left_;
  std::vector<Tick> start_, end_, ready_, open_;
  std::vector<std::int64_t> cursor_, epoch_left_, ended_now_;
  std::vector<GpuSlot> gpu_;
  std::vector<std::optional<Bubble>> held_;
  std::vector<WorkerState> workers_;
  std::vector<Task> tasks_;
  std::map<std::string, int> index_;
  std::vector<int> sub_order_;
  std::size_t next_sub_ = 0;
  std::vector<Rpc> rpcs_;
  std::vector<Timer> timers_;
  std::vector<Leak> leaks_;
  std::set<Tick> agenda_;
  std::int64_t seq_ = 0;
  Tick makespan_ = 0;
  RunTrace out_;
};

}  // namespace

RunTrace run_experiment(const ExperimentConfig& config, bool with_tasks, std::uint64_t seed) {
  Engine e(config, with_tasks, seed);
  RunTrace t = e.run();
  t.config = config;
  t.seed = seed;
  t.with_tasks = with_tasks;
  return t;
}

}  // namespace freeride
