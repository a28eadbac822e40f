// Side-task state machine, iterative/imperative interfaces and resource
// limits (reference: src/task.cpp:9-156, src/limits.cpp:5-26).
//
// The six legal edges of Fig. 4 are one 5x6 table instead of a switch; the
// program-directed gate compares doubles exactly as the reference does
// (task.cpp:94-95, limits.cpp:18) -- see DESIGN.md "float-fragile gate".
#include "freeride.hpp"

namespace freeride {

namespace {

constexpr int kStates = 5, kKinds = 6;
// kEdge[from][kind] = target state, or -1 when illegal (task.cpp:38-68).
constexpr int kEdge[kStates][kKinds] = {
    /* Submitted */ {1, -1, -1, -1, -1, -1},
    /* Created   */ {-1, 2, -1, -1, -1, 4},
    /* Paused    */ {-1, -1, 3, -1, -1, 4},
    /* Running   */ {-1, -1, -1, 3, 2, 4},
    /* Stopped   */ {-1, -1, -1, -1, -1, -1},
};

int edge(SideTaskState from, TransitionKind kind) {
  const int f = static_cast<int>(from), k = static_cast<int>(kind);
  if (f < 0 || f >= kStates || k < 0 || k >= kKinds) return -1;
  return kEdge[f][k];
}

}  // namespace

const char* to_string(SideTaskState s) {
  static const char* names[] = {"SUBMITTED", "CREATED", "PAUSED", "RUNNING", "STOPPED"};
  const int i = static_cast<int>(s);
  return i >= 0 && i < kStates ? names[i] : "?";
}

const char* to_string(TransitionKind k) {
  static const char* names[] = {"create", "init", "start", "run_next_step", "pause", "stop"};
  const int i = static_cast<int>(k);
  return i >= 0 && i < kKinds ? names[i] : "?";
}

IllegalTransition::IllegalTransition(SideTaskState f, TransitionKind k)
    : std::runtime_error(std::string("illegal transition ") + to_string(k) + " from state " +
                         to_string(f)),
      from(f),
      kind(k) {}

void SideTaskSpec::validate(const std::string& path) const {  // task.cpp:9-30
  if (id.empty()) throw ValidationError(path + ".id", "must be non-empty");
  if (per_step_duration <= 0) throw ValidationError(path + ".per_step_duration", "must be > 0");
  if (total_steps && *total_steps <= 0)
    throw ValidationError(path + ".total_steps", "must be > 0 when present");
  if (init_duration < 0) throw ValidationError(path + ".init_duration", "must be >= 0");
  if (memory_demand < 0.0) throw ValidationError(path + ".memory_demand", "must be >= 0");
  if (submit_time < 0) throw ValidationError(path + ".submit_time", "must be >= 0");
  if (misbehavior.kind == MisbehaviorKind::MemoryLeak && misbehavior.leak_rate_gib_per_s <= 0.0)
    throw ValidationError(path + ".misbehavior.rate_gib_per_s", "must be > 0 for a memory leak");
  if (memory_limit && *memory_limit < 0.0)
    throw ValidationError(path + ".memory_limit", "must be >= 0 when present");
  if (reference_throughput && *reference_throughput <= 0.0)
    throw ValidationError(path + ".reference_throughput", "must be > 0 when present");
}

bool transition_legal(SideTaskState from, TransitionKind kind) { return edge(from, kind) >= 0; }

SideTaskState transition_target(SideTaskState from, TransitionKind kind) {
  const int to = edge(from, kind);
  if (to < 0) throw IllegalTransition(from, kind);
  return static_cast<SideTaskState>(to);
}

// task.cpp:70-87: Init allocates memory_demand, Pause stamps last_paused,
// Stop releases memory; Pause/Stop end any in-flight step.
void apply_transition(SideTaskRuntime& rt, TransitionKind kind, Tick now) {
  rt.state = transition_target(rt.state, kind);
  if (kind == TransitionKind::InitSideTask) {
    rt.memory_allocated = rt.spec.memory_demand;
  } else if (kind == TransitionKind::PauseSideTask) {
    rt.last_paused = now;
    rt.busy_until.reset();
  } else if (kind == TransitionKind::StopSideTask) {
    rt.memory_allocated = 0.0;
    rt.busy_until.reset();
  }
}

IterativeDecision iterative_run(const SideTaskRuntime& rt, Tick bubble_end, Tick now,
                                double est_step_seconds, double tick_seconds,
                                Tick actual_step_ticks) {  // task.cpp:89-100
  if (rt.state != SideTaskState::Running) return {};
  const double remaining = ticks_to_seconds(bubble_end - now, tick_seconds);
  if (program_directed_gate(remaining, est_step_seconds) != Gate::Run) return {};
  return {true, now + actual_step_ticks};
}

Tick imperative_run(const SideTaskRuntime&, Tick now, Tick actual_kernel_ticks) {
  return now + actual_kernel_ticks;  // task.cpp:102-106
}

void LimitConfig::validate() const {  // limits.cpp:5-11
  if (grace_period <= 0) throw ValidationError("limits.grace_period", "must be > 0");
  if (memory_headroom < 0.0) throw ValidationError("limits.memory_headroom", "must be >= 0");
  if (reclamation_delay < 0) throw ValidationError("limits.reclamation_delay", "must be >= 0");
}

MemCheck check_memory(double alloc, double limit) {  // limits.cpp:13-15 (strict)
  return alloc > limit ? MemCheck::OomKill : MemCheck::Ok;
}

Gate program_directed_gate(double remaining, double est) {  // limits.cpp:17-19 (strict)
  return remaining > est ? Gate::Run : Gate::Yield;
}

Enforce framework_enforce(std::optional<Tick> last_paused, Tick issued, Tick now,
                          Tick grace) {  // limits.cpp:21-26
  if (now < issued + grace) return Enforce::Ok;
  return last_paused && *last_paused >= issued ? Enforce::Ok : Enforce::Kill;
}

}  // namespace freeride
