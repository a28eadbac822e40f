// freeride.hpp -- C++ host API of the B200-native bubble-harvesting path.
//
// Keeps the reference's API surface (namespace bubblesim in
// /root/reference/proj/include/bubblesim/*.hpp): same type names, field
// meaning, function names and error behaviour, re-implemented here with flat
// index arithmetic instead of std::map DAG bookkeeping.  The C-ABI
// (include/freeride.h) and the GPU runtime (csrc/runtime) sit on top of it.
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace freeride {

// ---------------------------------------------------------------- types.hpp
using Tick = std::int64_t;  // types.hpp:14

inline double ticks_to_seconds(Tick t, double tick_seconds) {  // types.hpp:16
  return static_cast<double>(t) * tick_seconds;
}

class ValidationError : public std::runtime_error {  // types.hpp:22-30
 public:
  ValidationError(std::string field, const std::string& what)
      : std::runtime_error(field + ": " + what), field_(std::move(field)) {}
  const std::string& field() const noexcept { return field_; }

 private:
  std::string field_;
};

class SchemaError : public std::runtime_error {  // types.hpp:34-42
 public:
  SchemaError(std::string path, const std::string& what)
      : std::runtime_error(path + ": " + what), path_(std::move(path)) {}
  const std::string& path() const noexcept { return path_; }

 private:
  std::string path_;
};

// types.hpp:44-58 -- whole-tick conversion with a 1e-6 tolerance.
Tick seconds_to_ticks(double seconds, double tick_seconds, const std::string& field);

// ------------------------------------------------------------- pipeline.hpp
struct PipelineConfig {  // pipeline.hpp:13-36
  int num_stages = 1;
  int num_micro_batches = 1;
  std::vector<Tick> fp_duration;
  std::vector<Tick> bp_duration;
  int num_epochs = 1;
  double gpu_memory_total = 0.0;
  std::vector<double> stage_memory;
  double tick_seconds = 0.001;

  Tick fp_ticks(int s) const { return fp_duration.size() == 1 ? fp_duration[0] : fp_duration[s]; }
  Tick bp_ticks(int s) const { return bp_duration.size() == 1 ? bp_duration[0] : bp_duration[s]; }
  double available_memory(int s) const { return gpu_memory_total - stage_memory[s]; }
  void validate() const;
};

enum class OpKind { FP = 0, BP = 1 };

struct OpEvent {  // pipeline.hpp:40-47
  int stage = 0;
  OpKind kind = OpKind::FP;
  int micro_batch = 1;
  int epoch = 0;
  Tick start = 0;
  Tick end = 0;
};

struct ScheduleTrace {  // pipeline.hpp:49-53
  std::vector<OpEvent> ops;
  std::vector<std::pair<Tick, Tick>> epoch_spans;
  PipelineConfig config;
};

enum class BubbleType { A = 0, B = 1, C = 2 };

struct Bubble {  // pipeline.hpp:58-67
  int stage = 0;
  int epoch = 0;
  Tick start = 0;
  Tick duration = 0;
  double available_memory = 0.0;
  BubbleType btype = BubbleType::A;
  Tick end() const { return start + duration; }
};

struct LinkedBubble {  // pipeline.hpp:102-106
  Bubble bubble;
  std::int64_t prev_op = -1;  // -1: leads the epoch
  std::int64_t next_op = -1;  // -1: trails the epoch
};

std::vector<std::pair<OpKind, int>> stage_issue_order(int stage, int num_stages, int m);
ScheduleTrace build_schedule(const PipelineConfig& config);
std::vector<LinkedBubble> extract_bubbles_linked(const ScheduleTrace& trace);
std::vector<Bubble> extract_bubbles(const ScheduleTrace& trace);
double bubble_rate(const ScheduleTrace& trace, const std::vector<Bubble>& bubbles);
double bubble_rate(int num_stages, const OpEvent* ops, std::size_t n_ops, const Bubble* b,
                   std::size_t n_b);
std::vector<double> default_stage_memory(int num_stages, double gpu_memory_total,
                                         double weight_mem, double activation_mem);

// Point-to-point plan of one stage's 1F1B loop for a real multi-GPU pipeline
// (fr_p2p_op in freeride.h): group g precedes op g and pairs op g-1's send
// with op g's receive.
struct P2POp {
  int group;
  bool is_send;
  int peer;
  OpKind kind;  // FP: activation, BP: gradient
  int micro_batch;
};
std::vector<P2POp> pipeline_p2p_plan(int stage, int num_stages, int num_micro_batches);

// ----------------------------------------------------------------- task.hpp
enum class SideTaskState { Submitted = 0, Created = 1, Paused = 2, Running = 3, Stopped = 4 };
enum class TransitionKind {
  CreateSideTask = 0, InitSideTask = 1, StartSideTask = 2, RunNextStep = 3,
  PauseSideTask = 4, StopSideTask = 5
};
enum class TaskInterface { Iterative = 0, Imperative = 1 };
enum class MisbehaviorKind { None = 0, IgnoresPause = 1, MemoryLeak = 2 };

struct Misbehavior {
  MisbehaviorKind kind = MisbehaviorKind::None;
  double leak_rate_gib_per_s = 0.0;
};

struct SideTaskSpec {  // task.hpp:33-50
  std::string id;
  TaskInterface interface_kind = TaskInterface::Iterative;
  Tick per_step_duration = 1;
  std::optional<std::int64_t> total_steps;
  Tick init_duration = 0;
  double memory_demand = 0.0;
  Misbehavior misbehavior;
  Tick submit_time = 0;
  std::optional<double> memory_limit;
  std::optional<double> reference_throughput;
  void validate(const std::string& path) const;
};

struct SideTaskRuntime {  // task.hpp:52-60
  SideTaskSpec spec;
  SideTaskState state = SideTaskState::Submitted;
  std::int64_t steps_completed = 0;
  double memory_allocated = 0.0;
  std::optional<Tick> last_paused;
  std::optional<int> assigned_worker;
  std::optional<Tick> busy_until;
};

class IllegalTransition : public std::runtime_error {  // task.hpp:62-67
 public:
  IllegalTransition(SideTaskState from, TransitionKind kind);
  SideTaskState from;
  TransitionKind kind;
};

bool transition_legal(SideTaskState from, TransitionKind kind);
SideTaskState transition_target(SideTaskState from, TransitionKind kind);
void apply_transition(SideTaskRuntime& rt, TransitionKind kind, Tick now);

struct IterativeDecision {
  bool run = false;
  Tick step_end = 0;
};

IterativeDecision iterative_run(const SideTaskRuntime& rt, Tick bubble_end, Tick now,
                                double est_step_seconds, double tick_seconds,
                                Tick actual_step_ticks);
Tick imperative_run(const SideTaskRuntime& rt, Tick now, Tick actual_kernel_ticks);

enum class Disposition {
  Rejected = 0, Completed = 1, KilledOom = 2, KilledPauseTimeout = 3, KilledInitTimeout = 4,
  Active = 5
};

const char* to_string(SideTaskState s);
const char* to_string(TransitionKind k);

// --------------------------------------------------------------- limits.hpp
struct LimitConfig {
  Tick grace_period = 100;
  double memory_headroom = 0.0;
  Tick reclamation_delay = 0;
  void validate() const;
};
enum class MemCheck { Ok = 0, OomKill = 1 };
enum class Gate { Run = 0, Yield = 1 };
enum class Enforce { Ok = 0, Kill = 1 };

MemCheck check_memory(double memory_allocated, double limit);
Gate program_directed_gate(double remaining_seconds, double est_step_seconds);
Enforce framework_enforce(std::optional<Tick> last_paused, Tick pause_issued_at, Tick now,
                          Tick grace_period);

// ------------------------------------------------------------- profiler.hpp
struct TaskProfile {
  std::string task_id;
  std::optional<double> est_per_step_duration;
  std::optional<double> max_per_step_duration;
  double est_memory = 0.0;
  int profiled_steps = 0;
};

struct StageBubbleProfile {
  std::vector<Tick> durations;
  double available_memory = 0.0;
};

struct BubbleProfile {
  std::vector<StageBubbleProfile> stages;
  double rate = 0.0;
};

struct ProfileOptions {
  int n_steps = 32;
  double step_jitter = 0.0;
  double tick_seconds = 0.001;
};

std::uint64_t stream_seed(std::uint64_t seed, const std::string& task_id, const char* salt);
Tick jittered_step_ticks(Tick base, double jitter, std::uint64_t& rng_state);
TaskProfile profile_task(const SideTaskSpec& spec, const ProfileOptions& opts,
                         std::uint64_t seed);
BubbleProfile profile_bubbles(const PipelineConfig& config);

// -------------------------------------------------------------- manager.hpp
struct WorkerState {  // manager.hpp:17-28
  int worker_id = 0;
  double gpu_mem = 0.0;
  std::deque<std::string> task_queue;
  std::optional<std::string> current_task;
  std::optional<Bubble> current_bubble;
  int task_count() const {
    return static_cast<int>(task_queue.size()) + (current_task ? 1 : 0);
  }
};

struct SubmitOutcome {
  bool assigned = false;
  int worker_id = -1;
};

struct TaskView {
  SideTaskState state = SideTaskState::Submitted;
  bool initializing = false;
};
using TaskLookup = std::function<TaskView(const std::string&)>;

enum class ManagerActionKind { IssueInit = 0, IssueStart = 1, IssuePause = 2, ArmInitGuard = 3 };
struct ManagerAction {
  ManagerActionKind kind;
  std::string task_id;
};

std::optional<int> select_worker(double task_memory, const std::vector<WorkerState>& workers);
SubmitOutcome submit_task(const TaskProfile& profile, std::vector<WorkerState>& workers);
std::vector<ManagerAction> on_bubble_started(WorkerState& worker, const Bubble& bubble,
                                             const TaskLookup& lookup);
std::vector<ManagerAction> on_bubble_ended(WorkerState& worker, Tick now,
                                           const TaskLookup& lookup);

// -------------------------------------------------------------- metrics.hpp
struct PriceConfig {
  double price_server_1 = 3.96;
  double price_server_2 = 0.18;
  void validate() const;
};

struct TaskWork {
  std::string id;
  double work = 0.0;
  std::optional<double> throughput_per_hour;
};

struct CostBreakdown {
  double c_no_side = 0.0;
  double c_extra = 0.0;
  double c_side_tasks = 0.0;
  double s = 0.0;
};

struct StageBreakdown {
  int stage = 0;
  Tick used_by_side_tasks = 0;
  Tick runtime_overhead = 0;
  Tick idle_oom = 0;
  Tick idle_insufficient_time = 0;
  Tick total() const {
    return used_by_side_tasks + runtime_overhead + idle_oom + idle_insufficient_time;
  }
};

// engine.hpp:15-65 record types
enum class ActivityKind { Init = 0, Step = 1, Kernel = 2, Check = 3 };
enum class KillReason { Oom = 0, PauseTimeout = 1, InitTimeout = 2 };

struct TransitionRecord {
  Tick t = 0;
  std::string task;
  TransitionKind kind = TransitionKind::CreateSideTask;
  int worker = -1;
};
using RpcRecord = TransitionRecord;

struct ActivityRecord {
  Tick start = 0;
  Tick end = 0;
  std::string task;
  int worker = -1;
  ActivityKind kind = ActivityKind::Step;
  bool clipped = false;
};

struct KillRecord {
  Tick t = 0;
  std::string task;
  int worker = -1;
  KillReason reason = KillReason::Oom;
};

struct AssignRecord {
  Tick t = 0;
  std::string task;
  int worker = -1;
};

struct DispositionRecord {
  std::string task;
  Disposition disposition = Disposition::Active;
  std::int64_t steps_completed = 0;
  std::optional<int> worker;
};

// What bubble_breakdown reads from a RunTrace (metrics.cpp:62-178).
struct BreakdownInput {
  int num_stages = 0;
  std::vector<TaskProfile> profiles;
  std::vector<Bubble> bubbles;
  std::vector<AssignRecord> assigns;
  std::vector<TransitionRecord> transitions;
  std::vector<ActivityRecord> activities;
};

// ---------------------------------------------------------------- engine.hpp
enum class GateEstimate { Mean = 0, Max = 1 };  // config.hpp:17

struct RuntimeOptions {  // config.hpp:19-27
  Tick check_overhead = 1;
  Tick rpc_latency = 0;
  double step_jitter = 0.0;
  int profile_steps = 32;
  GateEstimate gate_estimate = GateEstimate::Mean;
};

struct SweepGrid {  // config.hpp:29-35
  std::vector<int> micro_batches;
  std::vector<std::string> model_sizes;
  std::vector<int> batch_sizes;
};

struct ExperimentConfig {  // config.hpp:36-46 (JSON I/O: host/io.hpp)
  PipelineConfig pipeline;
  std::vector<SideTaskSpec> tasks;
  LimitConfig limits;
  PriceConfig prices;
  RuntimeOptions runtime;
  std::optional<SweepGrid> sweep;
  std::uint64_t seed = 0;
};

struct RunTrace {  // engine.hpp:75-92
  // RunMeta (engine.hpp:67-73)
  ExperimentConfig config;
  std::uint64_t seed = 0;
  bool with_tasks = false;
  std::vector<OpEvent> ops;
  std::vector<Bubble> bubbles;            // as signalled on the delayed timeline
  std::vector<AssignRecord> submits;      // worker -1
  std::vector<AssignRecord> assigns;
  std::vector<AssignRecord> rejects;      // worker -1
  std::vector<RpcRecord> rpcs;
  std::vector<TransitionRecord> transitions;
  std::vector<ActivityRecord> activities;
  std::vector<KillRecord> kills;
  std::vector<DispositionRecord> dispositions;
  std::vector<TaskProfile> profiles;
  Tick makespan = 0;
  // A trace recorded on the GPU (fr_harness_run_trace) rather than simulated:
  // op durations are measured, only the stages in it ran, side-task kernels
  // may co-run with an op (a step's tail past its bubble), and times from the
  // host / device-clock domains agree to within `tolerance` ticks.
  bool measured = false;
  Tick tolerance = 0;
};

// engine.hpp:97-98 -- the reference declares it and never implements it; the
// rules are SURVEY.md Appendix B with the ambiguities fixed in DESIGN.md §6.
RunTrace run_experiment(const ExperimentConfig& config, bool with_tasks, std::uint64_t seed);

double time_increase(double t_no_seconds, double t_with_seconds);
CostBreakdown cost_savings(double t_no_seconds, double delta_t, const std::vector<TaskWork>& work,
                           const PriceConfig& prices);
std::vector<StageBreakdown> bubble_breakdown(const BreakdownInput& in);

}  // namespace freeride
