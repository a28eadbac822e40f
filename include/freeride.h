/*
 * freeride.h -- C-ABI drop-in boundary of the B200-native bubble-harvesting
 * hot path (FreeRide, arXiv 2409.06941).
 *
 * Every entry point below replaces one function of the reference's C++ API
 * (`bubblesim`, /root/reference/proj/include/bubblesim/<module>.hpp); the cited
 * file:line is the declaration it stands in for.  The rules of the boundary:
 *
 *   - no exceptions cross it: every call returns an int status (FR_OK = 0);
 *     the reference's exception types map to status codes and the message /
 *     offending field are available from fr_last_error()/fr_last_error_field()
 *     (thread-local, valid until the next failing call on the same thread);
 *   - plain pointers and sizes only; caller-owned output buffers carry an
 *     explicit capacity and the required count is always written back, so a
 *     FR_ERR_CAPACITY return can be retried with a larger buffer;
 *   - task ids are NUL-terminated strings of at most FR_TASK_ID_MAX-1 bytes
 *     (the reference uses std::string; records here are fixed-size so they
 *     can be laid out as flat arrays / numpy structured dtypes);
 *   - GPU calls are asynchronous on the caller's stream (passed as void*,
 *     a cudaStream_t), never synchronise unless documented, and keep no
 *     global mutable state: one worker thread per GPU may call concurrently.
 *
 * Two libraries export this header:
 *   paper_2409_06941_b200/_lib/libfreeride.so   the product (host C++ + sm_100a)
 *   oracle/_ref/libbubblesim_ref.so             the reference's own sources
 *                                               behind a test-only shim (host
 *                                               rows only; GPU rows absent)
 */
#ifndef FREERIDE_H_
#define FREERIDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FR_ABI_VERSION 1
#define FR_TASK_ID_MAX 64

/* ------------------------------------------------------------------ status */
enum fr_status {
  FR_OK = 0,
  FR_ERR_VALIDATION = 1,         /* bubblesim::ValidationError  types.hpp:22   */
  FR_ERR_SCHEMA = 2,             /* bubblesim::SchemaError      types.hpp:34   */
  FR_ERR_INVARIANT = 3,          /* std::logic_error            pipeline.cpp:155 */
  FR_ERR_ILLEGAL_TRANSITION = 4, /* bubblesim::IllegalTransition task.hpp:62   */
  FR_ERR_CAPACITY = 5,           /* output buffer too small; count written back */
  FR_ERR_ARGUMENT = 6,           /* null pointer, bad enum, id too long        */
  FR_ERR_NOT_FOUND = 7,          /* unknown worker / task                      */
  FR_ERR_UNSUPPORTED = 8,        /* shape or mode the kernel does not cover    */
  FR_ERR_CUDA_BASE = 100         /* FR_ERR_CUDA_BASE + cudaError_t             */
};

int fr_abi_version(void);
const char* fr_last_error(void);
const char* fr_last_error_field(void);

typedef int64_t fr_tick; /* bubblesim::Tick  types.hpp:14 */

/* -------------------------------------------------------- pipeline (L1) */
enum fr_op_kind { FR_OP_FP = 0, FR_OP_BP = 1 };         /* pipeline.hpp:38 */
enum fr_bubble_type { FR_BUBBLE_A = 0, FR_BUBBLE_B = 1, FR_BUBBLE_C = 2 }; /* :55 */

/* bubblesim::PipelineConfig  pipeline.hpp:13-36 */
typedef struct fr_pipeline_config {
  int32_t num_stages;
  int32_t num_micro_batches;
  int32_t num_epochs;
  int32_t n_fp;               /* 1 (uniform) or num_stages */
  const fr_tick* fp_duration;
  int32_t n_bp;
  int32_t n_stage_memory;     /* must equal num_stages */
  const fr_tick* bp_duration;
  const double* stage_memory; /* GiB held by training, per stage */
  double gpu_memory_total;    /* GiB */
  double tick_seconds;
} fr_pipeline_config;

typedef struct fr_issue {     /* std::pair<OpKind,int>  pipeline.hpp:72 */
  int32_t kind;
  int32_t micro_batch;        /* 1-based */
} fr_issue;

typedef struct fr_op_event {  /* bubblesim::OpEvent  pipeline.hpp:40-47 */
  int32_t stage;
  int32_t kind;
  int32_t micro_batch;
  int32_t epoch;
  fr_tick start;
  fr_tick end;
} fr_op_event;

/* bubblesim::Bubble (pipeline.hpp:58-67) plus the detail::LinkedBubble links
 * (pipeline.hpp:102-106): prev_op / next_op index fr_build_schedule's ops,
 * -1 when the bubble leads / trails its epoch. */
typedef struct fr_bubble {
  int32_t stage;
  int32_t epoch;
  fr_tick start;
  fr_tick duration;
  double available_memory;
  int32_t btype;
  int32_t reserved;
  int64_t prev_op;
  int64_t next_op;
} fr_bubble;

/* PipelineConfig::validate  pipeline.hpp:35 */
int fr_pipeline_validate(const fr_pipeline_config* cfg);
/* stage_issue_order  pipeline.hpp:72 ; needs cap >= 2*m */
int fr_stage_issue_order(int32_t stage, int32_t num_stages, int32_t num_micro_batches,
                         fr_issue* out, int64_t cap, int64_t* n_out);
/* build_schedule  pipeline.hpp:78 ; ops cap >= 2*p*m*epochs, spans 2*epochs
 * (start,end) pairs.  Ops ordered by (start, stage, end, micro_batch). */
int fr_build_schedule(const fr_pipeline_config* cfg, fr_op_event* ops, int64_t cap,
                      int64_t* n_ops, fr_tick* epoch_spans);
/* detail::extract_bubbles_linked  pipeline.hpp:108 (extract_bubbles :84 drops
 * the links); cap >= epochs*p*(2m+1) always suffices. */
int fr_extract_bubbles(const fr_pipeline_config* cfg, const fr_op_event* ops, int64_t n_ops,
                       const fr_tick* epoch_spans, fr_bubble* out, int64_t cap,
                       int64_t* n_out);
/* bubble_rate  pipeline.hpp:87 */
int fr_bubble_rate(int32_t num_stages, const fr_op_event* ops, int64_t n_ops,
                   const fr_bubble* bubbles, int64_t n_bubbles, double* rate);
/* default_stage_memory  pipeline.hpp:91 ; out has num_stages entries */
int fr_default_stage_memory(int32_t num_stages, double gpu_memory_total, double weight_mem,
                            double activation_mem_per_microbatch, double* out);

/* -------------------------------------------------------- task model (L3) */
enum fr_task_state {          /* SideTaskState  task.hpp:12 */
  FR_SUBMITTED = 0, FR_CREATED = 1, FR_PAUSED = 2, FR_RUNNING = 3, FR_STOPPED = 4
};
enum fr_transition {          /* TransitionKind  task.hpp:15-22 */
  FR_CREATE_SIDE_TASK = 0, FR_INIT_SIDE_TASK = 1, FR_START_SIDE_TASK = 2,
  FR_RUN_NEXT_STEP = 3, FR_PAUSE_SIDE_TASK = 4, FR_STOP_SIDE_TASK = 5
};
enum fr_interface { FR_ITERATIVE = 0, FR_IMPERATIVE = 1 };          /* task.hpp:24 */
enum fr_misbehavior { FR_MB_NONE = 0, FR_MB_IGNORES_PAUSE = 1, FR_MB_MEMORY_LEAK = 2 }; /* :26 */
enum fr_disposition {         /* Disposition  task.hpp:97-104 */
  FR_DISP_REJECTED = 0, FR_DISP_COMPLETED = 1, FR_DISP_KILLED_OOM = 2,
  FR_DISP_KILLED_PAUSE_TIMEOUT = 3, FR_DISP_KILLED_INIT_TIMEOUT = 4, FR_DISP_ACTIVE = 5
};

/* bubblesim::SideTaskSpec  task.hpp:33-50 (std::optional -> has_* flag) */
typedef struct fr_side_task_spec {
  char id[FR_TASK_ID_MAX];
  int32_t interface_kind;
  int32_t misbehavior;
  int32_t has_total_steps;
  int32_t has_memory_limit;
  int32_t has_reference_throughput;
  int32_t reserved;
  fr_tick per_step_duration;
  int64_t total_steps;
  fr_tick init_duration;
  double memory_demand;
  double leak_rate_gib_per_s;
  fr_tick submit_time;
  double memory_limit;
  double reference_throughput;
} fr_side_task_spec;

/* bubblesim::SideTaskRuntime  task.hpp:52-60 (spec reduced to memory_demand,
 * the only field apply_transition reads) */
typedef struct fr_task_runtime {
  int32_t state;
  int32_t has_last_paused;
  int32_t has_assigned_worker;
  int32_t assigned_worker;
  int32_t has_busy_until;
  int32_t reserved;
  int64_t steps_completed;
  double memory_allocated;
  fr_tick last_paused;
  fr_tick busy_until;
  double memory_demand;
} fr_task_runtime;

typedef struct fr_iterative_decision { /* IterativeDecision  task.hpp:79-82 */
  int32_t run;
  int32_t reserved;
  fr_tick step_end;
} fr_iterative_decision;

/* SideTaskSpec::validate  task.hpp:49 ; path prefixes the error field */
int fr_side_task_validate(const fr_side_task_spec* spec, const char* path);
/* transition_legal  task.hpp:69 -> *legal = 0/1 */
int fr_transition_legal(int32_t from, int32_t kind, int32_t* legal);
/* transition_target  task.hpp:70 */
int fr_transition_target(int32_t from, int32_t kind, int32_t* to);
/* apply_transition  task.hpp:75 */
int fr_apply_transition(fr_task_runtime* rt, int32_t kind, fr_tick now);
/* iterative_run  task.hpp:87-89 -- the program-directed pre-step check */
int fr_iterative_run(const fr_task_runtime* rt, fr_tick bubble_end, fr_tick now,
                     double est_step_seconds, double tick_seconds, fr_tick actual_step_ticks,
                     fr_iterative_decision* out);
/* imperative_run  task.hpp:93 */
int fr_imperative_run(const fr_task_runtime* rt, fr_tick now, fr_tick actual_kernel_ticks,
                      fr_tick* kernel_end);

/* ------------------------------------------------------------ limits (L3) */
enum fr_gate { FR_GATE_RUN = 0, FR_GATE_YIELD = 1 };      /* limits.hpp:22 */
enum fr_memcheck { FR_MEM_OK = 0, FR_MEM_OOM_KILL = 1 };  /* limits.hpp:17 */
enum fr_enforce { FR_ENFORCE_OK = 0, FR_ENFORCE_KILL = 1 }; /* limits.hpp:28 */

typedef struct fr_limit_config {  /* LimitConfig  limits.hpp:9-15 */
  fr_tick grace_period;
  double memory_headroom;
  fr_tick reclamation_delay;
} fr_limit_config;

int fr_limit_config_validate(const fr_limit_config* cfg);
/* check_memory  limits.hpp:20 */
int fr_check_memory(double memory_allocated, double limit, int32_t* result);
/* program_directed_gate  limits.hpp:26 */
int fr_program_directed_gate(double remaining_seconds, double est_step_seconds, int32_t* gate);
/* framework_enforce  limits.hpp:34 ; has_last_paused=0 is std::nullopt */
int fr_framework_enforce(int32_t has_last_paused, fr_tick last_paused, fr_tick pause_issued_at,
                         fr_tick now, fr_tick grace_period, int32_t* result);

/* ---------------------------------------------------------- profiler (L2) */
typedef struct fr_profile_options { /* ProfileOptions  profiler.hpp:33-37 */
  int32_t n_steps;
  int32_t reserved;
  double step_jitter;
  double tick_seconds;
} fr_profile_options;

typedef struct fr_task_profile {    /* TaskProfile  profiler.hpp:15-21 */
  char task_id[FR_TASK_ID_MAX];
  int32_t has_est_per_step;         /* 0 for imperative tasks */
  int32_t profiled_steps;
  double est_per_step_duration;     /* seconds */
  double max_per_step_duration;     /* seconds */
  double est_memory;                /* GiB */
} fr_task_profile;

/* stream_seed  profiler.hpp:48 */
uint64_t fr_stream_seed(uint64_t seed, const char* task_id, const char* salt);
/* jittered_step_ticks  profiler.hpp:53 */
fr_tick fr_jittered_step_ticks(fr_tick base, double jitter, uint64_t* rng_state);
/* profile_task  profiler.hpp:41 */
int fr_profile_task(const fr_side_task_spec* spec, const fr_profile_options* opts,
                    uint64_t seed, fr_task_profile* out);
/* profile_bubbles  profiler.hpp:45 ; durations flattened per stage (sorted),
 * stage s owns durations[stage_offsets[s] .. stage_offsets[s+1]) ;
 * stage_offsets has p+1 entries, available_memory p entries. */
int fr_profile_bubbles(const fr_pipeline_config* cfg, fr_tick* durations, int64_t cap,
                       int64_t* stage_offsets, double* available_memory, double* rate);

/* ----------------------------------------------------------- manager (L4) */
/* The reference's caller-owned std::vector<WorkerState> (manager.hpp:17-28)
 * becomes an opaque handle owning one WorkerState per worker. */
typedef struct fr_manager fr_manager;

enum fr_action_kind {               /* ManagerActionKind  manager.hpp:54-59 */
  FR_ACT_ISSUE_INIT = 0, FR_ACT_ISSUE_START = 1, FR_ACT_ISSUE_PAUSE = 2,
  FR_ACT_ARM_INIT_GUARD = 3
};

typedef struct fr_task_view {       /* TaskView  manager.hpp:47-50 */
  int32_t state;
  int32_t initializing;
} fr_task_view;

typedef struct fr_manager_action {  /* ManagerAction  manager.hpp:61-64 */
  int32_t kind;
  char task_id[FR_TASK_ID_MAX];
} fr_manager_action;

/* TaskLookup  manager.hpp:52 ; return FR_OK or an error (propagated) */
typedef int (*fr_task_lookup_fn)(void* ctx, const char* task_id, fr_task_view* out);

typedef struct fr_worker_info {     /* WorkerState  manager.hpp:17-28 */
  int32_t worker_id;
  int32_t queue_len;
  int32_t has_current_task;
  int32_t has_current_bubble;
  double gpu_mem;
  char current_task[FR_TASK_ID_MAX];
  fr_bubble current_bubble;
} fr_worker_info;

int fr_manager_create(int32_t n_workers, const double* gpu_mem, fr_manager** out);
void fr_manager_destroy(fr_manager* mgr);
int fr_manager_worker_info(const fr_manager* mgr, int32_t worker, fr_worker_info* out);
/* i-th queued task id (0 = front, earliest submitted) */
int fr_manager_queue_at(const fr_manager* mgr, int32_t worker, int32_t i, char* buf,
                        int32_t cap);
/* mirror a remote worker's queue (distributed Alg. 1: every rank rebuilds the
 * gathered WorkerStates and runs the same deterministic select_worker) */
int fr_manager_push_task(fr_manager* mgr, int32_t worker, const char* task_id);
/* engine housekeeping (Appendix B rule 8): clear or set CurrentTask */
int fr_manager_set_current_task(fr_manager* mgr, int32_t worker, const char* task_id_or_null);
/* select_worker  manager.hpp:33 ; *worker = -1 when none qualifies */
int fr_select_worker(const fr_manager* mgr, double task_memory, int32_t* worker);
/* submit_task  manager.hpp:43 (Alg. 1) */
int fr_submit_task(fr_manager* mgr, const fr_task_profile* profile, int32_t* assigned,
                   int32_t* worker_id);
/* on_bubble_started  manager.hpp:69 (Alg. 2 lines 8-17) */
int fr_on_bubble_started(fr_manager* mgr, int32_t worker, const fr_bubble* bubble,
                         fr_task_lookup_fn lookup, void* ctx, fr_manager_action* out,
                         int32_t cap, int32_t* n_out);
/* on_bubble_ended  manager.hpp:76 (Alg. 2 lines 3-7) */
int fr_on_bubble_ended(fr_manager* mgr, int32_t worker, fr_tick now, fr_task_lookup_fn lookup,
                       void* ctx, fr_manager_action* out, int32_t cap, int32_t* n_out);

/* ----------------------------------------------------------- metrics (L6) */
typedef struct fr_price_config {    /* PriceConfig  metrics.hpp:16-21 */
  double price_server_1;
  double price_server_2;
} fr_price_config;

typedef struct fr_task_work {       /* TaskWork  metrics.hpp:27-31 */
  char id[FR_TASK_ID_MAX];
  double work;
  int32_t has_throughput;
  int32_t reserved;
  double throughput_per_hour;
} fr_task_work;

typedef struct fr_cost_breakdown {  /* CostBreakdown  metrics.hpp:33-38 */
  double c_no_side;
  double c_extra;
  double c_side_tasks;
  double s;
} fr_cost_breakdown;

typedef struct fr_stage_breakdown { /* StageBreakdown  metrics.hpp:51-62 */
  int32_t stage;
  int32_t reserved;
  fr_tick used_by_side_tasks;
  fr_tick runtime_overhead;
  fr_tick idle_oom;
  fr_tick idle_insufficient_time;
} fr_stage_breakdown;

/* RunTrace record types  engine.hpp:15-65 */
enum fr_activity_kind { FR_ACTIVITY_INIT = 0, FR_ACTIVITY_STEP = 1, FR_ACTIVITY_KERNEL = 2,
                        FR_ACTIVITY_CHECK = 3 };
enum fr_kill_reason { FR_KILL_OOM = 0, FR_KILL_PAUSE_TIMEOUT = 1, FR_KILL_INIT_TIMEOUT = 2 };

typedef struct fr_transition_record { /* TransitionRecord / RpcRecord engine.hpp:18-31 */
  fr_tick t;
  int32_t kind;
  int32_t worker;
  char task[FR_TASK_ID_MAX];
} fr_transition_record;

typedef struct fr_activity_record {   /* ActivityRecord  engine.hpp:33-40 */
  fr_tick start;
  fr_tick end;
  int32_t worker;
  int32_t kind;
  int32_t clipped;
  int32_t reserved;
  char task[FR_TASK_ID_MAX];
} fr_activity_record;

typedef struct fr_kill_record {       /* KillRecord  engine.hpp:42-47 */
  fr_tick t;
  int32_t worker;
  int32_t reason;
  char task[FR_TASK_ID_MAX];
} fr_kill_record;

typedef struct fr_assign_record {     /* SubmitRecord/AssignRecord engine.hpp:49-58 */
  fr_tick t;
  int32_t worker;                     /* -1 for submit / reject records */
  int32_t reserved;
  char task[FR_TASK_ID_MAX];
} fr_assign_record;

typedef struct fr_disposition_record { /* DispositionRecord  engine.hpp:60-65 */
  int32_t disposition;
  int32_t has_worker;
  int32_t worker;
  int32_t reserved;
  int64_t steps_completed;
  char task[FR_TASK_ID_MAX];
} fr_disposition_record;

/* The slice of RunTrace (engine.hpp:75-92) that bubble_breakdown reads. */
typedef struct fr_breakdown_input {
  int32_t num_stages;
  int32_t n_profiles;
  const fr_task_profile* profiles;
  int64_t n_bubbles;
  const fr_bubble* bubbles;
  int64_t n_assigns;
  const fr_assign_record* assigns;
  int64_t n_transitions;
  const fr_transition_record* transitions;
  int64_t n_activities;
  const fr_activity_record* activities;
} fr_breakdown_input;

/* ---------------------------------------- pipeline P2P plan (multi-GPU) */
/* One point-to-point operation of stage `stage`'s 1F1B loop (not in the
 * reference, which simulates stages on one timeline): at op
 * boundary `group` (0..2m; group g sits before op g, after op g-1) the stage
 * sends op g-1's output and receives op g's input in ONE send/recv group
 * (ncclGroupStart/End).  Pairing the two in one group is what keeps 1F1B
 * deadlock-free under rendezvous semantics (tests/test_p2p_plan.py). */
typedef struct fr_p2p_op {
  int32_t group;     /* op boundary index, 0..2m */
  int32_t is_send;   /* 1 send, 0 recv */
  int32_t peer;      /* stage +-1 */
  int32_t kind;      /* FR_OP_FP: activation, FR_OP_BP: gradient */
  int32_t micro_batch;
} fr_p2p_op;
/* ops in execution order; cap >= 4*m always suffices */
int fr_pipeline_p2p_plan(int32_t stage, int32_t num_stages, int32_t num_micro_batches,
                         fr_p2p_op* out, int64_t cap, int64_t* n_out);

/* ------------------------------------------------------------ engine (L5) */
typedef struct fr_runtime_options {  /* RuntimeOptions  config.hpp:19-27 */
  fr_tick check_overhead;
  fr_tick rpc_latency;
  double step_jitter;
  int32_t profile_steps;
  int32_t gate_estimate;             /* 0 mean, 1 max (GateEstimate config.hpp:17) */
} fr_runtime_options;

typedef struct fr_experiment_config { /* ExperimentConfig config.hpp:36-46 */
  fr_pipeline_config pipeline;
  const fr_side_task_spec* tasks;
  int32_t n_tasks;
  int32_t reserved;
  fr_limit_config limits;
  fr_runtime_options runtime;
} fr_experiment_config;

typedef struct fr_run_trace fr_run_trace; /* RunTrace engine.hpp:75-92 */

typedef struct fr_run_trace_counts {
  int64_t ops, bubbles, submits, assigns, rejects, rpcs, transitions, activities, kills,
      dispositions;
  fr_tick makespan;
} fr_run_trace_counts;

/* run_experiment  engine.hpp:97-98 (declared, never implemented by the
 * reference; rules in DESIGN.md §6).  Deterministic in (config, with_tasks, seed). */
int fr_run_experiment(const fr_experiment_config* cfg, int32_t with_tasks, uint64_t seed,
                      fr_run_trace** out);
void fr_run_trace_destroy(fr_run_trace* t);
int fr_run_trace_get_counts(const fr_run_trace* t, fr_run_trace_counts* out);
int fr_run_trace_ops(const fr_run_trace* t, fr_op_event* out, int64_t cap);
int fr_run_trace_bubbles(const fr_run_trace* t, fr_bubble* out, int64_t cap);
/* which: 0 submits, 1 assigns, 2 rejects */
int fr_run_trace_assigns(const fr_run_trace* t, int32_t which, fr_assign_record* out, int64_t cap);
/* which: 0 transitions, 1 rpcs */
int fr_run_trace_transitions(const fr_run_trace* t, int32_t which, fr_transition_record* out,
                             int64_t cap);
int fr_run_trace_activities(const fr_run_trace* t, fr_activity_record* out, int64_t cap);
int fr_run_trace_kills(const fr_run_trace* t, fr_kill_record* out, int64_t cap);
int fr_run_trace_dispositions(const fr_run_trace* t, fr_disposition_record* out, int64_t cap);
/* replay_check (engine.hpp:100-104): re-validates the module invariants over
 * the finished trace; violations joined by '\n' into buf (cap bytes,
 * NUL-terminated, truncated to fit), *n_violations = their count (0 = sound). */
int fr_run_trace_check(const fr_run_trace* t, char* buf, int64_t cap, int32_t* n_violations);
/* write_trace_file / read_trace_file (trace.hpp:19-20): the JSONL stream --
 * meta line (config, seed, profiles), records in timeline order,
 * dispositions, end line; byte-stable for identical runs. */
int fr_run_trace_write_jsonl(const fr_run_trace* t, const char* path);
int fr_run_trace_read_jsonl(const char* path, fr_run_trace** out);

/* time_increase  metrics.hpp:25 */
int fr_time_increase(double t_no_seconds, double t_with_seconds, double* out);
/* cost_savings  metrics.hpp:45 */
int fr_cost_savings(double t_no_seconds, double delta_t, const fr_task_work* work,
                    int32_t n_work, const fr_price_config* prices, fr_cost_breakdown* out);
/* bubble_breakdown  metrics.hpp:64 ; out has num_stages entries */
int fr_bubble_breakdown(const fr_breakdown_input* in, fr_stage_breakdown* out);

#ifdef __cplusplus
}
#endif

#endif /* FREERIDE_H_ */
