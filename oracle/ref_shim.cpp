// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Binds the reference's own compiled sources (/root/reference/proj/src/*.cpp,
// built by oracle/Makefile into oracle/_ref/) to the C-ABI of
// include/freeride.h, so tests can call the unmodified reference through the
// exact entry points the product exports and compare results byte for byte.
// Only host rows (pipeline, profiler, task, limits, manager, metrics) exist
// here; the reference has no engine .cpp and no GPU code.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "bubblesim/engine.hpp"
#include "bubblesim/limits.hpp"
#include "bubblesim/manager.hpp"
#include "bubblesim/metrics.hpp"
#include "bubblesim/pipeline.hpp"
#include "bubblesim/profiler.hpp"
#include "bubblesim/task.hpp"
#include "freeride.h"

using namespace bubblesim;

namespace {

thread_local std::string g_err;
thread_local std::string g_field;

int fail(int code, const std::string& msg, const std::string& field = "") {
  g_err = msg;
  g_field = field;
  return code;
}

struct CallbackError : std::runtime_error {
  int code;
  explicit CallbackError(int c) : std::runtime_error("lookup callback failed"), code(c) {}
};

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const ValidationError& e) {
    return fail(FR_ERR_VALIDATION, e.what(), e.field());
  } catch (const SchemaError& e) {
    return fail(FR_ERR_SCHEMA, e.what(), e.path());
  } catch (const IllegalTransition& e) {
    return fail(FR_ERR_ILLEGAL_TRANSITION, e.what());
  } catch (const CallbackError& e) {
    return e.code;
  } catch (const std::logic_error& e) {
    return fail(FR_ERR_INVARIANT, e.what());
  } catch (const std::exception& e) {
    return fail(FR_ERR_INVARIANT, e.what());
  }
}

PipelineConfig to_cfg(const fr_pipeline_config* c) {
  PipelineConfig cfg;
  cfg.num_stages = c->num_stages;
  cfg.num_micro_batches = c->num_micro_batches;
  cfg.num_epochs = c->num_epochs;
  cfg.fp_duration.assign(c->fp_duration, c->fp_duration + (c->fp_duration ? c->n_fp : 0));
  cfg.bp_duration.assign(c->bp_duration, c->bp_duration + (c->bp_duration ? c->n_bp : 0));
  cfg.stage_memory.assign(c->stage_memory,
                          c->stage_memory + (c->stage_memory ? c->n_stage_memory : 0));
  cfg.gpu_memory_total = c->gpu_memory_total;
  cfg.tick_seconds = c->tick_seconds;
  return cfg;
}

fr_op_event to_c(const OpEvent& o) {
  return fr_op_event{o.stage, static_cast<int32_t>(o.kind), o.micro_batch, o.epoch, o.start,
                     o.end};
}

OpEvent from_c(const fr_op_event& o) {
  OpEvent e;
  e.stage = o.stage;
  e.kind = static_cast<OpKind>(o.kind);
  e.micro_batch = o.micro_batch;
  e.epoch = o.epoch;
  e.start = o.start;
  e.end = o.end;
  return e;
}

Bubble from_c(const fr_bubble& b) {
  Bubble r;
  r.stage = b.stage;
  r.epoch = b.epoch;
  r.start = b.start;
  r.duration = b.duration;
  r.available_memory = b.available_memory;
  r.btype = static_cast<BubbleType>(b.btype);
  return r;
}

fr_bubble to_c(const Bubble& b, long long prev, long long next) {
  fr_bubble r{};
  r.stage = b.stage;
  r.epoch = b.epoch;
  r.start = b.start;
  r.duration = b.duration;
  r.available_memory = b.available_memory;
  r.btype = static_cast<int32_t>(b.btype);
  r.prev_op = prev;
  r.next_op = next;
  return r;
}

void copy_id(char* dst, const std::string& s) {
  std::memset(dst, 0, FR_TASK_ID_MAX);
  std::strncpy(dst, s.c_str(), FR_TASK_ID_MAX - 1);
}

SideTaskSpec to_spec(const fr_side_task_spec* s) {
  SideTaskSpec spec;
  spec.id = std::string(s->id, strnlen(s->id, FR_TASK_ID_MAX));
  spec.interface_kind = static_cast<TaskInterface>(s->interface_kind);
  spec.per_step_duration = s->per_step_duration;
  if (s->has_total_steps) spec.total_steps = s->total_steps;
  spec.init_duration = s->init_duration;
  spec.memory_demand = s->memory_demand;
  spec.misbehavior.kind = static_cast<MisbehaviorKind>(s->misbehavior);
  spec.misbehavior.leak_rate_gib_per_s = s->leak_rate_gib_per_s;
  spec.submit_time = s->submit_time;
  if (s->has_memory_limit) spec.memory_limit = s->memory_limit;
  if (s->has_reference_throughput) spec.reference_throughput = s->reference_throughput;
  return spec;
}

SideTaskRuntime to_rt(const fr_task_runtime* r) {
  SideTaskRuntime rt;
  rt.spec.memory_demand = r->memory_demand;
  rt.state = static_cast<SideTaskState>(r->state);
  rt.steps_completed = r->steps_completed;
  rt.memory_allocated = r->memory_allocated;
  if (r->has_last_paused) rt.last_paused = r->last_paused;
  if (r->has_assigned_worker) rt.assigned_worker = r->assigned_worker;
  if (r->has_busy_until) rt.busy_until = r->busy_until;
  return rt;
}

void from_rt(const SideTaskRuntime& rt, fr_task_runtime* r) {
  r->state = static_cast<int32_t>(rt.state);
  r->steps_completed = rt.steps_completed;
  r->memory_allocated = rt.memory_allocated;
  r->has_last_paused = rt.last_paused.has_value();
  r->last_paused = rt.last_paused.value_or(0);
  r->has_assigned_worker = rt.assigned_worker.has_value();
  r->assigned_worker = rt.assigned_worker.value_or(0);
  r->has_busy_until = rt.busy_until.has_value();
  r->busy_until = rt.busy_until.value_or(0);
}

}  // namespace

struct fr_manager {
  std::vector<WorkerState> workers;
};

extern "C" {

int fr_abi_version(void) { return FR_ABI_VERSION; }
const char* fr_last_error(void) { return g_err.c_str(); }
const char* fr_last_error_field(void) { return g_field.c_str(); }

int fr_pipeline_validate(const fr_pipeline_config* cfg) {
  if (!cfg) return fail(FR_ERR_ARGUMENT, "null config");
  return guard([&]() -> int {
    to_cfg(cfg).validate();
    return FR_OK;
  });
}

int fr_stage_issue_order(int32_t stage, int32_t num_stages, int32_t m, fr_issue* out,
                         int64_t cap, int64_t* n_out) {
  return guard([&]() -> int {
    auto order = stage_issue_order(stage, num_stages, m);
    *n_out = static_cast<int64_t>(order.size());
    if (static_cast<int64_t>(order.size()) > cap) return fail(FR_ERR_CAPACITY, "capacity");
    for (size_t i = 0; i < order.size(); ++i)
      out[i] = fr_issue{static_cast<int32_t>(order[i].first), order[i].second};
    return FR_OK;
  });
}

int fr_build_schedule(const fr_pipeline_config* cfg, fr_op_event* ops, int64_t cap,
                      int64_t* n_ops, fr_tick* spans) {
  return guard([&]() -> int {
    ScheduleTrace t = build_schedule(to_cfg(cfg));
    *n_ops = static_cast<int64_t>(t.ops.size());
    if (*n_ops > cap) return fail(FR_ERR_CAPACITY, "capacity");
    for (size_t i = 0; i < t.ops.size(); ++i) ops[i] = to_c(t.ops[i]);
    for (size_t e = 0; e < t.epoch_spans.size(); ++e) {
      spans[2 * e] = t.epoch_spans[e].first;
      spans[2 * e + 1] = t.epoch_spans[e].second;
    }
    return FR_OK;
  });
}

int fr_extract_bubbles(const fr_pipeline_config* cfg, const fr_op_event* ops, int64_t n_ops,
                       const fr_tick* spans, fr_bubble* out, int64_t cap, int64_t* n_out) {
  return guard([&]() -> int {
    ScheduleTrace t;
    t.config = to_cfg(cfg);
    for (int64_t i = 0; i < n_ops; ++i) t.ops.push_back(from_c(ops[i]));
    for (int e = 0; e < cfg->num_epochs; ++e) t.epoch_spans.push_back({spans[2 * e], spans[2 * e + 1]});
    auto lb = detail::extract_bubbles_linked(t);
    *n_out = static_cast<int64_t>(lb.size());
    if (*n_out > cap) return fail(FR_ERR_CAPACITY, "capacity");
    for (size_t i = 0; i < lb.size(); ++i) {
      out[i] = to_c(lb[i].bubble, lb[i].prev_op ? static_cast<long long>(*lb[i].prev_op) : -1,
                    lb[i].next_op ? static_cast<long long>(*lb[i].next_op) : -1);
    }
    return FR_OK;
  });
}

int fr_bubble_rate(int32_t p, const fr_op_event* ops, int64_t n_ops, const fr_bubble* b,
                   int64_t nb, double* rate) {
  return guard([&]() -> int {
    ScheduleTrace t;
    t.config.num_stages = p;
    for (int64_t i = 0; i < n_ops; ++i) t.ops.push_back(from_c(ops[i]));
    std::vector<Bubble> bs;
    for (int64_t i = 0; i < nb; ++i) bs.push_back(from_c(b[i]));
    *rate = bubble_rate(t, bs);
    return FR_OK;
  });
}

int fr_default_stage_memory(int32_t p, double total, double w, double a, double* out) {
  return guard([&]() -> int {
    auto v = default_stage_memory(p, total, w, a);
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    return FR_OK;
  });
}

int fr_side_task_validate(const fr_side_task_spec* spec, const char* path) {
  return guard([&]() -> int {
    to_spec(spec).validate(path ? path : "");
    return FR_OK;
  });
}

int fr_transition_legal(int32_t from, int32_t kind, int32_t* legal) {
  *legal = transition_legal(static_cast<SideTaskState>(from), static_cast<TransitionKind>(kind));
  return FR_OK;
}

int fr_transition_target(int32_t from, int32_t kind, int32_t* to) {
  return guard([&]() -> int {
    *to = static_cast<int32_t>(
        transition_target(static_cast<SideTaskState>(from), static_cast<TransitionKind>(kind)));
    return FR_OK;
  });
}

int fr_apply_transition(fr_task_runtime* r, int32_t kind, fr_tick now) {
  return guard([&]() -> int {
    SideTaskRuntime rt = to_rt(r);
    apply_transition(rt, static_cast<TransitionKind>(kind), now);
    from_rt(rt, r);
    return FR_OK;
  });
}

int fr_iterative_run(const fr_task_runtime* r, fr_tick bubble_end, fr_tick now, double est,
                     double tick, fr_tick actual, fr_iterative_decision* out) {
  return guard([&]() -> int {
    auto d = iterative_run(to_rt(r), bubble_end, now, est, tick, actual);
    out->run = d.run;
    out->reserved = 0;
    out->step_end = d.step_end;
    return FR_OK;
  });
}

int fr_imperative_run(const fr_task_runtime* r, fr_tick now, fr_tick actual, fr_tick* end) {
  *end = imperative_run(to_rt(r), now, actual);
  return FR_OK;
}

int fr_limit_config_validate(const fr_limit_config* c) {
  return guard([&]() -> int {
    LimitConfig l;
    l.grace_period = c->grace_period;
    l.memory_headroom = c->memory_headroom;
    l.reclamation_delay = c->reclamation_delay;
    l.validate();
    return FR_OK;
  });
}

int fr_check_memory(double alloc, double limit, int32_t* result) {
  *result = static_cast<int32_t>(check_memory(alloc, limit));
  return FR_OK;
}

int fr_program_directed_gate(double remaining, double est, int32_t* gate) {
  *gate = static_cast<int32_t>(program_directed_gate(remaining, est));
  return FR_OK;
}

int fr_framework_enforce(int32_t has_lp, fr_tick lp, fr_tick issued, fr_tick now,
                         fr_tick grace, int32_t* result) {
  std::optional<Tick> last;
  if (has_lp) last = lp;
  *result = static_cast<int32_t>(framework_enforce(last, issued, now, grace));
  return FR_OK;
}

uint64_t fr_stream_seed(uint64_t seed, const char* task_id, const char* salt) {
  return stream_seed(seed, task_id, salt);
}

fr_tick fr_jittered_step_ticks(fr_tick base, double jitter, uint64_t* rng) {
  std::uint64_t s = *rng;
  Tick t = jittered_step_ticks(base, jitter, s);
  *rng = s;
  return t;
}

int fr_profile_task(const fr_side_task_spec* spec, const fr_profile_options* o, uint64_t seed,
                    fr_task_profile* out) {
  return guard([&]() -> int {
    ProfileOptions opts;
    opts.n_steps = o->n_steps;
    opts.step_jitter = o->step_jitter;
    opts.tick_seconds = o->tick_seconds;
    TaskProfile p = profile_task(to_spec(spec), opts, seed);
    std::memset(out, 0, sizeof(*out));
    copy_id(out->task_id, p.task_id);
    out->has_est_per_step = p.est_per_step_duration.has_value();
    out->profiled_steps = p.profiled_steps;
    out->est_per_step_duration = p.est_per_step_duration.value_or(0.0);
    out->max_per_step_duration = p.max_per_step_duration.value_or(0.0);
    out->est_memory = p.est_memory;
    return FR_OK;
  });
}

int fr_profile_bubbles(const fr_pipeline_config* cfg, fr_tick* durations, int64_t cap,
                       int64_t* offsets, double* avail, double* rate) {
  return guard([&]() -> int {
    BubbleProfile bp = profile_bubbles(to_cfg(cfg));
    int64_t n = 0;
    for (auto& s : bp.stages) n += static_cast<int64_t>(s.durations.size());
    offsets[bp.stages.size()] = n;
    if (n > cap) return fail(FR_ERR_CAPACITY, "capacity");
    int64_t k = 0;
    for (size_t s = 0; s < bp.stages.size(); ++s) {
      offsets[s] = k;
      avail[s] = bp.stages[s].available_memory;
      for (Tick d : bp.stages[s].durations) durations[k++] = d;
    }
    *rate = bp.rate;
    return FR_OK;
  });
}

int fr_manager_create(int32_t n, const double* mem, fr_manager** out) {
  auto* m = new fr_manager;
  m->workers.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    m->workers[i].worker_id = i;
    m->workers[i].gpu_mem = mem[i];
  }
  *out = m;
  return FR_OK;
}

void fr_manager_destroy(fr_manager* m) { delete m; }

int fr_manager_worker_info(const fr_manager* m, int32_t w, fr_worker_info* out) {
  if (w < 0 || w >= static_cast<int32_t>(m->workers.size()))
    return fail(FR_ERR_NOT_FOUND, "worker");
  const WorkerState& ws = m->workers[w];
  std::memset(out, 0, sizeof(*out));
  out->worker_id = ws.worker_id;
  out->queue_len = static_cast<int32_t>(ws.task_queue.size());
  out->has_current_task = ws.current_task.has_value();
  if (ws.current_task) copy_id(out->current_task, *ws.current_task);
  out->has_current_bubble = ws.current_bubble.has_value();
  if (ws.current_bubble) out->current_bubble = to_c(*ws.current_bubble, -1, -1);
  out->gpu_mem = ws.gpu_mem;
  return FR_OK;
}

int fr_manager_queue_at(const fr_manager* m, int32_t w, int32_t i, char* buf, int32_t cap) {
  if (w < 0 || w >= static_cast<int32_t>(m->workers.size()))
    return fail(FR_ERR_NOT_FOUND, "worker");
  const auto& q = m->workers[w].task_queue;
  if (i < 0 || i >= static_cast<int32_t>(q.size())) return fail(FR_ERR_NOT_FOUND, "index");
  if (static_cast<int32_t>(q[i].size()) + 1 > cap) return fail(FR_ERR_CAPACITY, "capacity");
  std::memcpy(buf, q[i].c_str(), q[i].size() + 1);
  return FR_OK;
}

int fr_manager_set_current_task(fr_manager* m, int32_t w, const char* id) {
  if (w < 0 || w >= static_cast<int32_t>(m->workers.size()))
    return fail(FR_ERR_NOT_FOUND, "worker");
  if (id)
    m->workers[w].current_task = std::string(id);
  else
    m->workers[w].current_task.reset();
  return FR_OK;
}

int fr_select_worker(const fr_manager* m, double task_memory, int32_t* worker) {
  auto s = select_worker(task_memory, m->workers);
  *worker = s ? *s : -1;
  return FR_OK;
}

int fr_submit_task(fr_manager* m, const fr_task_profile* p, int32_t* assigned, int32_t* wid) {
  TaskProfile tp;
  tp.task_id = std::string(p->task_id, strnlen(p->task_id, FR_TASK_ID_MAX));
  tp.est_memory = p->est_memory;
  tp.profiled_steps = p->profiled_steps;
  SubmitOutcome o = submit_task(tp, m->workers);
  *assigned = o.assigned;
  *wid = o.worker_id;
  return FR_OK;
}

static TaskLookup make_lookup(fr_task_lookup_fn fn, void* ctx) {
  return [fn, ctx](const std::string& id) {
    fr_task_view v{};
    int rc = fn(ctx, id.c_str(), &v);
    if (rc != FR_OK) throw CallbackError(rc);
    TaskView tv;
    tv.state = static_cast<SideTaskState>(v.state);
    tv.initializing = v.initializing != 0;
    return tv;
  };
}

static int emit_actions(const std::vector<ManagerAction>& acts, fr_manager_action* out,
                        int32_t cap, int32_t* n_out) {
  *n_out = static_cast<int32_t>(acts.size());
  if (*n_out > cap) return fail(FR_ERR_CAPACITY, "capacity");
  for (size_t i = 0; i < acts.size(); ++i) {
    out[i].kind = static_cast<int32_t>(acts[i].kind);
    copy_id(out[i].task_id, acts[i].task_id);
  }
  return FR_OK;
}

int fr_on_bubble_started(fr_manager* m, int32_t w, const fr_bubble* b, fr_task_lookup_fn fn,
                         void* ctx, fr_manager_action* out, int32_t cap, int32_t* n_out) {
  if (w < 0 || w >= static_cast<int32_t>(m->workers.size()))
    return fail(FR_ERR_NOT_FOUND, "worker");
  return guard([&]() -> int {
    auto acts = on_bubble_started(m->workers[w], from_c(*b), make_lookup(fn, ctx));
    return emit_actions(acts, out, cap, n_out);
  });
}

int fr_on_bubble_ended(fr_manager* m, int32_t w, fr_tick now, fr_task_lookup_fn fn, void* ctx,
                       fr_manager_action* out, int32_t cap, int32_t* n_out) {
  if (w < 0 || w >= static_cast<int32_t>(m->workers.size()))
    return fail(FR_ERR_NOT_FOUND, "worker");
  return guard([&]() -> int {
    auto acts = on_bubble_ended(m->workers[w], now, make_lookup(fn, ctx));
    return emit_actions(acts, out, cap, n_out);
  });
}

int fr_time_increase(double t_no, double t_with, double* out) {
  return guard([&]() -> int {
    *out = time_increase(t_no, t_with);
    return FR_OK;
  });
}

int fr_cost_savings(double t_no, double dt, const fr_task_work* work, int32_t n,
                    const fr_price_config* prices, fr_cost_breakdown* out) {
  return guard([&]() -> int {
    std::vector<TaskWork> w;
    for (int i = 0; i < n; ++i) {
      TaskWork tw;
      tw.id = std::string(work[i].id, strnlen(work[i].id, FR_TASK_ID_MAX));
      tw.work = work[i].work;
      if (work[i].has_throughput) tw.throughput_per_hour = work[i].throughput_per_hour;
      w.push_back(tw);
    }
    PriceConfig pc;
    pc.price_server_1 = prices->price_server_1;
    pc.price_server_2 = prices->price_server_2;
    CostBreakdown cb = cost_savings(t_no, dt, w, pc);
    out->c_no_side = cb.c_no_side;
    out->c_extra = cb.c_extra;
    out->c_side_tasks = cb.c_side_tasks;
    out->s = cb.s;
    return FR_OK;
  });
}

int fr_bubble_breakdown(const fr_breakdown_input* in, fr_stage_breakdown* out) {
  return guard([&]() -> int {
    RunTrace t;
    t.meta.config.pipeline.num_stages = in->num_stages;
    for (int i = 0; i < in->n_profiles; ++i) {
      TaskProfile tp;
      tp.task_id = in->profiles[i].task_id;
      tp.est_memory = in->profiles[i].est_memory;
      t.meta.profiles.push_back(tp);
    }
    for (int64_t i = 0; i < in->n_bubbles; ++i) t.bubbles.push_back(from_c(in->bubbles[i]));
    for (int64_t i = 0; i < in->n_assigns; ++i) {
      AssignRecord a;
      a.t = in->assigns[i].t;
      a.task = in->assigns[i].task;
      a.worker = in->assigns[i].worker;
      t.assigns.push_back(a);
    }
    for (int64_t i = 0; i < in->n_transitions; ++i) {
      TransitionRecord r;
      r.t = in->transitions[i].t;
      r.task = in->transitions[i].task;
      r.kind = static_cast<TransitionKind>(in->transitions[i].kind);
      r.worker = in->transitions[i].worker;
      t.transitions.push_back(r);
    }
    for (int64_t i = 0; i < in->n_activities; ++i) {
      ActivityRecord a;
      a.start = in->activities[i].start;
      a.end = in->activities[i].end;
      a.task = in->activities[i].task;
      a.worker = in->activities[i].worker;
      a.kind = static_cast<ActivityKind>(in->activities[i].kind);
      a.clipped = in->activities[i].clipped != 0;
      t.activities.push_back(a);
    }
    auto bd = bubble_breakdown(t);
    for (size_t s = 0; s < bd.size(); ++s) {
      out[s].stage = bd[s].stage;
      out[s].reserved = 0;
      out[s].used_by_side_tasks = bd[s].used_by_side_tasks;
      out[s].runtime_overhead = bd[s].runtime_overhead;
      out[s].idle_oom = bd[s].idle_oom;
      out[s].idle_insufficient_time = bd[s].idle_insufficient_time;
    }
    return FR_OK;
  });
}

}  // extern "C"
