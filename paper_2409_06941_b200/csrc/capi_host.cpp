// C-ABI (include/freeride.h) over the product's C++ host core.  No exception
// crosses this boundary: each entry point maps the reference's exception
// types onto status codes and records message + field thread-locally.
#include <cstring>
#include <string>
#include <vector>

#include "freeride.h"
#include "host/freeride.hpp"
#include "capi_util.hpp"

using namespace freeride;

namespace frcapi {
std::string& last_error() {
  thread_local std::string s;
  return s;
}
std::string& last_field() {
  thread_local std::string s;
  return s;
}
}  // namespace frcapi

namespace {

PipelineConfig to_cfg(const fr_pipeline_config* c) {
  PipelineConfig cfg;
  cfg.num_stages = c->num_stages;
  cfg.num_micro_batches = c->num_micro_batches;
  cfg.num_epochs = c->num_epochs;
  if (c->fp_duration) cfg.fp_duration.assign(c->fp_duration, c->fp_duration + c->n_fp);
  if (c->bp_duration) cfg.bp_duration.assign(c->bp_duration, c->bp_duration + c->n_bp);
  if (c->stage_memory) cfg.stage_memory.assign(c->stage_memory, c->stage_memory + c->n_stage_memory);
  cfg.gpu_memory_total = c->gpu_memory_total;
  cfg.tick_seconds = c->tick_seconds;
  return cfg;
}

fr_op_event op_out(const OpEvent& o) {
  return fr_op_event{o.stage, static_cast<int32_t>(o.kind), o.micro_batch, o.epoch, o.start, o.end};
}

OpEvent op_in(const fr_op_event& c) {
  OpEvent o;
  o.stage = c.stage;
  o.kind = static_cast<OpKind>(c.kind);
  o.micro_batch = c.micro_batch;
  o.epoch = c.epoch;
  o.start = c.start;
  o.end = c.end;
  return o;
}

std::string id_in(const char* s) { return std::string(s, strnlen(s, FR_TASK_ID_MAX)); }

SideTaskSpec spec_in(const fr_side_task_spec* s) {
  SideTaskSpec spec;
  spec.id = id_in(s->id);
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

SideTaskRuntime rt_in(const fr_task_runtime* r) {
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

void rt_out(const SideTaskRuntime& rt, fr_task_runtime* r) {
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

bool valid_state(int32_t s) { return s >= 0 && s <= 4; }
bool valid_kind(int32_t k) { return k >= 0 && k <= 5; }

}  // namespace

struct fr_manager {
  std::vector<WorkerState> workers;
};

extern "C" {

int fr_abi_version(void) { return FR_ABI_VERSION; }
const char* fr_last_error(void) { return frcapi::last_error().c_str(); }
const char* fr_last_error_field(void) { return frcapi::last_field().c_str(); }

int fr_pipeline_validate(const fr_pipeline_config* cfg) {
  if (!cfg) return frcapi::fail(FR_ERR_ARGUMENT, "null config");
  return frcapi::guard([&]() -> int {
    to_cfg(cfg).validate();
    return FR_OK;
  });
}

int fr_stage_issue_order(int32_t stage, int32_t p, int32_t m, fr_issue* out, int64_t cap,
                         int64_t* n_out) {
  return frcapi::guard([&]() -> int {
    const auto seq = stage_issue_order(stage, p, m);
    *n_out = static_cast<int64_t>(seq.size());
    if (*n_out > cap) return frcapi::fail(FR_ERR_CAPACITY, "issue order needs 2*m entries");
    for (std::size_t i = 0; i < seq.size(); ++i)
      out[i] = fr_issue{static_cast<int32_t>(seq[i].first), seq[i].second};
    return FR_OK;
  });
}

int fr_build_schedule(const fr_pipeline_config* cfg, fr_op_event* ops, int64_t cap,
                      int64_t* n_ops, fr_tick* spans) {
  if (!cfg || !n_ops) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    const ScheduleTrace t = build_schedule(to_cfg(cfg));
    *n_ops = static_cast<int64_t>(t.ops.size());
    if (*n_ops > cap) return frcapi::fail(FR_ERR_CAPACITY, "schedule needs 2*p*m*epochs ops");
    for (std::size_t i = 0; i < t.ops.size(); ++i) ops[i] = op_out(t.ops[i]);
    for (std::size_t e = 0; e < t.epoch_spans.size(); ++e) {
      spans[2 * e] = t.epoch_spans[e].first;
      spans[2 * e + 1] = t.epoch_spans[e].second;
    }
    return FR_OK;
  });
}

int fr_extract_bubbles(const fr_pipeline_config* cfg, const fr_op_event* ops, int64_t n_ops,
                       const fr_tick* spans, fr_bubble* out, int64_t cap, int64_t* n_out) {
  if (!cfg || !n_out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (n_ops < 0 || cap < 0) return frcapi::fail(FR_ERR_VALIDATION, "counts must be >= 0", n_ops < 0 ? "n_ops" : "cap");
  if ((n_ops > 0 && !ops) || !spans || (cap > 0 && !out)) return frcapi::fail(FR_ERR_ARGUMENT, "null buffer");
  return frcapi::guard([&]() -> int {
    ScheduleTrace t;
    t.config = to_cfg(cfg);
    t.config.validate();  // num_epochs >= 1 bounds the reads of spans
    t.ops.reserve(static_cast<std::size_t>(n_ops));
    for (int64_t i = 0; i < n_ops; ++i) t.ops.push_back(op_in(ops[i]));
    for (int e = 0; e < cfg->num_epochs; ++e) t.epoch_spans.push_back({spans[2 * e], spans[2 * e + 1]});
    const auto lb = extract_bubbles_linked(t);
    *n_out = static_cast<int64_t>(lb.size());
    if (*n_out > cap) return frcapi::fail(FR_ERR_CAPACITY, "bubble buffer too small");
    for (std::size_t i = 0; i < lb.size(); ++i) out[i] = frcapi::bubble_out(lb[i].bubble, lb[i].prev_op, lb[i].next_op);
    return FR_OK;
  });
}

int fr_bubble_rate(int32_t p, const fr_op_event* ops, int64_t n_ops, const fr_bubble* b,
                   int64_t nb, double* rate) {
  if (!rate || (n_ops > 0 && !ops) || (nb > 0 && !b)) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    std::vector<OpEvent> o;
    for (int64_t i = 0; i < n_ops; ++i) o.push_back(op_in(ops[i]));
    std::vector<Bubble> bs;
    for (int64_t i = 0; i < nb; ++i) bs.push_back(frcapi::bubble_in(b[i]));
    *rate = bubble_rate(p, o.data(), o.size(), bs.data(), bs.size());
    return FR_OK;
  });
}

int fr_default_stage_memory(int32_t p, double total, double w, double a, double* out) {
  return frcapi::guard([&]() -> int {
    const auto v = default_stage_memory(p, total, w, a);
    std::copy(v.begin(), v.end(), out);
    return FR_OK;
  });
}

int fr_pipeline_p2p_plan(int32_t stage, int32_t p, int32_t m, fr_p2p_op* out, int64_t cap,
                         int64_t* n_out) {
  if (!n_out) return frcapi::fail(FR_ERR_ARGUMENT, "null count");
  return frcapi::guard([&]() -> int {
    const auto plan = pipeline_p2p_plan(stage, p, m);
    *n_out = static_cast<int64_t>(plan.size());
    if (*n_out > cap) return frcapi::fail(FR_ERR_CAPACITY, "p2p plan needs up to 4*m entries");
    for (std::size_t i = 0; i < plan.size(); ++i)
      out[i] = fr_p2p_op{plan[i].group, plan[i].is_send ? 1 : 0, plan[i].peer,
                         static_cast<int32_t>(plan[i].kind), plan[i].micro_batch};
    return FR_OK;
  });
}

int fr_side_task_validate(const fr_side_task_spec* spec, const char* path) {
  return frcapi::guard([&]() -> int {
    spec_in(spec).validate(path ? path : "");
    return FR_OK;
  });
}

int fr_transition_legal(int32_t from, int32_t kind, int32_t* legal) {
  *legal = valid_state(from) && valid_kind(kind) &&
           transition_legal(static_cast<SideTaskState>(from), static_cast<TransitionKind>(kind));
  return FR_OK;
}

int fr_transition_target(int32_t from, int32_t kind, int32_t* to) {
  return frcapi::guard([&]() -> int {
    *to = static_cast<int32_t>(
        transition_target(static_cast<SideTaskState>(from), static_cast<TransitionKind>(kind)));
    return FR_OK;
  });
}

int fr_apply_transition(fr_task_runtime* r, int32_t kind, fr_tick now) {
  if (!r) return frcapi::fail(FR_ERR_ARGUMENT, "null runtime");
  return frcapi::guard([&]() -> int {
    SideTaskRuntime rt = rt_in(r);
    apply_transition(rt, static_cast<TransitionKind>(kind), now);
    rt_out(rt, r);
    return FR_OK;
  });
}

int fr_iterative_run(const fr_task_runtime* r, fr_tick bubble_end, fr_tick now, double est,
                     double tick, fr_tick actual, fr_iterative_decision* out) {
  const IterativeDecision d = iterative_run(rt_in(r), bubble_end, now, est, tick, actual);
  out->run = d.run;
  out->reserved = 0;
  out->step_end = d.step_end;
  return FR_OK;
}

int fr_imperative_run(const fr_task_runtime* r, fr_tick now, fr_tick actual, fr_tick* end) {
  *end = imperative_run(rt_in(r), now, actual);
  return FR_OK;
}

int fr_limit_config_validate(const fr_limit_config* c) {
  return frcapi::guard([&]() -> int {
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

int fr_framework_enforce(int32_t has_lp, fr_tick lp, fr_tick issued, fr_tick now, fr_tick grace,
                         int32_t* result) {
  *result = static_cast<int32_t>(
      framework_enforce(has_lp ? std::optional<Tick>(lp) : std::nullopt, issued, now, grace));
  return FR_OK;
}

uint64_t fr_stream_seed(uint64_t seed, const char* task_id, const char* salt) {
  return stream_seed(seed, task_id ? task_id : "", salt ? salt : "");
}

fr_tick fr_jittered_step_ticks(fr_tick base, double jitter, uint64_t* rng) {
  std::uint64_t s = *rng;
  const Tick t = jittered_step_ticks(base, jitter, s);
  *rng = s;
  return t;
}

int fr_profile_task(const fr_side_task_spec* spec, const fr_profile_options* o, uint64_t seed,
                    fr_task_profile* out) {
  return frcapi::guard([&]() -> int {
    ProfileOptions opts;
    opts.n_steps = o->n_steps;
    opts.step_jitter = o->step_jitter;
    opts.tick_seconds = o->tick_seconds;
    const TaskProfile p = profile_task(spec_in(spec), opts, seed);
    frcapi::profile_out(p, out);
    return FR_OK;
  });
}

int fr_profile_bubbles(const fr_pipeline_config* cfg, fr_tick* durations, int64_t cap,
                       int64_t* offsets, double* avail, double* rate) {
  return frcapi::guard([&]() -> int {
    const BubbleProfile bp = profile_bubbles(to_cfg(cfg));
    int64_t n = 0;
    for (const auto& s : bp.stages) n += static_cast<int64_t>(s.durations.size());
    offsets[bp.stages.size()] = n;
    if (n > cap) return frcapi::fail(FR_ERR_CAPACITY, "duration buffer too small");
    int64_t k = 0;
    for (std::size_t s = 0; s < bp.stages.size(); ++s) {
      offsets[s] = k;
      avail[s] = bp.stages[s].available_memory;
      for (Tick d : bp.stages[s].durations) durations[k++] = d;
    }
    *rate = bp.rate;
    return FR_OK;
  });
}

int fr_manager_create(int32_t n, const double* mem, fr_manager** out) {
  if (n < 0 || (!mem && n > 0) || !out) return frcapi::fail(FR_ERR_ARGUMENT, "bad manager args");
  auto* m = new fr_manager;
  m->workers.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    m->workers[i].worker_id = i;
    m->workers[i].gpu_mem = mem[i];
  }
  *out = m;
  return FR_OK;
}

void fr_manager_destroy(fr_manager* m) { delete m; }

static WorkerState* worker_of(const fr_manager* m, int32_t w) {
  if (!m || w < 0 || w >= static_cast<int32_t>(m->workers.size())) return nullptr;
  return const_cast<WorkerState*>(&m->workers[static_cast<std::size_t>(w)]);
}

int fr_manager_worker_info(const fr_manager* m, int32_t w, fr_worker_info* out) {
  const WorkerState* ws = worker_of(m, w);
  if (!ws) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker");
  std::memset(out, 0, sizeof(*out));
  out->worker_id = ws->worker_id;
  out->queue_len = static_cast<int32_t>(ws->task_queue.size());
  out->has_current_task = ws->current_task.has_value();
  if (ws->current_task) frcapi::copy_id(out->current_task, *ws->current_task);
  out->has_current_bubble = ws->current_bubble.has_value();
  if (ws->current_bubble) out->current_bubble = frcapi::bubble_out(*ws->current_bubble, -1, -1);
  out->gpu_mem = ws->gpu_mem;
  return FR_OK;
}

int fr_manager_queue_at(const fr_manager* m, int32_t w, int32_t i, char* buf, int32_t cap) {
  const WorkerState* ws = worker_of(m, w);
  if (!ws) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker");
  if (i < 0 || i >= static_cast<int32_t>(ws->task_queue.size()))
    return frcapi::fail(FR_ERR_NOT_FOUND, "queue index out of range");
  const std::string& id = ws->task_queue[static_cast<std::size_t>(i)];
  if (static_cast<int32_t>(id.size()) + 1 > cap) return frcapi::fail(FR_ERR_CAPACITY, "id buffer");
  std::memcpy(buf, id.c_str(), id.size() + 1);
  return FR_OK;
}

int fr_manager_push_task(fr_manager* m, int32_t w, const char* id) {
  WorkerState* ws = worker_of(m, w);
  if (!ws || !id) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker / null id");
  ws->task_queue.push_back(id_in(id));
  return FR_OK;
}

int fr_manager_set_current_task(fr_manager* m, int32_t w, const char* id) {
  WorkerState* ws = worker_of(m, w);
  if (!ws) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker");
  if (id)
    ws->current_task = id_in(id);
  else
    ws->current_task.reset();
  return FR_OK;
}

int fr_select_worker(const fr_manager* m, double task_memory, int32_t* worker) {
  if (!m) return frcapi::fail(FR_ERR_ARGUMENT, "null manager");
  const auto s = select_worker(task_memory, m->workers);
  *worker = s ? *s : -1;
  return FR_OK;
}

int fr_submit_task(fr_manager* m, const fr_task_profile* p, int32_t* assigned, int32_t* wid) {
  if (!m || !p) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  TaskProfile tp = frcapi::profile_in(p);
  const SubmitOutcome o = submit_task(tp, m->workers);
  *assigned = o.assigned;
  *wid = o.worker_id;
  return FR_OK;
}

int fr_on_bubble_started(fr_manager* m, int32_t w, const fr_bubble* b, fr_task_lookup_fn fn,
                         void* ctx, fr_manager_action* out, int32_t cap, int32_t* n_out) {
  WorkerState* ws = worker_of(m, w);
  if (!ws) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker");
  return frcapi::guard([&]() -> int {
    const auto acts = on_bubble_started(*ws, frcapi::bubble_in(*b), frcapi::lookup_of(fn, ctx));
    return frcapi::actions_out(acts, out, cap, n_out);
  });
}

int fr_on_bubble_ended(fr_manager* m, int32_t w, fr_tick now, fr_task_lookup_fn fn, void* ctx,
                       fr_manager_action* out, int32_t cap, int32_t* n_out) {
  WorkerState* ws = worker_of(m, w);
  if (!ws) return frcapi::fail(FR_ERR_NOT_FOUND, "no such worker");
  return frcapi::guard([&]() -> int {
    const auto acts = on_bubble_ended(*ws, now, frcapi::lookup_of(fn, ctx));
    return frcapi::actions_out(acts, out, cap, n_out);
  });
}

int fr_time_increase(double t_no, double t_with, double* out) {
  return frcapi::guard([&]() -> int {
    *out = time_increase(t_no, t_with);
    return FR_OK;
  });
}

int fr_cost_savings(double t_no, double dt, const fr_task_work* work, int32_t n,
                    const fr_price_config* prices, fr_cost_breakdown* out) {
  return frcapi::guard([&]() -> int {
    std::vector<TaskWork> w;
    for (int i = 0; i < n; ++i) {
      TaskWork tw;
      tw.id = id_in(work[i].id);
      tw.work = work[i].work;
      if (work[i].has_throughput) tw.throughput_per_hour = work[i].throughput_per_hour;
      w.push_back(std::move(tw));
    }
    PriceConfig pc;
    pc.price_server_1 = prices->price_server_1;
    pc.price_server_2 = prices->price_server_2;
    const CostBreakdown cb = cost_savings(t_no, dt, w, pc);
    *out = fr_cost_breakdown{cb.c_no_side, cb.c_extra, cb.c_side_tasks, cb.s};
    return FR_OK;
  });
}

int fr_bubble_breakdown(const fr_breakdown_input* in, fr_stage_breakdown* out) {
  if (!in || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    BreakdownInput bi;
    bi.num_stages = in->num_stages;
    for (int i = 0; i < in->n_profiles; ++i) bi.profiles.push_back(frcapi::profile_in(&in->profiles[i]));
    for (int64_t i = 0; i < in->n_bubbles; ++i) bi.bubbles.push_back(frcapi::bubble_in(in->bubbles[i]));
    for (int64_t i = 0; i < in->n_assigns; ++i)
      bi.assigns.push_back({in->assigns[i].t, id_in(in->assigns[i].task), in->assigns[i].worker});
    for (int64_t i = 0; i < in->n_transitions; ++i)
      bi.transitions.push_back({in->transitions[i].t, id_in(in->transitions[i].task),
                                static_cast<TransitionKind>(in->transitions[i].kind),
                                in->transitions[i].worker});
    for (int64_t i = 0; i < in->n_activities; ++i) {
      const fr_activity_record& a = in->activities[i];
      bi.activities.push_back({a.start, a.end, id_in(a.task), a.worker,
                               static_cast<ActivityKind>(a.kind), a.clipped != 0});
    }
    const auto bd = bubble_breakdown(bi);
    for (std::size_t s = 0; s < bd.size(); ++s)
      out[s] = fr_stage_breakdown{bd[s].stage, 0, bd[s].used_by_side_tasks, bd[s].runtime_overhead,
                                  bd[s].idle_oom, bd[s].idle_insufficient_time};
    return FR_OK;
  });
}

}  // extern "C"
