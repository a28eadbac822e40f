// C-ABI of the simulated dispatch engine (fr_run_experiment and the RunTrace
// getters).
#include <algorithm>
#include <cstring>
#include <memory>

#include "capi_util.hpp"
#include "freeride.h"
#include "host/freeride.hpp"
#include "host/io.hpp"

using namespace freeride;

#include "run_trace.hpp"

namespace {

PipelineConfig cfg_in(const fr_pipeline_config* c) {
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

SideTaskSpec spec_in(const fr_side_task_spec* s) {
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

template <class V>
int sized(const V& v, int64_t cap) {
  if (static_cast<int64_t>(v.size()) > cap) return frcapi::fail(FR_ERR_CAPACITY, "record buffer too small");
  return FR_OK;
}

}  // namespace

extern "C" {

int fr_run_experiment(const fr_experiment_config* c, int32_t with_tasks, uint64_t seed,
                      fr_run_trace** out) {
  if (!c || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    ExperimentConfig ec;
    ec.pipeline = cfg_in(&c->pipeline);
    for (int i = 0; i < c->n_tasks; ++i) ec.tasks.push_back(spec_in(&c->tasks[i]));
    ec.limits.grace_period = c->limits.grace_period;
    ec.limits.memory_headroom = c->limits.memory_headroom;
    ec.limits.reclamation_delay = c->limits.reclamation_delay;
    ec.limits.validate();
    ec.runtime.check_overhead = c->runtime.check_overhead;
    ec.runtime.rpc_latency = c->runtime.rpc_latency;
    ec.runtime.step_jitter = c->runtime.step_jitter;
    ec.runtime.profile_steps = c->runtime.profile_steps;
    ec.runtime.gate_estimate = static_cast<GateEstimate>(c->runtime.gate_estimate);
    if (ec.runtime.check_overhead < 0) throw ValidationError("runtime.check_overhead", "must be >= 0");
    if (ec.runtime.rpc_latency < 0) throw ValidationError("runtime.rpc_latency", "must be >= 0");
    if (ec.runtime.profile_steps < 1) throw ValidationError("runtime.profile_steps", "must be >= 1");
    ec.seed = seed;
    auto tr = std::make_unique<fr_run_trace>();
    tr->t = run_experiment(ec, with_tasks != 0, seed);
    *out = tr.release();
    return FR_OK;
  });
}

void fr_run_trace_destroy(fr_run_trace* t) { delete t; }

int fr_run_trace_get_counts(const fr_run_trace* t, fr_run_trace_counts* o) {
  if (!t || !o) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  const RunTrace& r = t->t;
  *o = fr_run_trace_counts{static_cast<int64_t>(r.ops.size()), static_cast<int64_t>(r.bubbles.size()),
                           static_cast<int64_t>(r.submits.size()), static_cast<int64_t>(r.assigns.size()),
                           static_cast<int64_t>(r.rejects.size()), static_cast<int64_t>(r.rpcs.size()),
                           static_cast<int64_t>(r.transitions.size()), static_cast<int64_t>(r.activities.size()),
                           static_cast<int64_t>(r.kills.size()), static_cast<int64_t>(r.dispositions.size()),
                           r.makespan};
  return FR_OK;
}

int fr_run_trace_ops(const fr_run_trace* t, fr_op_event* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  if (sized(t->t.ops, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < t->t.ops.size(); ++i) {
    const OpEvent& o = t->t.ops[i];
    out[i] = fr_op_event{o.stage, static_cast<int32_t>(o.kind), o.micro_batch, o.epoch, o.start, o.end};
  }
  return FR_OK;
}

int fr_run_trace_bubbles(const fr_run_trace* t, fr_bubble* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  if (sized(t->t.bubbles, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < t->t.bubbles.size(); ++i) out[i] = frcapi::bubble_out(t->t.bubbles[i], -1, -1);
  return FR_OK;
}

int fr_run_trace_assigns(const fr_run_trace* t, int32_t which, fr_assign_record* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  const auto& v = which == 0 ? t->t.submits : which == 1 ? t->t.assigns : t->t.rejects;
  if (sized(v, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[i] = fr_assign_record{v[i].t, v[i].worker, 0, {}};
    frcapi::copy_id(out[i].task, v[i].task);
  }
  return FR_OK;
}

int fr_run_trace_transitions(const fr_run_trace* t, int32_t which, fr_transition_record* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  const auto& v = which == 0 ? t->t.transitions : t->t.rpcs;
  if (sized(v, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[i] = fr_transition_record{v[i].t, static_cast<int32_t>(v[i].kind), v[i].worker, {}};
    frcapi::copy_id(out[i].task, v[i].task);
  }
  return FR_OK;
}

int fr_run_trace_activities(const fr_run_trace* t, fr_activity_record* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  const auto& v = t->t.activities;
  if (sized(v, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[i] = fr_activity_record{v[i].start, v[i].end, v[i].worker, static_cast<int32_t>(v[i].kind),
                                v[i].clipped ? 1 : 0, 0, {}};
    frcapi::copy_id(out[i].task, v[i].task);
  }
  return FR_OK;
}

int fr_run_trace_kills(const fr_run_trace* t, fr_kill_record* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  const auto& v = t->t.kills;
  if (sized(v, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[i] = fr_kill_record{v[i].t, v[i].worker, static_cast<int32_t>(v[i].reason), {}};
    frcapi::copy_id(out[i].task, v[i].task);
  }
  return FR_OK;
}

int fr_run_trace_dispositions(const fr_run_trace* t, fr_disposition_record* out, int64_t cap) {
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null trace");
  const auto& v = t->t.dispositions;
  if (sized(v, cap)) return FR_ERR_CAPACITY;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[i] = fr_disposition_record{static_cast<int32_t>(v[i].disposition), v[i].worker.has_value(),
                                   v[i].worker.value_or(-1), 0, v[i].steps_completed, {}};
    frcapi::copy_id(out[i].task, v[i].task);
  }
  return FR_OK;
}

int fr_run_trace_check(const fr_run_trace* t, char* buf, int64_t cap, int32_t* n) {
  if (!t || !n) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    const std::vector<std::string> v = replay_check(t->t);
    *n = static_cast<int32_t>(v.size());
    if (buf && cap > 0) {
      std::string all;
      for (const auto& s : v) all += s + "\n";
      const std::size_t k = std::min<std::size_t>(all.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, all.data(), k);
      buf[k] = 0;
    }
    return FR_OK;
  });
}

int fr_run_trace_write_jsonl(const fr_run_trace* t, const char* path) {
  if (!t || !path) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    write_trace_file(t->t, path);
    return FR_OK;
  });
}

int fr_run_trace_read_jsonl(const char* path, fr_run_trace** out) {
  if (!path || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  return frcapi::guard([&]() -> int {
    auto tr = std::make_unique<fr_run_trace>();
    tr->t = read_trace_file(path);
    *out = tr.release();
    return FR_OK;
  });
}

}  // extern "C"
