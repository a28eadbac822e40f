// Experiment config <-> JSON (reference config.hpp:19-56; schema SPEC.md:525,
// DESIGN.md §6b).
#include <fstream>
#include <sstream>

#include "io.hpp"

// json::need / get_* return references into the document, never into their
// (temporary) path argument; GCC 13's heuristic cannot see that.
#pragma GCC diagnostic ignored "-Wdangling-reference"

namespace freeride {

namespace {

using json::Value;

Tick ticks(const Value& v, double tick, const std::string& path) {
  return seconds_to_ticks(json::get_number(v, path), tick, path.substr(path.find('.') + 1));
}

Value secs(Tick t, double tick) { return Value::number(ticks_to_seconds(t, tick)); }

const Value* opt(const Value& obj, const char* key) {
  const Value* v = obj.find(key);
  return v && !v->is_null() ? v : nullptr;
}

template <class F>
void each(const Value& arr, const std::string& path, F f) {
  const auto& a = json::get_array(arr, path);
  for (std::size_t k = 0; k < a.size(); ++k) f(a[k], path + "[" + std::to_string(k) + "]");
}

const char* iface_name(TaskInterface i) { return i == TaskInterface::Imperative ? "imperative" : "iterative"; }

}  // namespace

bool apply_model_preset(const std::string& name, int batch_size, PipelineConfig& p) {
  // Illustrative nanoGPT-like presets, per micro-batch of 4 sequences: larger
  // models leave less memory and shorter bubbles per stage (§2.2.1).
  struct Preset { const char* name; double fp, bp, weight, act; };
  static const Preset presets[] = {{"1.2B", 0.220, 0.347, 20.0, 6.5},
                                   {"3.6B", 0.200, 0.320, 28.0, 7.0},
                                   {"6B", 0.180, 0.300, 34.0, 7.5}};
  for (const Preset& pr : presets) {
    if (name != pr.name) continue;
    const double f = batch_size > 0 ? batch_size / 4.0 : 1.0;
    p.fp_duration = {seconds_to_ticks(pr.fp * f, p.tick_seconds, "sweep.batch_sizes")};
    p.bp_duration = {seconds_to_ticks(pr.bp * f, p.tick_seconds, "sweep.batch_sizes")};
    p.stage_memory = default_stage_memory(p.num_stages, p.gpu_memory_total, pr.weight, pr.act * f);
    return true;
  }
  return false;
}

void validate_experiment(const ExperimentConfig& c) {
  c.pipeline.validate();
  c.limits.validate();
  c.prices.validate();
  for (std::size_t k = 0; k < c.tasks.size(); ++k) {
    c.tasks[k].validate("tasks[" + std::to_string(k) + "]");
    for (std::size_t j = 0; j < k; ++j)
      if (c.tasks[j].id == c.tasks[k].id)
        throw ValidationError("tasks[" + std::to_string(k) + "].id", "duplicate task id");
  }
  if (c.runtime.check_overhead < 0) throw ValidationError("runtime.check_overhead", "must be >= 0");
  if (c.runtime.rpc_latency < 0) throw ValidationError("runtime.rpc_latency", "must be >= 0");
  if (c.runtime.profile_steps < 1) throw ValidationError("runtime.profile_steps", "must be >= 1");
  if (c.runtime.step_jitter < 0 || c.runtime.step_jitter >= 1)
    throw ValidationError("runtime.step_jitter", "must be in [0, 1)");
  if (c.sweep) {
    if (c.sweep->micro_batches.empty() && c.sweep->model_sizes.empty() && c.sweep->batch_sizes.empty())
      throw ValidationError("sweep", "a sweep needs at least one non-empty axis");
    for (int m : c.sweep->micro_batches)
      if (m < 1) throw ValidationError("sweep.micro_batches", "must be >= 1");
    for (int b : c.sweep->batch_sizes)
      if (b < 1) throw ValidationError("sweep.batch_sizes", "must be >= 1");
    PipelineConfig probe = c.pipeline;
    for (const auto& n : c.sweep->model_sizes)
      if (!apply_model_preset(n, 4, probe))
        throw ValidationError("sweep.model_sizes", "unknown preset '" + n + "' (1.2B, 3.6B, 6B)");
  }
}

ExperimentConfig experiment_from_json(const Value& doc) {
  ExperimentConfig c;
  if (doc.kind != Value::Kind::Object) throw SchemaError("$", "expected an object");
  const Value& pj = json::need(doc, "pipeline", "$");
  PipelineConfig& p = c.pipeline;
  p.num_stages = static_cast<int>(json::get_int(json::need(pj, "num_stages", "$.pipeline"), "$.pipeline.num_stages"));
  p.num_micro_batches = static_cast<int>(json::get_int(json::need(pj, "num_micro_batches", "$.pipeline"), "$.pipeline.num_micro_batches"));
  if (const Value* v = opt(pj, "num_epochs")) p.num_epochs = static_cast<int>(json::get_int(*v, "$.pipeline.num_epochs"));
  if (const Value* v = opt(pj, "tick_seconds")) p.tick_seconds = json::get_number(*v, "$.pipeline.tick_seconds");
  if (!(p.tick_seconds > 0)) throw ValidationError("pipeline.tick_seconds", "must be > 0");
  p.gpu_memory_total = json::get_number(json::need(pj, "gpu_memory_total", "$.pipeline"), "$.pipeline.gpu_memory_total");
  each(json::need(pj, "fp_duration", "$.pipeline"), "$.pipeline.fp_duration",
       [&](const Value& v, const std::string& path) { p.fp_duration.push_back(ticks(v, p.tick_seconds, path)); });
  each(json::need(pj, "bp_duration", "$.pipeline"), "$.pipeline.bp_duration",
       [&](const Value& v, const std::string& path) { p.bp_duration.push_back(ticks(v, p.tick_seconds, path)); });
  if (const Value* v = opt(pj, "stage_memory")) {
    each(*v, "$.pipeline.stage_memory",
         [&](const Value& x, const std::string& path) { p.stage_memory.push_back(json::get_number(x, path)); });
  } else {
    const Value& mm = json::need(pj, "memory_model", "$.pipeline");
    p.stage_memory = default_stage_memory(
        p.num_stages, p.gpu_memory_total,
        json::get_number(json::need(mm, "weight", "$.pipeline.memory_model"), "$.pipeline.memory_model.weight"),
        json::get_number(json::need(mm, "activation_per_microbatch", "$.pipeline.memory_model"),
                         "$.pipeline.memory_model.activation_per_microbatch"));
  }
  const double tick = p.tick_seconds;
  if (const Value* tj = opt(doc, "tasks")) {
    each(*tj, "$.tasks", [&](const Value& t, const std::string& path) {
      SideTaskSpec s;
      s.id = json::get_string(json::need(t, "id", path), path + ".id");
      if (const Value* v = opt(t, "interface")) {
        const std::string n = json::get_string(*v, path + ".interface");
        if (n == "iterative") s.interface_kind = TaskInterface::Iterative;
        else if (n == "imperative") s.interface_kind = TaskInterface::Imperative;
        else throw SchemaError(path + ".interface", "expected iterative | imperative");
      }
      s.per_step_duration = ticks(json::need(t, "per_step_duration", path), tick, path + ".per_step_duration");
      if (const Value* v = opt(t, "total_steps")) s.total_steps = json::get_int(*v, path + ".total_steps");
      if (const Value* v = opt(t, "init_duration")) s.init_duration = ticks(*v, tick, path + ".init_duration");
      s.memory_demand = json::get_number(json::need(t, "memory_demand", path), path + ".memory_demand");
      if (const Value* v = opt(t, "misbehavior")) {
        const std::string mp = path + ".misbehavior";
        const std::string k = json::get_string(json::need(*v, "kind", mp), mp + ".kind");
        if (k == "none") s.misbehavior.kind = MisbehaviorKind::None;
        else if (k == "ignores_pause") s.misbehavior.kind = MisbehaviorKind::IgnoresPause;
        else if (k == "memory_leak") {
          s.misbehavior.kind = MisbehaviorKind::MemoryLeak;
          s.misbehavior.leak_rate_gib_per_s = json::get_number(json::need(*v, "rate", mp), mp + ".rate");
        } else throw SchemaError(mp + ".kind", "expected none | ignores_pause | memory_leak");
      }
      if (const Value* v = opt(t, "submit_time")) s.submit_time = ticks(*v, tick, path + ".submit_time");
      if (const Value* v = opt(t, "memory_limit")) s.memory_limit = json::get_number(*v, path + ".memory_limit");
      if (const Value* v = opt(t, "reference_throughput"))
        s.reference_throughput = json::get_number(*v, path + ".reference_throughput");
      c.tasks.push_back(s);
    });
  }
  if (const Value* lj = opt(doc, "limits")) {
    if (const Value* v = opt(*lj, "grace_period")) c.limits.grace_period = ticks(*v, tick, "$.limits.grace_period");
    if (const Value* v = opt(*lj, "memory_headroom")) c.limits.memory_headroom = json::get_number(*v, "$.limits.memory_headroom");
    if (const Value* v = opt(*lj, "reclamation_delay")) c.limits.reclamation_delay = ticks(*v, tick, "$.limits.reclamation_delay");
  }
  if (const Value* pr = opt(doc, "prices")) {
    if (const Value* v = opt(*pr, "price_server_1")) c.prices.price_server_1 = json::get_number(*v, "$.prices.price_server_1");
    if (const Value* v = opt(*pr, "price_server_2")) c.prices.price_server_2 = json::get_number(*v, "$.prices.price_server_2");
  }
  if (const Value* rj = opt(doc, "runtime")) {
    if (const Value* v = opt(*rj, "check_overhead")) c.runtime.check_overhead = ticks(*v, tick, "$.runtime.check_overhead");
    if (const Value* v = opt(*rj, "rpc_latency")) c.runtime.rpc_latency = ticks(*v, tick, "$.runtime.rpc_latency");
    if (const Value* v = opt(*rj, "step_jitter")) c.runtime.step_jitter = json::get_number(*v, "$.runtime.step_jitter");
    if (const Value* v = opt(*rj, "profile_steps")) c.runtime.profile_steps = static_cast<int>(json::get_int(*v, "$.runtime.profile_steps"));
    if (const Value* v = opt(*rj, "gate_estimate")) {
      const std::string g = json::get_string(*v, "$.runtime.gate_estimate");
      if (g == "mean") c.runtime.gate_estimate = GateEstimate::Mean;
      else if (g == "max") c.runtime.gate_estimate = GateEstimate::Max;
      else throw SchemaError("$.runtime.gate_estimate", "expected mean | max");
    }
  }
  if (const Value* sj = opt(doc, "sweep")) {
    SweepGrid g;
    if (const Value* v = opt(*sj, "micro_batches"))
      each(*v, "$.sweep.micro_batches", [&](const Value& x, const std::string& path) {
        g.micro_batches.push_back(static_cast<int>(json::get_int(x, path)));
      });
    if (const Value* v = opt(*sj, "model_sizes"))
      each(*v, "$.sweep.model_sizes", [&](const Value& x, const std::string& path) {
        g.model_sizes.push_back(json::get_string(x, path));
      });
    if (const Value* v = opt(*sj, "batch_sizes"))
      each(*v, "$.sweep.batch_sizes", [&](const Value& x, const std::string& path) {
        g.batch_sizes.push_back(static_cast<int>(json::get_int(x, path)));
      });
    c.sweep = g;
  }
  if (const Value* v = opt(doc, "seed")) c.seed = static_cast<std::uint64_t>(json::get_int(*v, "$.seed"));
  validate_experiment(c);
  return c;
}

ExperimentConfig load_experiment(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw SchemaError(path, "cannot read config file");
  std::stringstream ss;
  ss << f.rdbuf();
  return experiment_from_json(json::parse(ss.str()));
}

json::Value experiment_to_json(const ExperimentConfig& c) {
  const double tick = c.pipeline.tick_seconds;
  Value doc = Value::object();
  Value& p = doc.set("pipeline", Value::object());
  p.set("num_stages", Value::integer(c.pipeline.num_stages));
  p.set("num_micro_batches", Value::integer(c.pipeline.num_micro_batches));
  p.set("num_epochs", Value::integer(c.pipeline.num_epochs));
  p.set("tick_seconds", Value::number(tick));
  p.set("gpu_memory_total", Value::number(c.pipeline.gpu_memory_total));
  Value& fp = p.set("fp_duration", Value::array());
  for (Tick t : c.pipeline.fp_duration) fp.push(secs(t, tick));
  Value& bp = p.set("bp_duration", Value::array());
  for (Tick t : c.pipeline.bp_duration) bp.push(secs(t, tick));
  Value& sm = p.set("stage_memory", Value::array());
  for (double m : c.pipeline.stage_memory) sm.push(Value::number(m));
  Value& ts = doc.set("tasks", Value::array());
  for (const SideTaskSpec& s : c.tasks) {
    Value t = Value::object();
    t.set("id", Value::string(s.id));
    t.set("interface", Value::string(iface_name(s.interface_kind)));
    t.set("per_step_duration", secs(s.per_step_duration, tick));
    t.set("total_steps", s.total_steps ? Value::integer(*s.total_steps) : Value::null());
    t.set("init_duration", secs(s.init_duration, tick));
    t.set("memory_demand", Value::number(s.memory_demand));
    Value mb = Value::object();
    mb.set("kind", Value::string(s.misbehavior.kind == MisbehaviorKind::None ? "none"
                                 : s.misbehavior.kind == MisbehaviorKind::IgnoresPause ? "ignores_pause"
                                                                                        : "memory_leak"));
    if (s.misbehavior.kind == MisbehaviorKind::MemoryLeak)
      mb.set("rate", Value::number(s.misbehavior.leak_rate_gib_per_s));
    t.set("misbehavior", mb);
    t.set("submit_time", secs(s.submit_time, tick));
    t.set("memory_limit", s.memory_limit ? Value::number(*s.memory_limit) : Value::null());
    t.set("reference_throughput", s.reference_throughput ? Value::number(*s.reference_throughput) : Value::null());
    ts.push(t);
  }
  Value& l = doc.set("limits", Value::object());
  l.set("grace_period", secs(c.limits.grace_period, tick));
  l.set("memory_headroom", Value::number(c.limits.memory_headroom));
  l.set("reclamation_delay", secs(c.limits.reclamation_delay, tick));
  Value& pr = doc.set("prices", Value::object());
  pr.set("price_server_1", Value::number(c.prices.price_server_1));
  pr.set("price_server_2", Value::number(c.prices.price_server_2));
  Value& r = doc.set("runtime", Value::object());
  r.set("check_overhead", secs(c.runtime.check_overhead, tick));
  r.set("rpc_latency", secs(c.runtime.rpc_latency, tick));
  r.set("step_jitter", Value::number(c.runtime.step_jitter));
  r.set("profile_steps", Value::integer(c.runtime.profile_steps));
  r.set("gate_estimate", Value::string(c.runtime.gate_estimate == GateEstimate::Max ? "max" : "mean"));
  if (c.sweep) {
    Value& g = doc.set("sweep", Value::object());
    Value& m = g.set("micro_batches", Value::array());
    for (int x : c.sweep->micro_batches) m.push(Value::integer(x));
    Value& ms = g.set("model_sizes", Value::array());
    for (const auto& x : c.sweep->model_sizes) ms.push(Value::string(x));
    Value& b = g.set("batch_sizes", Value::array());
    for (int x : c.sweep->batch_sizes) b.push(Value::integer(x));
  }
  doc.set("seed", Value::integer(static_cast<std::int64_t>(c.seed)));
  return doc;
}

}  // namespace freeride
