// Run-trace stream (reference trace.hpp:16-22) and the
// metrics report (metrics.hpp:87, report_to_json trace.hpp:22).
#include <algorithm>
#include <fstream>
#include <map>
#include <sstream>

#include "io.hpp"

// json::need / get_* return references into the document, never into their
// (temporary) path argument; GCC 13's heuristic cannot see that.
#pragma GCC diagnostic ignored "-Wdangling-reference"

namespace freeride {

namespace {

using json::Value;

const char* kind_name(OpKind k) { return k == OpKind::FP ? "FP" : "BP"; }
const char* btype_name(BubbleType b) { return b == BubbleType::A ? "A" : b == BubbleType::B ? "B" : "C"; }
const char* act_name(ActivityKind k) {
  static const char* n[] = {"init", "step", "kernel", "check"};
  return n[static_cast<int>(k)];
}
const char* reason_name(KillReason r) {
  static const char* n[] = {"oom", "pause-timeout", "init-timeout"};
  return n[static_cast<int>(r)];
}
const char* disp_name(Disposition d) {
  static const char* n[] = {"rejected", "completed", "killed-oom", "killed-pause-timeout",
                            "killed-init-timeout", "active"};
  return n[static_cast<int>(d)];
}

template <class E, std::size_t N>
E lookup(const std::string& s, const char* const (&names)[N], const std::string& path) {
  for (std::size_t k = 0; k < N; ++k)
    if (s == names[k]) return static_cast<E>(k);
  throw SchemaError(path, "unknown value '" + s + "'");
}

Value opt_num(const std::optional<double>& v) { return v ? Value::number(*v) : Value::null(); }

Value profile_json(const TaskProfile& p) {
  Value o = Value::object();
  o.set("task_id", Value::string(p.task_id));
  o.set("est_per_step_duration", opt_num(p.est_per_step_duration));
  o.set("max_per_step_duration", opt_num(p.max_per_step_duration));
  o.set("est_memory", Value::number(p.est_memory));
  o.set("profiled_steps", Value::integer(p.profiled_steps));
  return o;
}

struct Rec {
  Tick t;
  int rank;
  std::size_t idx;
  Value v;
};

Value tr_rec(const char* type, const TransitionRecord& r) {
  Value o = Value::object();
  o.set("type", Value::string(type));
  o.set("t", Value::integer(r.t));
  o.set("task", Value::string(r.task));
  o.set("kind", Value::string(to_string(r.kind)));
  o.set("worker", Value::integer(r.worker));
  return o;
}

Value as_rec(const char* type, const AssignRecord& r) {
  Value o = Value::object();
  o.set("type", Value::string(type));
  o.set("t", Value::integer(r.t));
  o.set("task", Value::string(r.task));
  o.set("worker", Value::integer(r.worker));
  return o;
}

}  // namespace

void write_trace_jsonl(const RunTrace& tr, std::ostream& out) {
  Value meta = Value::object();
  meta.set("type", Value::string("meta"));
  meta.set("config", experiment_to_json(tr.config));
  meta.set("seed", Value::integer(static_cast<std::int64_t>(tr.seed)));
  meta.set("with_tasks", Value::boolean(tr.with_tasks));
  Value& pf = meta.set("profiles", Value::array());
  for (const TaskProfile& p : tr.profiles) pf.push(profile_json(p));
  if (tr.measured) {  // only in GPU traces: simulated traces stay byte-identical
    meta.set("measured", Value::boolean(true));
    meta.set("tolerance", Value::integer(tr.tolerance));
  }
  out << json::dump(meta) << '\n';

  std::vector<Rec> recs;
  for (std::size_t i = 0; i < tr.ops.size(); ++i) {
    const OpEvent& o = tr.ops[i];
    Value v = Value::object();
    v.set("type", Value::string("op"));
    v.set("stage", Value::integer(o.stage));
    v.set("kind", Value::string(kind_name(o.kind)));
    v.set("mb", Value::integer(o.micro_batch));
    v.set("epoch", Value::integer(o.epoch));
    v.set("start", Value::integer(o.start));
    v.set("end", Value::integer(o.end));
    recs.push_back({o.start, 0, i, v});
  }
  for (std::size_t i = 0; i < tr.bubbles.size(); ++i) {
    const Bubble& b = tr.bubbles[i];
    Value v = Value::object();
    v.set("type", Value::string("bubble"));
    v.set("stage", Value::integer(b.stage));
    v.set("epoch", Value::integer(b.epoch));
    v.set("start", Value::integer(b.start));
    v.set("duration", Value::integer(b.duration));
    v.set("available_memory", Value::number(b.available_memory));
    v.set("btype", Value::string(btype_name(b.btype)));
    recs.push_back({b.start, 1, i, v});
  }
  for (std::size_t i = 0; i < tr.submits.size(); ++i) recs.push_back({tr.submits[i].t, 2, i, as_rec("submit", tr.submits[i])});
  for (std::size_t i = 0; i < tr.assigns.size(); ++i) recs.push_back({tr.assigns[i].t, 3, i, as_rec("assign", tr.assigns[i])});
  for (std::size_t i = 0; i < tr.rejects.size(); ++i) recs.push_back({tr.rejects[i].t, 4, i, as_rec("reject", tr.rejects[i])});
  for (std::size_t i = 0; i < tr.rpcs.size(); ++i) recs.push_back({tr.rpcs[i].t, 5, i, tr_rec("rpc", tr.rpcs[i])});
  for (std::size_t i = 0; i < tr.transitions.size(); ++i)
    recs.push_back({tr.transitions[i].t, 6, i, tr_rec("transition", tr.transitions[i])});
  for (std::size_t i = 0; i < tr.activities.size(); ++i) {
    const ActivityRecord& a = tr.activities[i];
    Value v = Value::object();
    v.set("type", Value::string("activity"));
    v.set("start", Value::integer(a.start));
    v.set("end", Value::integer(a.end));
    v.set("task", Value::string(a.task));
    v.set("worker", Value::integer(a.worker));
    v.set("kind", Value::string(act_name(a.kind)));
    v.set("clipped", Value::boolean(a.clipped));
    recs.push_back({a.start, 7, i, v});
  }
  for (std::size_t i = 0; i < tr.kills.size(); ++i) {
    const KillRecord& k = tr.kills[i];
    Value v = Value::object();
    v.set("type", Value::string("kill"));
    v.set("t", Value::integer(k.t));
    v.set("task", Value::string(k.task));
    v.set("worker", Value::integer(k.worker));
    v.set("reason", Value::string(reason_name(k.reason)));
    recs.push_back({k.t, 8, i, v});
  }
  std::stable_sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.rank != b.rank) return a.rank < b.rank;
    return a.idx < b.idx;
  });
  for (const Rec& r : recs) out << json::dump(r.v) << '\n';
  for (const DispositionRecord& d : tr.dispositions) {
    Value v = Value::object();
    v.set("type", Value::string("disposition"));
    v.set("task", Value::string(d.task));
    v.set("disposition", Value::string(disp_name(d.disposition)));
    v.set("steps", Value::integer(d.steps_completed));
    v.set("worker", d.worker ? Value::integer(*d.worker) : Value::null());
    out << json::dump(v) << '\n';
  }
  Value end = Value::object();
  end.set("type", Value::string("end"));
  end.set("makespan", Value::integer(tr.makespan));
  out << json::dump(end) << '\n';
}

RunTrace read_trace_jsonl(std::istream& in) {
  static const char* const kinds[] = {"FP", "BP"};
  static const char* const btypes[] = {"A", "B", "C"};
  static const char* const acts[] = {"init", "step", "kernel", "check"};
  static const char* const reasons[] = {"oom", "pause-timeout", "init-timeout"};
  static const char* const disps[] = {"rejected", "completed", "killed-oom", "killed-pause-timeout",
                                      "killed-init-timeout", "active"};
  static const char* const tks[] = {"create", "init", "start", "run_next_step", "pause", "stop"};
  RunTrace tr;
  std::string line;
  std::size_t n = 0;
  bool meta = false, end = false;
  while (std::getline(in, line)) {
    ++n;
    if (line.empty()) continue;
    const std::string path = "$line" + std::to_string(n);
    const Value v = json::parse(line);
    const std::string type = json::get_string(json::need(v, "type", path), path + ".type");
    auto I = [&](const char* k) { return json::get_int(json::need(v, k, path), path + "." + k); };
    auto S = [&](const char* k) -> std::string { return json::get_string(json::need(v, k, path), path + "." + k); };
    if (end) throw SchemaError(path, "record after the end line");
    if (type == "meta") {
      tr.config = experiment_from_json(json::need(v, "config", path));
      tr.seed = static_cast<std::uint64_t>(I("seed"));
      tr.with_tasks = json::get_bool(json::need(v, "with_tasks", path), path + ".with_tasks");
      for (const Value& p : json::get_array(json::need(v, "profiles", path), path + ".profiles")) {
        TaskProfile tp;
        tp.task_id = json::get_string(json::need(p, "task_id", path), path + ".task_id");
        const Value& e = json::need(p, "est_per_step_duration", path);
        if (!e.is_null()) tp.est_per_step_duration = json::get_number(e, path);
        const Value& m = json::need(p, "max_per_step_duration", path);
        if (!m.is_null()) tp.max_per_step_duration = json::get_number(m, path);
        tp.est_memory = json::get_number(json::need(p, "est_memory", path), path);
        tp.profiled_steps = static_cast<int>(json::get_int(json::need(p, "profiled_steps", path), path));
        tr.profiles.push_back(tp);
      }
      if (const Value* m = v.find("measured")) tr.measured = json::get_bool(*m, path + ".measured");
      if (const Value* t = v.find("tolerance")) tr.tolerance = json::get_int(*t, path + ".tolerance");
      meta = true;
      continue;
    }
    if (!meta) throw SchemaError(path, "the meta line must come first");
    if (type == "op") {
      tr.ops.push_back(OpEvent{static_cast<int>(I("stage")), lookup<OpKind>(S("kind"), kinds, path + ".kind"),
                               static_cast<int>(I("mb")), static_cast<int>(I("epoch")), I("start"), I("end")});
    } else if (type == "bubble") {
      tr.bubbles.push_back(Bubble{static_cast<int>(I("stage")), static_cast<int>(I("epoch")), I("start"),
                                  I("duration"),
                                  json::get_number(json::need(v, "available_memory", path), path),
                                  lookup<BubbleType>(S("btype"), btypes, path + ".btype")});
    } else if (type == "submit" || type == "assign" || type == "reject") {
      AssignRecord r{I("t"), S("task"), static_cast<int>(I("worker"))};
      (type == "submit" ? tr.submits : type == "assign" ? tr.assigns : tr.rejects).push_back(r);
    } else if (type == "rpc" || type == "transition") {
      TransitionRecord r{I("t"), S("task"), lookup<TransitionKind>(S("kind"), tks, path + ".kind"),
                         static_cast<int>(I("worker"))};
      (type == "rpc" ? tr.rpcs : tr.transitions).push_back(r);
    } else if (type == "activity") {
      tr.activities.push_back(ActivityRecord{I("start"), I("end"), S("task"), static_cast<int>(I("worker")),
                                             lookup<ActivityKind>(S("kind"), acts, path + ".kind"),
                                             json::get_bool(json::need(v, "clipped", path), path)});
    } else if (type == "kill") {
      tr.kills.push_back(KillRecord{I("t"), S("task"), static_cast<int>(I("worker")),
                                    lookup<KillReason>(S("reason"), reasons, path + ".reason")});
    } else if (type == "disposition") {
      DispositionRecord d;
      d.task = S("task");
      d.disposition = lookup<Disposition>(S("disposition"), disps, path + ".disposition");
      d.steps_completed = I("steps");
      const Value& w = json::need(v, "worker", path);
      if (!w.is_null()) d.worker = static_cast<int>(json::get_int(w, path + ".worker"));
      tr.dispositions.push_back(d);
    } else if (type == "end") {
      tr.makespan = I("makespan");
      end = true;
    } else {
      throw SchemaError(path + ".type", "unknown record type '" + type + "'");
    }
  }
  if (!meta || !end) throw SchemaError("$", "trace needs a meta line and an end line");
  return tr;
}

void write_trace_file(const RunTrace& trace, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw SchemaError(path, "cannot write trace file");
  write_trace_jsonl(trace, f);
}

RunTrace read_trace_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw SchemaError(path, "cannot read trace file");
  return read_trace_jsonl(f);
}

BreakdownInput breakdown_input(const RunTrace& t) {
  BreakdownInput bi;
  bi.num_stages = t.config.pipeline.num_stages;
  bi.profiles = t.profiles;
  bi.bubbles = t.bubbles;
  bi.assigns = t.assigns;
  bi.transitions = t.transitions;
  bi.activities = t.activities;
  return bi;
}

MetricsReport build_report(const RunTrace& base, const RunTrace& with) {
  MetricsReport r;
  const double tick = with.config.pipeline.tick_seconds;
  r.t_no = ticks_to_seconds(base.makespan, tick);
  r.t_with = ticks_to_seconds(with.makespan, tick);
  r.delta_t = time_increase(r.t_no, r.t_with);
  Tick bsum = 0;
  for (const Bubble& b : base.bubbles) bsum += b.duration;
  // metrics.cpp:212-219: the baseline makespan is the wall time
  r.bubble_rate = base.makespan > 0
                      ? static_cast<double>(bsum) / (static_cast<double>(with.config.pipeline.num_stages) *
                                                     static_cast<double>(base.makespan))
                      : 0.0;
  std::vector<TaskWork> work;
  r.has_cost = true;
  for (const DispositionRecord& d : with.dispositions) {
    TaskWork w;
    w.id = d.task;
    w.work = static_cast<double>(d.steps_completed);
    for (const SideTaskSpec& s : with.config.tasks)
      if (s.id == d.task) w.throughput_per_hour = s.reference_throughput;
    if (w.work > 0 && !w.throughput_per_hour) r.has_cost = false;
    work.push_back(w);
  }
  if (r.has_cost) r.cost = cost_savings(r.t_no, r.delta_t, work, with.config.prices);
  r.breakdown = bubble_breakdown(breakdown_input(with));
  r.dispositions = with.dispositions;
  return r;
}

json::Value report_to_json(const MetricsReport& r, double tick_seconds) {
  Value o = Value::object();
  o.set("t_no_side_tasks_s", Value::number(r.t_no));
  o.set("t_with_side_tasks_s", Value::number(r.t_with));
  o.set("delta_t", Value::number(r.delta_t));
  o.set("bubble_rate", Value::number(r.bubble_rate));
  if (r.has_cost) {
    Value& c = o.set("cost", Value::object());
    c.set("c_no_side", Value::number(r.cost.c_no_side));
    c.set("c_extra", Value::number(r.cost.c_extra));
    c.set("c_side_tasks", Value::number(r.cost.c_side_tasks));
    c.set("s", Value::number(r.cost.s));
  } else {
    o.set("cost", Value::null());  // a task with work states no reference_throughput
  }
  Value& b = o.set("breakdown", Value::array());
  Tick used = 0, total = 0;
  for (const StageBreakdown& s : r.breakdown) {
    Value x = Value::object();
    x.set("stage", Value::integer(s.stage));
    x.set("used_by_side_tasks_s", Value::number(ticks_to_seconds(s.used_by_side_tasks, tick_seconds)));
    x.set("runtime_overhead_s", Value::number(ticks_to_seconds(s.runtime_overhead, tick_seconds)));
    x.set("idle_oom_s", Value::number(ticks_to_seconds(s.idle_oom, tick_seconds)));
    x.set("idle_insufficient_time_s", Value::number(ticks_to_seconds(s.idle_insufficient_time, tick_seconds)));
    b.push(x);
    used += s.used_by_side_tasks;
    total += s.total();
  }
  o.set("fill", Value::number(total > 0 ? static_cast<double>(used) / static_cast<double>(total) : 0.0));
  Value& d = o.set("dispositions", Value::array());
  for (const DispositionRecord& x : r.dispositions) {
    Value e = Value::object();
    e.set("task", Value::string(x.task));
    e.set("disposition", Value::string(disp_name(x.disposition)));
    e.set("steps", Value::integer(x.steps_completed));
    d.push(e);
  }
  return o;
}

}  // namespace freeride
