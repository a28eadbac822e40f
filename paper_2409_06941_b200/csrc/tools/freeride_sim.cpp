// freeride-sim: the reference's command-line front end (cli.hpp:10-31,
// SPEC.md:519-557), over this repo's simulated engine and its JSON config /
// JSONL trace formats:
//
//   freeride-sim profile <config> [--out <path>|-]
//   freeride-sim run     <config> --out <dir> [--seed N] [--format json-lines|csv]
//   freeride-sim sweep   <config> --out <dir> [--jobs K] [--format json-lines|csv]
//   freeride-sim check   <trace.jsonl>
//
// Exit codes (cli.hpp:10-13): 0 ok, 1 infeasible/validation, 2 schema/parse,
// 3 replay_check violation (a bug).  Default out dir: $FREERIDE_OUT.
#include <sys/stat.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <mutex>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "host/io.hpp"

using namespace freeride;
using json::Value;

namespace {

constexpr int kExitOk = 0, kExitValidation = 1, kExitSchema = 2, kExitViolation = 3;
enum class TableFormat { Csv, JsonLines };

void mkdirs(const std::string& dir) {
  std::string cur;
  for (std::size_t i = 0; i <= dir.size(); ++i) {
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty()) ::mkdir(cur.c_str(), 0755);
    }
    if (i < dir.size()) cur += dir[i];
  }
}

void write_text(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw SchemaError(path, "cannot write");
  f << text;
}

int check_traces(const std::vector<const RunTrace*>& ts, const std::vector<std::string>& names) {
  int bad = 0;
  for (std::size_t k = 0; k < ts.size(); ++k)
    for (const std::string& v : replay_check(*ts[k])) {
      std::cerr << names[k] << ": " << v << "\n";
      ++bad;
    }
  return bad ? kExitViolation : kExitOk;
}

// cmd_profile (cli.hpp:18): bubble profile + per-task profiles
int cmd_profile(const std::string& config_path, const std::string& out_path) {
  const ExperimentConfig c = load_experiment(config_path);
  const BubbleProfile bp = profile_bubbles(c.pipeline);
  Value doc = Value::object();
  doc.set("bubble_rate", Value::number(bp.rate));
  Value& st = doc.set("stages", Value::array());
  for (std::size_t s = 0; s < bp.stages.size(); ++s) {
    Value x = Value::object();
    x.set("stage", Value::integer(static_cast<std::int64_t>(s)));
    Value& d = x.set("bubble_durations_s", Value::array());
    for (Tick t : bp.stages[s].durations) d.push(Value::number(ticks_to_seconds(t, c.pipeline.tick_seconds)));
    x.set("available_memory", Value::number(bp.stages[s].available_memory));
    st.push(x);
  }
  Value& tp = doc.set("tasks", Value::array());
  ProfileOptions po;
  po.n_steps = c.runtime.profile_steps;
  po.step_jitter = c.runtime.step_jitter;
  po.tick_seconds = c.pipeline.tick_seconds;
  for (const SideTaskSpec& s : c.tasks) {
    const TaskProfile p = profile_task(s, po, c.seed);
    Value x = Value::object();
    x.set("task_id", Value::string(p.task_id));
    x.set("est_per_step_duration", p.est_per_step_duration ? Value::number(*p.est_per_step_duration) : Value::null());
    x.set("max_per_step_duration", p.max_per_step_duration ? Value::number(*p.max_per_step_duration) : Value::null());
    x.set("est_memory", Value::number(p.est_memory));
    x.set("profiled_steps", Value::integer(p.profiled_steps));
    tp.push(x);
  }
  const std::string text = json::dump(doc) + "\n";
  if (out_path == "-") std::cout << text;
  else write_text(out_path, text);
  return kExitOk;
}

std::string table_row(const std::vector<std::pair<std::string, Value>>& cols, TableFormat f, bool header) {
  if (f == TableFormat::JsonLines) {
    Value o = Value::object();
    for (const auto& [k, v] : cols) o.set(k, v);
    return json::dump(o) + "\n";
  }
  std::string out;
  for (std::size_t i = 0; i < cols.size(); ++i) {
    if (i) out += ',';
    out += header ? cols[i].first : (cols[i].second.kind == Value::Kind::String ? cols[i].second.s
                                                                               : json::dump(cols[i].second));
  }
  return out + "\n";
}

struct RunOut {
  RunTrace base, with;
  MetricsReport report;
};

RunOut run_pair(const ExperimentConfig& c, std::uint64_t seed) {
  RunOut r;
  r.base = run_experiment(c, false, seed);
  r.with = run_experiment(c, true, seed);
  r.report = build_report(r.base, r.with);
  return r;
}

void write_run(const RunOut& r, const std::string& dir, TableFormat fmt, double tick) {
  mkdirs(dir);
  write_trace_file(r.base, dir + "/baseline.trace.jsonl");
  write_trace_file(r.with, dir + "/treatment.trace.jsonl");
  write_text(dir + "/report.json", json::dump(report_to_json(r.report, tick)) + "\n");
  std::string table;
  for (std::size_t i = 0; i < r.report.breakdown.size(); ++i) {
    const StageBreakdown& s = r.report.breakdown[i];
    std::vector<std::pair<std::string, Value>> cols = {
        {"stage", Value::integer(s.stage)},
        {"used_by_side_tasks_s", Value::number(ticks_to_seconds(s.used_by_side_tasks, tick))},
        {"runtime_overhead_s", Value::number(ticks_to_seconds(s.runtime_overhead, tick))},
        {"idle_oom_s", Value::number(ticks_to_seconds(s.idle_oom, tick))},
        {"idle_insufficient_time_s", Value::number(ticks_to_seconds(s.idle_insufficient_time, tick))}};
    if (i == 0 && fmt == TableFormat::Csv) table += table_row(cols, fmt, true);
    table += table_row(cols, fmt, false);
  }
  write_text(dir + (fmt == TableFormat::Csv ? "/breakdown.csv" : "/breakdown.jsonl"), table);
}

// cmd_run (cli.hpp:22-23)
int cmd_run(const std::string& config_path, const std::string& out_dir, std::optional<std::uint64_t> seed,
            TableFormat fmt) {
  ExperimentConfig c = load_experiment(config_path);
  const RunOut r = run_pair(c, seed.value_or(c.seed));
  write_run(r, out_dir, fmt, c.pipeline.tick_seconds);
  return check_traces({&r.base, &r.with}, {"baseline", "treatment"});
}

// cmd_sweep (cli.hpp:27-28): cartesian grid, one isolated run per point
int cmd_sweep(const std::string& config_path, const std::string& out_dir, int jobs, TableFormat fmt) {
  const ExperimentConfig c = load_experiment(config_path);
  if (!c.sweep) throw ValidationError("sweep", "config has no sweep grid");
  struct Point { int mb; std::string model; int batch; };
  std::vector<Point> pts;
  const std::vector<int> mbs = c.sweep->micro_batches.empty() ? std::vector<int>{c.pipeline.num_micro_batches}
                                                              : c.sweep->micro_batches;
  const std::vector<std::string> models = c.sweep->model_sizes.empty() ? std::vector<std::string>{""}
                                                                       : c.sweep->model_sizes;
  const std::vector<int> batches = c.sweep->batch_sizes.empty() ? std::vector<int>{0} : c.sweep->batch_sizes;
  for (int mb : mbs)
    for (const auto& md : models)
      for (int b : batches) pts.push_back({mb, md, b});
  std::vector<std::optional<RunOut>> res(pts.size());
  std::vector<std::string> err(pts.size());
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (std::size_t i; (i = next++) < pts.size();) {
      try {
        ExperimentConfig pc = c;
        pc.sweep.reset();
        pc.pipeline.num_micro_batches = pts[i].mb;
        if (!pts[i].model.empty() || pts[i].batch > 0)
          apply_model_preset(pts[i].model.empty() ? "1.2B" : pts[i].model, pts[i].batch > 0 ? pts[i].batch : 4,
                             pc.pipeline);
        validate_experiment(pc);
        res[i] = run_pair(pc, pc.seed);
      } catch (const std::exception& e) {
        err[i] = e.what();
      }
    }
  };
  std::vector<std::thread> th;
  for (int j = 0; j < std::max(1, jobs); ++j) th.emplace_back(worker);
  for (auto& t : th) t.join();
  mkdirs(out_dir);
  std::string table;
  int rc = kExitOk;
  for (std::size_t i = 0; i < pts.size(); ++i) {
    if (!res[i]) {
      std::cerr << "point " << i << ": " << err[i] << "\n";
      rc = std::max(rc, kExitValidation);
      continue;
    }
    const std::string dir = out_dir + "/point" + std::to_string(i);
    write_run(*res[i], dir, fmt, c.pipeline.tick_seconds);
    Tick used = 0, total = 0;
    for (const StageBreakdown& s : res[i]->report.breakdown) used += s.used_by_side_tasks, total += s.total();
    std::vector<std::pair<std::string, Value>> cols = {
        {"point", Value::integer(static_cast<std::int64_t>(i))},
        {"micro_batches", Value::integer(pts[i].mb)},
        {"model_size", Value::string(pts[i].model)},
        {"batch_size", Value::integer(pts[i].batch)},
        {"bubble_rate", Value::number(res[i]->report.bubble_rate)},
        {"delta_t", Value::number(res[i]->report.delta_t)},
        {"s", res[i]->report.has_cost ? Value::number(res[i]->report.cost.s) : Value::null()},
        {"fill", Value::number(total > 0 ? double(used) / double(total) : 0.0)}};
    if (table.empty() && fmt == TableFormat::Csv) table += table_row(cols, fmt, true);
    table += table_row(cols, fmt, false);
    rc = std::max(rc, check_traces({&res[i]->base, &res[i]->with}, {dir + "/baseline", dir + "/treatment"}));
  }
  write_text(out_dir + (fmt == TableFormat::Csv ? "/sweep.csv" : "/sweep.jsonl"), table);
  return rc;
}

// cmd_check (cli.hpp:31)
int cmd_check(const std::string& trace_path) {
  const RunTrace t = read_trace_file(trace_path);
  const int rc = check_traces({&t}, {trace_path});
  if (rc == kExitOk) std::cout << "ok: " << trace_path << "\n";
  return rc;
}

int usage() {
  std::cerr << "usage: freeride-sim profile <config> [--out <path>|-]\n"
               "       freeride-sim run <config> --out <dir> [--seed N] [--format json-lines|csv]\n"
               "       freeride-sim sweep <config> --out <dir> [--jobs K] [--format json-lines|csv]\n"
               "       freeride-sim check <trace.jsonl>\n";
  return kExitSchema;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1], target = argv[2];
  std::string out = std::getenv("FREERIDE_OUT") ? std::getenv("FREERIDE_OUT") : "";
  std::optional<std::uint64_t> seed;
  int jobs = 1;
  TableFormat fmt = TableFormat::Csv;
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw SchemaError(a, "missing value");
      return argv[++i];
    };
    try {
      if (a == "--out") out = val();
      else if (a == "--seed") seed = std::stoull(val());
      else if (a == "--jobs") jobs = std::stoi(val());
      else if (a == "--format") {
        const std::string f = val();
        if (f == "csv") fmt = TableFormat::Csv;
        else if (f == "json-lines") fmt = TableFormat::JsonLines;
        else throw SchemaError("--format", "expected csv | json-lines");
      } else {
        throw SchemaError(a, "unknown flag");
      }
    } catch (const SchemaError& e) {
      std::cerr << "error: " << e.what() << "\n";
      return usage();
    } catch (const std::exception& e) {
      std::cerr << "error: " << a << ": " << e.what() << "\n";
      return kExitSchema;
    }
  }
  try {
    if (cmd == "profile") return cmd_profile(target, out.empty() ? "-" : out);
    if (cmd == "run" || cmd == "sweep") {
      if (out.empty()) throw SchemaError("--out", "an output directory is required");
      return cmd == "run" ? cmd_run(target, out, seed, fmt) : cmd_sweep(target, out, jobs, fmt);
    }
    if (cmd == "check") return cmd_check(target);
    return usage();
  } catch (const ValidationError& e) {
    std::cerr << "validation error: " << e.what() << "\n";
    return kExitValidation;
  } catch (const SchemaError& e) {
    std::cerr << "schema error: " << e.what() << "\n";
    return kExitSchema;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitViolation;
  }
}
