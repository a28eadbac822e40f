// Experiment config, run-trace stream, report and replay_check -- the
// reference's config.hpp:52-56, trace.hpp:16-22, engine.hpp:100-104 and
// metrics.hpp:87 (declared there, never implemented).
#pragma once

#include <iosfwd>
#include <string>
#include <vector>

#include "freeride.hpp"
#include "json.hpp"

namespace freeride {

// config.hpp:52-56.  Shape problems throw SchemaError(path); well-formed
// documents violating invariants throw ValidationError(field).  Durations
// are simulated seconds (whole ticks, seconds_to_ticks), memory GiB.
ExperimentConfig experiment_from_json(const json::Value& doc);
ExperimentConfig load_experiment(const std::string& path);
json::Value experiment_to_json(const ExperimentConfig& config);  // deterministic
void validate_experiment(const ExperimentConfig& config);

// trace.hpp:16-20: a meta line, one record per line in timeline order, the
// dispositions and an end line with the makespan.  Byte-stable.
void write_trace_jsonl(const RunTrace& trace, std::ostream& out);
RunTrace read_trace_jsonl(std::istream& in);
void write_trace_file(const RunTrace& trace, const std::string& path);
RunTrace read_trace_file(const std::string& path);

// metrics.hpp:87 build_report: ΔT, S, per-stage breakdown, bubble rate --
// every field recomputable from the two traces.
struct MetricsReport {
  double t_no = 0.0, t_with = 0.0, delta_t = 0.0, bubble_rate = 0.0;
  CostBreakdown cost;
  bool has_cost = false;  // S needs every task with work to state reference_throughput
  std::vector<StageBreakdown> breakdown;
  std::vector<DispositionRecord> dispositions;
};
BreakdownInput breakdown_input(const RunTrace& trace);
MetricsReport build_report(const RunTrace& baseline, const RunTrace& treatment);
json::Value report_to_json(const MetricsReport& report, double tick_seconds);

// engine.hpp:100-104: re-validates the module invariants over a finished
// trace (dependency soundness, GPU and state exclusivity, transition
// legality, memory lifecycle, step accounting, breakdown conservation).
// Empty = sound.
std::vector<std::string> replay_check(const RunTrace& trace);

// Named model-size presets for sweeps (SweepGrid::model_sizes).
bool apply_model_preset(const std::string& name, int batch_size, PipelineConfig& p);

}  // namespace freeride
