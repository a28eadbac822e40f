// Per-stage 1F1B bubble timeline (reference: src/pipeline.cpp:27-296).
//
// The reference builds a generic DAG keyed by std::map<tuple> and runs a LIFO
// worklist.  Here every op of the 2*p*m*E grid has a closed-form flat index
//   id(e, s, kind, mb) = ((e*p + s)*2 + kind)*m + (mb-1)
// and its <=3 predecessors / <=3 successors are computed arithmetically from
// the per-stage issue order, so the schedule is one Kahn pass over int arrays
// (no allocation per edge, no map lookups).  Earliest-start times are the
// longest-path fixpoint of the DAG, unique regardless of processing order, so
// results equal the reference's bit for bit.
#include <algorithm>
#include <cmath>
#include <limits>
#include <tuple>

#include "freeride.hpp"

namespace freeride {

Tick seconds_to_ticks(double seconds, double tick_seconds, const std::string& field) {
  if (!(tick_seconds > 0.0)) throw ValidationError("tick_seconds", "must be > 0");
  const double q = seconds / tick_seconds;
  const double r = std::round(q);
  if (std::abs(q - r) > 1e-6)
    throw ValidationError(field, "duration " + std::to_string(seconds) +
                                     " is not a whole number of ticks (tick_seconds=" +
                                     std::to_string(tick_seconds) + ")");
  return static_cast<Tick>(r);
}

namespace {

void check_durations(const std::vector<Tick>& v, int p, const char* field) {
  if (v.size() != 1 && v.size() != static_cast<std::size_t>(p))
    throw ValidationError(field, "override list must have one entry per stage");
  for (Tick d : v)
    if (d <= 0) throw ValidationError(field, "durations must be > 0");
}

}  // namespace

void PipelineConfig::validate() const {  // pipeline.cpp:27-49
  if (num_stages < 1) throw ValidationError("num_stages", "must be >= 1");
  if (num_micro_batches < 1) throw ValidationError("num_micro_batches", "must be >= 1");
  if (num_epochs < 1) throw ValidationError("num_epochs", "must be >= 1");
  if (!(tick_seconds > 0.0)) throw ValidationError("tick_seconds", "must be > 0");
  if (fp_duration.empty()) throw ValidationError("fp_duration", "missing");
  if (bp_duration.empty()) throw ValidationError("bp_duration", "missing");
  check_durations(fp_duration, num_stages, "fp_duration");
  check_durations(bp_duration, num_stages, "bp_duration");
  if (gpu_memory_total < 0.0) throw ValidationError("gpu_memory_total", "must be >= 0");
  if (stage_memory.size() != static_cast<std::size_t>(num_stages))
    throw ValidationError("stage_memory", "must have one entry per stage");
  for (int s = 0; s < num_stages; ++s) {
    if (stage_memory[s] < 0.0) throw ValidationError("stage_memory", "entries must be >= 0");
    if (stage_memory[s] > gpu_memory_total)
      throw ValidationError("stage_memory",
                            "stage " + std::to_string(s) + " exceeds gpu_memory_total");
  }
}

// pipeline.cpp:51-72: warm-up min(m, p-s) FPs, BP/FP alternation, BP drain;
// a single stage accumulates all FPs before its BPs.
std::vector<std::pair<OpKind, int>> stage_issue_order(int stage, int p, int m) {
  std::vector<std::pair<OpKind, int>> seq;
  if (m <= 0) return seq;
  seq.reserve(static_cast<std::size_t>(2 * m));
  const int warm = p == 1 ? m : std::min(m, p - stage);
  int f = 1, b = 1;
  for (; f <= warm; ++f) seq.emplace_back(OpKind::FP, f);
  if (p == 1) {
    for (; b <= m; ++b) seq.emplace_back(OpKind::BP, b);
    return seq;
  }
  while (f <= m) {
    seq.emplace_back(OpKind::BP, b++);
    seq.emplace_back(OpKind::FP, f++);
  }
  for (; b <= m; ++b) seq.emplace_back(OpKind::BP, b);
  return seq;
}

ScheduleTrace build_schedule(const PipelineConfig& cfg) {
  cfg.validate();
  const int p = cfg.num_stages, m = cfg.num_micro_batches, E = cfg.num_epochs;
  const std::int64_t per_epoch = 2LL * p * m;
  const std::int64_t n = per_epoch * E;
  auto id = [&](std::int64_t e, std::int64_t s, int k, std::int64_t mb) {
    return ((e * p + s) * 2 + k) * m + (mb - 1);
  };

  // Issue order per stage and each (s, kind, mb)'s slot in it.
  std::vector<std::vector<std::pair<OpKind, int>>> order(p);
  std::vector<int> slot(static_cast<std::size_t>(per_epoch));  // [(s*2+k)*m + mb-1]
  for (int s = 0; s < p; ++s) {
    order[s] = stage_issue_order(s, p, m);
    for (int i = 0; i < 2 * m; ++i) {
      const auto& [k, mb] = order[s][i];
      slot[(static_cast<std::size_t>(s) * 2 + static_cast<int>(k)) * m + (mb - 1)] = i;
    }
  }

  // Successors of one op (<= 3): next on stage (wrapping into the next
  // epoch), the cross-stage consumer, and BP(s,mb) for an FP.
  auto successors = [&](std::int64_t e, int s, int k, int mb, std::int64_t* out) {
    int c = 0;
    const int i = slot[(static_cast<std::size_t>(s) * 2 + k) * m + (mb - 1)];
    if (i + 1 < 2 * m) {
      const auto& [nk, nmb] = order[s][i + 1];
      out[c++] = id(e, s, static_cast<int>(nk), nmb);
    } else if (e + 1 < E) {
      const auto& [nk, nmb] = order[s][0];
      out[c++] = id(e + 1, s, static_cast<int>(nk), nmb);
    }
    if (k == 0) {
      if (s + 1 < p) out[c++] = id(e, s + 1, 0, mb);
      out[c++] = id(e, s, 1, mb);
    } else if (s > 0) {
      out[c++] = id(e, s - 1, 1, mb);
    }
    return c;
  };

  std::vector<int> indeg(static_cast<std::size_t>(n), 0);
  std::vector<Tick> ready_at(static_cast<std::size_t>(n), 0);
  std::vector<Tick> start(static_cast<std::size_t>(n), 0);
  std::int64_t succ[3];
  for (std::int64_t e = 0; e < E; ++e)
    for (int s = 0; s < p; ++s)
      for (int k = 0; k < 2; ++k)
        for (int mb = 1; mb <= m; ++mb) {
          const int c = successors(e, s, k, mb, succ);
          for (int j = 0; j < c; ++j) indeg[static_cast<std::size_t>(succ[j])]++;
        }

  std::vector<std::int64_t> stack;
  stack.reserve(static_cast<std::size_t>(p) * 2);
  for (std::int64_t v = 0; v < n; ++v)
    if (indeg[static_cast<std::size_t>(v)] == 0) stack.push_back(v);
  std::int64_t done = 0;
  while (!stack.empty()) {
    const std::int64_t v = stack.back();
    stack.pop_back();
    ++done;
    const int mb = static_cast<int>(v % m) + 1;
    const int k = static_cast<int>((v / m) % 2);
    const int s = static_cast<int>((v / (2LL * m)) % p);
    const std::int64_t e = v / per_epoch;
    const Tick st = ready_at[static_cast<std::size_t>(v)];
    start[static_cast<std::size_t>(v)] = st;
    const Tick fin = st + (k == 0 ? cfg.fp_ticks(s) : cfg.bp_ticks(s));
    const int c = successors(e, s, k, mb, succ);
    for (int j = 0; j < c; ++j) {
      const auto u = static_cast<std::size_t>(succ[j]);
      if (ready_at[u] < fin) ready_at[u] = fin;
      if (--indeg[u] == 0) stack.push_back(succ[j]);
    }
  }
  if (done != n) throw std::logic_error("dependency cycle in pipeline schedule");

  ScheduleTrace trace;
  trace.config = cfg;
  trace.ops.resize(static_cast<std::size_t>(n));
  for (std::int64_t v = 0; v < n; ++v) {
    OpEvent& o = trace.ops[static_cast<std::size_t>(v)];
    o.micro_batch = static_cast<int>(v % m) + 1;
    o.kind = static_cast<OpKind>((v / m) % 2);
    o.stage = static_cast<int>((v / (2LL * m)) % p);
    o.epoch = static_cast<int>(v / per_epoch);
    o.start = start[static_cast<std::size_t>(v)];
    o.end = o.start + (o.kind == OpKind::FP ? cfg.fp_ticks(o.stage) : cfg.bp_ticks(o.stage));
  }
  // Total order: same-stage ops never share a start, so (start, stage) alone
  // is already unique; end and micro_batch complete the reference's key.
  std::sort(trace.ops.begin(), trace.ops.end(), [](const OpEvent& a, const OpEvent& b) {
    return std::tie(a.start, a.stage, a.end, a.micro_batch) <
           std::tie(b.start, b.stage, b.end, b.micro_batch);
  });
  trace.epoch_spans.assign(static_cast<std::size_t>(E),
                           {std::numeric_limits<Tick>::max(), Tick{0}});
  for (const OpEvent& o : trace.ops) {
    auto& sp = trace.epoch_spans[static_cast<std::size_t>(o.epoch)];
    sp.first = std::min(sp.first, o.start);
    sp.second = std::max(sp.second, o.end);
  }
  return trace;
}

// pipeline.cpp:180-249: maximal idle gaps per (epoch, stage), classified
// A (leading/trailing), B (before the stage's first BP), C (other).
std::vector<LinkedBubble> extract_bubbles_linked(const ScheduleTrace& trace) {
  const PipelineConfig& cfg = trace.config;
  const int p = cfg.num_stages, E = cfg.num_epochs;
  const std::size_t cells = static_cast<std::size_t>(p) * static_cast<std::size_t>(E);
  // CSR bucket of op indices per (epoch, stage), preserving time order.
  std::vector<std::int64_t> head(cells + 1, 0);
  for (const OpEvent& o : trace.ops) {
    if (o.epoch < 0 || o.epoch >= E || o.stage < 0 || o.stage >= p)
      throw ValidationError("ops", "op outside the configured epochs/stages");
    head[static_cast<std::size_t>(o.epoch) * p + o.stage + 1]++;
  }
  for (std::size_t c = 0; c < cells; ++c) head[c + 1] += head[c];
  std::vector<std::int64_t> fill(head.begin(), head.end() - 1);
  std::vector<std::int64_t> bucket(trace.ops.size());
  for (std::size_t i = 0; i < trace.ops.size(); ++i) {
    const OpEvent& o = trace.ops[i];
    bucket[static_cast<std::size_t>(fill[static_cast<std::size_t>(o.epoch) * p + o.stage]++)] =
        static_cast<std::int64_t>(i);
  }

  std::vector<LinkedBubble> out;
  for (int e = 0; e < E; ++e) {
    const Tick span_lo = trace.epoch_spans[e].first, span_hi = trace.epoch_spans[e].second;
    for (int s = 0; s < p; ++s) {
      const std::size_t c = static_cast<std::size_t>(e) * p + s;
      const double avail = cfg.available_memory(s);
      std::int64_t first_bp = -1;
      for (std::int64_t j = head[c]; j < head[c + 1]; ++j)
        if (trace.ops[static_cast<std::size_t>(bucket[j])].kind == OpKind::BP) {
          first_bp = bucket[j];
          break;
        }
      Tick cursor = span_lo;
      std::int64_t prev = -1;
      auto gap = [&](Tick lo, Tick hi, BubbleType t, std::int64_t a, std::int64_t b) {
        if (hi > lo) out.push_back(LinkedBubble{Bubble{s, e, lo, hi - lo, avail, t}, a, b});
      };
      for (std::int64_t j = head[c]; j < head[c + 1]; ++j) {
        const std::int64_t i = bucket[j];
        const OpEvent& o = trace.ops[static_cast<std::size_t>(i)];
        if (o.start > cursor) {
          const BubbleType t =
              prev < 0 ? BubbleType::A : (i == first_bp ? BubbleType::B : BubbleType::C);
          gap(cursor, o.start, t, prev, i);
        }
        cursor = o.end;
        prev = i;
      }
      gap(cursor, span_hi, BubbleType::A, prev, -1);
    }
  }
  // (start, stage) is unique: bubbles on one stage are disjoint.
  std::sort(out.begin(), out.end(), [](const LinkedBubble& a, const LinkedBubble& b) {
    return a.bubble.start != b.bubble.start ? a.bubble.start < b.bubble.start
                                            : a.bubble.stage < b.bubble.stage;
  });
  return out;
}

std::vector<Bubble> extract_bubbles(const ScheduleTrace& trace) {
  std::vector<Bubble> v;
  for (const LinkedBubble& lb : extract_bubbles_linked(trace)) v.push_back(lb.bubble);
  return v;
}

// pipeline.cpp:261-275: total bubble time over p x (last end - first start).
double bubble_rate(int p, const OpEvent* ops, std::size_t n_ops, const Bubble* b,
                   std::size_t n_b) {
  if (n_ops == 0) return 0.0;
  Tick lo = ops[0].start, hi = 0;
  for (std::size_t i = 0; i < n_ops; ++i) {
    lo = std::min(lo, ops[i].start);
    hi = std::max(hi, ops[i].end);
  }
  const Tick wall = hi - lo;
  if (wall <= 0) return 0.0;
  Tick idle = 0;
  for (std::size_t i = 0; i < n_b; ++i) idle += b[i].duration;
  return static_cast<double>(idle) / (static_cast<double>(p) * static_cast<double>(wall));
}

double bubble_rate(const ScheduleTrace& trace, const std::vector<Bubble>& bubbles) {
  return bubble_rate(trace.config.num_stages, trace.ops.data(), trace.ops.size(),
                     bubbles.data(), bubbles.size());
}

// pipeline.cpp:277-296: stage s holds w + (p - s) a, clamped to the GPU.
std::vector<double> default_stage_memory(int p, double total, double w, double a) {
  if (p < 1) throw ValidationError("num_stages", "must be >= 1");
  if (total < 0 || w < 0 || a < 0) throw ValidationError("memory_model", "inputs must be >= 0");
  const double peak = w + p * a;
  if (peak > total)
    throw ValidationError("memory_model", "infeasible: weight_mem + p * activation_mem (" +
                                              std::to_string(peak) +
                                              ") exceeds gpu_memory_total (" +
                                              std::to_string(total) + ")");
  std::vector<double> mem(static_cast<std::size_t>(p));
  for (int s = 0; s < p; ++s) mem[s] = std::min(w + (p - s) * a, total);
  return mem;
}

}  // namespace freeride

namespace freeride {

// 1F1B point-to-point plan of one stage (see freeride.h fr_p2p_op): group g
// (0..2m) precedes op g; it sends op g-1's output (FP -> stage+1 activation,
// BP -> stage-1 gradient) and receives op g's input (FP <- stage-1, BP <-
// stage+1).  Send first, then recv, inside one group.
std::vector<P2POp> pipeline_p2p_plan(int stage, int p, int m) {
  if (p < 1 || m < 1 || stage < 0 || stage >= p)
    throw ValidationError("stage", "need 0 <= stage < num_stages and m >= 1");
  const auto order = stage_issue_order(stage, p, m);
  std::vector<P2POp> plan;
  const int n = static_cast<int>(order.size());
  for (int g = 0; g <= n; ++g) {
    if (g > 0) {
      const auto [k, mb] = order[g - 1];
      if (k == OpKind::FP && stage + 1 < p) plan.push_back({g, true, stage + 1, OpKind::FP, mb});
      if (k == OpKind::BP && stage > 0) plan.push_back({g, true, stage - 1, OpKind::BP, mb});
    }
    if (g < n) {
      const auto [k, mb] = order[g];
      if (k == OpKind::FP && stage > 0) plan.push_back({g, false, stage - 1, OpKind::FP, mb});
      if (k == OpKind::BP && stage + 1 < p) plan.push_back({g, false, stage + 1, OpKind::BP, mb});
    }
  }
  return plan;
}

}  // namespace freeride
