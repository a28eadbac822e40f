// ΔT, cost savings S and the bubble-time breakdown (reference:
// src/metrics.cpp:11-178).
//
// The reference classifies each bubble by scanning every activity of the
// stage for every bubble and every idle piece (O(bubbles x activities^2)).
// Here each stage's intervals are sorted once and a bubble visits only the
// intervals that overlap it (back-scan bounded by a prefix max of ends);
// coverage of idle pieces is a +1/-1 sweep over the cut points and the
// serviceable-task count is a prefix sum -- same integers, near-linear time,
// so the breakdown of a full 128-epoch run is cheap enough to report live.
#include <algorithm>
#include <map>
#include <set>

#include "freeride.hpp"

namespace freeride {

void PriceConfig::validate() const {  // metrics.cpp:11-16
  if (!(price_server_1 > 0.0)) throw ValidationError("prices.price_server_1", "must be > 0");
  if (!(price_server_2 > 0.0)) throw ValidationError("prices.price_server_2", "must be > 0");
}

double time_increase(double t_no, double t_with) {  // metrics.cpp:18-22
  if (!(t_no > 0.0)) throw ValidationError("t_no_side", "baseline time must be > 0");
  return (t_with - t_no) / t_no;
}

CostBreakdown cost_savings(double t_no, double delta_t, const std::vector<TaskWork>& work,
                           const PriceConfig& prices) {  // metrics.cpp:24-44
  prices.validate();
  CostBreakdown cb;
  cb.c_no_side = prices.price_server_1 * (t_no / 3600.0);
  cb.c_extra = delta_t * cb.c_no_side;
  for (const TaskWork& w : work) {
    if (w.work <= 0.0) continue;
    if (!w.throughput_per_hour || !(*w.throughput_per_hour > 0.0))
      throw ValidationError("tasks." + w.id + ".reference_throughput",
                            "required for a task with nonzero work");
    cb.c_side_tasks += prices.price_server_2 * (w.work / *w.throughput_per_hour);
  }
  if (!(cb.c_no_side > 0.0)) throw ValidationError("t_no_side", "baseline cost must be > 0");
  cb.s = (cb.c_side_tasks - cb.c_extra) / cb.c_no_side;
  return cb;
}

namespace {

struct Span {
  Tick lo, hi;
};

// Intervals of one stage sorted by start, with a running max of ends so a
// query can stop scanning backwards once nothing earlier reaches `lo`.
struct SpanIndex {
  std::vector<Span> v;
  std::vector<Tick> max_hi;

  void finish() {
    std::sort(v.begin(), v.end(), [](const Span& a, const Span& b) { return a.lo < b.lo; });
    max_hi.resize(v.size());
    Tick m = 0;
    for (std::size_t i = 0; i < v.size(); ++i) max_hi[i] = m = (i ? std::max(m, v[i].hi) : v[i].hi);
  }

  template <class F>
  void overlapping(Tick lo, Tick hi, F&& f) const {  // iv.hi > lo && iv.lo < hi
    auto it = std::lower_bound(v.begin(), v.end(), hi,
                               [](const Span& s, Tick t) { return s.lo < t; });
    for (std::ptrdiff_t i = (it - v.begin()) - 1; i >= 0; --i) {
      if (max_hi[static_cast<std::size_t>(i)] <= lo) break;
      const Span& s = v[static_cast<std::size_t>(i)];
      if (s.hi > lo) f(s);
    }
  }
};

}  // namespace

std::vector<StageBreakdown> bubble_breakdown(const BreakdownInput& in) {  // metrics.cpp:62-178
  const int p = in.num_stages;
  std::vector<StageBreakdown> out(static_cast<std::size_t>(p));
  for (int s = 0; s < p; ++s) out[s].stage = s;
  auto stage_of = [&](int w) {
    if (w < 0 || w >= p) throw ValidationError("trace.worker", "worker outside the pipeline");
    return static_cast<std::size_t>(w);
  };

  std::map<std::string, double> est;
  for (const TaskProfile& tp : in.profiles) est[tp.task_id] = tp.est_memory;

  // Serviceable-task count per worker: +1 on assignment, -1 on StopSideTask.
  std::vector<std::vector<std::pair<Tick, int>>> ev(static_cast<std::size_t>(p));
  std::vector<std::set<std::string>> assigned(static_cast<std::size_t>(p));
  for (const AssignRecord& a : in.assigns) {
    ev[stage_of(a.worker)].push_back({a.t, +1});
    assigned[stage_of(a.worker)].insert(a.task);
  }
  for (const TransitionRecord& t : in.transitions)
    if (t.kind == TransitionKind::StopSideTask && t.worker >= 0) ev[stage_of(t.worker)].push_back({t.t, -1});
  std::vector<std::vector<Tick>> ev_t(static_cast<std::size_t>(p));
  std::vector<std::vector<int>> ev_sum(static_cast<std::size_t>(p));
  for (int s = 0; s < p; ++s) {
    std::sort(ev[s].begin(), ev[s].end());
    int run = 0;
    for (const auto& [t, d] : ev[s]) {
      ev_t[s].push_back(t);
      ev_sum[s].push_back(run += d);
    }
  }

  std::vector<SpanIndex> used(static_cast<std::size_t>(p)), over(static_cast<std::size_t>(p)),
      busy(static_cast<std::size_t>(p));
  for (const ActivityRecord& a : in.activities) {
    if (a.end <= a.start) continue;
    const std::size_t s = stage_of(a.worker);
    const bool gpu_work = a.kind == ActivityKind::Step || a.kind == ActivityKind::Kernel;
    (gpu_work ? used[s] : over[s]).v.push_back({a.start, a.end});
    busy[s].v.push_back({a.start, a.end});
  }
  for (int s = 0; s < p; ++s) {
    used[s].finish();
    over[s].finish();
    busy[s].finish();
  }

  std::vector<Tick> cuts;
  std::vector<std::pair<Tick, int>> sweep;
  for (const Bubble& b : in.bubbles) {
    const std::size_t s = stage_of(b.stage);
    StageBreakdown& sb = out[s];
    const Tick lo = b.start, hi = b.end();
    auto clip = [&](const Span& iv) { return std::max<Tick>(0, std::min(iv.hi, hi) - std::max(iv.lo, lo)); };
    used[s].overlapping(lo, hi, [&](const Span& iv) { sb.used_by_side_tasks += clip(iv); });
    over[s].overlapping(lo, hi, [&](const Span& iv) { sb.runtime_overhead += clip(iv); });

    // Vacuously OOM when nothing was ever assigned here (metrics.cpp:123-134).
    bool oom = true;
    for (const std::string& id : assigned[s]) {
      auto it = est.find(id);
      if ((it == est.end() ? 0.0 : it->second) < b.available_memory) {
        oom = false;
        break;
      }
    }

    cuts.assign({lo, hi});
    sweep.clear();
    busy[s].overlapping(lo, hi, [&](const Span& iv) {
      const Tick a = std::clamp(iv.lo, lo, hi), z = std::clamp(iv.hi, lo, hi);
      cuts.push_back(a);
      cuts.push_back(z);
      sweep.push_back({a, +1});
      sweep.push_back({z, -1});
    });
    const auto& et = ev_t[s];
    for (auto it = std::upper_bound(et.begin(), et.end(), lo); it != et.end() && *it < hi; ++it)
      cuts.push_back(*it);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    std::sort(sweep.begin(), sweep.end());

    std::size_t k = 0;
    int cover = 0;
    for (std::size_t i = 0; i + 1 < cuts.size(); ++i) {
      const Tick a = cuts[i], z = cuts[i + 1];
      while (k < sweep.size() && sweep[k].first <= a) cover += sweep[k++].second;
      if (cover > 0) continue;  // inside some activity
      auto ub = std::upper_bound(et.begin(), et.end(), a);
      const int live = ub == et.begin() ? 0 : ev_sum[s][static_cast<std::size_t>(ub - et.begin()) - 1];
      if (live > 0 || !oom)
        sb.idle_insufficient_time += z - a;
      else
        sb.idle_oom += z - a;
    }
  }
  return out;
}

}  // namespace freeride
