// The GPU bubble-harvesting runtime: one stage of a 1F1B pipeline of real
// tensor-core GEMMs on a high-priority stream, and one side-task worker
// that serves bubbles with bounded steps on a low-priority stream.
//
// This is the real-time counterpart of the reference's missing engine
// (engine.hpp:94-98, semantics SPEC.md:466-517 / SURVEY.md Appendix B):
//  * bubble signals come from the device (timeline.cu gap kernels) through a
//    host-mapped ring: BubbleStarted when the stage's previous op completes,
//    BubbleEnded when the next op's dependency arrives;
//  * the manager runs Alg. 2 (on_bubble_started / on_bubble_ended) over this
//    GPU's WorkerState, the task runs the five-state machine through
//    apply_transition, and every RunNextStep passes iterative_run's
//    program-directed gate (strict double compare, task.cpp:89-100) with the
//    *projected* device start time of the step as `now`, so steps can be
//    queued back to back without idling the GPU between them;
//  * a pause takes effect when the in-flight steps drain (last_paused is the
//    drain time) and framework_enforce (limits.cpp:21-26) judges it after the
//    grace period;
//  * imperative tasks (vtable interface_kind = FR_IMPERATIVE, imperative_run
//    task.cpp:102-106) run one preemptible GPU workload from StartSideTask on;
//    the pause is delivered on the device: the gap kernel that observes the
//    next op's dependency raises the bubble-end word the workload polls
//    between work items, so it lands within one work item (SPEC.md:170 allows
//    one kernel) without waiting for the host to see BubbleEnded.
// Everything is timed on the device (globaltimer / CUDA events).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.hpp"
#include "freeride_gpu.h"
#include "host/freeride.hpp"
#include "run_trace.hpp"
#include "runtime/standin.hpp"
#include "runtime/timeline.cuh"

using namespace freeride;
using namespace freeride::rt;

#define FR_CUDA_TRY_H(expr)                                                                  \
  do {                                                                                       \
    const cudaError_t fr_e_ = (expr);                                                        \
    if (fr_e_ != cudaSuccess)                                                                \
      return frcapi::fail(FR_ERR_CUDA_BASE + static_cast<int>(fr_e_),                        \
                          std::string(#expr) + ": " + cudaGetErrorString(fr_e_));            \
  } while (0)

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

std::int64_t host_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct HookError : std::runtime_error {
  int code;
  HookError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

void hook(int rc, const char* name) {
  if (rc != FR_OK) throw HookError(rc, std::string("side-task hook ") + name + " failed");
}

constexpr double kTick = 1e-9;  // runtime ticks are nanoseconds
constexpr std::uint32_t kRingSlots = 1u << 16;
constexpr std::uint32_t kBubbleIds = 1024;  // bubble ids per epoch in a ring code
constexpr Tick kGraceTicks = 100'000'000;  // LimitConfig::grace_period (0.1 s), ns ticks
constexpr double kGiB = 1024.0 * 1024.0 * 1024.0;

// Makes `pool` the device's current memory pool for the scope, so the
// stream-ordered allocations a task's hooks make (cudaMallocAsync) are
// accounted to the task.  Only the worker thread allocates while a run is in
// flight (the training program is captured graphs + fixed buffers).
struct PoolScope {
  int dev;
  cudaMemPool_t prev = nullptr;
  bool active = false;
  PoolScope(int d, cudaMemPool_t pool) : dev(d) {
    if (pool && cudaDeviceGetMemPool(&prev, dev) == cudaSuccess &&
        cudaDeviceSetMemPool(dev, pool) == cudaSuccess)
      active = true;
  }
  ~PoolScope() {
    if (active) cudaDeviceSetMemPool(dev, prev);
  }
};

struct Task {
  std::string id;
  fr_side_task_vtable vt{};
  void* user = nullptr;
  SideTaskRuntime rt;
  TaskProfile prof;
  bool initializing = false;
  double init_host_us = 0.0;  // host time of the last init hook call (FR_HARNESS_TRACE)
  double est_scale = 1.0;     // ΔT controller: measured / profiled step time at the current SM budget
  bool imperative() const { return vt.interface_kind == FR_IMPERATIVE; }
  cudaEvent_t init_a = nullptr, init_b = nullptr;
  bool init_recorded = false;
  int device = 0;
  cudaMemPool_t pool = nullptr;  // every allocation the task's hooks make
  double mem_limit = 0.0;        // GiB: profiled est_memory + headroom (check_memory)
  Disposition disp = Disposition::Active;
  double used_gib() const {
    std::size_t used = 0;
    if (pool) cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    return static_cast<double>(used) / kGiB;
  }
  ~Task() {
    if (init_a) cudaEventDestroy(init_a);
    if (init_b) cudaEventDestroy(init_b);
    if (vt.destroy && user) {
      PoolScope ps(device, pool);
      vt.destroy(user);
    }
    if (pool) cudaMemPoolDestroy(pool);
  }
};

// One timed record: `n` consecutive RunNextStep calls of `task` between the
// events a and b (n > 1 with cfg.step_group: no event between the steps).
struct StepRec {
  cudaEvent_t a, b;
  Task* task;
  int n = 1;
};

// Peer-linked pipeline mailbox (transport 1): one device allocation per
// stage, written by its neighbours.  Flags (uint32, the global epoch + 1 of
// the message) for dir 0 = FP input from stage s-1, dir 1 = BP input from
// stage s+1, dir 2 = epoch-end token from stage s-1, one per micro-batch;
// then the message slots of dirs 0 and 1.
constexpr std::size_t kFlagArea = 4096;
constexpr std::uint64_t kLinkTimeoutNs = 20'000'000'000ull;  // dependency-wait watchdog
constexpr int kMaxMb = 256;

struct Mailbox {
  char* base = nullptr;
  std::size_t msg_stride = 0;
  int m = 0;
  std::uint32_t* flag(int dir, int mb0) const {
    return reinterpret_cast<std::uint32_t*>(base) + dir * kMaxMb + mb0;
  }
  void* slot(int dir, int mb0) const {
    return base + kFlagArea + (static_cast<std::size_t>(dir) * m + mb0) * msg_stride;
  }
};

}  // namespace

struct fr_harness {
  fr_harness_config cfg{};
  int device = 0;
  cudaStream_t train = nullptr, side = nullptr;
  std::unique_ptr<StandIn> standin;
  RingSlot* ring = nullptr;       // host view
  RingSlot* ring_dev = nullptr;   // device view
  TimelineCtl* ctl = nullptr;
  std::uint64_t* stamp = nullptr;  // mapped
  std::uint32_t* flag = nullptr;   // mapped
  std::uint64_t* stamp_dev = nullptr;
  std::uint32_t* flag_dev = nullptr;
  std::uint32_t* pgate = nullptr;      // host-mapped gate of the standalone step profile
  std::uint32_t* pgate_dev = nullptr;
  std::uint32_t pgate_seq = 0;
  // transport 1 (peer-linked pipeline)
  Mailbox mbox, prev_mbox, next_mbox;
  std::size_t mbox_bytes = 0, msg_bytes = 0;
  bool linked = false;
  std::uint32_t epoch_base = 0;    // global epochs run so far (message sequence numbers)
  std::int64_t clock_off = 0;      // device_ns = host_ns + clock_off
  double clock_err = 0;
  std::int64_t launch_lat = 5000;  // host launch -> device start, ns

  // schedule of this stage (one epoch, undelayed)
  PipelineConfig pcfg;
  Tick fp = 0, bp = 0, span = 0;
  double fp_tflops = 0, bp_tflops = 0, rate = 0, avail = 0;
  std::vector<OpEvent> ops;              // issue order
  std::vector<std::int64_t> ready;       // dependency-ready offset per op
  std::vector<int> gap_bubble;           // per gap (2m+1): bubble index or -1
  std::vector<Bubble> bubbles;           // this stage, one epoch, relative ticks

  std::vector<WorkerState> workers;      // this process serves one worker
  std::map<std::string, std::unique_ptr<Task>> tasks;

  // The last run's decision records (device ns, absolute; converted to ns
  // from the run start -- ctl->run0_ns -- on export).
  struct SignalRec {
    std::int64_t t = 0;
    int kind = 0;  // 0 started, 1 ended
    std::uint32_t id = 0;
    std::int64_t duration = 0;
    bool looked_up = false, deferred = false;
    std::string task;
    TaskView view;
    std::vector<ManagerAction> acts;
  };
  struct GateRec {
    std::int64_t now = 0, bubble_end = 0, step_end = 0;
    double est = 0;
    std::int64_t est_ticks = 0;
    bool run = false;
    int signal = -1;
    std::string task;
  };
  std::vector<SignalRec> sig_log;
  std::vector<GateRec> gate_log;
  std::vector<TransitionRecord> tr_log;
  // per tr_log entry: step records completed when it was applied (a pause or
  // stop lands only after them; the export lifts its host-clock stamp to
  // their device end, see fr_harness_run_trace)
  std::vector<std::size_t> tr_recs_done;
  std::vector<std::size_t> rec_slices;  // per step record of the last run: first slice in step_se
  std::vector<KillRecord> kill_log;
  std::map<std::string, SideTaskState> run_start_state;
  std::vector<std::pair<std::string, std::pair<double, double>>> init_log;  // event seconds
  std::int64_t run0_dev = 0;
  bool last_with_tasks = false;
  int last_epochs = 0;
  // reclamation_delay: killed tasks whose pool pages are still held, and when they go
  std::vector<std::pair<Task*, std::int64_t>> reclaim;
  void reclaim_due(std::int64_t now) {
    for (auto it = reclaim.begin(); it != reclaim.end();) {
      if (now >= it->second) {
        if (it->first->pool) cudaMemPoolTrimTo(it->first->pool, 0);
        it = reclaim.erase(it);
      } else {
        ++it;
      }
    }
  }

  // last run
  std::vector<double> op_se, bubble_se, step_se;
  std::int64_t last_side_steps = 0, last_train_ops = 0;
  std::vector<cudaEvent_t> pool;
  std::size_t pool_used = 0;

  cudaEvent_t ev() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      ck(cudaEventCreate(&e), "cudaEventCreate");
      pool.push_back(e);
    }
    return pool[pool_used++];
  }

  ~fr_harness() {
    if (train) cudaStreamSynchronize(train);
    if (side) cudaStreamSynchronize(side);
    tasks.clear();
    standin.reset();
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (ring) cudaFreeHost(ring);
    if (stamp) cudaFreeHost(stamp);
    if (flag) cudaFreeHost(flag);
    if (pgate) cudaFreeHost(pgate);
    if (ctl) cudaFree(ctl);
    if (mbox.base) cudaFree(mbox.base);
    if (train) cudaStreamDestroy(train);
    if (side) cudaStreamDestroy(side);
  }

  void calibrate() {
    // device_ns - host_ns is bracketed by [g - t1, g - t0] for every stamp;
    // keep the tightest lower bound (error <= device->host visibility).
    std::int64_t lo = INT64_MIN, hi = INT64_MAX, best_rtt = INT64_MAX, lat = 0;
    for (std::uint32_t i = 1; i <= 64; ++i) {
      const std::int64_t t0 = host_ns();
      launch_stamp(stamp_dev, flag_dev, i, side);
      while (*reinterpret_cast<volatile std::uint32_t*>(flag) != i) {
      }
      const std::int64_t t1 = host_ns();
      const auto g = static_cast<std::int64_t>(*reinterpret_cast<volatile std::uint64_t*>(stamp));
      lo = std::max(lo, g - t1);
      hi = std::min(hi, g - t0);
      if (t1 - t0 < best_rtt) {
        best_rtt = t1 - t0;
      }
      lat = (i == 1) ? (g - t0) : std::min(lat, g - t0);
    }
    clock_off = lo;
    clock_err = static_cast<double>(std::max<std::int64_t>(0, hi - lo));
    launch_lat = std::max<std::int64_t>(1000, lat - lo);  // host call -> device start
  }

  std::int64_t dev_now() const { return host_ns() + clock_off; }

  void build_schedule_from(Tick fpt, Tick bpt) {
    const int p = cfg.num_stages, m = cfg.num_micro_batches, s = cfg.stage;
    pcfg = PipelineConfig{};
    pcfg.num_stages = p;
    pcfg.num_micro_batches = m;
    pcfg.fp_duration = {fpt};
    pcfg.bp_duration = {bpt};
    pcfg.num_epochs = 1;
    pcfg.tick_seconds = kTick;
    pcfg.gpu_memory_total = cfg.gpu_memory_total;
    const double gib = 1024.0 * 1024.0 * 1024.0;
    const double w = cfg.weight_mem >= 0 ? cfg.weight_mem
                                         : static_cast<double>(standin->weight_bytes()) * 8.0 / gib;
    const double a = cfg.activation_mem >= 0
                         ? cfg.activation_mem
                         : static_cast<double>(standin->activation_bytes()) / gib;
    pcfg.stage_memory = default_stage_memory(p, cfg.gpu_memory_total, w, a);
    const ScheduleTrace tr = build_schedule(pcfg);
    const auto linked = extract_bubbles_linked(tr);
    std::vector<Bubble> all;
    for (const auto& lb : linked) all.push_back(lb.bubble);
    rate = bubble_rate(tr, all);
    span = tr.epoch_spans[0].second - tr.epoch_spans[0].first;
    avail = pcfg.available_memory(s);
    fp = fpt;
    bp = bpt;
    // this stage's ops in issue order with their cross-stage ready times
    ops.clear();
    ready.clear();
    std::map<std::tuple<int, int, int>, const OpEvent*> at;  // (stage, kind, mb)
    for (const OpEvent& o : tr.ops) at[{o.stage, static_cast<int>(o.kind), o.micro_batch}] = &o;
    for (const auto& [k, mb] : stage_issue_order(s, p, m)) {
      const OpEvent* o = at.at({s, static_cast<int>(k), mb});
      ops.push_back(*o);
      std::int64_t r = 0;
      if (k == OpKind::FP && s > 0) r = at.at({s - 1, 0, mb})->end;
      if (k == OpKind::BP && s < p - 1) r = at.at({s + 1, 1, mb})->end;
      ready.push_back(r);
    }
    // map each of this stage's bubbles to the gap it occupies
    gap_bubble.assign(ops.size() + 1, -1);
    bubbles.clear();
    for (const auto& lb : linked) {
      if (lb.bubble.stage != s) continue;
      int gap = static_cast<int>(ops.size());  // trailing
      if (lb.next_op >= 0) {
        const OpEvent& nx = tr.ops[static_cast<std::size_t>(lb.next_op)];
        for (std::size_t i = 0; i < ops.size(); ++i)
          if (ops[i].kind == nx.kind && ops[i].micro_batch == nx.micro_batch) gap = static_cast<int>(i);
      }
      gap_bubble[static_cast<std::size_t>(gap)] = static_cast<int>(bubbles.size());
      bubbles.push_back(lb.bubble);
    }
  }

  Tick measure_op(bool is_fp, int reps) {
    std::vector<float> ms;
    for (int i = 0; i < reps + 2; ++i) {
      cudaEvent_t a = ev(), b = ev();
      ck(cudaEventRecord(a, train), "record");
      is_fp ? standin->launch_fp(train) : standin->launch_bp(train);
      ck(cudaEventRecord(b, train), "record");
      ck(cudaEventSynchronize(b), "sync");
      float t = 0;
      ck(cudaEventElapsedTime(&t, a, b), "elapsed");
      if (i >= 2) ms.push_back(t);
    }
    pool_used = 0;
    std::sort(ms.begin(), ms.end());
    return static_cast<Tick>(std::llround(static_cast<double>(ms[ms.size() / 2]) * 1e6));
  }

  // Bubble profiler (§4.3: "runs DeepSpeed ... and automatically
  // measures each bubble's duration"): first re-derive the op durations the
  // stage actually shows inside a pipeline (idle gaps let the GPU boost, so
  // back-to-back op timing is pessimistic), rebuild the schedule from them,
  // then dry-run `epochs` epochs and take each bubble's median duration as
  // its profiled duration -- the value StartSideTask carries as bubble end.
  void profile_in_pipeline(int epochs) {
    if (epochs <= 0) return;
    fr_run_report rep{};
    auto median = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v.empty() ? 0.0 : v[v.size() / 2];
    };
    for (int pass = 0; pass < 2; ++pass) {
      run(epochs, false, &rep);
      std::vector<double> fpd, bpd;
      for (std::size_t i = 0; i < op_se.size() / 2; ++i)
        (ops[i % ops.size()].kind == OpKind::FP ? fpd : bpd).push_back(op_se[2 * i + 1] - op_se[2 * i]);
      const Tick f = cfg.fp_ticks_override > 0 ? fp : static_cast<Tick>(std::llround(median(fpd) / kTick));
      const Tick b = cfg.bp_ticks_override > 0 ? bp : static_cast<Tick>(std::llround(median(bpd) / kTick));
      build_schedule_from(f, b);
    }
    run(epochs, false, &rep);
    bubbles_from_last_run();
  }

  // Each profiled bubble duration := its median over the last run's epochs
  // (used after a warm-up run *with* side tasks too: ops run slightly slower
  // when bubbles are busy, so the bubbles the worker will see are shorter).
  int bubbles_from_last_run() {
    const std::size_t nb = bubbles.size();
    if (nb == 0) return 0;
    const std::size_t epochs = bubble_se.size() / 2 / nb;
    if (epochs == 0 || bubble_se.size() / 2 != nb * epochs) return 0;
    for (std::size_t j = 0; j < nb; ++j) {
      std::vector<double> d;
      for (std::size_t e = 0; e < epochs; ++e) {
        const std::size_t k = e * nb + j;
        d.push_back(bubble_se[2 * k + 1] - bubble_se[2 * k]);
      }
      std::sort(d.begin(), d.end());
      bubbles[j].duration = static_cast<Tick>(std::llround(d[d.size() / 2] / kTick));
    }
    return static_cast<int>(epochs);
  }

  // GateEstimate (config.hpp:17,24): profiled mean by default, max if asked.
  double gate_est(const Task& t) const {
    return t.est_scale * (cfg.gate_estimate == 1 ? t.prof.max_per_step_duration.value_or(0.0)
                                                 : t.prof.est_per_step_duration.value_or(0.0));
  }

  // ---- ΔT-budgeted harvesting (cfg.dt_budget > 0)
  // On a power-capped B200 the pipeline's GEMMs run faster when their bubbles
  // idle (the power controller banks the idle time as boost); every joule a
  // side task spends in a bubble comes out of that boost.  The stage's own
  // ops are the sensor: each op's duration against the same op in the last
  // run without side tasks (op_ref) -> EWMA of the slowdown; the actuator is
  // the side tasks' SM budget (the same bytes moved by fewer SMs draw far
  // less power).  Multiplicative decrease above the budget, additive
  // increase well below it, a hold of 4 ops after every change.
  std::vector<double> op_ref;  // seconds per op index, last run without side tasks
  int ctrl_sms = 0;            // current SM budget (0: not started)
  double ctrl_ewma = 0.0;
  int ctrl_hold = 0;
  int sm_count = 148;
  void apply_sms(int sms) {
    const int old = ctrl_sms > 0 ? ctrl_sms : sm_count;
    ctrl_sms = sms;
    for (auto& kv : tasks) {
      Task& t = *kv.second;
      if (!t.vt.set_sm_budget || t.rt.state == SideTaskState::Stopped) continue;
      hook(t.vt.set_sm_budget(t.user, sms >= sm_count ? 0 : sms), "set_sm_budget");
      // step time grows sub-linearly as SMs go (per-SM bandwidth rises):
      // a first guess until measured steps re-anchor it
      t.est_scale *= std::pow(static_cast<double>(old) / static_cast<double>(sms), 0.7);
    }
  }
  void control(double growth) {
    const double a = 1.0 / 16.0;  // ~2 epochs of a 4-stage stage's 8 ops: the per-op clock jitter averages out
    ctrl_ewma = (1 - a) * ctrl_ewma + a * growth;
    if (ctrl_hold > 0) {
      --ctrl_hold;
      return;
    }
    const int lo = cfg.min_side_sms > 0 ? cfg.min_side_sms : 2;
    int next = ctrl_sms;
    if (ctrl_ewma > cfg.dt_budget) next = std::max(lo, static_cast<int>(ctrl_sms * 0.8));
    else if (ctrl_ewma < 0.5 * cfg.dt_budget) next = std::min(sm_count, ctrl_sms + std::max(2, ctrl_sms / 8));
    if (next != ctrl_sms) {
      apply_sms(next);
      ctrl_hold = 8;
    }
  }

  std::vector<Task*> step_task;  // task of each step of the last run (groups: equal slices)

  TaskView lookup(const std::string& id) const {
    auto it = tasks.find(id);
    if (it == tasks.end()) throw frcapi::CallbackStatus(FR_ERR_NOT_FOUND);
    return TaskView{it->second->rt.state, it->second->initializing};
  }

  void run(int epochs, bool with_tasks, fr_run_report* rep);
};

namespace {

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
  return static_cast<double>(ms) * 1e-3;
}

}  // namespace

void fr_harness::run(int epochs, bool with_tasks, fr_run_report* rep) {
  if (cfg.transport == 1 && !linked)
    throw std::runtime_error("peer-linked harness: call fr_harness_link before running");
  pool_used = 0;
  sig_log.clear();
  gate_log.clear();
  tr_log.clear();
  tr_recs_done.clear();
  kill_log.clear();
  init_log.clear();
  run_start_state.clear();
  for (const auto& kv : tasks) run_start_state[kv.first] = kv.second->rt.state;
  last_with_tasks = with_tasks;
  last_epochs = epochs;
  std::memset(ring, 0, sizeof(RingSlot) * kRingSlots);
  ck(cudaMemset(&ctl->end_seq, 0, 2 * sizeof(std::uint32_t)), "end_seq / link_timeouts reset");
  // the wait kernels' L1/shared split: max-L1 only if every task wants it
  bool all_l1 = false;
  for (const auto& kv : tasks) {
    if (kv.second->rt.state == SideTaskState::Stopped) continue;
    if (kv.second->vt.carveout_hint != 0) {
      all_l1 = false;
      break;
    }
    all_l1 = true;
  }
  set_wait_kernel_carveout(all_l1 ? cudaSharedmemCarveoutMaxL1 : cudaSharedmemCarveoutMaxShared);
  calibrate();
  reclaim_due(dev_now());
  // this harness's streams only: a device-wide sync would wait on a linked
  // neighbour's dependency spin in the same process (deadlock)
  ck(cudaStreamSynchronize(train), "pre-run sync");
  ck(cudaStreamSynchronize(side), "pre-run sync");
  const int nops = static_cast<int>(ops.size());
  const int ngaps = nops + 1;

  // ---- training-stream program for all epochs (enqueued by its own thread,
  //      as a training framework would, so the worker never blocks on it)
  struct EpochEvents {
    std::vector<cudaEvent_t> op_start, op_end;
    std::vector<cudaEvent_t> send_a, send_b;  // transport 1: the op's message copy to its neighbour
    cudaEvent_t end;
  };
  std::vector<EpochEvents> eev(static_cast<std::size_t>(epochs));
  for (auto& e : eev) {
    e.op_start.resize(static_cast<std::size_t>(nops));
    e.op_end.resize(static_cast<std::size_t>(nops));
    for (int i = 0; i < nops; ++i) {
      e.op_start[i] = ev();
      e.op_end[i] = ev();
    }
    if (cfg.transport == 1) {
      e.send_a.resize(static_cast<std::size_t>(nops));
      e.send_b.resize(static_cast<std::size_t>(nops));
      for (int i = 0; i < nops; ++i) {
        e.send_a[i] = ev();
        e.send_b[i] = ev();
      }
    }
    e.end = ev();
  }
  cudaEvent_t run_start = ev();
  std::int64_t n_events = 0;
  for (int g = 0; g < ngaps; ++g)
    if (gap_bubble[static_cast<std::size_t>(g)] >= 0) n_events += 2;
  n_events *= epochs;
  if (n_events >= static_cast<std::int64_t>(kRingSlots))
    throw std::runtime_error("too many epochs for the event ring in one run");

  std::atomic<bool> train_failed{false};
  std::atomic<std::int64_t> enq_ops{0};  // ops whose end event the trainer has recorded
  std::string train_err;
  std::thread trainer([&] {
    try {
      ck(cudaSetDevice(device), "cudaSetDevice");
      ck(cudaEventRecord(run_start, train), "record");
      std::int64_t slot = 0;
      if (cfg.transport == 1) {
        // Peer-linked 1F1B: wait on this stage's mailbox flag for the op's
        // cross-stage input, run the op, copy its output into the
        // neighbour's mailbox slot (copy engine over NVLink / peer memory,
        // no SMs) and raise the neighbour's flag.  The epoch-end token runs
        // down the chain from stage 0 (the last stage to finish an epoch).
        const int p = cfg.num_stages, st = cfg.stage;
        for (int e = 0; e < epochs; ++e) {
          const std::uint32_t seq = epoch_base + static_cast<std::uint32_t>(e) + 1;
          for (int g = 0; g < ngaps; ++g) {
            LinkWaitArgs a{};
            a.ctl = ctl;
            a.ring = ring_dev;
            a.ring_mask = kRingSlots - 1;
            a.slot_start = a.slot_end = -1;
            a.seq = seq;
            a.mode = (e == 0 && g == 0) ? 2 : 0;
            a.timeout_ns = kLinkTimeoutNs;
            const int b = gap_bubble[static_cast<std::size_t>(g)];
            if (b >= 0) {
              const std::uint32_t id = static_cast<std::uint32_t>(e) * kBubbleIds + static_cast<std::uint32_t>(b);
              a.slot_start = slot++;
              a.slot_end = slot++;
              a.code_start = ring_code(kEvBubbleStart, id);
              a.code_end = ring_code(kEvBubbleEnd, id);
              a.end_token = id + 1;
            }
            if (g < nops) {
              const OpEvent& op = ops[static_cast<std::size_t>(g)];
              const int mb0 = op.micro_batch - 1;
              if (op.kind == OpKind::FP && st > 0) a.flag = mbox.flag(0, mb0);
              if (op.kind == OpKind::BP && st < p - 1) a.flag = mbox.flag(1, mb0);
              if (a.flag || b >= 0) launch_link_wait(a, train);
              ck(cudaEventRecord(eev[e].op_start[g], train), "record");
              op.kind == OpKind::FP ? standin->launch_fp(train) : standin->launch_bp(train);
              ck(cudaEventRecord(eev[e].op_end[g], train), "record");
              enq_ops.fetch_add(1, std::memory_order_release);
              const Mailbox* to = nullptr;
              int dir = 0;
              if (op.kind == OpKind::FP && st < p - 1) to = &next_mbox, dir = 0;
              if (op.kind == OpKind::BP && st > 0) to = &prev_mbox, dir = 1;
              if (to) {
                ck(cudaEventRecord(eev[e].send_a[g], train), "record");
                ck(cudaMemcpyAsync(to->slot(dir, mb0), standin->output(), msg_bytes,
                                   cudaMemcpyDefault, train), "send");
                ck(cudaEventRecord(eev[e].send_b[g], train), "record");
                launch_link_signal(to->flag(dir, mb0), seq, train);
              }
            } else {
              if (st > 0) a.flag = mbox.flag(2, 0);
              if (a.flag || b >= 0) launch_link_wait(a, train);
              if (st < p - 1) launch_link_signal(next_mbox.flag(2, 0), seq, train);
              ck(cudaEventRecord(eev[e].end, train), "record");
            }
          }
        }
        ck(cudaGetLastError(), "training enqueue");
        return;
      }
      for (int e = 0; e < epochs; ++e) {
        for (int g = 0; g < ngaps; ++g) {
          GapArgs a{};
          a.ctl = ctl;
          a.ring = ring_dev;
          a.ring_mask = kRingSlots - 1;
          const int b = gap_bubble[static_cast<std::size_t>(g)];
          a.slot_start = a.slot_end = -1;
          if (b >= 0) {
            const std::uint32_t id = static_cast<std::uint32_t>(e) * kBubbleIds + static_cast<std::uint32_t>(b);
            a.slot_start = slot++;
            a.slot_end = slot++;
            a.code_start = ring_code(kEvBubbleStart, id);
            a.code_end = ring_code(kEvBubbleEnd, id);
            a.end_token = id + 1;  // bubble ids grow monotonically through the run
          }
          a.span_ns = span;
          if (g < nops) {
            a.mode = (e == 0 && g == 0) ? 2 : 0;
            a.ready_ns = ready[static_cast<std::size_t>(g)];
            launch_gap(a, train);
            ck(cudaEventRecord(eev[e].op_start[g], train), "record");
            ops[static_cast<std::size_t>(g)].kind == OpKind::FP ? standin->launch_fp(train)
                                                               : standin->launch_bp(train);
            ck(cudaEventRecord(eev[e].op_end[g], train), "record");
            enq_ops.fetch_add(1, std::memory_order_release);
          } else {
            a.mode = 1;
            a.ready_ns = 0;
            launch_gap(a, train);
            ck(cudaEventRecord(eev[e].end, train), "record");
          }
        }
      }
      ck(cudaGetLastError(), "training enqueue");
    } catch (const std::exception& ex) {
      train_err = ex.what();
      train_failed = true;
    }
  });

  // ---- the worker: Alg. 2 + iterative interface, in real time
  WorkerState& ws = workers[0];
  // Alg. 2's task lookup, remembering what it showed the manager (signal log)
  std::string seen_id;
  TaskView seen_view;
  bool looked = false;
  const auto view = [&](const std::string& id) {
    TaskView v = lookup(id);
    if (!looked) {
      looked = true;
      seen_id = id;
      seen_view = v;
    }
    return v;
  };
  // every transition the worker applies, stamped (device ns) for the run
  // trace.  Stamps are the decision's device time (a BubbleStarted's signal
  // time, a step's projected start, a pause's drain) made non-decreasing per
  // task, so the trace's time order is the order they were applied in (a
  // BubbleStarted held while a pause drained is applied after that pause).
  std::map<std::string, std::int64_t> last_stamp;
  std::size_t recs_done = 0;  // step records [0, recs_done) have completed
  const auto trans = [&](Task& t, TransitionKind k, std::int64_t now) {
    auto it = last_stamp.find(t.id);
    if (it != last_stamp.end()) now = std::max(now, it->second);
    last_stamp[t.id] = now;
    apply_transition(t.rt, k, now);
    tr_log.push_back(TransitionRecord{now, t.id, k, cfg.stage});
    tr_recs_done.push_back(recs_done);
  };
  const auto log_signal = [&](std::int64_t t, int kind, std::uint32_t id, std::int64_t dur, bool deferred,
                              const std::vector<ManagerAction>& acts) {
    SignalRec r;
    r.t = t;
    r.kind = kind;
    r.id = id;
    r.duration = dur;
    r.deferred = deferred;
    r.looked_up = looked;
    r.task = looked ? seen_id : std::string();
    r.view = seen_view;
    r.acts = acts;
    sig_log.push_back(std::move(r));
    looked = false;
  };
  int cur_signal = -1;                 // the BubbleStarted that started the running task
  Task* guard_task = nullptr;          // ArmInitGuard (manager.hpp:58): init in flight at a bubble end
  std::int64_t guard_due = 0;
  const Tick grace = cfg.grace_ns > 0 ? cfg.grace_ns : kGraceTicks;
  std::vector<StepRec> steps;
  std::deque<std::size_t> inflight;  // indices into steps
  std::vector<std::pair<std::int64_t, std::int64_t>> init_spans;
  Task* running = nullptr;
  std::int64_t bubble_end_dev = 0;   // device ns (profiled end)
  std::int64_t proj_end_dev = 0;     // projected end of the queued steps
  bool pause_pending = false, gate_closed = false, kill_judged = false;
  std::int64_t pause_issued_dev = 0;
  std::int64_t launched = 0, completed = 0, pauses = 0, kills = 0;
  double dispatch_ns = 0;
  std::int64_t next_slot = 0;
  double units = 0;
  // Step groups: up to G consecutive steps of a task go out between one pair
  // of timing events.  An event between two kernels serialises them (the next
  // launch waits for the event), which costs ~2-3 us per step and defeats a
  // kernel's programmatic dependent launch; grouped steps run back to back.
  const int group = std::max(1, cfg.step_group);
  const int depth = std::max(std::max(1, cfg.max_inflight_steps), group > 1 ? 2 * group : 1);
  std::int64_t inflight_steps = 0;  // dispatched, not yet completed (all records)
  std::int64_t open_rec = -1;       // record still collecting steps (no end event yet)
  auto close_group = [&] {
    if (open_rec < 0) return;
    ck(cudaEventRecord(steps[static_cast<std::size_t>(open_rec)].b, side), "record");
    inflight.push_back(static_cast<std::size_t>(open_rec));
    open_rec = -1;
  };

  auto task_of = [&](const std::string& id) -> Task& { return *tasks.at(id); };
  // the op-slowdown sensor runs whenever a no-task reference exists (its mean
  // is reported as op_growth); the controller acts on it only with a budget
  const bool sensing = with_tasks && op_ref.size() == static_cast<std::size_t>(nops);
  const bool controlled = sensing && cfg.dt_budget > 0;
  if (controlled && ctrl_sms == 0) {
    ctrl_sms = cfg.side_sms > 0 ? std::min(cfg.side_sms, sm_count) : sm_count;
    ctrl_ewma = 0.0;
  }
  std::int64_t meas_idx = 0;          // next op whose duration feeds the controller
  double growth_sum = 0, sms_sum = 0;
  std::int64_t growth_n = 0;
  const auto measure_ops = [&] {
    const std::int64_t ready = enq_ops.load(std::memory_order_acquire);
    while (meas_idx < ready) {
      const std::size_t e = static_cast<std::size_t>(meas_idx / nops), g = static_cast<std::size_t>(meas_idx % nops);
      const cudaError_t q = cudaEventQuery(eev[e].op_end[g]);
      if (q == cudaErrorNotReady) break;
      ck(q, "op event");
      const double d = elapsed_s(eev[e].op_start[g], eev[e].op_end[g]);
      const double growth = d / op_ref[g] - 1.0;
      growth_sum += growth;
      sms_sum += ctrl_sms;
      ++growth_n;
      if (controlled) control(growth);
      ++meas_idx;
    }
  };
  // imperative work is counted by the workload itself (rows, pixels, ...)
  std::map<Task*, double> work_before;
  for (auto& kv : tasks)
    if (kv.second->imperative() && kv.second->vt.work_done && with_tasks) {
      double u = 0;
      hook(kv.second->vt.work_done(kv.second->user, side, &u), "work_done");
      work_before[kv.second.get()] = u;
    }
  std::uint32_t cur_token = 0;  // bubble-end token the running imperative workload stops at
  auto stop_task = [&](Task& t, Tick now) {
    trans(t, TransitionKind::StopSideTask, now);
    {
      PoolScope ps(device, t.pool);
      hook(t.vt.stop ? t.vt.stop(t.user) : FR_OK, "stop");
    }
    t.disp = Disposition::Completed;
    if (ws.current_task && *ws.current_task == t.id) ws.current_task.reset();  // Appendix B rule 8
    if (running == &t) running = nullptr;
  };
  std::int64_t kills_oom = 0, kills_timeout = 0, kills_init = 0;
  std::function<void(Task&, Disposition)> kill;  // defined below (needs drain_completions)
  auto drain_completions = [&] {
    while (!inflight.empty()) {
      const cudaError_t q = cudaEventQuery(steps[inflight.front()].b);
      if (q == cudaErrorNotReady) break;
      ck(q, "step event");
      Task* st = steps[inflight.front()].task;
      const int n = steps[inflight.front()].n;
      if (controlled && !st->imperative() && n > 0) {
        const double prof_est = cfg.gate_estimate == 1 ? st->prof.max_per_step_duration.value_or(0.0)
                                                       : st->prof.est_per_step_duration.value_or(0.0);
        const double per = elapsed_s(steps[inflight.front()].a, steps[inflight.front()].b) / n;
        if (prof_est > 0 && per > 0) st->est_scale = 0.7 * st->est_scale + 0.3 * (per / prof_est);
      }
      recs_done = std::max(recs_done, inflight.front() + 1);
      inflight.pop_front();
      inflight_steps -= n;
      completed += n;
      if (!st->imperative()) units += n * st->vt.work_units_per_step;  // the completing steps' own task
      st->rt.steps_completed += n;  // counted at step end (task.hpp:55); imperative: kernels
      // Re-anchor the projection: the next queued step started when this one
      // ended (~now), so drift from mis-estimated step times cannot build up.
      if (!inflight.empty() && !st->imperative()) {
        const double est = gate_est(*st);
        proj_end_dev = std::max<std::int64_t>(
            proj_end_dev, dev_now() + static_cast<std::int64_t>(std::llround(est / kTick)) *
                                          inflight_steps);
      }
      if (running && !running->imperative()) {
        int32_t done = 0;
        if (running->vt.finished) hook(running->vt.finished(running->user, running->rt.steps_completed, &done), "finished");
        if (done) stop_task(*running, dev_now());
      }
    }
  };
  // Framework-enforced kill (limits.cpp:13-26): cancel the task's in-flight
  // work (its cancel hook), drain its stream, StopSideTask, release its pool.
  kill = [&](Task& t, Disposition d) {
    const std::int64_t t_kill = dev_now();
    kill_log.push_back(KillRecord{t_kill, t.id, cfg.stage,
                                  d == Disposition::KilledOom ? KillReason::Oom
                                  : d == Disposition::KilledPauseTimeout ? KillReason::PauseTimeout
                                                                         : KillReason::InitTimeout});
    if (t.vt.cancel) hook(t.vt.cancel(t.user), "cancel");
    ck(cudaStreamSynchronize(side), "kill drain");
    drain_completions();
    if (t.rt.state != SideTaskState::Stopped) {
      trans(t, TransitionKind::StopSideTask, t_kill);
      PoolScope ps(device, t.pool);
      hook(t.vt.stop ? t.vt.stop(t.user) : FR_OK, "stop");
    }
    ck(cudaStreamSynchronize(side), "kill release");
    // memory goes back after LimitConfig::reclamation_delay (limits.hpp:12)
    if (cfg.reclamation_delay_ns > 0)
      reclaim.emplace_back(&t, t_kill + cfg.reclamation_delay_ns);
    else if (t.pool)
      cudaMemPoolTrimTo(t.pool, 0);
    if (guard_task == &t) guard_task = nullptr;
    t.disp = d;
    t.initializing = false;
    if (ws.current_task && *ws.current_task == t.id) ws.current_task.reset();  // Appendix B rule 8
    ws.task_queue.erase(std::remove(ws.task_queue.begin(), ws.task_queue.end(), t.id), ws.task_queue.end());
    if (running == &t) running = nullptr;
    pause_pending = false;
    gate_closed = false;
    ++kills;
    ++(d == Disposition::KilledOom ? kills_oom : d == Disposition::KilledPauseTimeout ? kills_timeout : kills_init);
  };
  auto oom = [&](Task& t) {  // check_memory (limits.cpp:13-15), strict exceedance
    if (check_memory(t.used_gib(), t.mem_limit) == MemCheck::OomKill) {
      kill(t, Disposition::KilledOom);
      return true;
    }
    return false;
  };
  auto finish_pause = [&] {
    if (!pause_pending || !inflight.empty()) return;
    pause_pending = false;
    if (running && running->rt.state == SideTaskState::Running) {
      const Tick now = dev_now();
      trans(*running, TransitionKind::PauseSideTask, now);
      hook(running->vt.pause ? running->vt.pause(running->user) : FR_OK, "pause");
      ++pauses;
    }
    running = nullptr;
  };
  auto finish_init = [&] {
    for (auto& kv : tasks) {
      Task& t = *kv.second;
      if (!t.initializing) continue;
      const cudaError_t q = cudaEventQuery(t.init_b);
      if (q == cudaErrorNotReady) continue;
      ck(q, "init event");
      t.initializing = false;
      trans(t, TransitionKind::InitSideTask, dev_now());
      t.rt.assigned_worker = 0;
      if (guard_task == &t) guard_task = nullptr;  // the init landed before the guard fired
    }
  };

  // Alg. 2 lines 8-17 on a BubbleStarted signal at device time t_dev.
  bool deferred_start = false;
  std::int64_t deferred_t = 0;
  std::uint32_t deferred_id = 0;
  auto start_bubble = [&](std::int64_t t_dev, std::uint32_t id, bool deferred) {
    const Bubble& pb = bubbles[id % kBubbleIds];
    Bubble b = pb;
    b.epoch = static_cast<int>(id / kBubbleIds);
    b.start = t_dev;
    looked = false;
    const std::vector<ManagerAction> acts = on_bubble_started(ws, b, view);
    log_signal(t_dev, 0, id, pb.duration, deferred, acts);
    for (const ManagerAction& act : acts) {
      Task& t = task_of(act.task_id);
      if (act.kind == ManagerActionKind::IssueInit) {
        if (!t.init_a) {
          ck(cudaEventCreate(&t.init_a), "init event");
          ck(cudaEventCreate(&t.init_b), "init event");
        }
        ck(cudaEventRecord(t.init_a, side), "record");
        {
          const auto h0 = std::chrono::steady_clock::now();
          PoolScope ps(device, t.pool);
          hook(t.vt.init(t.user, side), "init");
          t.init_host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
        }
        ck(cudaEventRecord(t.init_b, side), "record");
        t.initializing = true;
        t.init_recorded = true;
        oom(t);
      } else if (act.kind == ManagerActionKind::IssueStart) {
        trans(t, TransitionKind::StartSideTask, t_dev);
        cur_signal = static_cast<int>(sig_log.size()) - 1;
        hook(t.vt.start ? t.vt.start(t.user) : FR_OK, "start");
        running = &t;
        // StartSideTask carries the bubble end (§4.5); a harvest
        // fraction < 1 hands the gate only the bubble's first part
        const double frac = cfg.harvest_fraction > 0 && cfg.harvest_fraction < 1 ? cfg.harvest_fraction : 1.0;
        bubble_end_dev = t_dev + static_cast<std::int64_t>(std::llround(frac * static_cast<double>(pb.duration)));
        proj_end_dev = 0;
        gate_closed = false;
        cur_token = id + 1;
      }
    }
  };

  while (true) {
    if (train_failed) {
      trainer.join();
      throw std::runtime_error("training stream: " + train_err);
    }
    // 1. bubble signals from the device
    volatile RingSlot* sl = ring + (static_cast<std::uint64_t>(next_slot) & (kRingSlots - 1));
    // acquire: the payload (code, t_ns) is read only after the published seq
    // (the device writes it behind a system-scope fence); on a weakly ordered
    // host (aarch64) plain loads could pair a stale payload with a fresh seq
    if (next_slot < n_events &&
        __atomic_load_n(const_cast<std::uint32_t*>(&sl->seq), __ATOMIC_ACQUIRE) ==
            static_cast<std::uint32_t>(next_slot + 1)) {
      const std::uint32_t code = sl->code;
      const auto t_dev = static_cast<std::int64_t>(sl->t_ns);
      const std::int64_t seen = host_ns();
      ++next_slot;
      clock_off = std::max(clock_off, t_dev - seen);  // causality tightens the bound
      const std::uint32_t kind = code >> 28, id = code & 0x0FFFFFFFu;
      if (with_tasks && kind == kEvBubbleStart && pause_pending) {
        // The previous bubble's pause is still draining (a step in flight):
        // hold this BubbleStarted until the pause lands, so Alg. 2 sees the
        // task PAUSED exactly as it would had the pause been instantaneous.
        deferred_start = true;
        deferred_t = t_dev;
        deferred_id = id;
      } else if (with_tasks && kind == kEvBubbleStart) {
        start_bubble(t_dev, id, false);
      } else if (with_tasks && kind == kEvBubbleEnd && deferred_start) {
        deferred_start = false;  // the held bubble ended before the pause landed
        looked = false;
        log_signal(t_dev, 1, id, 0, true, on_bubble_ended(ws, t_dev, view));
      } else if (with_tasks && kind == kEvBubbleEnd) {
        looked = false;
        const std::vector<ManagerAction> acts = on_bubble_ended(ws, t_dev, view);
        log_signal(t_dev, 1, id, 0, false, acts);
        for (const ManagerAction& act : acts) {
          if (act.kind == ManagerActionKind::IssuePause) {
            pause_pending = true;
            kill_judged = false;
            pause_issued_dev = t_dev;
          } else if (act.kind == ManagerActionKind::ArmInitGuard) {
            // engine rule: at issue + grace the init
            // must have landed, else KilledInitTimeout
            guard_task = &task_of(act.task_id);
            guard_due = t_dev + grace;
          }
        }
      }
    }
    if (with_tasks && deferred_start && !pause_pending) {
      deferred_start = false;
      start_bubble(deferred_t, deferred_id, true);
    }
    if (!with_tasks && next_slot >= n_events) break;
    // 2. step completions, init completion, pause drains
    if (with_tasks) {
      drain_completions();
      finish_init();
      finish_pause();
      if (sensing) measure_ops();
      // 3a. imperative: one preemptible workload at a time (each loops over
      // its input until the device-side stop; a queued second launch would
      // only run -- and exit -- after the next op has taken the SMs)
      while (running && running->imperative() && !pause_pending &&
             running->rt.state == SideTaskState::Running && inflight.empty()) {
        const std::int64_t h0 = host_ns();
        imperative_run(running->rt, h0 + clock_off, 0);  // RUNNING precondition (task.cpp:102)
        fr_preempt pre{&ctl->end_seq, cur_token, 0};
        StepRec r{ev(), ev(), running};
        ck(cudaEventRecord(r.a, side), "record");
        {
          PoolScope ps(device, running->pool);
          hook(running->vt.run_gpu_workload(running->user, side, &pre), "run_gpu_workload");
        }
        ck(cudaEventRecord(r.b, side), "record");
        steps.push_back(r);
        inflight.push_back(steps.size() - 1);
        ++inflight_steps;
        ++launched;
        dispatch_ns += static_cast<double>(host_ns() - h0);
        if (oom(*r.task)) break;
      }
      // 3b. iterative dispatch: the program-directed gate at the projected start time
      while (running && !running->imperative() && !pause_pending && !gate_closed &&
             running->rt.state == SideTaskState::Running &&
             inflight_steps < depth) {
        const std::int64_t h0 = host_ns();
        const std::int64_t now = h0 + clock_off;
        const std::int64_t start = std::max(now + launch_lat, proj_end_dev);
        const double est = gate_est(*running);
        const Tick est_ticks = static_cast<Tick>(std::llround(est / kTick));
        const IterativeDecision d = iterative_run(running->rt, bubble_end_dev, start, est, kTick, est_ticks);
        {
          GateRec g;
          g.now = start;
          g.bubble_end = bubble_end_dev;
          g.est = est;
          g.est_ticks = est_ticks;
          g.run = d.run;
          g.step_end = d.step_end;
          g.signal = cur_signal;
          g.task = running->id;
          gate_log.push_back(std::move(g));
        }
        if (!d.run) {
          gate_closed = true;  // yield until the next transition
          break;
        }
        const bool extend = open_rec >= 0 && steps[static_cast<std::size_t>(open_rec)].task == running &&
                            steps[static_cast<std::size_t>(open_rec)].n < group;
        if (!extend) {
          close_group();
          steps.push_back(StepRec{ev(), ev(), running, 0});
          open_rec = static_cast<std::int64_t>(steps.size()) - 1;
          ck(cudaEventRecord(steps.back().a, side), "record");
        }
        {
          PoolScope ps(device, running->pool);
          hook(running->vt.run_next_step(running->user, side), "run_next_step");
        }
        StepRec& r = steps[static_cast<std::size_t>(open_rec)];
        ++r.n;
        Task* rt = r.task;
        if (r.n >= group) close_group();
        trans(*running, TransitionKind::RunNextStep, start);
        ++inflight_steps;
        proj_end_dev = d.step_end;
        ++launched;
        dispatch_ns += static_cast<double>(host_ns() - h0);
        if (oom(*rt)) break;
      }
      close_group();  // nothing else may enter the side stream inside a group
      // framework-enforced limit: a pause not observed within the grace
      // period is a Kill (limits.cpp:21-26): the task's cancel hook stops its
      // in-flight kernels (cooperative ones exit at once), then it is stopped
      // and its memory pool released.
      // the init guard: InitSideTask still running one grace period after the
      // bubble it was issued in ended -> KilledInitTimeout (engine.hpp:16)
      if (guard_task) {
        finish_init();
        if (guard_task && guard_task->initializing && dev_now() >= guard_due) {
          Task* g = guard_task;
          guard_task = nullptr;
          kill(*g, Disposition::KilledInitTimeout);
        }
      }
      if (!reclaim.empty()) reclaim_due(dev_now());
      if (pause_pending && !kill_judged && running &&
          framework_enforce(running->rt.last_paused, pause_issued_dev, dev_now(), grace) == Enforce::Kill) {
        kill_judged = true;
        kill(*running, Disposition::KilledPauseTimeout);
      }
      if (next_slot >= n_events && inflight.empty() && !pause_pending && !guard_task) break;
    }
  }
  trainer.join();
  if (train_failed) throw std::runtime_error("training stream: " + train_err);
  ck(cudaStreamSynchronize(train), "train sync");
  ck(cudaStreamSynchronize(side), "side sync");
  drain_completions();
  finish_init();
  for (auto& kv : tasks) {  // StopSideTask freed the task's memory: give the pages back
    const bool held = std::any_of(reclaim.begin(), reclaim.end(),
                                  [&](const auto& x) { return x.first == kv.second.get(); });
    if (kv.second->rt.state == SideTaskState::Stopped && kv.second->pool && !held)
      cudaMemPoolTrimTo(kv.second->pool, 0);
  }
  if (cfg.transport == 1) {
    std::uint32_t timeouts = 0;
    ck(cudaMemcpy(&timeouts, &ctl->link_timeouts, sizeof(timeouts), cudaMemcpyDeviceToHost), "timeouts");
    if (timeouts)
      throw std::runtime_error("peer-linked pipeline: " + std::to_string(timeouts) +
                               " dependency waits timed out (a neighbour stage never signalled)");
  }
  {
    std::uint64_t r0 = 0;
    ck(cudaMemcpy(&r0, &ctl->run0_ns, sizeof(r0), cudaMemcpyDeviceToHost), "run0");
    run0_dev = static_cast<std::int64_t>(r0);
  }
  for (auto& [t, before] : work_before) {
    double u = before;
    hook(t->vt.work_done(t->user, side, &u), "work_done");
    units += u - before;
  }

  // ---- device-timed accounting
  op_se.clear();
  bubble_se.clear();
  step_se.clear();
  BreakdownInput bi;
  bi.num_stages = 1;
  cudaEvent_t prev_end = run_start;  // the leading bubble starts at the epoch base
  for (int e = 0; e < epochs; ++e) {
    for (int i = 0; i < nops; ++i) {
      const double a = elapsed_s(run_start, eev[e].op_start[i]);
      const double b = elapsed_s(run_start, eev[e].op_end[i]);
      op_se.push_back(a);
      op_se.push_back(b);
      if (gap_bubble[static_cast<std::size_t>(i)] >= 0) {
        bubble_se.push_back(elapsed_s(run_start, prev_end));
        bubble_se.push_back(a);
      }
      prev_end = eev[e].op_end[i];
    }
    if (gap_bubble[static_cast<std::size_t>(nops)] >= 0) {
      bubble_se.push_back(elapsed_s(run_start, prev_end));
      bubble_se.push_back(elapsed_s(run_start, eev[e].end));
    }
    prev_end = eev[e].end;
  }
  step_task.clear();
  rec_slices.clear();
  for (const StepRec& r : steps) {  // a group of n back-to-back steps: n equal slices
    rec_slices.push_back(step_se.size() / 2);
    const double a = elapsed_s(run_start, r.a), b = elapsed_s(run_start, r.b);
    const int n = std::max(1, r.n);
    for (int i = 0; i < n; ++i) {
      step_se.push_back(a + (b - a) * i / n);
      step_se.push_back(a + (b - a) * (i + 1) / n);
      step_task.push_back(r.task);
    }
  }
  const double makespan = elapsed_s(run_start, eev[static_cast<std::size_t>(epochs) - 1].end);
  if (!with_tasks) {  // the ΔT controller's reference: each op's median duration without side tasks
    op_ref.assign(static_cast<std::size_t>(nops), 0.0);
    for (int g = 0; g < nops; ++g) {
      std::vector<double> d;
      for (int e = 0; e < epochs; ++e) {
        const std::size_t k = static_cast<std::size_t>(e) * nops + g;
        d.push_back(op_se[2 * k + 1] - op_se[2 * k]);
      }
      std::sort(d.begin(), d.end());
      op_ref[static_cast<std::size_t>(g)] = d[d.size() / 2];
    }
  } else if (!op_ref.empty()) {  // every op of the run against the reference (report)
    growth_sum = 0;
    growth_n = 0;
    for (std::size_t k = 0; k < op_se.size() / 2; ++k) {
      growth_sum += (op_se[2 * k + 1] - op_se[2 * k]) / op_ref[k % static_cast<std::size_t>(nops)] - 1.0;
      ++growth_n;
    }
  }
  double bubble_total = 0, used = 0, step_total = 0, worst = 0;
  for (std::size_t i = 0; i < bubble_se.size(); i += 2) bubble_total += bubble_se[i + 1] - bubble_se[i];
  std::size_t bi_idx = 0;
  for (std::size_t i = 0; i < step_se.size(); i += 2) {
    const double a = step_se[i], b = step_se[i + 1];
    step_total += b - a;
    while (bi_idx + 2 < bubble_se.size() && bubble_se[bi_idx + 1] <= a) bi_idx += 2;
    double in = 0;
    for (std::size_t j = bi_idx; j < bubble_se.size() && bubble_se[j] < b; j += 2)
      in += std::max(0.0, std::min(b, bubble_se[j + 1]) - std::max(a, bubble_se[j]));
    used += in;
    if (bi_idx < bubble_se.size() && b > bubble_se[bi_idx + 1] && a < bubble_se[bi_idx + 1])
      worst = std::max(worst, b - bubble_se[bi_idx + 1]);
  }
  // bubble_breakdown (metrics.hpp:64) over the measured timeline, ns ticks
  auto tick_of = [](double s) { return static_cast<Tick>(std::llround(s / kTick)); };
  for (std::size_t i = 0; i < bubble_se.size(); i += 2)
    bi.bubbles.push_back(Bubble{0, 0, tick_of(bubble_se[i]), tick_of(bubble_se[i + 1]) - tick_of(bubble_se[i]), avail, BubbleType::C});
  for (auto& kv : tasks) {
    bi.profiles.push_back(kv.second->prof);
    if (kv.second->rt.assigned_worker || kv.second->rt.state != SideTaskState::Submitted)
      bi.assigns.push_back(AssignRecord{0, kv.first, 0});
    if (kv.second->init_recorded && with_tasks) {
      const double a = elapsed_s(run_start, kv.second->init_a);
      const double b = elapsed_s(run_start, kv.second->init_b);
      if (b > 0) bi.activities.push_back(ActivityRecord{tick_of(std::max(0.0, a)), tick_of(b), kv.first, 0, ActivityKind::Init, false});
      if (b > 0) init_log.push_back({kv.first, {std::max(0.0, a), b}});
      if (std::getenv("FR_HARNESS_TRACE"))
        std::fprintf(stderr, "[harness] %s InitSideTask on device %.3f..%.3f ms after run start (hook %.0f us on host)\n",
                     kv.first.c_str(), a * 1e3, b * 1e3, kv.second->init_host_us);
      kv.second->init_recorded = false;
    }
  }
  for (std::size_t i = 0; i < step_se.size(); i += 2)
    bi.activities.push_back(ActivityRecord{tick_of(step_se[i]), tick_of(step_se[i + 1]), "step", 0, ActivityKind::Step, false});
  const std::vector<StageBreakdown> bd = bubble_breakdown(bi);

  std::memset(rep, 0, sizeof(*rep));
  rep->epochs = epochs;
  rep->with_tasks = with_tasks;
  rep->makespan_s = makespan;
  rep->bubble_s = bubble_total;
  rep->used_s = used;
  rep->overrun_s = step_total - used;
  rep->work_units = units;
  rep->steps_launched = launched;
  rep->steps_completed = completed;
  rep->dispatch_host_us = launched ? dispatch_ns / static_cast<double>(launched) * 1e-3 : 0.0;
  rep->max_step_overrun_s = worst;
  rep->breakdown = fr_stage_breakdown{0, 0, bd[0].used_by_side_tasks, bd[0].runtime_overhead, bd[0].idle_oom, bd[0].idle_insufficient_time};
  rep->pauses = pauses;
  rep->kills = kills;
  rep->kills_oom = kills_oom;
  rep->kills_pause_timeout = kills_timeout;
  rep->kills_init_timeout = kills_init;
  if (cfg.transport == 1) {  // stage-to-stage exchange: each message's copy-engine transfer
    double t = 0;
    std::int64_t n = 0;
    for (int e = 0; e < epochs; ++e)
      for (int g = 0; g < nops; ++g) {
        const OpEvent& op = ops[static_cast<std::size_t>(g)];
        const bool sends = (op.kind == OpKind::FP && cfg.stage < cfg.num_stages - 1) ||
                           (op.kind == OpKind::BP && cfg.stage > 0);
        if (!sends) continue;
        t += elapsed_s(eev[e].send_a[g], eev[e].send_b[g]);
        ++n;
      }
    rep->exchange_messages = n;
    rep->exchange_us = n ? t / static_cast<double>(n) * 1e6 : 0.0;
    rep->exchange_gbps = t > 0 ? static_cast<double>(msg_bytes) * static_cast<double>(n) / t * 1e-9 : 0.0;
  }
  rep->op_growth = growth_n ? growth_sum / static_cast<double>(growth_n) : 0.0;
  rep->side_sms_mean = controlled && meas_idx ? sms_sum / static_cast<double>(meas_idx)
                                              : (cfg.side_sms > 0 ? cfg.side_sms : sm_count);
  rep->side_sms_final = controlled ? ctrl_sms : (cfg.side_sms > 0 ? cfg.side_sms : sm_count);
  last_side_steps = launched;
  last_train_ops = static_cast<std::int64_t>(epochs) * nops;
  epoch_base += static_cast<std::uint32_t>(epochs);
}

extern "C" {

int fr_harness_create(const fr_harness_config* cfg, fr_harness** out) {
  if (!cfg || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (cfg->stage < 0 || cfg->stage >= cfg->num_stages)
    return frcapi::fail(FR_ERR_VALIDATION, "stage must be in [0, num_stages)", "stage");
  if (cfg->num_micro_batches < 1 || 2 * cfg->num_micro_batches + 1 >= static_cast<int>(kBubbleIds) ||
      cfg->num_micro_batches > kMaxMb)
    return frcapi::fail(FR_ERR_VALIDATION, "num_micro_batches out of range", "num_micro_batches");
  if (cfg->transport != 0 && cfg->transport != 1)
    return frcapi::fail(FR_ERR_VALIDATION, "transport must be 0 (replica) or 1 (peer-linked)", "transport");
  auto h = std::make_unique<fr_harness>();
  return frcapi::guard([&]() -> int {
    h->cfg = *cfg;
    ck(cudaGetDevice(&h->device), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device), "SM count");
    configure_timeline_kernels();
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    ck(cudaStreamCreateWithPriority(&h->train, cudaStreamNonBlocking, hi), "train stream");
    ck(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, lo), "side stream");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h->ring), sizeof(RingSlot) * kRingSlots, cudaHostAllocMapped), "ring");
    std::memset(h->ring, 0, sizeof(RingSlot) * kRingSlots);
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->ring_dev), h->ring, 0), "ring dev");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h->stamp), 64, cudaHostAllocMapped), "stamp");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h->flag), 64, cudaHostAllocMapped), "flag");
    *h->flag = 0;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h->pgate), 64, cudaHostAllocMapped), "profile gate");
    *h->pgate = 0;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->pgate_dev), h->pgate, 0), "profile gate dev");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->stamp_dev), h->stamp, 0), "stamp dev");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->flag_dev), h->flag, 0), "flag dev");
    ck(cudaMalloc(&h->ctl, sizeof(TimelineCtl)), "ctl");
    ck(cudaMemset(h->ctl, 0, sizeof(TimelineCtl)), "ctl");
    StandInShape shape;
    shape.layers = cfg->layers;
    shape.hidden = cfg->hidden;
    shape.tokens = cfg->tokens;
    shape.ffn_mult = cfg->ffn_mult > 0 ? cfg->ffn_mult : 4;
    h->standin = std::make_unique<StandIn>(shape);
    h->standin->capture(h->train);
    const int reps = std::max(1, cfg->profile_reps);
    const Tick f = cfg->fp_ticks_override > 0 ? cfg->fp_ticks_override : h->measure_op(true, reps);
    const Tick b = cfg->bp_ticks_override > 0 ? cfg->bp_ticks_override : h->measure_op(false, reps);
    h->fp_tflops = h->standin->fp_flops() / (static_cast<double>(h->measure_op(true, 3)) * kTick) * 1e-12;
    h->bp_tflops = h->standin->bp_flops() / (static_cast<double>(h->measure_op(false, 3)) * kTick) * 1e-12;
    h->build_schedule_from(f, b);
    if (cfg->transport == 1) {
      // mailbox: flags, then FP-in and BP-in slots per micro-batch
      h->msg_bytes = h->standin->message_bytes();
      h->mbox.m = cfg->num_micro_batches;
      h->mbox.msg_stride = (h->msg_bytes + 255) & ~static_cast<std::size_t>(255);
      h->mbox_bytes = kFlagArea + 2 * static_cast<std::size_t>(h->mbox.m) * h->mbox.msg_stride;
      ck(cudaMalloc(&h->mbox.base, h->mbox_bytes), "mailbox");
      ck(cudaMemset(h->mbox.base, 0, kFlagArea), "mailbox flags");
      h->prev_mbox = h->next_mbox = h->mbox;  // geometry; bases set by fr_harness_link
      h->prev_mbox.base = h->next_mbox.base = nullptr;
    } else {
      h->profile_in_pipeline(cfg->profile_epochs);  // linked: dry-run after fr_harness_link
    }
    h->workers.resize(1);
    h->workers[0].worker_id = 0;
    h->workers[0].gpu_mem = h->avail;
    h->calibrate();
    *out = h.release();
    return FR_OK;
  });
}

int fr_harness_mailbox(const fr_harness* h, void** base, int64_t* bytes) {
  if (!h || !base) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (h->cfg.transport != 1) return frcapi::fail(FR_ERR_UNSUPPORTED, "mailbox exists only with transport 1");
  *base = h->mbox.base;
  if (bytes) *bytes = static_cast<int64_t>(h->mbox_bytes);
  return FR_OK;
}

int fr_harness_link(fr_harness* h, void* prev_mailbox, void* next_mailbox) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (h->cfg.transport != 1) return frcapi::fail(FR_ERR_UNSUPPORTED, "link needs transport 1");
  const int s = h->cfg.stage, p = h->cfg.num_stages;
  if ((s > 0) != (prev_mailbox != nullptr) || (s < p - 1) != (next_mailbox != nullptr))
    return frcapi::fail(FR_ERR_VALIDATION, "a stage links exactly its existing neighbours", "mailbox");
  // a neighbour on another GPU of this process: its mailbox is written by
  // this GPU's copy engine and read by our flag waits -> peer access both
  // ways over NVLink (IPC-opened mailboxes already have it:
  // cudaIpcMemLazyEnablePeerAccess)
  for (void* q : {prev_mailbox, next_mailbox}) {
    if (!q) continue;
    cudaPointerAttributes at{};
    FR_CUDA_TRY_H(cudaPointerGetAttributes(&at, q));
    if (at.type != cudaMemoryTypeDevice || at.device == h->device) continue;
    int can = 0;
    FR_CUDA_TRY_H(cudaDeviceCanAccessPeer(&can, h->device, at.device));
    if (!can)
      return frcapi::fail(FR_ERR_UNSUPPORTED, "no peer access from GPU " + std::to_string(h->device) + " to GPU " +
                                                  std::to_string(at.device) + " (NVLink / P2P required)");
    const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) FR_CUDA_TRY_H(e);
    cudaGetLastError();  // clear the sticky "already enabled"
  }
  h->prev_mbox.base = static_cast<char*>(prev_mailbox);
  h->next_mbox.base = static_cast<char*>(next_mailbox);
  h->linked = true;
  return FR_OK;
}

int fr_ipc_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  cudaIpcMemHandle_t hd;
  FR_CUDA_TRY_H(cudaIpcGetMemHandle(&hd, dev_ptr));
  std::memcpy(handle_out, &hd, sizeof(hd));
  return FR_OK;
}

int fr_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  FR_CUDA_TRY_H(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  return FR_OK;
}

int fr_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return FR_OK;
  FR_CUDA_TRY_H(cudaIpcCloseMemHandle(dev_ptr));
  return FR_OK;
}

int fr_harness_destroy(fr_harness* h) {
  delete h;
  return FR_OK;
}

int fr_harness_get_profile(const fr_harness* h, fr_harness_profile* out) {
  if (!h || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  std::memset(out, 0, sizeof(*out));
  out->fp_ticks = h->fp;
  out->bp_ticks = h->bp;
  out->epoch_span = h->span;
  for (const Bubble& b : h->bubbles) out->stage_bubble_ticks += b.duration;
  out->bubble_rate = h->rate;
  out->available_memory = h->avail;
  out->fp_tflops = h->fp_tflops;
  out->bp_tflops = h->bp_tflops;
  out->n_bubbles = static_cast<int32_t>(h->bubbles.size());
  out->clock_offset_err_ns = h->clock_err;
  return FR_OK;
}

int fr_harness_stage_bubbles(const fr_harness* h, fr_bubble* out, int32_t cap, int32_t* n) {
  if (!h || !n) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *n = static_cast<int32_t>(h->bubbles.size());
  if (*n > cap) return frcapi::fail(FR_ERR_CAPACITY, "bubble buffer too small");
  for (std::size_t i = 0; i < h->bubbles.size(); ++i) out[i] = frcapi::bubble_out(h->bubbles[i], -1, -1);
  return FR_OK;
}

int fr_harness_submit(fr_harness* h, const char* task_id, const fr_side_task_vtable* vt,
                      void* user, double mem, int32_t profile_steps, fr_task_profile* prof_out,
                      int32_t* assigned) {
  if (!h || !task_id || !vt || !vt->init || (!vt->run_next_step && vt->interface_kind != FR_IMPERATIVE))
    return frcapi::fail(FR_ERR_ARGUMENT, "null argument / missing hook");
  if (h->tasks.count(task_id)) return frcapi::fail(FR_ERR_VALIDATION, "duplicate task id", "id");
  auto t = std::make_unique<Task>();
  t->id = task_id;
  t->vt = *vt;
  t->user = user;
  return frcapi::guard([&]() -> int {
    t->rt.spec.id = task_id;
    t->rt.spec.memory_demand = mem;
    // profile_task (profiler.hpp:41): run the body standalone, time each
    // RunNextStep on the device, est = mean, max = worst (ns ticks).
    const bool imperative = vt->interface_kind == FR_IMPERATIVE;
    if (imperative && (!vt->run_gpu_workload || !vt->work_done))
      throw HookError(FR_ERR_ARGUMENT, "imperative task without run_gpu_workload / work_done");
    t->rt.spec.interface_kind = imperative ? TaskInterface::Imperative : TaskInterface::Iterative;
    t->device = h->device;
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = h->device;
    ck(cudaMemPoolCreate(&t->pool, &pp), "task memory pool");
    std::uint64_t keep = UINT64_MAX;  // cache freed memory inside the pool (no device sync on reuse)
    cudaMemPoolSetAttribute(t->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    PoolScope ps(h->device, t->pool);
    if (vt->set_sm_budget) hook(vt->set_sm_budget(user, std::max(0, h->cfg.side_sms)), "set_sm_budget");
    hook(vt->create ? vt->create(user) : FR_OK, "create");
    hook(vt->init(user, h->side), "init");
    const int n = imperative ? 0 : std::max(1, profile_steps);
    for (int i = 0; i < (imperative ? 0 : 2); ++i) hook(vt->run_next_step(user, h->side), "run_next_step");
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
    // FR_HARNESS_NO_PROFILE_GATE=1: no host-released gate before the profiled
    // steps.  A profiler that serialises launches (ncu) blocks in the gate
    // kernel's launch, so the host never releases it; the profile then
    // includes hook host time, which is what ncu runs accept.
    static const bool no_gate = [] {
      const char* e = std::getenv("FR_HARNESS_NO_PROFILE_GATE");
      return e && std::atoi(e) != 0;
    }();
    for (int i = 0; i < n; ++i) {
      // The side stream is held by a flag wait until the hook has returned:
      // a hook that stalls the host (a cudaMallocAsync growing its pool
      // maps memory for 0.4-23 ms) must not be timed as GPU step time --
      // an inflated estimate closes the gate for every bubble.
      LinkWaitArgs w{};
      w.ctl = h->ctl;
      w.slot_start = w.slot_end = -1;
      w.flag = h->pgate_dev;
      w.seq = ++h->pgate_seq;
      w.timeout_ns = 5'000'000'000ull;
      if (!no_gate) launch_link_wait(w, h->side);
      cudaEvent_t a = h->ev(), b = h->ev();
      ck(cudaEventRecord(a, h->side), "record");
      hook(vt->run_next_step(user, h->side), "run_next_step");
      ck(cudaEventRecord(b, h->side), "record");
      __atomic_store_n(h->pgate, w.seq, __ATOMIC_RELEASE);
      ck(cudaEventSynchronize(b), "profile step");  // standalone: one step at a time
      evs.push_back({a, b});
    }
    Tick busy = 0, longest = 0;
    for (auto& [a, b] : evs) {
      const Tick d = static_cast<Tick>(std::llround(elapsed_s(a, b) / kTick));
      busy += d;
      longest = std::max(longest, d);
    }
    h->pool_used = 0;
    hook(vt->stop ? vt->stop(user) : FR_OK, "stop");  // profiling instance torn down
    ck(cudaStreamSynchronize(h->side), "profile sync");
    // GPU memory consumption (§4.3): the pool's high-water mark
    // while the task was initialised and stepped standalone
    std::size_t high = 0;
    cudaMemPoolGetAttribute(t->pool, cudaMemPoolAttrUsedMemHigh, &high);
    std::uint64_t zero = 0;
    cudaMemPoolSetAttribute(t->pool, cudaMemPoolAttrUsedMemHigh, &zero);
    TaskProfile p;
    p.task_id = task_id;
    p.profiled_steps = n;
    if (!imperative) {  // the profiler does not time imperative tasks
      p.est_per_step_duration = ticks_to_seconds(busy, kTick) / n;
      p.max_per_step_duration = ticks_to_seconds(longest, kTick);
    }
    p.est_memory = std::max(mem, static_cast<double>(high) / kGiB);
    t->prof = p;
    t->mem_limit = p.est_memory + std::max(0.0, h->cfg.memory_headroom_gib);
    const SubmitOutcome o = submit_task(p, h->workers);  // Alg. 1
    if (assigned) *assigned = o.assigned;
    if (prof_out) frcapi::profile_out(p, prof_out);
    if (o.assigned) {
      apply_transition(t->rt, TransitionKind::CreateSideTask, 0);
      hook(vt->create ? vt->create(user) : FR_OK, "create");
      h->tasks[task_id] = std::move(t);
      // The profiling instance's pages stay mapped in the task's pool (the
      // worker reserved est_memory for it under Alg. 1): InitSideTask then
      // reuses them instead of growing the pool inside a bubble, which
      // stalls the dispatch thread 3-23 ms for the image task's 0.5 GB
      // (FR_HARNESS_TRACE) and once cost a whole 2-epoch warm-up.
    } else {
      cudaMemPoolTrimTo(t->pool, 0);
      t->user = nullptr;  // rejected: ownership stays with the caller
      t->disp = Disposition::Rejected;
    }
    return FR_OK;
  });
}

int fr_harness_run(fr_harness* h, int32_t epochs, int32_t with_tasks, fr_run_report* out) {
  if (!h || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (epochs < 1) return frcapi::fail(FR_ERR_VALIDATION, "epochs must be >= 1", "epochs");
  try {
    ck(cudaSetDevice(h->device), "cudaSetDevice");  // any calling thread
    h->run(epochs, with_tasks != 0, out);
    return FR_OK;
  } catch (const HookError& e) {
    return frcapi::fail(e.code, e.what());
  } catch (const std::exception& e) {
    return frcapi::fail(FR_ERR_INVARIANT, e.what());
  }
}

int fr_harness_set_harvest_fraction(fr_harness* h, double fraction) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (!(fraction >= 0.0 && fraction <= 1.0))
    return frcapi::fail(FR_ERR_VALIDATION, "harvest fraction must be in [0, 1]", "harvest_fraction");
  h->cfg.harvest_fraction = fraction;
  return FR_OK;
}

int fr_harness_set_side_sms(fr_harness* h, int32_t sms) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (sms < 0) return frcapi::fail(FR_ERR_VALIDATION, "side_sms must be >= 0", "side_sms");
  h->cfg.side_sms = sms;
  h->ctrl_sms = 0;  // the ΔT controller restarts from this budget
  for (auto& kv : h->tasks)
    if (kv.second->vt.set_sm_budget) {
      const int rc = kv.second->vt.set_sm_budget(kv.second->user, sms);
      if (rc != FR_OK) return rc;
    }
  return FR_OK;
}

int fr_harness_set_dt_budget(fr_harness* h, double budget) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (!(budget >= 0.0 && budget < 1.0)) return frcapi::fail(FR_ERR_VALIDATION, "dt_budget in [0, 1)", "dt_budget");
  h->cfg.dt_budget = budget;
  h->ctrl_sms = 0;
  return FR_OK;
}

int fr_harness_task_memory(const fr_harness* h, const char* task_id, double* used_gib, double* reserved_gib) {
  if (!h || !task_id) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto it = h->tasks.find(task_id);
  if (it == h->tasks.end()) return frcapi::fail(FR_ERR_NOT_FOUND, "unknown task");
  const Task& t = *it->second;
  std::size_t used = 0, reserved = 0;
  if (t.pool) {
    cudaMemPoolGetAttribute(t.pool, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaMemPoolGetAttribute(t.pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  }
  if (used_gib) *used_gib = static_cast<double>(used) / kGiB;
  if (reserved_gib) *reserved_gib = static_cast<double>(reserved) / kGiB;
  return FR_OK;
}

int fr_harness_reprofile_bubbles(fr_harness* h) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (h->bubbles_from_last_run() == 0)
    return frcapi::fail(FR_ERR_VALIDATION, "no complete run to profile bubbles from", "run");
  return FR_OK;
}

int fr_harness_stop_task(fr_harness* h, const char* task_id) {
  if (!h || !task_id) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto it = h->tasks.find(task_id);
  if (it == h->tasks.end()) return frcapi::fail(FR_ERR_NOT_FOUND, "unknown task");
  Task& t = *it->second;
  return frcapi::guard([&]() -> int {
    if (t.rt.state != SideTaskState::Stopped) {
      apply_transition(t.rt, TransitionKind::StopSideTask, 0);  // {CREATED,PAUSED,RUNNING} -> STOPPED
      PoolScope ps(h->device, t.pool);
      if (t.rt.memory_allocated == 0.0 && t.vt.stop) hook(t.vt.stop(t.user), "stop");
    }
    WorkerState& ws = h->workers[0];
    if (ws.current_task && *ws.current_task == t.id) ws.current_task.reset();  // Appendix B rule 8
    ws.task_queue.erase(std::remove(ws.task_queue.begin(), ws.task_queue.end(), t.id), ws.task_queue.end());
    ck(cudaStreamSynchronize(h->side), "side sync");
    return FR_OK;
  });
}

int fr_harness_reprofile(fr_harness* h, const char* task_id, fr_task_profile* out) {
  if (!h || !task_id) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto it = h->tasks.find(task_id);
  if (it == h->tasks.end()) return frcapi::fail(FR_ERR_NOT_FOUND, "unknown task");
  Task& t = *it->second;
  Tick busy = 0, longest = 0;
  int n = 0;
  for (std::size_t i = 0; i < h->step_task.size(); ++i) {
    if (h->step_task[i] != &t) continue;
    const Tick d = static_cast<Tick>(std::llround((h->step_se[2 * i + 1] - h->step_se[2 * i]) / kTick));
    busy += d;
    longest = std::max(longest, d);
    ++n;
  }
  if (n == 0) return frcapi::fail(FR_ERR_VALIDATION, "task ran no step in the last run", "task");
  t.prof.profiled_steps = n;
  t.prof.est_per_step_duration = ticks_to_seconds(busy, kTick) / n;
  t.prof.max_per_step_duration = ticks_to_seconds(longest, kTick);
  if (out) frcapi::profile_out(t.prof, out);
  return FR_OK;
}

int fr_harness_task_status(const fr_harness* h, const char* task_id, int32_t* state,
                           int32_t* disposition, double* memory_used_gib) {
  if (!h || !task_id) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto it = h->tasks.find(task_id);
  if (it == h->tasks.end()) return frcapi::fail(FR_ERR_NOT_FOUND, "unknown task");
  const Task& t = *it->second;
  if (state) *state = static_cast<int32_t>(t.rt.state);
  if (disposition) *disposition = static_cast<int32_t>(t.disp);
  if (memory_used_gib) *memory_used_gib = t.used_gib();
  return FR_OK;
}

int fr_harness_run_trace(const fr_harness* h, fr_run_trace** out) {
  if (!h || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (!h->last_with_tasks || h->last_epochs < 1)
    return frcapi::fail(FR_ERR_VALIDATION, "the last run had no side tasks", "run");
  return frcapi::guard([&]() -> int {
    auto tr = std::make_unique<fr_run_trace>();
    RunTrace& r = tr->t;
    const int s = h->cfg.stage;
    const auto tick_of = [](double sec) { return static_cast<Tick>(std::llround(sec / kTick)); };
    const auto rel = [h](std::int64_t t_dev) { return static_cast<Tick>(t_dev - h->run0_dev); };
    r.measured = true;
    r.tolerance = 20'000;  // host-clock stamps vs device events (calibrated offset + polling)
    r.with_tasks = true;
    ExperimentConfig& ec = r.config;
    ec.pipeline = h->pcfg;
    ec.pipeline.num_epochs = h->last_epochs;
    ec.limits.grace_period = h->cfg.grace_ns > 0 ? h->cfg.grace_ns : kGraceTicks;
    ec.limits.memory_headroom = std::max(0.0, h->cfg.memory_headroom_gib);
    ec.limits.reclamation_delay = std::max<std::int64_t>(0, h->cfg.reclamation_delay_ns);
    ec.runtime.check_overhead = 0;
    ec.runtime.gate_estimate = h->cfg.gate_estimate == 1 ? GateEstimate::Max : GateEstimate::Mean;
    std::map<std::string, std::int64_t> steps;
    for (const auto& kv : h->tasks) {
      const Task& t = *kv.second;
      SideTaskSpec spec = t.rt.spec;
      spec.per_step_duration = static_cast<Tick>(std::llround(t.prof.est_per_step_duration.value_or(0.0) / kTick));
      ec.tasks.push_back(spec);
      r.profiles.push_back(t.prof);
      r.submits.push_back(AssignRecord{0, t.id, -1});
      r.assigns.push_back(AssignRecord{0, t.id, s});
      // the transitions that brought the task to its state at the run start
      auto it = h->run_start_state.find(t.id);
      const SideTaskState st0 = it == h->run_start_state.end() ? SideTaskState::Created : it->second;
      std::vector<TransitionKind> pre;
      if (st0 != SideTaskState::Submitted) pre.push_back(TransitionKind::CreateSideTask);
      if (st0 == SideTaskState::Paused || st0 == SideTaskState::Running) pre.push_back(TransitionKind::InitSideTask);
      if (st0 == SideTaskState::Running) pre.push_back(TransitionKind::StartSideTask);
      if (st0 == SideTaskState::Stopped) pre.push_back(TransitionKind::StopSideTask);
      for (TransitionKind k : pre) r.transitions.push_back(TransitionRecord{0, t.id, k, s});
    }
    // A pause (or stop) is applied once the task's in-flight steps have
    // drained; its stamp is the host clock mapped to the device's, which
    // trails the device by the polling latency (~10 us).  It cannot have
    // landed before those steps ended, so it is lifted to their device end,
    // and the task's later stamps keep their order.
    std::map<std::string, Tick> floor_of;
    for (std::size_t i = 0; i < h->tr_log.size(); ++i) {
      const TransitionRecord& x = h->tr_log[i];
      Tick t = rel(x.t);
      const std::size_t done = i < h->tr_recs_done.size() ? h->tr_recs_done[i] : 0;
      if ((x.kind == TransitionKind::PauseSideTask || x.kind == TransitionKind::StopSideTask) && done > 0 &&
          done <= h->rec_slices.size()) {
        const std::size_t end_slice = done < h->rec_slices.size() ? h->rec_slices[done] : h->step_se.size() / 2;
        if (end_slice > 0) t = std::max(t, tick_of(h->step_se[2 * end_slice - 1]));
      }
      Tick& fl = floor_of[x.task];
      t = std::max(t, fl);
      fl = t;
      r.transitions.push_back(TransitionRecord{t, x.task, x.kind, x.worker});
    }
    std::stable_sort(r.transitions.begin(), r.transitions.end(),
                     [](const TransitionRecord& a, const TransitionRecord& b) { return a.t < b.t; });
    const std::size_t nops = h->ops.size();
    for (std::size_t i = 0; i < h->op_se.size() / 2; ++i) {
      const OpEvent& o = h->ops[i % nops];
      r.ops.push_back(OpEvent{s, o.kind, o.micro_batch, static_cast<int>(i / nops), tick_of(h->op_se[2 * i]),
                              tick_of(h->op_se[2 * i + 1])});
    }
    const std::size_t nb = h->bubbles.size();
    for (std::size_t k = 0; nb && k < h->bubble_se.size() / 2; ++k) {
      const Tick a = tick_of(h->bubble_se[2 * k]), b = tick_of(h->bubble_se[2 * k + 1]);
      r.bubbles.push_back(Bubble{s, static_cast<int>(k / nb), a, b - a, h->avail, h->bubbles[k % nb].btype});
    }
    for (const auto& [id, se] : h->init_log)
      r.activities.push_back(ActivityRecord{tick_of(se.first), tick_of(se.second), id, s, ActivityKind::Init, false});
    for (std::size_t i = 0; i < h->step_task.size(); ++i) {
      const Task* t = h->step_task[i];
      r.activities.push_back(ActivityRecord{tick_of(h->step_se[2 * i]), tick_of(h->step_se[2 * i + 1]), t->id, s,
                                            t->imperative() ? ActivityKind::Kernel : ActivityKind::Step, false});
      ++steps[t->id];
    }
    for (const KillRecord& k : h->kill_log) r.kills.push_back(KillRecord{rel(k.t), k.task, k.worker, k.reason});
    for (const auto& kv : h->tasks)
      r.dispositions.push_back(DispositionRecord{kv.first, kv.second->disp, steps[kv.first], s});
    for (const OpEvent& o : r.ops) r.makespan = std::max(r.makespan, o.end);
    *out = tr.release();
    return FR_OK;
  });
}

int fr_harness_gate_log(const fr_harness* h, fr_gate_record* out, int64_t cap, int64_t* n) {
  if (!h || !n) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *n = static_cast<int64_t>(h->gate_log.size());
  if (*n > cap) return frcapi::fail(FR_ERR_CAPACITY, "gate record buffer too small");
  for (std::size_t i = 0; i < h->gate_log.size(); ++i) {
    const auto& g = h->gate_log[i];
    fr_gate_record& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.now = g.now - h->run0_dev;
    o.bubble_end = g.bubble_end - h->run0_dev;
    o.est_seconds = g.est;
    o.step_ticks = g.est_ticks;
    o.run = g.run;
    o.signal = g.signal;
    o.step_end = g.run ? g.step_end - h->run0_dev : 0;
    frcapi::copy_id(o.task, g.task);
  }
  return FR_OK;
}

int fr_harness_signal_log(const fr_harness* h, fr_signal_record* out, int64_t cap, int64_t* n) {
  if (!h || !n) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *n = static_cast<int64_t>(h->sig_log.size());
  if (*n > cap) return frcapi::fail(FR_ERR_CAPACITY, "signal record buffer too small");
  for (std::size_t i = 0; i < h->sig_log.size(); ++i) {
    const auto& g = h->sig_log[i];
    fr_signal_record& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.t = g.t - h->run0_dev;
    o.kind = g.kind;
    o.epoch = static_cast<int32_t>(g.id / kBubbleIds);
    o.bubble = static_cast<int32_t>(g.id % kBubbleIds);
    o.looked_up = g.looked_up;
    o.duration = g.duration;
    o.view_state = static_cast<int32_t>(g.view.state);
    o.view_initializing = g.view.initializing;
    o.n_actions = static_cast<int32_t>(std::min<std::size_t>(4, g.acts.size()));
    for (int k = 0; k < o.n_actions; ++k) o.actions[k] = static_cast<int32_t>(g.acts[static_cast<std::size_t>(k)].kind);
    o.deferred = g.deferred;
    frcapi::copy_id(o.task, g.task);
  }
  return FR_OK;
}

int fr_harness_timeline(const fr_harness* h, int32_t which, double* se, int64_t cap, int64_t* n) {
  if (!h || !n) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  const std::vector<double>* v = which == 0 ? &h->op_se : which == 1 ? &h->bubble_se : &h->step_se;
  *n = static_cast<int64_t>(v->size() / 2);
  if (*n > cap) return frcapi::fail(FR_ERR_CAPACITY, "timeline buffer too small");
  std::copy(v->begin(), v->end(), se);
  return FR_OK;
}

int fr_harness_launches(const fr_harness* h, int64_t* side_steps, int64_t* training_ops) {
  if (!h) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (side_steps) *side_steps = h->last_side_steps;
  if (training_ops) *training_ops = h->last_train_ops;
  return FR_OK;
}

}  // extern "C"
