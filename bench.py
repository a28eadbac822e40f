"""Benchmark of the bubble-harvesting hot path (BASELINE.json metric):

  side-task edges/s & px/s per bubble-second at <= 1 % pipeline ΔT,
  HBM GB/s vs peak

Pipeline: a 4-stage 1F1B pipeline (m = 4) whose stages are nanoGPT-1.2B-
shaped bf16 GEMM stand-ins (6 layers x h 2048 per stage, 8192 tokens per
micro-batch).  One GPU replays every stage in turn ("replica mode",
SURVEY.md §7); with --gpus N each rank is an independent replica (no
collective on the data path) -> scaling "weak".

Headline workload (BASELINE.json configs[1]): the image resize + watermark
side task (64 synthetic 4K RGB frames -> 1080p, RGBA watermark, 16 frames per
RunNextStep), run on an SM budget (IMG_SMS) that holds the pipeline's ΔT
under 1 %: on a power-capped B200 every joule a side task spends in a bubble
is taken from the boost the pipeline's GEMMs get out of their idle bubbles,
and the same bytes moved by fewer SMs cost far less power (
"image_full_gpu" under workloads is the same task on all 148 SMs).  The same run also measures configs[0] (PageRank, RMAT-20,
two pull iterations per step), configs[2] (Graph-SGD, Orkut shape, rank
16, 2^22 edges per step), configs[3] (mixed, 3.6B-shaped stages) and the
image task through the imperative interface (device-preempted workload)
under "workloads".

ΔT is the PIPELINE's: the per-stage FP / BP op durations measured with and
without the side task go through build_schedule (the reference's 1F1B DAG)
and the makespan growth is reported (`delta_t`, paper_2409_06941_b200/
pipeline_dt.py); the per-stage replica makespan growths are reported beside
it (`delta_t_stage_max`).

A bench *step* is one training iteration (epoch) of all 4 stages with the
side task harvesting its bubbles.  Per stage and workload: the bubble
profiler dry-runs the pipeline (harness creation), the task is profiled
standalone then submitted (Alg. 1), W warm-up epochs run with it (InitSideTask
lands in a bubble; the per-step duration is then re-profiled in-situ), then K
epochs without side tasks (ΔT baseline, bubble-seconds denominator) and K
timed epochs with them.  All times are device times (CUDA events, %globaltimer).

  value  = side-task output px completed / baseline bubble-seconds
           (summed over ranks / max over ranks' bubble-seconds)
  e2e    = the same through the host-buffer path: frames in pinned host
           memory, H2D + kernel + D2H inside every RunNextStep (1 frame/step)
  --impl reference : the CPU restatement of the side task (oracle) on this
           box's host cores, same metric (CPU px per second of work).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STAGES = 4
MICRO_BATCHES = 4
SHAPE = dict(layers=6, hidden=2048, tokens=8192, ffn_mult=4)        # nanoGPT-1.2B / 4 stages
SHAPE_36B = dict(layers=9, hidden=2880, tokens=8192, ffn_mult=4)    # nanoGPT-3.6B / 4 stages
LAYERS_6B, HIDDEN_6B = 32, 4096                                       # nanoGPT-6B (configs[4])
FRAMES = dict(sw=3840, sh=2160, dw=1920, dh=1080)
BATCH = 64
IMAGES_PER_STEP = int(os.environ.get("FR_IMAGES_PER_STEP", "16"))   # ~95 us steps (step size vs fill vs ΔT)
# Power-aware harvesting: every stage's worker runs the live
# ΔT controller -- it times its stage's ops as they complete and sizes the
# side task's SM budget so they run at most DT_BUDGET slower than without
# side tasks -- starting from the budgets the sweeps found (image 16 SMs,
# Graph-SGD 20, PageRank all 148; scripts/harvest_sweep.py).  How much power
# a bubble can take differs from box to box (image at a fixed 16 SMs: +0.3 %
# on one, +1.6 % on another), so a fixed budget cannot hold the ΔT
# everywhere.  FR_DT_BUDGET=0 runs the fixed budgets instead.
DT_BUDGET = float(os.environ.get("FR_DT_BUDGET", "0.004"))
IMG_SMS = int(os.environ.get("FR_IMG_SMS", "8"))
SGD_SMS = int(os.environ.get("FR_SGD_SMS", "20"))
E2E_SMS = int(os.environ.get("FR_E2E_SMS", "4"))     # K5 SMs + copy-ahead depth (2 ring slots per SM-equivalent): PCIe DMA during compute costs dT too
PAIRS = int(os.environ.get("FR_DT_PAIRS", "8"))           # (baseline, harvest) pairs for the headline ΔT (ABBA order)
PAIRS_OTHER = int(os.environ.get("FR_DT_PAIRS_OTHER", "4"))   # ... for every other workload
STEP_GROUP = int(os.environ.get("FR_STEP_GROUP", "3"))   # steps between one pair of timing events
E2E_IMAGES_PER_STEP = 1
E2E_RING = int(os.environ.get("FR_E2E_RING", "128"))   # device staging slots: the copy engines run ahead of the steps
OUT_PX = FRAMES["dw"] * FRAMES["dh"]
K5_WARP_INSTR_PER_PX = 0.938   # img_resize2x_wm_ws in a harvest on all SMs, ncu instruction count (profiles/r2s_k5ws_harvest_ncu.txt; round 1: 1.434)
PR = dict(scale=20, edge_factor=16, seed=1, iters_per_step=2)
SGD = dict(V=3072441, E=117185083, k=16, edge_seed=2, init_seed=3,
           edges_per_step=int(os.environ.get("FR_SGD_EDGES_PER_STEP", str(1 << 22))))
METRIC = "side-task px/s per bubble-sec at <=1% pipeline dT (image 4K->1080p+watermark); HBM GB/s vs peak"
UNIT = "px/bubble-s"
WORKLOAD = ("image resize+watermark side task (64x 3840x2160 RGB -> 1920x1080, RGBA watermark), "
            "harvesting a 4-stage 1F1B pipeline (m=4) of nanoGPT-1.2B-shaped bf16 GEMM stand-ins, "
            "every stage replayed per GPU (replica mode)")


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Clocks:
    """Samples SM clock + throttle reasons during the timed region (NVML)."""

    NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x2: "applications_clocks_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _loop(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                if nv.nvmlDeviceGetUtilizationRates(self._h).gpu > 0:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def load_ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_image_step.json")) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("images_per_launch")
    except OSError:
        return None, None


# ----------------------------------------------------------- CPU baselines
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import sidetasks_oracle  # noqa: E402  (oracle: CPU baseline legs only)
    return sidetasks_oracle.load()


def _timed(fn, seconds):
    fn()  # warm
    t0, reps = time.perf_counter(), 0
    while True:
        fn()
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return reps, el


def cpu_image(seconds, images=IMAGES_PER_STEP):
    o = _oracle()
    src = o.img_generate(images, FRAMES["sw"], FRAMES["sh"], seed=1)
    wm = o.img_generate_watermark(FRAMES["dw"], FRAMES["dh"], seed=7)
    reps, el = _timed(lambda: o.img_resize_watermark(src, wm, FRAMES["dw"], FRAMES["dh"]), seconds)
    return {"value": reps * images * OUT_PX / el, "unit": "px/s", "cores": os.cpu_count(), "kind": "port",
            "seconds": el, "sample": f"{reps} x {images} frames 3840x2160->1920x1080 (+watermark), "
                                     f"oracle/sidetasks.c OpenMP on {os.cpu_count()} host threads"}


def cpu_pagerank(seconds, csr):
    o = _oracle()
    off, col, outdeg = csr
    reps, el = _timed(lambda: o.pr_run(off, col, outdeg, 1, 0.85), seconds)
    return {"value": reps * len(col) / el, "unit": "edges/s", "cores": os.cpu_count(), "kind": "port",
            "seconds": el, "sample": f"{reps} pull iterations, RMAT-20 (E={len(col)}), fp64, "
                                     f"OpenMP on {os.cpu_count()} host threads"}


def cpu_sgd(seconds, edges=1 << 24):
    o = _oracle()
    u, v, r = o.sgd_edges(SGD["V"], edges, seed=SGD["edge_seed"])
    u, v, r = o.sgd_group_by_user(SGD["V"], u, v, r, window=SGD["edges_per_step"])   # the GPU task's layout
    L = o.sgd_init(SGD["V"], SGD["k"], seed=SGD["init_seed"])
    reps, el = _timed(lambda: o.sgd_epoch(u, v, r, L, 0.01, 0.05, nthreads=0), seconds)
    return {"value": reps * edges / el, "unit": "edges/s", "cores": os.cpu_count(), "kind": "port",
            "seconds": el, "sample": f"{reps} passes over {edges} Orkut-shaped edges (V={SGD['V']}, k=16, "
                                     f"by-user layout), Hogwild OpenMP on {os.cpu_count()} host threads"}


def bench_config(ws):
    """the workload both arms report (the reference arm runs the same op on
    the same frames and step size on the host cores)"""
    return {"workload": WORKLOAD, "stages": STAGES, "micro_batches": MICRO_BATCHES, "stage_shape": SHAPE,
            "frames": BATCH, "images_per_step": IMAGES_PER_STEP,
            "step": "one 1F1B epoch of all 4 stages (replayed) with the side task",
            "parallelism": f"replicas x{ws}", "step_group": STEP_GROUP, "dt_budget": DT_BUDGET,
            "side_sms_start": IMG_SMS, "l2": "image inputs 1.6 GB per batch > 126 MB L2; no flush needed"}


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# ---------------------------------------------------------------- harvest
def _sum_reports(rs):
    """several run reports of the same length as one (sums; means of the rates)"""
    out = dict(rs[0])
    for k in ("makespan_s", "bubble_s", "used_s", "overrun_s", "work_units", "steps_launched", "steps_completed",
              "pauses", "kills"):
        out[k] = sum(r[k] for r in rs)
    out["side_sms_mean"] = statistics.fmean(r["side_sms_mean"] for r in rs)
    return out


def harvest(h, name, task, K, W, sms=0, kinds=None, budget=0.0, pairs=1):
    """submit + warm-up + ΔT baseline + timed harvest on one stage replica;
    `sms`: the side task's SM budget (the ΔT controller's start when
    budget > 0); `kinds`: the stage's issue-order op kinds, for the per-stage
    mean FP / BP op durations of both runs; `pairs`: (baseline, harvest)
    run pairs of K epochs each, averaged -- the run-to-run drift of the
    GEMMs' power state is +-0.4 % (scripts/dt_noise_diag.py), so the pipeline
    ΔT of one pair carries that noise and `pairs` shrinks it by sqrt(pairs)"""
    from paper_2409_06941_b200 import pipeline_dt as PD
    h.set_dt_budget(budget)
    h.set_side_sms(sms)
    ok, tprof = h.submit(name, task, profile_steps=32)
    if not ok:
        raise RuntimeError(f"{name}: rejected by Alg. 1")
    # warm-up: InitSideTask lands in a bubble, then the per-step duration is
    # re-profiled in-situ from the warm-up's steps (a warm-up whose bubbles
    # all went to Init is repeated, at most twice)
    for attempt in range(3):
        warm = h.run(max(W, 1), True)
        if warm["steps_completed"] > 0:
            h.reprofile(name)
            break
    else:
        print(f"bench: {name} ran no step in {3 * max(W, 1)} warm-up epochs "
              f"({h.task_status(name)}); keeping the standalone profile", file=sys.stderr)
    bases, withs, ob, ow, durs = [], [], [], [], []
    for i in range(pairs):
        # ABBA order (baseline first in even pairs, harvest first in odd ones):
        # a drift of the power / thermal state over the run (the GPU warming
        # up) then cancels from the averaged ΔT instead of biasing it
        for with_tasks in ((False, True) if i % 2 == 0 else (True, False)):
            if with_tasks:
                withs.append(h.run(K, True))
                if kinds:
                    ow.append(PD.op_means(h.timeline(0), kinds))
                durs += [b - a for a, b in h.timeline(2)]
            else:
                bases.append(h.run(K, False))
                if kinds:
                    ob.append(PD.op_means(h.timeline(0), kinds))
    base, r = _sum_reports(bases), _sum_reports(withs)
    mean2 = (lambda xs: tuple(statistics.fmean(x[i] for x in xs) for i in range(2))) if kinds else None
    ops_base = mean2(ob) if kinds else None
    ops_with = mean2(ow) if kinds else None
    side, train = h.launches()
    h.stop_task(name)
    return {"base": base, "with": r, "durs": durs, "side": side, "train_ops": train, "pairs": pairs,
            "ops_base": ops_base, "ops_with": ops_with, "ops_base_runs": ob, "ops_with_runs": ow,
            "sms": r["side_sms_mean"], "budget": budget,
            "units_per_step": task.units_per_step, "bytes_per_step": task.bytes_per_step,
            "h2d": task.h2d_per_step, "d2h": task.d2h_per_step, "est_step_s": tprof["est_per_step_duration"]}


def ours(args):
    import torch
    ws, rank, local = dist_env()
    # one rank per GPU; FR_DIST_BACKEND=gloo + more ranks than GPUs is the
    # single-GPU rehearsal of the multi-rank path (ranks share a device)
    device = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("FR_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    K, W = args.steps, args.warmup
    from paper_2409_06941_b200 import api as host_api
    from paper_2409_06941_b200 import pipeline_dt as PD
    A = host_api()
    names = (["image", "image_full_gpu", "image_imperative", "pagerank", "pagerank_full_gpu", "sgd", "sgd_full_gpu"]
             + ([] if args.no_e2e else ["image_e2e"]))
    # the imperative workload runs through whole bubbles (99.7 % fill): more joules per SM-equivalent,
    # so its controller starts at half the iterative image task's budget
    sms_of = {"image": IMG_SMS, "image_imperative": max(2, IMG_SMS // 2), "image_e2e": E2E_SMS, "sgd": SGD_SMS}
    runs = {n: [] for n in names}
    stage_prof = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(device) as clk:
        for s in range(STAGES):
            h = gpu.Harness(num_stages=STAGES, num_micro_batches=MICRO_BATCHES, stage=s, step_group=STEP_GROUP,
                            **SHAPE)
            stage_prof.append(h.profile())
            kinds = PD.issue_kinds(A, s, STAGES, MICRO_BATCHES)
            for n in names:
                if n in ("image", "image_full_gpu"):
                    task = gpu.ImageTask(batch=BATCH, images_per_step=IMAGES_PER_STEP, **FRAMES)
                elif n == "image_imperative":
                    task = gpu.ImageTask(batch=BATCH, images_per_step=IMAGES_PER_STEP, imperative=True, **FRAMES)
                elif n == "image_e2e":
                    task = gpu.ImageTask(batch=BATCH, images_per_step=E2E_IMAGES_PER_STEP, host_io=True,
                                         host_ring=E2E_RING, **FRAMES)
                elif n in ("pagerank", "pagerank_full_gpu"):
                    task = gpu.PageRankTask(**PR)
                else:
                    task = gpu.SgdTask(**SGD)
                runs[n].append(harvest(h, n, task, K, W, sms=sms_of.get(n, 0), kinds=kinds,
                                       budget=0.0 if n.endswith("_full_gpu") else DT_BUDGET,
                                       pairs=PAIRS if n in ("image", "image_e2e")
                                       else 1 if n.endswith("_full_gpu") else PAIRS_OTHER))
            h.close()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    def agg(rs):
        return dict(units=sum(r["with"]["work_units"] for r in rs),
                    bubble_s=sum(r["base"]["bubble_s"] for r in rs),
                    t_no=sum(r["base"]["makespan_s"] for r in rs),
                    t_with=sum(r["with"]["makespan_s"] for r in rs),
                    stage_dT=[(r["with"]["makespan_s"] - r["base"]["makespan_s"]) / r["base"]["makespan_s"] for r in rs],
                    ops_base={i: r["ops_base"] for i, r in enumerate(rs)},
                    ops_with={i: r["ops_with"] for i, r in enumerate(rs)},
                    used=sum(r["with"]["used_s"] for r in rs),
                    bubble_with=sum(r["with"]["bubble_s"] for r in rs),
                    overrun=sum(r["with"]["overrun_s"] for r in rs),
                    pauses=sum(r["with"]["pauses"] for r in rs),
                    steps=sum(r["with"]["steps_completed"] for r in rs),
                    launches=sum(r["side"] for r in rs),
                    sms=statistics.fmean(r["sms"] for r in rs), budget=rs[0]["budget"],
                    mean_step_s=statistics.fmean(d for r in rs for d in r["durs"]) if any(r["durs"] for r in rs) else None,
                    bytes_per_step=rs[0]["bytes_per_step"], units_per_step=rs[0]["units_per_step"],
                    h2d=sum(r["h2d"] * r["with"]["steps_completed"] for r in rs),
                    d2h=sum(r["d2h"] * r["with"]["steps_completed"] for r in rs))

    def pipe_dt(rs, p, m, epochs):
        """the linked pipeline's ΔT from the replicas' op durations (pipeline_dt)"""
        base = {r_["stage"]: r_["ops_base"] for r_ in rs}
        with_ = {r_["stage"]: r_["ops_with"] for r_ in rs}
        return PD.critical_path_dt(A, p, m, epochs, base, with_)

    local_res = {n: agg(runs[n]) for n in names}
    for n in names:
        local_res[n]["pipeline"] = pipe_dt([dict(r_, stage=i) for i, r_ in enumerate(runs[n])], STAGES,
                                           MICRO_BATCHES, K)
    # the measurement's noise floor: pipeline ΔT between consecutive baseline
    # runs (no side task in either) of the headline workload
    npairs = min(len(r_["ops_base_runs"]) for r_ in runs["image"])
    local_res["image"]["null_dT"] = [
        PD.critical_path_dt(A, STAGES, MICRO_BATCHES, K, {i: r_["ops_base_runs"][j] for i, r_ in enumerate(runs["image"])},
                            {i: r_["ops_base_runs"][j + 1] for i, r_ in enumerate(runs["image"])})["dT"]
        for j in range(npairs - 1)]
    # per-pair pipeline ΔTs of the headline: their spread is the estimate's
    # standard error (the GPU's clock transients hit runs at random)
    for n in names:   # every workload: its pairs' pipeline ΔTs (spread -> standard error)
        npn = min(len(r_["ops_with_runs"]) for r_ in runs[n])
        local_res[n]["pair_dT"] = [
            PD.critical_path_dt(A, STAGES, MICRO_BATCHES, K, {i: r_["ops_base_runs"][j] for i, r_ in enumerate(runs[n])},
                                {i: r_["ops_with_runs"][j] for i, r_ in enumerate(runs[n])})["dT"]
            for j in range(npn)]
    local_res["clocks"] = clk.summary()
    local_res["l2_gbps"] = gpu.l2_read_gbps()   # PageRank's working set is L2-resident: its roofline
    local_res["gap_kernels"] = sum(r["train_ops"] // (2 * MICRO_BATCHES) * (2 * MICRO_BATCHES + 1)
                                   for r in runs["image"])
    local_res["stages"] = [{"stage": s, "fp_ms": p["fp_ticks"] / 1e6, "bp_ms": p["bp_ticks"] / 1e6,
                            "fp_tflops": p["fp_tflops"], "bp_tflops": p["bp_tflops"],
                            "bubble_ms_per_epoch": p["stage_bubble_ticks"] / 1e6,
                            "dT": {n: local_res[n]["stage_dT"][s] for n in names},
                            "op_growth_image": local_res["image"]["pipeline"]["op_growth"][s],
                            "fill_image": runs["image"][s]["with"]["used_s"] / runs["image"][s]["with"]["bubble_s"],
                            "breakdown_image": runs["image"][s]["with"]["breakdown"]}
                           for s, p in enumerate(stage_prof)]
    # configs[3]: mixed side tasks over a 3.6B-shaped pipeline, placed by Alg. 1
    mixed = None
    if not args.no_mixed:
        probe = gpu.Harness(num_stages=STAGES, num_micro_batches=MICRO_BATCHES, stage=0,
                            profile_epochs=0, profile_reps=1, **SHAPE_36B)
        avail = [probe.profile()["available_memory"]]
        probe.close()
        specs = [("pagerank", lambda: gpu.PageRankTask(**PR), 0), ("sgd", lambda: gpu.SgdTask(**SGD), SGD_SMS),
                 ("image", lambda: gpu.ImageTask(batch=BATCH, images_per_step=IMAGES_PER_STEP, **FRAMES), IMG_SMS),
                 ("pagerank2", lambda: gpu.PageRankTask(**PR), 0)]
        from paper_2409_06941_b200.bubblesim import TaskProfile
        mem = {"pagerank": 0.3, "pagerank2": 0.3, "sgd": 1.6, "image": 2.2}
        wstates = A.workers([avail[0]] * STAGES)   # replica: every stage sees its own GPU's memory
        placement = {}
        for name, _, _ in specs:
            o = A.submit_task(TaskProfile(name, 1e-4, 1e-4, mem[name], 32), wstates)
            placement[name] = o.worker_id if o.assigned else None
        mixed = {"placement": placement, "stages": []}
        mruns = []
        for name, make, sms in specs:
            s = placement[name]
            if s is None:
                continue
            h = gpu.Harness(num_stages=STAGES, num_micro_batches=MICRO_BATCHES, stage=s, step_group=STEP_GROUP,
                            **SHAPE_36B)
            r = harvest(h, name, make(), K, W, sms=sms, kinds=PD.issue_kinds(A, s, STAGES, MICRO_BATCHES),
                        budget=DT_BUDGET, pairs=PAIRS_OTHER)
            h.close()
            mruns.append(dict(r, stage=s))
            mixed["stages"].append({"stage": s, "task": name, "units_per_bubble_s": r["with"]["work_units"] / r["base"]["bubble_s"],
                                    "unit": "px" if name == "image" else "edges", "side_sms_mean": r["sms"],
                                    "dT": (r["with"]["makespan_s"] - r["base"]["makespan_s"]) / r["base"]["makespan_s"],
                                    "fill": r["with"]["used_s"] / r["with"]["bubble_s"]})
        mixed["dT_stage_max"] = max(x["dT"] for x in mixed["stages"])
        if len({r_["stage"] for r_ in mruns}) == STAGES:
            mixed["dT_pipeline"] = pipe_dt(mruns, STAGES, MICRO_BATCHES, K)["dT"]
            mp = [PD.critical_path_dt(A, STAGES, MICRO_BATCHES, K, {r_["stage"]: r_["ops_base_runs"][j] for r_ in mruns},
                                      {r_["stage"]: r_["ops_with_runs"][j] for r_ in mruns})["dT"]
                  for j in range(min(len(r_["ops_with_runs"]) for r_ in mruns))]
            mixed["dT_pairs"] = mp
            mixed["dT_se"] = statistics.stdev(mp) / len(mp) ** 0.5 if len(mp) > 1 else None
        mixed["fill_mean"] = statistics.fmean(x["fill"] for x in mixed["stages"])
    local_res["mixed"] = mixed
    # configs[4] at N = 1: every stage of the 8-stage, m = 8 pipeline of
    # nanoGPT-6B-shaped stages (32/8 layers of h = 4096 each) replayed in turn;
    # its runs are 4 epochs, so the ΔT controller starts lower (half the
    # image task's start) -- from 8 SM-equivalents it measured +0.6-1.2 %
    c5 = None
    if not args.no_c5:
        K5 = min(K, 4)
        c5runs, prof = [], None
        for s in range(8):
            h = gpu.Harness(num_stages=8, num_micro_batches=8, stage=s, layers=LAYERS_6B // 8, hidden=HIDDEN_6B,
                            tokens=8192, ffn_mult=4, step_group=STEP_GROUP, profile_epochs=2)
            prof = prof or h.profile()
            r = harvest(h, "image", gpu.ImageTask(batch=BATCH, images_per_step=IMAGES_PER_STEP, **FRAMES), K5, W,
                        sms=max(2, IMG_SMS // 2), kinds=PD.issue_kinds(A, s, 8, 8), budget=DT_BUDGET, pairs=PAIRS_OTHER)
            h.close()
            c5runs.append(dict(r, stage=s))
        pipe = pipe_dt(c5runs, 8, 8, K5)
        c5_pairs = [PD.critical_path_dt(A, 8, 8, K5, {r_["stage"]: r_["ops_base_runs"][j] for r_ in c5runs},
                                        {r_["stage"]: r_["ops_with_runs"][j] for r_ in c5runs})["dT"]
                    for j in range(min(len(r_["ops_with_runs"]) for r_ in c5runs))]
        c5 = {"bubble_rate": prof["bubble_rate"], "fp_ms": prof["fp_ticks"] / 1e6, "bp_ms": prof["bp_ticks"] / 1e6,
              "epochs": K5, "side_sms_mean": statistics.fmean(r_["sms"] for r_ in c5runs),
              "units_per_bubble_s": sum(r_["with"]["work_units"] for r_ in c5runs) / sum(r_["base"]["bubble_s"] for r_ in c5runs),
              "dT_pipeline": pipe["dT"], "dT_pairs": c5_pairs,
              "dT_se": statistics.stdev(c5_pairs) / len(c5_pairs) ** 0.5 if len(c5_pairs) > 1 else None,
              "dT_stage_max": max((r_["with"]["makespan_s"] - r_["base"]["makespan_s"]) / r_["base"]["makespan_s"] for r_ in c5runs),
              "fill": sum(r_["with"]["used_s"] for r_ in c5runs) / sum(r_["with"]["bubble_s"] for r_ in c5runs)}
    local_res["c5"] = c5
    # configs[4] / SURVEY §8(e): with N > 1 GPUs, additionally a REAL N-stage
    # pipeline (6B-shaped stages, rank s = stage s) whose activations and
    # gradients travel through the peer-linked mailboxes (NVLink), one
    # image side-task worker per GPU
    linked = None
    if dist and not args.no_linked:
        from paper_2409_06941_b200 import distributed as D
        shape = dict(layers=max(1, LAYERS_6B // ws), hidden=HIDDEN_6B, tokens=8192, ffn_mult=4)
        try:   # a failure here (e.g. a peer link timing out) must not cost the replica numbers
            linked = D.linked_harvest(
                lambda: gpu.ImageTask(batch=BATCH, images_per_step=IMAGES_PER_STEP, **FRAMES),
                shape, num_micro_batches=max(MICRO_BATCHES, ws), epochs=K, warmup=W, task_name="image",
                step_group=STEP_GROUP, side_sms=IMG_SMS, dt_budget=DT_BUDGET)
            linked["shape"] = shape
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            print(f"[bench] rank {rank}: linked pipeline failed: {e!r}", file=sys.stderr, flush=True)
            linked = {"stage": rank, "error": repr(e)[:300], "shape": shape}
    local_res["linked"] = linked
    csr = None
    if rank == 0 and not args.no_cpu:
        g = gpu.PageRankGraph(scale=PR["scale"], edge_factor=PR["edge_factor"], seed=PR["seed"])
        csr = tuple(t.cpu().numpy() for t in g.csr())
        del g
    results = [local_res]
    if dist:
        results = [None] * ws
        dist.all_gather_object(results, local_res)
    if rank == 0:
        emit(args, results, ws, names, csr)
    if dist:
        dist.destroy_process_group()


def emit(args, results, ws, names, csr):
    K, W = args.steps, args.warmup
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm = peaks.get("hbm_gbs") or 6650.0
    psrc = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"

    def rate(n):
        return sum(r[n]["units"] for r in results) / max(r[n]["bubble_s"] for r in results)

    def dT(n):
        """the pipeline's ΔT (build_schedule over the measured op durations), max over ranks"""
        return max(r[n]["pipeline"]["dT"] for r in results)

    def dT_stages(n):
        return max(x for r in results for x in r[n]["stage_dT"])

    def se(xs):
        return statistics.stdev(xs) / len(xs) ** 0.5 if len(xs) > 1 else None

    def dT_fields(n):
        pairs = results[0][n].get("pair_dT") or []
        return {"dT": dT(n), "dT_se": se(pairs), "dT_pairs": pairs, "dT_stage_max": dT_stages(n),
                "dT_stages": results[0][n]["stage_dT"], "side_sms_mean": results[0][n]["sms"],
                "dt_budget": results[0][n]["budget"],
                "dT_budget_met": (dT(n) <= 0.01) if results[0][n]["budget"] > 0 else None}

    def fill(n):
        return sum(r[n]["used"] for r in results) / sum(r[n]["bubble_with"] for r in results)

    def roof(n, kernel, bound="hbm"):
        a = results[0][n]
        if not a["mean_step_s"]:
            return None
        achieved = a["bytes_per_step"] / a["mean_step_s"] / 1e9
        return {"bound": bound, "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "kernel": kernel, "alg_bytes_per_launch": a["bytes_per_step"],
                "mean_launch_us": a["mean_step_s"] * 1e6, "peak_source": psrc}

    traffic, timgs = load_ncu_traffic()
    if traffic and timgs and timgs != IMAGES_PER_STEP:
        traffic = traffic / timgs * IMAGES_PER_STEP
    # The dominant kernel's HBM roofline: K5 on every SM, launched by the
    # runtime in the bubbles of this run (workload image_full_gpu).  The
    # headline runs the same kernel on the ΔT controller's budget (DESIGN.md
    # §5c): there the bound is the GPU's power budget, not HBM or issue --
    # that operating point (SM-equivalents, GB/s, fraction of HBM) sits beside it.
    image_roof = roof("image_full_gpu", f"img_resize2x_wm_ws ({IMAGES_PER_STEP} frames/launch, all 148 SMs, "
                                        "in-pipeline)") or {}
    image_roof["traffic"] = traffic
    op = roof("image", f"img_resize2x_wm_ws ({IMAGES_PER_STEP} frames/launch, in-pipeline, ΔT-controlled budget)")
    if op:
        sms = results[0]["image"]["sms"] or 148
        image_roof["operating_point"] = {
            "sm_equivalents": sms, "ctas": 3 * sms, "achieved": op["achieved"], "unit": "GB/s",
            "mean_launch_us": op["mean_launch_us"], "hbm_frac": op["frac"],
            "bound": "the GPU power budget (ΔT controller): every joule the side task spends in a bubble "
                     "comes out of the GEMMs' boost clock",
            "how": f"{sms:.1f} SM-equivalents = {3 * sms:.0f} one-pipeline CTAs spread one per SM; "
                   f"{K5_WARP_INSTR_PER_PX} warp-instructions per output pixel (ncu)"}
    cpu = cpu_image(args.cpu_seconds) if not args.no_cpu else None
    if cpu:
        cpu.update(cpu_info())
    e2e = None
    if "image_e2e" in names:
        e2e = {"value": rate("image_e2e"), "unit": UNIT,
               # a step = one 1F1B epoch of all 4 stages (replayed), as for the headline; the e2e leg runs
               # K epochs in each of its PAIRS harvest runs
               "h2d_bytes_per_step": sum(r["image_e2e"]["h2d"] for r in results) / (K * PAIRS),
               "d2h_bytes_per_step": sum(r["image_e2e"]["d2h"] for r in results) / (K * PAIRS),
               **dT_fields("image_e2e"), "fill": fill("image_e2e"),
               "path": f"fr_image_task host_io=1: pinned host frames -> {E2E_RING}-slot device ring filled by the "
                       "copy engines ahead of the steps (also while the pipeline computes; copy-ahead depth 2 slots "
                       "per SM-equivalent of the ΔT controller's budget) -> K5 -> D2H per frame"}
    # PageRank and Graph-SGD kernel rooflines: on all SMs, launched by the
    # runtime in this run's bubbles (workloads *_full_gpu), like K5's; their
    # ΔT-controlled operating points are the workloads' values
    pr_roof = roof("pagerank_full_gpu", "pr_pull_kernel (2 launches of 1 iteration per step, all 148 SMs, "
                                        "in-pipeline); working set L2-resident: latency-bound gathers, not HBM")
    if pr_roof:
        l2 = results[0]["l2_gbps"]
        pr_roof["l2"] = {"achieved": pr_roof["achieved"], "peak": l2, "unit": "GB/s", "frac": pr_roof["achieved"] / l2,
                         "peak_source": "measured in this run: coalesced 16 B ld.global.cg sweeps of a 48 MB "
                                        "L2-resident buffer (fr_l2_read_probe)"}
    workloads = {
        "pagerank": {"config": "configs[0]: RMAT scale 20 (edge factor 16, seed 1), pull, d=0.85, 2 iterations/step",
                     "value": rate("pagerank"), "unit": "edges/bubble-s", **dT_fields("pagerank"),
                     "fill": fill("pagerank"),
                     "roofline": pr_roof,
                     "cpu_baseline": cpu_pagerank(args.cpu_seconds / 2, csr) if csr is not None else None},
        "sgd": {"config": f"configs[2]: Orkut shape V=3,072,441 E=117,185,083 k=16, {SGD['edges_per_step']} edges/step, "
                          "by-user layout (fr_sgd_group_by_user)",
                "value": rate("sgd"), "unit": "edges/bubble-s", **dT_fields("sgd"), "fill": fill("sgd"),
                "roofline": dict(roof("sgd_full_gpu", f"sgd_user_kernel<16> ({SGD['edges_per_step']} edges/launch, "
                                                      "all 148 SMs, in-pipeline; "
                                             "alg bytes 12 + 128 per edge + 128 per L_u load; item blocks keep "
                                             "L_v in L2, so part of them never reaches DRAM)") or {},
                                 traffic=63.6 * SGD["edges_per_step"],
                                 traffic_source="profiles/r2_sgd_harvest_ncu.txt (inside a harvest, all SMs: "
                                                "266.7 MB DRAM per 2^22-edge step)"),
                "cpu_baseline": cpu_sgd(args.cpu_seconds / 2) if not args.no_cpu else None},
    }
    for n, unit in (("pagerank_full_gpu", "edges/bubble-s"), ("sgd_full_gpu", "edges/bubble-s")):
        workloads[n] = {"config": f"{n[:-9]} with the side task on all 148 SMs (no ΔT budget): the kernel's "
                                  "roofline is measured here", "value": rate(n), "unit": unit, **dT_fields(n),
                        "fill": fill(n)}
    imp = results[0]["image_imperative"]
    workloads["image_imperative"] = {
        "config": "configs[1] through the imperative interface (RunGpuWorkload): one preemptible K5 "
                  "workload per bubble over the 64-frame batch, paused on the device per output row",
        "value": rate("image_imperative"), "unit": UNIT, **dT_fields("image_imperative"),
        "fill": fill("image_imperative"),
        "overrun_per_pause_us": sum(r["image_imperative"]["overrun"] for r in results)
        / max(1, sum(r["image_imperative"]["pauses"] for r in results)) * 1e6,
        "alg_GBps_in_bubbles": imp["units"] / OUT_PX * (FRAMES["sw"] * FRAMES["sh"] * 3 + OUT_PX * 3)
        / max(1e-12, imp["used"] + imp["overrun"]) / 1e9,
        "workload_launches": imp["launches"]}
    workloads["image_full_gpu"] = {
        "config": "configs[1] with the side task on all 148 SMs: the most px per bubble-second, but the "
                  "power its HBM streaming draws slows every GEMM of the pipeline (DESIGN.md §5c)",
        "value": rate("image_full_gpu"), "unit": UNIT, **dT_fields("image_full_gpu"), "fill": fill("image_full_gpu"),
        "roofline": roof("image_full_gpu", f"img_resize2x_wm_ws ({IMAGES_PER_STEP} frames/launch, 148 SMs, "
                                           "in-pipeline)")}
    launches = sum(r[n]["launches"] for r in results for n in names) + sum(r["gap_kernels"] for r in results)
    line = {
        "metric": METRIC, "value": rate("image"), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": max(r["image"]["t_with"] for r in results) / (K * PAIRS) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded counter-based frames/watermark, RMAT graph, Orkut-shaped ratings)",
        "config": bench_config(ws),
        "side_sms_mean": results[0]["image"]["sms"],
        "delta_t": dT("image"),
        "delta_t_def": "pipeline makespan growth: per-stage mean FP/BP op durations with vs without the side task "
                       "(every stage replayed) through build_schedule (pipeline_dt.critical_path_dt)",
        "delta_t_stage_max": dT_stages("image"), "delta_t_stages": results[0]["image"]["stage_dT"],
        "dT_budget_met": dT("image") <= 0.01, "fill": fill("image"),
        "delta_t_pairs": PAIRS,
        "delta_t_pair_values": results[0]["image"]["pair_dT"],
        "delta_t_se": se(results[0]["image"]["pair_dT"]),
        "delta_t_noise": {"null_dT": results[0]["image"]["null_dT"],
                          "how": "pipeline ΔT between the baseline runs (no side task in either) of successive ABBA pairs"},
        "overrun_frac": sum(r["image"]["overrun"] for r in results) / max(1e-12, sum(r["image"]["used"] for r in results)),
        "bubble_s_per_step": max(r["image"]["bubble_s"] for r in results) / (K * PAIRS),
        "px_per_step": sum(r["image"]["units"] for r in results) / (K * PAIRS),
        "roofline": image_roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": results[0]["clocks"],
        "gpu_launches": launches, "workloads": workloads, "stages": results[0]["stages"],
    }
    errs = [r["linked"]["error"] for r in results if r.get("linked") and "error" in r["linked"]]
    if errs:
        workloads["pipeline_linked"] = {"error": errs[0], "ranks_failed": len(errs)}
    elif results[0].get("linked"):
        ls = [r["linked"] for r in results]
        t_no = max(x["base"]["makespan_s"] for x in ls)
        workloads["pipeline_linked"] = {
            "config": f"configs[4]-style: real {ws}-stage 1F1B pipeline (m={max(MICRO_BATCHES, ws)}), "
                      f"nanoGPT-6B-shaped stages {ls[0]['shape']}, activations/gradients through "
                      "peer-linked mailboxes (copy engine over NVLink), image side task on every stage",
            "value": sum(x["with"]["work_units"] for x in ls) / max(x["base"]["bubble_s"] for x in ls),
            "unit": UNIT, "dT": (max(x["with"]["makespan_s"] for x in ls) - t_no) / t_no,
            "fill": sum(x["with"]["used_s"] for x in ls) / sum(x["with"]["bubble_s"] for x in ls),
            "bubble_rate": ls[0]["profile"]["bubble_rate"],
            "exchange": {"messages": sum(x["with"]["exchange_messages"] for x in ls),
                         "us_per_message": statistics.fmean(x["with"]["exchange_us"] for x in ls if x["with"]["exchange_messages"]),
                         "GBps": statistics.fmean(x["with"]["exchange_gbps"] for x in ls if x["with"]["exchange_messages"]),
                         "how": "copy engine, mailbox slot on the neighbour GPU (NVLink peer memory)"},
            "stages": [{"stage": x["stage"], "dT": (x["with"]["makespan_s"] - x["base"]["makespan_s"])
                        / x["base"]["makespan_s"], "fill": x["with"]["used_s"] / max(1e-12, x["with"]["bubble_s"])}
                       for x in ls]}
    if not args.no_cpu:
        # host hot path: ours vs the reference's own sources
        # (oracle/_ref) as the CPU baseline, same C-ABI, C++ time only
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import host_path_bench  # noqa: E402
        from paper_2409_06941_b200 import api as host_api
        from paper_2409_06941_b200.bubblesim import BubbleSim, PipelineConfig
        import ctypes
        ref_so = os.path.join(ROOT, "oracle", "_ref", "libbubblesim_ref.so")
        ref = BubbleSim(ctypes.CDLL(ref_so)) if os.path.exists(ref_so) else None
        hp = {}
        for name, (p, m) in {"C1_p4_m4_128ep": (4, 4), "C5_p8_m8_128ep": (8, 8)}.items():
            cfg = PipelineConfig(p, m, [220], [347], 128, 48.0, [1.0] * p, 1e-3)
            (b, x), n_ops, n_b = host_path_bench.time_host(host_api(), cfg)
            row = {"ops": n_ops, "bubbles": n_b, "build_schedule_ms": b * 1e3, "extract_bubbles_ms": x * 1e3}
            if ref:
                (rb, rx), _, _ = host_path_bench.time_host(ref, cfg)
                row["cpu_baseline"] = {"kind": "reference", "cores": 1, "build_schedule_ms": rb * 1e3,
                                       "extract_bubbles_ms": rx * 1e3, "speedup": (rb + rx) / (b + x)}
            hp[name] = row
        workloads["host_path"] = hp
    if results[0].get("c5"):
        workloads["c5_stage_replay"] = dict(
            results[0]["c5"], unit=UNIT,
            config="configs[4] at one GPU: every stage of an 8-stage m=8 1F1B pipeline of nanoGPT-6B-shaped "
                   f"stages (4 layers x h 4096 each) replayed in turn, image side task, {IMAGES_PER_STEP} "
                   "frames/step; dT_pipeline through build_schedule over the 8 stages' op durations")
    if results[0].get("mixed"):
        workloads["mixed"] = dict(results[0]["mixed"],
                                  config="configs[3]: PageRank + SGD + Image + PageRank on a "
                                         "nanoGPT-3.6B-shaped 4-stage pipeline, placed by Alg. 1")
    print(json.dumps(line), flush=True)


def reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    per = max(1.0, args.cpu_seconds / max(1, K))
    for _ in range(W):
        cpu_image(min(per, 1.0))
    vals = [cpu_image(per) for _ in range(K)]
    v = statistics.fmean(x["value"] for x in vals)
    secs = sum(x["seconds"] for x in vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": secs / K * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded counter-based frames/watermark)",
            "impl": "reference",
            "config": bench_config(ws),
            "cpu_baseline": {"value": v, "unit": "px/s", "cores": vals[0]["cores"], "kind": "port",
                             "sample": vals[0]["sample"], **cpu_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the reference ships no side-task code (task.hpp:36-38); this is the CPU restatement "
                    "(oracle/sidetasks.c) -- every CPU second of work counted as a bubble-second"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-mixed", action="store_true")
    ap.add_argument("--no-linked", action="store_true", help="skip the real N-stage pipeline (N > 1)")
    ap.add_argument("--no-c5", action="store_true", help="skip the 8-stage 6B-shaped stage replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
