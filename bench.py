"""Benchmark of the bubble-harvesting hot path (BASELINE.json metric):

  side-task px/s per bubble-second at <= 1 % pipeline ΔT, HBM GB/s vs peak

Workload (BASELINE.json configs[1]): the image resize + watermark side task
(64 synthetic 4K RGB frames -> 1080p, RGBA watermark) harvesting the bubbles
of a 4-stage 1F1B pipeline (m = 4) whose stages are nanoGPT-1.2B-shaped
bf16 GEMM stand-ins (6 layers x h 2048 per stage, 8192 tokens per
micro-batch).  One GPU replays every stage of the pipeline in turn ("replica
mode"); with --gpus N each rank is an independent replica
(no collective on the data path) -> scaling "weak".

A bench *step* is one training iteration (epoch) of all 4 stages with the
side task harvesting its bubbles.  Per stage: the bubble profiler dry-runs
the pipeline, the task is profiled standalone then submitted (Alg. 1), W
warm-up epochs run with the task (InitSideTask lands in a bubble; the task's
per-step duration is re-profiled in-situ), then K epochs without side tasks
(the ΔT baseline and the bubble-seconds denominator) and K timed epochs with
them.  All times are device times (CUDA events / %globaltimer).

  value  = side-task output px completed / baseline bubble-seconds
           (summed over ranks / max over ranks' bubble-seconds)
  e2e    = the same through the host-buffer path: frames in pinned host
           memory, H2D + kernel + D2H inside every RunNextStep
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
SHAPE = dict(layers=6, hidden=2048, tokens=8192, ffn_mult=4)
FRAMES = dict(sw=3840, sh=2160, dw=1920, dh=1080)
BATCH = 64
IMAGES_PER_STEP = 8
E2E_IMAGES_PER_STEP = 1
OUT_PX = FRAMES["dw"] * FRAMES["dh"]
SRC_BYTES = FRAMES["sw"] * FRAMES["sh"] * 3
DST_BYTES = OUT_PX * 3
PREPARED_WM_BYTES = OUT_PX * 8
METRIC = "side-task px/s per bubble-sec at <=1% pipeline dT (image 4K->1080p+watermark); HBM GB/s vs peak"
UNIT = "px/bubble-s"
WORKLOAD = ("image resize+watermark side task (64x 3840x2160 RGB -> 1920x1080, RGBA watermark), "
            "harvesting a 4-stage 1F1B pipeline (m=4) of nanoGPT-1.2B-shaped bf16 GEMM stand-ins, "
            "every stage replayed per GPU (replica mode)")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """Samples SM clock + throttle reasons during the timed region (NVML)."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

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
        names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}
        while not self._stop.is_set():
            try:
                util = nv.nvmlDeviceGetUtilizationRates(self._h).gpu
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                if util > 0:
                    self.samples.append(mhz)
                for bit, name in names.items():
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
    p = os.path.join(ROOT, "profiles", "ncu_image_step.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("images_per_launch")
    except OSError:
        return None, None


def cpu_image_throughput(seconds: float, images: int = IMAGES_PER_STEP):
    """The CPU restatement (oracle/sidetasks.c, OpenMP over all host threads)
    on a bounded sample: the same 8-frame step repeated for ~`seconds`."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import sidetasks_oracle  # noqa: E402  (oracle: CPU baseline leg only)
    o = sidetasks_oracle.load()
    src = o.img_generate(images, FRAMES["sw"], FRAMES["sh"], seed=1)
    wm = o.img_generate_watermark(FRAMES["dw"], FRAMES["dh"], seed=7)
    o.img_resize_watermark(src, wm, FRAMES["dw"], FRAMES["dh"])  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        o.img_resize_watermark(src, wm, FRAMES["dw"], FRAMES["dh"])
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": reps * images * OUT_PX / el, "unit": "px/s", "cores": os.cpu_count(),
            "kind": "port", "seconds": el,
            "sample": f"{reps} x {images} frames 3840x2160->1920x1080 (+watermark), "
                      f"oracle/sidetasks.c OpenMP on {os.cpu_count()} host threads"}


def run_stage(gpu, stage, K, W, host_io):
    h = gpu.Harness(num_stages=STAGES, num_micro_batches=MICRO_BATCHES, stage=stage, **SHAPE)
    prof = h.profile()
    # host-buffer steps are PCIe-bound (25 MB H2D per frame): one frame per
    # step keeps a step well inside the ~3 ms type-C bubbles
    ips = E2E_IMAGES_PER_STEP if host_io else IMAGES_PER_STEP
    task = gpu.ImageTask(batch=BATCH, images_per_step=ips, host_io=host_io, **FRAMES)
    ok, tprof = h.submit("image", task, profile_steps=32)
    if not ok:
        raise RuntimeError(f"stage {stage}: image task rejected by Alg. 1")
    h.run(max(W, 1), True)
    h.reprofile("image")       # per-step duration measured in bubbles, under load
    base = h.run(K, False)
    r = h.run(K, True)
    steps = h.timeline(2)
    durs = [b - a for a, b in steps]
    side, train = h.launches()
    out = {"stage": stage, "profile": prof, "task_profile": tprof, "base": base, "with": r,
           "step_durs": durs, "gap_kernels": train // (2 * MICRO_BATCHES) * (2 * MICRO_BATCHES + 1),
           "side_launches": side, "units_per_step": task.units_per_step,
           "bytes_per_step": task.bytes_per_step, "h2d": task.h2d_per_step, "d2h": task.d2h_per_step}
    h.close()
    return out


def ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    K, W = args.steps, args.warmup

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        dev = [run_stage(gpu, s, K, W, host_io=False) for s in range(STAGES)]
    torch.cuda.synchronize()
    e2e_runs = [run_stage(gpu, s, K, W, host_io=True) for s in range(STAGES)] if not args.no_e2e else []
    if dist:
        dist.barrier()

    def agg(runs):
        px = sum(r["with"]["work_units"] for r in runs)
        bub = sum(r["base"]["bubble_s"] for r in runs)
        t_no = sum(r["base"]["makespan_s"] for r in runs)
        t_w = sum(r["with"]["makespan_s"] for r in runs)
        used = sum(r["with"]["used_s"] for r in runs)
        bub_w = sum(r["with"]["bubble_s"] for r in runs)
        over = sum(r["with"]["overrun_s"] for r in runs)
        return dict(px=px, bubble_s=bub, t_no=t_no, t_with=t_w, used=used, bubble_with=bub_w, overrun=over,
                    steps=sum(r["with"]["steps_completed"] for r in runs))

    a = agg(dev)
    durs = [d for r in dev for d in r["step_durs"]]
    mean_dur = statistics.fmean(durs) if durs else float("nan")
    local_res = {
        "px": a["px"], "bubble_s": a["bubble_s"], "t_no": a["t_no"], "t_with": a["t_with"],
        "used": a["used"], "bubble_with": a["bubble_with"], "overrun": a["overrun"], "steps": a["steps"],
        "mean_step_s": mean_dur, "clocks": clk.summary(),
        "gpu_launches": sum(r["side_launches"] + r["gap_kernels"] for r in dev),
        "e2e": agg(e2e_runs) if e2e_runs else None,
        "e2e_h2d": sum(r["h2d"] * r["with"]["steps_completed"] for r in e2e_runs),
        "e2e_d2h": sum(r["d2h"] * r["with"]["steps_completed"] for r in e2e_runs),
        "stages": [{"stage": r["stage"], "fp_ms": r["profile"]["fp_ticks"] / 1e6,
                    "bp_ms": r["profile"]["bp_ticks"] / 1e6, "fp_tflops": r["profile"]["fp_tflops"],
                    "bp_tflops": r["profile"]["bp_tflops"],
                    "dT": (r["with"]["makespan_s"] - r["base"]["makespan_s"]) / r["base"]["makespan_s"],
                    "fill": r["with"]["used_s"] / r["with"]["bubble_s"] if r["with"]["bubble_s"] else 0.0,
                    "est_step_us": r["task_profile"]["est_per_step_duration"] * 1e6,
                    "breakdown": r["with"]["breakdown"]} for r in dev],
        "bytes_per_step": dev[0]["bytes_per_step"],
    }
    results = [local_res]
    if dist:
        results = [None] * ws
        dist.all_gather_object(results, local_res)
    if rank == 0:
        emit(args, results, ws)
    if dist:
        dist.destroy_process_group()


def emit(args, results, ws):
    K, W = args.steps, args.warmup
    px = sum(r["px"] for r in results)
    bub = max(r["bubble_s"] for r in results)
    value = px / bub
    t_no = max(r["t_no"] for r in results)
    t_with = max(r["t_with"] for r in results)
    r0 = results[0]
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    achieved = r0["bytes_per_step"] / r0["mean_step_s"] / 1e9
    traffic, traffic_imgs = load_ncu_traffic()
    if traffic and traffic_imgs and traffic_imgs != IMAGES_PER_STEP:
        traffic = traffic / traffic_imgs * IMAGES_PER_STEP
    cpu = cpu_image_throughput(args.cpu_seconds) if not args.no_cpu else None
    e2e = None
    if all(r["e2e"] for r in results):
        e_px = sum(r["e2e"]["px"] for r in results)
        e_bub = max(r["e2e"]["bubble_s"] for r in results)
        e2e = {"value": e_px / e_bub, "unit": UNIT,
               "h2d_bytes_per_step": sum(r["e2e_h2d"] for r in results) / (K * STAGES),
               "d2h_bytes_per_step": sum(r["e2e_d2h"] for r in results) / (K * STAGES),
               "dT": (max(r["e2e"]["t_with"] for r in results) - max(r["e2e"]["t_no"] for r in results))
               / max(r["e2e"]["t_no"] for r in results),
               "fill": sum(r["e2e"]["used"] for r in results) / sum(r["e2e"]["bubble_with"] for r in results),
               "path": "fr_image_task host_io=1: pinned host frames, H2D + K5 + D2H per RunNextStep"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": t_with / K * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded counter-based frames/watermark)",
        "config": {"workload": WORKLOAD, "stages": STAGES, "micro_batches": MICRO_BATCHES,
                   "stage_shape": SHAPE, "frames": BATCH, "images_per_step": IMAGES_PER_STEP,
                   "step": "one 1F1B epoch of all 4 stages (replayed) with the side task",
                   "parallelism": f"replicas x{ws}",
                   "l2": "inputs 1.6 GB per batch > 126 MB L2; no flush needed"},
        "delta_t": (t_with - t_no) / t_no,
        "fill": sum(r["used"] for r in results) / sum(r["bubble_with"] for r in results),
        "overrun_frac": sum(r["overrun"] for r in results) / max(1e-12, sum(r["used"] for r in results)),
        "bubble_s_per_step": bub / K, "px_per_step": px / K,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": "img_resize2x_wm_tma (8 frames/launch, in-pipeline)",
                     "alg_bytes_per_launch": r0["bytes_per_step"],
                     "mean_launch_us": r0["mean_step_s"] * 1e6,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": r0["clocks"],
        "gpu_launches": sum(r["gpu_launches"] for r in results),
        "stages": r0["stages"],
    }
    print(json.dumps(line), flush=True)


def reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    per = max(1.0, args.cpu_seconds / max(1, K))
    for _ in range(W):
        cpu_image_throughput(min(per, 1.0))
    vals = [cpu_image_throughput(per) for _ in range(K)]
    v = statistics.fmean(x["value"] for x in vals)
    secs = sum(x["seconds"] for x in vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": secs / K * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded counter-based frames/watermark)",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "frames": BATCH, "images_per_step": IMAGES_PER_STEP},
            "cpu_baseline": {"value": v, "unit": "px/s", "cores": vals[0]["cores"], "kind": "port",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the reference ships no side-task code (task.hpp:36-38); this is the CPU "
                    "restatement (oracle/sidetasks.c) every CPU second of which is a bubble-second"}
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
