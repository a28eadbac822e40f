"""Device-timed microbenchmark of the K5 image step (CUDA events on the
launching stream).  Usage: python scripts/img_microbench.py [n_per_step] [reps]
env FR_IMG_MAX_SMS: the plan's SM budget (fr_img_plan_set_max_sms)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    per_step = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    batch = 64
    plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
    plan.set_max_sms(int(os.environ.get("FR_IMG_MAX_SMS", "0")))
    src = gpu.img_generate(batch, 3840, 2160, seed=1)
    wm = gpu.img_generate_watermark(1920, 1080, seed=7)
    dst = torch.empty((batch, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    s = gpu.low_priority_stream()
    wmp = plan.prepare(wm, stream=s)
    torch.cuda.synchronize()
    steps = batch // per_step
    for _ in range(3):
        for i in range(steps):
            sl = slice(i * per_step, (i + 1) * per_step)
            plan.run_prepared(src[sl], dst[sl], wmp, stream=s)
    s.synchronize()
    if len(sys.argv) > 3 and sys.argv[3] == "chain1":   # one event between consecutive steps
        n = reps * steps
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        ev[0].record(s)
        for k in range(n):
            i = k % steps
            plan.run_prepared(src[i * per_step:(i + 1) * per_step], dst[i * per_step:(i + 1) * per_step], wmp,
                              stream=s)
            ev[k + 1].record(s)
        s.synchronize()
        ts = sorted(ev[k].elapsed_time(ev[k + 1]) * 1e-3 for k in range(n))
        med = ts[len(ts) // 2]
        alg = per_step * (24883200 + 6220800) + wmp.numel()
        print(json.dumps({"per_step": per_step, "mode": "chain1", "median_s": med, "alg_GBps": alg / med / 1e9}))
        return
    if len(sys.argv) > 3 and sys.argv[3] == "chain":   # steps back to back, events only around each batch pass
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record(s)
            for i in range(steps):
                sl = slice(i * per_step, (i + 1) * per_step)
                plan.run_prepared(src[sl], dst[sl], wmp, stream=s)
            b.record(s)
        s.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e-3 / steps for a, b in ev)
        med = ts[len(ts) // 2]
        alg = per_step * (24883200 + 6220800) + wmp.numel()
        print(json.dumps({"per_step": per_step, "mode": "chain", "median_s": med, "alg_GBps": alg / med / 1e9}))
        return
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps * steps)]
    k = 0
    for _ in range(reps):
        for i in range(steps):
            sl = slice(i * per_step, (i + 1) * per_step)
            ev[k][0].record(s)
            plan.run_prepared(src[sl], dst[sl], wmp, stream=s)
            ev[k][1].record(s)
            k += 1
    s.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e-3 for a, b in ev)
    med = ts[len(ts) // 2]
    alg = per_step * (24883200 + 6220800) + wmp.numel()
    print(json.dumps({"per_step": per_step, "median_s": med, "min_s": ts[0],
                      "alg_GBps": alg / med / 1e9, "px_per_s": per_step * 2073600 / med,
                      "path": plan.path}))


if __name__ == "__main__":
    main()
