"""Why is K5 slower inside bubbles than alone?  Per-step durations inside a
harness run (stage 1 of the bench pipeline) vs the same 8-frame launches
alone, and alone right after a burst of stand-in GEMM ops (power state)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def pct(xs):
    xs = sorted(xs)
    return {"p10": xs[len(xs) // 10] * 1e6, "p50": xs[len(xs) // 2] * 1e6, "p90": xs[9 * len(xs) // 10] * 1e6,
            "n": len(xs)}


def alone(plan, src, dst, wmp, s, reps=40):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for k, (a, b) in enumerate(ev):
        sl = slice((k % 8) * 8, (k % 8) * 8 + 8)
        a.record(s)
        plan.run_prepared(src[sl], dst[sl], wmp, stream=s)
        b.record(s)
    s.synchronize()
    return [a.elapsed_time(b) * 1e-3 for a, b in ev]


def main():
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192)
    task = gpu.ImageTask(batch=64, images_per_step=8)
    h.submit("image", task, profile_steps=16)
    h.run(3, True)
    r = h.run(6, True)
    steps = [b - a for a, b in h.timeline(2)]
    out = {"in_bubbles": pct(steps), "fill": r["used_s"] / r["bubble_s"]}
    h.close()
    plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
    src = gpu.img_generate(64, 3840, 2160, seed=1)
    wm = gpu.img_generate_watermark(1920, 1080, seed=7)
    dst = torch.empty((64, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    s = gpu.low_priority_stream()
    wmp = plan.prepare(wm, stream=s)
    torch.cuda.synchronize()
    alone(plan, src, dst, wmp, s, 10)
    out["alone"] = pct(alone(plan, src, dst, wmp, s))
    # after a GEMM burst: ~200 ms of bf16 matmuls, then the image launches
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(120):
        a @ a
    out["after_gemm_burst"] = pct(alone(plan, src, dst, wmp, s))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
