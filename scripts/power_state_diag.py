"""Is a side-task step slower right after a sustained tensor-core burst (the
power controller holding clocks down) than on an idle GPU?  Times SGD and
image steps cold-idle vs immediately after ~300 ms of bf16 GEMMs (synced)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def timed(fn, s, n=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    s.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def main():
    s = gpu.low_priority_stream()
    p = gpu.SgdProblem()
    plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
    src = gpu.img_generate(16, 3840, 2160, seed=1)
    wm = gpu.img_generate_watermark(1920, 1080, seed=7)
    dst = torch.empty((16, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    wmp = plan.prepare(wm, stream=s)
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    sgd = lambda: p.step(0, 1 << 21, stream=s)
    img = lambda: plan.run_prepared(src, dst, wmp, stream=s)
    out = {}
    for name, fn in (("sgd", sgd), ("image16", img)):
        timed(fn, s, 3)
        time.sleep(0.5)
        idle = timed(fn, s)
        for _ in range(150):
            a @ a
        torch.cuda.synchronize()
        hot = timed(fn, s)
        out[name] = {"idle_us": idle, "after_gemm_us": hot, "slowdown": hot / idle}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
