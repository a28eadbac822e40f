"""Is HBM streaming slower right after tensor-core bursts?  Alternate GEMM
bursts and image steps on one stream (no harness), time each image step, and
sample NVML SM/memory clocks + power."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def sampler(stop, out):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.005)


def main():
    plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
    src = gpu.img_generate(64, 3840, 2160)
    dst = torch.empty((64, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    wmp = plan.prepare(gpu.img_generate_watermark(1920, 1080))
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def img_steps(n):
        ev = []
        for k in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            i = (k % 8) * 8
            e0.record()
            plan.run_prepared(src[i:i + 8], dst[i:i + 8], wmp)
            e1.record()
            ev.append((e0, e1))
        return ev

    stop, samples = threading.Event(), []
    th = threading.Thread(target=sampler, args=(stop, samples))
    th.start()
    res = {}
    lo, hi = torch.cuda.Stream.priority_range()
    hs = torch.cuda.Stream(priority=hi)
    ls = torch.cuda.Stream(priority=lo)
    for mode in ["idle", "after_gemm", "idle_again", "spinner_hi", "lowpri_alone"]:
        evs = []
        for rep in range(30):
            if mode == "after_gemm":
                for _ in range(6):
                    torch.matmul(a, b)   # ~4 ms of tensor-core work
            if mode in ("spinner_hi", "lowpri_alone"):
                torch.cuda.synchronize()
                if mode == "spinner_hi":
                    with torch.cuda.stream(hs):
                        torch.cuda._sleep(8_000_000)  # resident high-priority spin kernel
                with torch.cuda.stream(ls):
                    evs += img_steps(40)
                torch.cuda.synchronize()
                continue
            evs += img_steps(40)         # ~2-3 ms of streaming
            if mode != "after_gemm":
                torch.cuda._sleep(5_000_000)
        torch.cuda.synchronize()
        d = [e0.elapsed_time(e1) * 1e3 for e0, e1 in evs]
        first = [d[i] for i in range(0, len(d), 40)]
        res[mode] = {"step_us_med": statistics.median(d), "first_step_us_med": statistics.median(first),
                     "last10_us_med": statistics.median([d[i] for i in range(len(d)) if i % 40 >= 30])}
    stop.set()
    th.join()
    sm = [x[0] for x in samples]
    mem = [x[1] for x in samples]
    pw = [x[2] for x in samples]
    res["nvml"] = {"sm_mhz_deciles": statistics.quantiles(sm, n=10), "mem_mhz_set": sorted(set(mem)),
                   "power_w_max": max(pw), "power_w_med": statistics.median(pw)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
