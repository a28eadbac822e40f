"""Energy per output pixel of the K5 step (NVML total-energy counter), the
quantity a ΔT budget actually rations.  Back-to-back 16-frame
launches on the low-priority stream for SECONDS; idle power measured first
(same duration, nothing running) and subtracted -> dynamic nJ per pixel.
Usage: python scripts/img_energy.py [seconds]   env: FR_IMG_MAX_SMS, FR_IMG_PIPES, FR_IMG_CFG, FR_IMG_MATH
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    import pynvml
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(0)
    plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
    plan.set_max_sms(int(os.environ.get("FR_IMG_MAX_SMS", "0")))
    batch, per = 64, 16
    src = gpu.img_generate(batch, 3840, 2160, seed=1)
    wm = gpu.img_generate_watermark(1920, 1080, seed=7)
    dst = torch.empty((batch, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    s = gpu.low_priority_stream()
    wmp = plan.prepare(wm, stream=s)
    torch.cuda.synchronize()

    def burst(n):
        for k in range(n):
            i = k % (batch // per)
            plan.run_prepared(src[i * per:(i + 1) * per], dst[i * per:(i + 1) * per], wmp, stream=s)

    burst(8)
    s.synchronize()
    # launches per second, to size the timed loop
    t0 = time.perf_counter()
    burst(40)
    s.synchronize()
    rate = 40 / (time.perf_counter() - t0)
    time.sleep(1.0)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
    time.sleep(secs)
    idle_w = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e0) / 1e3 / secs
    n = max(10, int(rate * secs))
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
    t0 = time.perf_counter()
    burst(n)
    s.synchronize()
    el = time.perf_counter() - t0
    joules = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e0) / 1e3
    px = n * per * 1920 * 1080
    out = {"sms": int(os.environ.get("FR_IMG_MAX_SMS", "0")), "pipes": os.environ.get("FR_IMG_PIPES", "1"),
           "cfg": os.environ.get("FR_IMG_CFG", "ws"), "math": os.environ.get("FR_IMG_MATH", "1"),
           "px_per_s": px / el, "watts": joules / el, "idle_w": idle_w,
           "nj_per_px": joules / px * 1e9, "dyn_nj_per_px": (joules - idle_w * el) / px * 1e9,
           "sm_mhz": pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
