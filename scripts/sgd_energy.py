"""Energy per edge of the Graph-SGD step (NVML), like scripts/img_energy.py:
back-to-back 2^22-edge steps (by-user layout, the task's) for SECONDS, idle
power subtracted.  Usage: python scripts/sgd_energy.py [seconds] [sms ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    budgets = [int(x) for x in sys.argv[2:]] or [0]
    import pynvml
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(0)
    p = gpu.SgdProblem(by_user=True)
    s = gpu.low_priority_stream()
    chunk = 1 << 22
    n = p.E // chunk
    torch.cuda.synchronize()
    time.sleep(1.0)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
    time.sleep(secs)
    idle_w = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e0) / 1e3 / secs
    for sms in budgets:
        p.set_max_sms(sms)
        k = 0

        def burst(m):
            nonlocal k
            for _ in range(m):
                j = k % n
                p.step(j * chunk, (j + 1) * chunk, stream=s)
                k += 1

        burst(4)
        s.synchronize()
        t0 = time.perf_counter()
        burst(20)
        s.synchronize()
        rate = 20 / (time.perf_counter() - t0)
        m = max(10, int(rate * secs))
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
        t0 = time.perf_counter()
        burst(m)
        s.synchronize()
        el = time.perf_counter() - t0
        j = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e0) / 1e3
        edges = m * chunk
        print(json.dumps({"sms": sms, "edges_per_s": edges / el, "watts": j / el, "idle_w": idle_w,
                          "nj_per_edge": j / edges * 1e9, "dyn_nj_per_edge": (j - idle_w * el) / edges * 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
