"""Where does the noise of the pipeline ΔT come from?  One stage of the bench
pipeline, a long sequence of runs (B = no side task, H = image task at a fixed
budget) in the pattern given; per run, every epoch's mean FP and BP op
duration, and the GPU's temperature / power / SM clock (NVML) after the run.

Usage: python scripts/dt_epoch_diag.py [stage] [K] [pattern] [side_sms]
       e.g. 0 8 BBHHBBHHBBHHBBHHBBHH 11 -> JSON lines, one per run
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_06941_b200 import api, gpu  # noqa: E402
from paper_2409_06941_b200 import pipeline_dt as P  # noqa: E402


def main():
    stage = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    pattern = sys.argv[3] if len(sys.argv) > 3 else "BH" * 10
    sms = int(sys.argv[4]) if len(sys.argv) > 4 else 11
    torch.cuda.set_device(0)
    import pynvml
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(0)
    a = api()
    kinds = P.issue_kinds(a, stage, 4, 4)
    n = len(kinds)
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=6, hidden=2048, tokens=8192,
                    ffn_mult=4, step_group=3, side_sms=sms)
    ok, _ = h.submit("image", gpu.ImageTask(batch=64, images_per_step=16), profile_steps=16)
    assert ok
    h.run(3, True)
    h.reprofile("image")
    for i, c in enumerate(pattern):
        r = h.run(K, c == "H")
        ops = h.timeline(0)
        ep = []
        for e in range(K):
            ep.append(P.op_means(ops[e * n:(e + 1) * n], kinds))
        durs = [b - a for a, b in ops]
        med = sorted(durs[j] for j in range(len(durs)) if kinds[j % n] == 0)[len(durs) // (2 * 2)]
        slow = [(j // n, j % n, round(d * 1e3, 3), round((ops[j][0] - ops[j - 1][1]) * 1e6, 1) if j else None)
                for j, d in enumerate(durs) if kinds[j % n] == 0 and d > 1.05 * med]
        print(json.dumps({"i": i, "kind": c, "epochs": ep, "makespan_s": r["makespan_s"], "slow_fp": slow,
                          "temp_c": pynvml.nvmlDeviceGetTemperature(nv, pynvml.NVML_TEMPERATURE_GPU),
                          "power_w": pynvml.nvmlDeviceGetPowerUsage(nv) / 1000.0,
                          "sm_mhz": pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM),
                          "px": r["work_units"]}), flush=True)
    h.close()


if __name__ == "__main__":
    main()
