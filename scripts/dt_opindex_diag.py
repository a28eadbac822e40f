"""Which ops of a stage grow when its bubbles are harvested?  One stage, a
fixed side-task budget, ABBA (baseline, harvest) pairs; per op index of the
stage's 1F1B epoch: mean duration with / without, and whether a bubble
precedes the op (a harvested bubble's last step may still hold SMs when the
op becomes ready).  Separates a per-bubble transition cost (growth only on
ops right after a bubble) from a power cost (growth on every op).
Usage: python scripts/dt_opindex_diag.py TASK STAGE SMS [pairs] [K]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

from paper_2409_06941_b200 import api, gpu  # noqa: E402
from paper_2409_06941_b200 import pipeline_dt as P  # noqa: E402
from harvest_sweep import make  # noqa: E402


def main():
    name, stage, sms = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    pairs = int(sys.argv[4]) if len(sys.argv) > 4 else 6
    K = int(sys.argv[5]) if len(sys.argv) > 5 else 8
    torch.cuda.set_device(0)
    a = api()
    kinds = P.issue_kinds(a, stage, 4, 4)
    n = len(kinds)
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=6, hidden=2048, tokens=8192,
                    ffn_mult=4, step_group=3, side_sms=sms)
    ok, _ = h.submit(name, make(name), profile_steps=16)
    assert ok
    h.run(2, False)
    h.run(2, True)
    h.reprofile(name)
    dur = {False: [[] for _ in range(n)], True: [[] for _ in range(n)]}
    gaps = {False: [[] for _ in range(n)], True: [[] for _ in range(n)]}
    rep = []
    for i in range(pairs):
        for wt in ((False, True) if i % 2 == 0 else (True, False)):
            r = h.run(K, wt)
            ops = h.timeline(0)
            for j, (s0, s1) in enumerate(ops):
                dur[wt][j % n].append(s1 - s0)
                if j:
                    gaps[wt][j % n].append(s0 - ops[j - 1][1])
            if wt:
                rep.append({k: r[k] for k in ("overrun_s", "used_s", "bubble_s", "op_growth", "steps_completed")})
    bub = h.profile()
    out = {"task": name, "stage": stage, "sms": sms, "ops": []}
    for j in range(n):
        b, w = statistics.fmean(dur[False][j]), statistics.fmean(dur[True][j])
        out["ops"].append({"j": j, "kind": "FP" if kinds[j] == 0 else "BP", "base_ms": b * 1e3, "growth": w / b - 1,
                           "gap_base_us": statistics.fmean(gaps[False][j]) * 1e6 if gaps[False][j] else None,
                           "gap_with_us": statistics.fmean(gaps[True][j]) * 1e6 if gaps[True][j] else None})
    out["runs"] = rep
    print(json.dumps(out), flush=True)
    h.close()


if __name__ == "__main__":
    main()
