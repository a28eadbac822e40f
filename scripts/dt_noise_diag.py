"""How noisy is the pipeline ΔT measurement?  Every stage of the bench
pipeline: R consecutive runs of K epochs WITHOUT side tasks; the pipeline ΔT
(pipeline_dt.critical_path_dt) between runs i and i+1 is pure measurement
noise (power / thermal drift, GEMM jitter).  Then the same with the image
task at a fixed SM budget, measured two ways: sequential (K base epochs, then
K harvested) and interleaved (base / harvested alternating in runs of 2).

Usage: python scripts/dt_noise_diag.py [K] [R] [side_sms]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_06941_b200 import api, gpu  # noqa: E402
from paper_2409_06941_b200 import pipeline_dt as P  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    sms = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    torch.cuda.set_device(0)
    a = api()
    p, m = 4, 4
    null = [dict() for _ in range(R)]
    seq_b, seq_w, il_b, il_w = {}, {}, {}, {}
    for s in range(p):
        h = gpu.Harness(num_stages=p, num_micro_batches=m, stage=s, layers=6, hidden=2048, tokens=8192,
                        ffn_mult=4, step_group=3, side_sms=sms)
        kinds = P.issue_kinds(a, s, p, m)
        for i in range(R):
            h.run(K, False)
            null[i][s] = P.op_means(h.timeline(0), kinds)
        ok, _ = h.submit("image", gpu.ImageTask(batch=64, images_per_step=16), profile_steps=16)
        assert ok
        h.run(3, True)
        h.reprofile("image")
        h.run(K, False)
        seq_b[s] = P.op_means(h.timeline(0), kinds)
        h.run(K, True)
        seq_w[s] = P.op_means(h.timeline(0), kinds)
        bb, ww = [], []
        for _ in range(K // 2):
            h.run(2, False)
            bb.append(P.op_means(h.timeline(0), kinds))
            h.run(2, True)
            ww.append(P.op_means(h.timeline(0), kinds))
        il_b[s] = tuple(statistics.fmean(x[i] for x in bb) for i in range(2))
        il_w[s] = tuple(statistics.fmean(x[i] for x in ww) for i in range(2))
        h.close()
    nulls = [P.critical_path_dt(a, p, m, K, null[i], null[i + 1])["dT"] for i in range(R - 1)]
    out = {"K": K, "side_sms": sms, "null_dT": nulls,
           "null_sd": statistics.pstdev(nulls) if len(nulls) > 1 else None,
           "sequential_dT": P.critical_path_dt(a, p, m, K, seq_b, seq_w)["dT"],
           "interleaved_dT": P.critical_path_dt(a, p, m, K, il_b, il_w)["dT"]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
