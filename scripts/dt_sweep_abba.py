"""Pipeline ΔT vs a FIXED side-task budget, measured the way bench.py measures
the headline (every stage replayed, ABBA-ordered (baseline, harvest) pairs,
per-pair critical-path ΔT -> mean and standard error).  Also prints the
mean op growth the harness's own controller sensor saw (run report).
Usage: python scripts/dt_sweep_abba.py TASK SMS_LIST [pairs] [K]
   e.g. python scripts/dt_sweep_abba.py image16 4,6,8,12 6 8
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
    name = sys.argv[1]
    smss = [int(x) for x in sys.argv[2].split(",")]
    pairs = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    K = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    budget = float(os.environ.get("FR_DT_BUDGET", "0"))
    p, m = 4, 4
    torch.cuda.set_device(0)
    a = api()
    res = {n: {"b": [dict() for _ in range(pairs)], "w": [dict() for _ in range(pairs)], "units": 0.0,
               "bubble_s": 0.0, "sensor": [], "sms": []} for n in smss}
    for s in range(p):
        h = gpu.Harness(num_stages=p, num_micro_batches=m, stage=s, layers=6, hidden=2048, tokens=8192,
                        ffn_mult=4, step_group=3, dt_budget=budget)
        kinds = P.issue_kinds(a, s, p, m)
        ok, _ = h.submit(name, make(name), profile_steps=16)
        assert ok
        frac = float(os.environ.get("FR_HARVEST_FRACTION", "1"))   # the gate sees the first f of each bubble
        for n in smss:
            h.set_side_sms(n)
            h.set_harvest_fraction(frac)
            h.run(2, False)
            h.run(2, True)
            try:
                h.reprofile(name)
            except Exception:  # noqa: BLE001
                pass
            R = res[n]
            for i in range(pairs):
                for wt in ((False, True) if i % 2 == 0 else (True, False)):
                    r = h.run(K, wt)
                    om = P.op_means(h.timeline(0), kinds)
                    if wt:
                        R["w"][i][s] = om
                        R["units"] += r["work_units"]
                        R["sensor"].append(r["op_growth"])
                        R["sms"].append(r["side_sms_mean"])
                    else:
                        R["b"][i][s] = om
                        R["bubble_s"] += r["bubble_s"]
        h.close()
    for n in smss:
        R = res[n]
        d = [P.critical_path_dt(a, p, m, K, R["b"][i], R["w"][i])["dT"] for i in range(pairs)]
        print(json.dumps({"task": name, "side_sms": n, "budget": budget,
                          "harvest_fraction": float(os.environ.get("FR_HARVEST_FRACTION", "1")), "units_per_bubble_s": R["units"] / R["bubble_s"],
                          "dT_mean": statistics.fmean(d), "dT_se": statistics.stdev(d) / len(d) ** 0.5,
                          "dT_pairs": d, "sensor_growth_mean": statistics.fmean(R["sensor"]),
                          "sms_mean": statistics.fmean(R["sms"])}), flush=True)


if __name__ == "__main__":
    main()
