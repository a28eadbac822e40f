"""Operating points of bubble harvesting on a power-capped B200: side-task
throughput per bubble-second vs pipeline (critical-path) ΔT.

Every stage of the bench pipeline is replayed in turn; per stage and harvest
fraction f (the gate sees the first f of every bubble): a run without and a
run with the side task.  The per-stage mean FP / BP durations of both runs go
through build_schedule (pipeline_dt.critical_path_dt) -> the linked
pipeline's ΔT; throughput = units / bubble-seconds over all stages.

Usage: python scripts/harvest_sweep.py TASK FRACTIONS [epochs] [stages] [SMS]
  TASK in image16 | image8 | image4 | e2e128 | e2e8 | pagerank | sgd | spin ; FRACTIONS e.g. 1,0.5,0.25;
  SMS: side-task SM budgets to try (fr_harness_set_side_sms), e.g. 0,74,37 (0 = all);
       env FR_DT_BUDGET=0.007 turns on the harness's ΔT controller (SMS = its start)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_06941_b200 import api, gpu  # noqa: E402
from paper_2409_06941_b200 import pipeline_dt as P  # noqa: E402


def make(name):
    if name.startswith("e2e"):   # e2eR: the host-I/O image task (pinned host frames, R-slot device ring)
        return gpu.ImageTask(batch=64, images_per_step=1, host_io=True, host_ring=int(name[3:] or 128))
    if name.startswith("imp"):   # impN: the imperative (device-preempted) image task over a 64-frame batch
        return gpu.ImageTask(batch=64, images_per_step=int(name[3:] or 16), imperative=True)
    if name.startswith("image"):
        return gpu.ImageTask(batch=64, images_per_step=int(name[5:] or 16))
    if name.startswith("pagerank"):   # pagerankN: N iterations per step (default 2)
        return gpu.PageRankTask(scale=20, edge_factor=16, seed=1, iters_per_step=int(name[8:] or 2))
    if name == "sgd":
        return gpu.SgdTask(edges_per_step=1 << 22)
    if name == "spin":
        return gpu.SyntheticTask(step_ns=100_000, memory_demand_gib=0.1)
    raise ValueError(name)


def main():
    name = sys.argv[1]
    fracs = [float(x) for x in sys.argv[2].split(",")]
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    stages = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 and sys.argv[4] else [0, 1, 2, 3]
    smss = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0]
    pts = [(f, n) for n in smss for f in fracs]
    p, m = 4, 4
    torch.cuda.set_device(0)
    a = api()
    res = {pt: {"base": {}, "with": {}, "units": 0.0, "bubble_s": 0.0, "stage_dT": {}, "fill": {}} for pt in pts}
    for s in stages:
        h = gpu.Harness(num_stages=p, num_micro_batches=m, stage=s, layers=6, hidden=2048, tokens=8192,
                        ffn_mult=4, step_group=3, dt_budget=float(os.environ.get("FR_DT_BUDGET", "0")))
        kinds = P.issue_kinds(a, s, p, m)
        ok, _ = h.submit(name, make(name), profile_steps=16)
        assert ok
        for f, n in pts:
            h.set_side_sms(n)
            h.set_harvest_fraction(1.0)
            h.run(2, False)          # the controller's op reference
            h.run(2, True)           # warm at this budget, then re-profile the step
            try:
                h.reprofile(name)
            except Exception:  # noqa: BLE001
                pass
            h.set_harvest_fraction(f)
            base = h.run(K, False)
            ob = h.timeline(0)
            r = h.run(K, True)
            ow = h.timeline(0)
            R = res[(f, n)]
            R["base"][s] = P.op_means(ob, kinds)
            R["with"][s] = P.op_means(ow, kinds)
            R["units"] += r["work_units"]
            R["bubble_s"] += base["bubble_s"]
            R["stage_dT"][s] = (r["makespan_s"] - base["makespan_s"]) / base["makespan_s"]
            R["fill"][s] = r["used_s"] / r["bubble_s"]
            R.setdefault("sms_mean", {})[s] = r["side_sms_mean"]
            R.setdefault("growth_rep", {})[s] = r["op_growth"]
        h.close()
    out = []
    for f, n in pts:
        R = res[(f, n)]
        row = {"task": name, "fraction": f, "side_sms": n,
               "units_per_bubble_s": R["units"] / R["bubble_s"],
               "stage_dT_max": max(R["stage_dT"].values()), "fill": R["fill"],
               "sms_mean": R.get("sms_mean"), "op_growth_reported": R.get("growth_rep"),
               "op_growth": {s: (R["with"][s][0] / R["base"][s][0] - 1, R["with"][s][1] / R["base"][s][1] - 1)
                             for s in R["base"]}}
        if len(R["base"]) == p:
            row["critical_path_dT"] = P.critical_path_dt(a, p, m, K, R["base"], R["with"])["dT"]
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
