"""Step duration / inter-step gap inside bubbles vs dispatch depth."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    for depth in [int(x) for x in os.environ.get("DEPTHS", "1,2,3,4").split(",")]:
        for ips in [int(x) for x in os.environ.get("IPS", "8").split(",")]:
            h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, max_inflight_steps=depth)
            h.submit("image", gpu.ImageTask(images_per_step=ips), profile_steps=16)
            h.run(3, True)
            h.reprofile("image")
            if os.environ.get("REBUB", "1") == "1":
                h.reprofile_bubbles()
            base = h.run(6, False)
            r = h.run(6, True)
            st = h.timeline(2)
            durs = [(b - a) * 1e6 for a, b in st]
            gaps = [(st[i + 1][0] - st[i][1]) * 1e6 for i in range(len(st) - 1) if st[i + 1][0] - st[i][1] < 50e-6]
            print(json.dumps({"depth": depth, "ips": ips, "step_us_med": statistics.median(durs),
                              "step_us_p10": statistics.quantiles(durs, n=10)[0],
                              "gap_us_med": statistics.median(gaps) if gaps else None,
                              "fill": r["used_s"] / r["bubble_s"], "overrun_frac": r["overrun_s"] / r["used_s"],
                              "dT": (r["makespan_s"] - base["makespan_s"]) / base["makespan_s"],
                              "px_per_bubble_s": r["work_units"] / base["bubble_s"],
                              "dispatch_us": r["dispatch_host_us"]}), flush=True)
            h.close()


if __name__ == "__main__":
    main()
