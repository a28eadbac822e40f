"""Why do a stage's GEMM ops run slower when its bubbles are harvested?

Stage `s` of the bench pipeline, one harness per side task; per task: median
FP / BP op duration with vs without the task, stage ΔT, fill, and NVML power /
SM clock sampled separately during the base and the harvested run.  Tasks:
the image step (16 and 4 frames), a synthetic spin task (every SM held, no
memory traffic, ~no power), PageRank and Graph-SGD.

Usage: python scripts/power_dt_diag.py [stage] [epochs] [tasks,...]
"""
import os
import statistics
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


class Sampler:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.p, self.c = [], []

    def __enter__(self):
        self.stop = threading.Event()
        self.p, self.c = [], []

        def loop():
            while not self.stop.is_set():
                try:
                    self.p.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                    self.c.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                except Exception:  # noqa: BLE001
                    pass
                self.stop.wait(0.02)
        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()

    def summary(self):
        return (statistics.fmean(self.p) if self.p else 0.0, statistics.median(self.c) if self.c else 0)


def op_durs(h, nops=8):
    ops = h.timeline(0)
    fp = [b - a for i, (a, b) in enumerate(ops) if (i % nops) < 4]
    bp = [b - a for i, (a, b) in enumerate(ops) if (i % nops) >= 4]
    return statistics.median(fp), statistics.median(bp)


def make(name):
    if name == "image16":
        return gpu.ImageTask(batch=64, images_per_step=16)
    if name == "image4":
        return gpu.ImageTask(batch=64, images_per_step=4)
    if name == "spin":
        return gpu.SyntheticTask(step_ns=200_000, memory_demand_gib=0.1)
    if name == "pagerank":
        return gpu.PageRankTask(scale=20, edge_factor=16, seed=1, iters_per_step=2)
    if name == "sgd":
        return gpu.SgdTask(edges_per_step=1 << 22)
    raise ValueError(name)


def main():
    stage = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["spin", "image16", "image4", "pagerank", "sgd"]
    torch.cuda.set_device(0)
    smp = Sampler()
    for n in names:
        h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=6, hidden=2048, tokens=8192,
                        ffn_mult=4, step_group=3)
        ok, _ = h.submit(n, make(n), profile_steps=16)
        assert ok
        h.run(3, True)
        try:
            h.reprofile(n)
        except Exception:  # noqa: BLE001
            pass
        with smp:
            base = h.run(K, False)
        pb, cb = smp.summary()
        fb, bb = op_durs(h)
        with smp:
            r = h.run(K, True)
        pw, cw = smp.summary()
        fw, bw = op_durs(h)
        dT = (r["makespan_s"] - base["makespan_s"]) / base["makespan_s"]
        print(f"{n:9s} stage {stage}: dT {dT*100:+.3f} %  fill {r['used_s']/r['bubble_s']:.3f}  "
              f"FP {fb*1e3:.3f}->{fw*1e3:.3f} ms ({(fw/fb-1)*100:+.1f} %)  BP {bb*1e3:.3f}->{bw*1e3:.3f} ms "
              f"({(bw/bb-1)*100:+.1f} %)  power {pb:.0f}->{pw:.0f} W  sm clock {cb}->{cw} MHz", flush=True)
        h.close()


if __name__ == "__main__":
    main()
