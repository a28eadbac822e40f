"""What SM clock does the GPU run at inside pipeline bubbles?  A Python side
task launches a clock probe before each image step; compare with idle."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


class ProbeImage(gpu.PythonTask):
    work_units_per_step = 8 * 1920 * 1080

    def __init__(self):
        super().__init__()
        self.memory_gib = 2.0
        self.k = 0

    def init(self, stream):
        s = torch.cuda.ExternalStream(stream)
        with torch.cuda.stream(s):
            self.plan = gpu.ImagePlan(3840, 2160, 1920, 1080)
            self.src = gpu.img_generate(64, 3840, 2160, stream=stream)
            self.dst = torch.empty((64, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
            self.wmp = self.plan.prepare(gpu.img_generate_watermark(1920, 1080, stream=stream), stream=stream)
            self.probe = torch.zeros((1 << 16, 2), dtype=torch.int64, device="cuda")

    def run_next_step(self, stream):
        i = (self.k % 8) * 8
        gpu.check(gpu.glib().fr_clock_probe(self.probe[self.k % (1 << 16)].data_ptr(), 20000, stream))
        self.plan.run_prepared(self.src[i:i + 8], self.dst[i:i + 8], self.wmp, stream=stream)
        self.k += 1


def main():
    # idle clock
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    gpu.check(gpu.glib().fr_clock_probe(out.data_ptr(), 200000, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    c, ns = out.tolist()
    print(json.dumps({"idle_mhz": c / ns * 1e3}))
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=int(os.environ.get("STAGE", "1")))
    t = ProbeImage()
    h.submit("probe", t, profile_steps=8)
    h.run(2, True)
    t.k = 0
    t.probe.zero_()
    r = h.run(4, True)
    n = min(t.k, 1 << 16)
    pr = t.probe[:n].cpu().tolist()
    mhz = [c / ns * 1e3 for c, ns in pr if ns > 0]
    steps = h.timeline(2)
    durs = [(b - a) * 1e6 for a, b in steps]
    print(json.dumps({"in_bubble_mhz_median": statistics.median(mhz), "min": min(mhz), "max": max(mhz),
                      "deciles": [round(x) for x in statistics.quantiles(mhz, n=10)],
                      "step_us_median": statistics.median(durs), "fill": r["used_s"] / r["bubble_s"]}))
    # and a back-to-back idle-GPU run of the same steps for comparison
    s = gpu.low_priority_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(64)]
    for a, b in ev:
        a.record(s)
        t.run_next_step(s.cuda_stream)
        b.record(s)
    s.synchronize()
    print(json.dumps({"idle_step_us_median": statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)}))


if __name__ == "__main__":
    main()
