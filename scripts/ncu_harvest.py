"""ncu inside a harvest: one stage of the bench pipeline
with a side task; after the warm-up, the timed 2-epoch run is bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off -k regex:<kernel>`
captures the side-task kernel (and the stand-in GEMMs) launched by the
harness in its bubbles -- not a standalone microbenchmark.  Run with
FR_HARNESS_NO_PROFILE_GATE=1 (the standalone step profile's host gate would
deadlock under ncu's serialised launches).

Usage: FR_HARNESS_NO_PROFILE_GATE=1 ncu ... python scripts/ncu_harvest.py image|pagerank|sgd [side_sms]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "image"
sms = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if name == "image":
    task = gpu.ImageTask(batch=64, images_per_step=16)
elif name == "pagerank":
    task = gpu.PageRankTask(scale=20, edge_factor=16, seed=1, iters_per_step=2)
else:
    task = gpu.SgdTask(edges_per_step=1 << 22)
h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192, step_group=3,
                profile_epochs=1, side_sms=sms)
h.submit(name, task, profile_steps=4)
h.run(2, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = h.run(2, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: r[k] for k in ("steps_completed", "used_s", "bubble_s", "makespan_s")})
h.close()
