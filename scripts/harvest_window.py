"""One image harvest run (bench stage shape) bracketed by cudaProfilerStart/
Stop, so `ncu --profile-from-start off` lists exactly the launches of the
timed region: the stand-in GEMMs, gap kernels and K5 steps of 2 epochs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402

# the bench's configuration: 16 frames per step, step groups of 3
h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192, step_group=3)
h.submit("image", gpu.ImageTask(batch=64, images_per_step=16), profile_steps=16)
h.run(3, True)
h.reprofile("image")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = h.run(2, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: r[k] for k in ("steps_completed", "used_s", "bubble_s", "makespan_s")})
h.close()
