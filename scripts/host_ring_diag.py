"""Drive the host_io image task's hooks directly (no harness) and check every
output frame against the oracle after each Init..Stop lifetime."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import sidetasks_oracle  # noqa: E402
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    ring = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    orc = sidetasks_oracle.load()
    src = orc.img_generate(6, 3840, 2160, seed=41)
    wm = orc.img_generate_watermark(1920, 1080, seed=41 ^ 0x77)
    want = orc.img_resize_watermark(src, wm, 1920, 1080)
    t = gpu.ImageTask(batch=6, images_per_step=2, host_io=True, seed=41, host_ring=ring)
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    assert t.vt.create(t.user) == 0
    for life, nsteps in enumerate([8, 3, 5, 3]):
        assert t.vt.init(t.user, sp) == 0
        for _ in range(nsteps):
            assert t.vt.run_next_step(t.user, sp) == 0
        s.synchronize()
        out = t.host_outputs()
        bad = [i for i in range(6) if not np.array_equal(out[i], want[i])]
        print("life", life, "steps", nsteps, "bad frames", bad, flush=True)
        assert t.vt.stop(t.user) == 0
        s.synchronize()


if __name__ == "__main__":
    main()
