"""Does a resident 1-warp spinning kernel (like the stage's dependency wait)
slow a side-task step?  SGD / image steps alone vs with torch.cuda._sleep
spinning on a high-priority stream."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def timed(fn, s, n=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    s.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def main():
    s = gpu.low_priority_stream()
    hi = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
    p = gpu.SgdProblem()
    sgd = lambda: p.step(0, 1 << 21, stream=s)
    timed(sgd, s, 3)
    alone = timed(sgd, s)
    with torch.cuda.stream(hi):
        torch.cuda._sleep(400_000_000)  # ~0.2 s of one spinning thread
    busy = timed(sgd, s)
    torch.cuda.synchronize()
    print(json.dumps({"sgd_alone_us": alone, "sgd_with_spinner_us": busy}))


if __name__ == "__main__":
    main()
