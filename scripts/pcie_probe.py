"""PCIe H2D/D2H bandwidth from pinned memory: one copy vs the same bytes split
over two streams, and H2D + D2H concurrently (full duplex)."""
import json
import torch

n = 24883200 * 4
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 4, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def one():
    d.copy_(h, non_blocking=True)


def two():
    with torch.cuda.stream(s1):
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[n // 2:].copy_(h[n // 2:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


print(json.dumps({"h2d_one_GBps": bw(one, n), "h2d_two_streams_GBps": bw(two, n),
                  "h2d_with_concurrent_d2h_GBps": bw(duplex, n)}))
