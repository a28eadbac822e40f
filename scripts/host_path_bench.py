"""Host hot path: build_schedule + extract_bubbles_linked
on the product library vs the reference's own compiled sources
(oracle/_ref, the CPU baseline), through the same C-ABI with preallocated
buffers so only the C++ work is timed.  Prints one JSON line."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_06941_b200 import _abi as A  # noqa: E402
from paper_2409_06941_b200 import api  # noqa: E402
from paper_2409_06941_b200.bubblesim import BubbleSim, PipelineConfig, _Cfg  # noqa: E402


def time_host(api_, cfg, reps=15):
    c = _Cfg(cfg)
    cap = 2 * cfg.num_stages * cfg.num_micro_batches * cfg.num_epochs
    ops = (A.OpEventC * cap)()
    spans = (A.tick * (2 * cfg.num_epochs))()
    bcap = cfg.num_epochs * cfg.num_stages * (2 * cfg.num_micro_batches + 1)
    out = (A.BubbleC * bcap)()
    n, nb = C.c_int64(), C.c_int64()
    lib = api_.lib
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        api_._check(lib.fr_build_schedule(C.byref(c.c), ops, cap, C.byref(n), spans))
        t1 = time.perf_counter()
        api_._check(lib.fr_extract_bubbles(C.byref(c.c), ops, n.value, spans, out, bcap, C.byref(nb)))
        t2 = time.perf_counter()
        best.append((t1 - t0, t2 - t1))
    best.sort(key=lambda x: x[0] + x[1])
    return best[len(best) // 2], n.value, nb.value


def main():
    ours = api()
    ref_path = os.path.join(ROOT, "oracle", "_ref", "libbubblesim_ref.so")
    ref = BubbleSim(C.CDLL(ref_path)) if os.path.exists(ref_path) else None
    res = {}
    for name, (p, m, e) in {"C1_p4_m4_128ep": (4, 4, 128), "C5_p8_m8_128ep": (8, 8, 128)}.items():
        cfg = PipelineConfig(p, m, [220], [347], e, 48.0, [1.0] * p, 1e-3)
        (b, x), n_ops, n_b = time_host(ours, cfg)
        row = {"ops": n_ops, "bubbles": n_b, "ours_build_ms": b * 1e3, "ours_extract_ms": x * 1e3}
        if ref:
            (rb, rx), _, _ = time_host(ref, cfg)
            row.update(ref_build_ms=rb * 1e3, ref_extract_ms=rx * 1e3, speedup=(rb + rx) / (b + x))
        res[name] = row
    print(json.dumps(res))


if __name__ == "__main__":
    main()
