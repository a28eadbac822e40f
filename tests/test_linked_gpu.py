"""Peer-linked pipeline transport (transport=1):
real stage-to-stage activation/gradient messages through neighbour
mailboxes (copy engine + release flag), dependency waits on the stage's own
flags, and the epoch-end token down the chain.  On one B200 the stages
share the device: in one process (two harnesses, two threads) and across two
processes through CUDA IPC -- the same code path a multi-GPU run takes with
NVLink peer pointers."""
import os
import threading

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SMALL = dict(layers=2, hidden=2048, tokens=8192, profile_reps=2)   # ms-scale ops: bubbles the gate can use


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


def run_all(hs, epochs, with_tasks):
    out, errs = [None] * len(hs), []

    def go(i):
        try:
            out[i] = hs[i].run(epochs, with_tasks)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=go, args=(i,)) for i in range(len(hs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "linked pipeline deadlocked"
    if errs:
        raise errs[0]
    return out


def flags(g, ptr, m):
    from paper_2409_06941_b200.gpu import _dev_copy
    f = _dev_copy(ptr, 3 * 256, torch.int32).cpu()
    return [f[d * 256: d * 256 + m].tolist() for d in range(3)]


@pytest.mark.parametrize("p,m", [(2, 4), (3, 3)])
def test_linked_in_process(g, p, m):
    hs = [g.Harness(num_stages=p, num_micro_batches=m, stage=s, transport="linked", **SMALL)
          for s in range(p)]
    boxes = [h.mailbox() for h in hs]
    for s, h in enumerate(hs):
        h.link(boxes[s - 1] if s > 0 else None, boxes[s + 1] if s < p - 1 else None)
    reps = run_all(hs, 2, False)               # dry run, then the bubble profiler
    for h in hs:
        h.reprofile_bubbles()
    reps = run_all(hs, 3, False)
    total = 5                                  # global epochs so far = message sequence
    for s in range(p):
        fl = flags(g, boxes[s], m)
        assert fl[0] == ([total] * m if s > 0 else [0] * m)          # FP inputs from s-1
        assert fl[1] == ([total] * m if s < p - 1 else [0] * m)      # BP inputs from s+1
        assert fl[2][0] == (total if s > 0 else 0)                   # epoch-end token
    for s, (h, r) in enumerate(zip(hs, reps)):
        assert r["makespan_s"] > 0
        n_b = len(h.stage_bubbles())
        assert len(h.timeline(1)) == 3 * n_b   # every profiled bubble signalled each epoch
    # harvest: an image task on the last stage (its leading/trailing bubbles)
    task = g.ImageTask(sw=1920, sh=1080, dw=960, dh=540, batch=4, images_per_step=1)
    ok, _ = hs[-1].submit("img", task, profile_steps=4)
    assert ok
    reps = run_all(hs, 3, True)
    assert reps[-1]["steps_completed"] > 0 and reps[-1]["used_s"] > 0
    for h in hs:
        h.close()


def _ipc_stage(stage, q_out, q_in, res):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    h = gpu.Harness(num_stages=2, num_micro_batches=2, stage=stage, transport="linked",
                    layers=1, hidden=512, tokens=1024, profile_reps=1)
    q_out.put(gpu.ipc_handle(h.mailbox()))
    peer = gpu.ipc_open(q_in.get(timeout=60))
    h.link(peer if stage == 1 else None, peer if stage == 0 else None)
    r = h.run(2, False)
    res.put((stage, r["makespan_s"], flags(gpu, h.mailbox(), 2)))
    q_out.put("done")
    q_in.get(timeout=60)                  # keep the mailbox alive until the peer finished
    gpu.ipc_close(peer)
    h.close()


def test_linked_across_processes_ipc(g):
    ctx = mp.get_context("spawn")
    a, b, res = ctx.Queue(), ctx.Queue(), ctx.Queue()
    ps = [ctx.Process(target=_ipc_stage, args=(0, a, b, res)),
          ctx.Process(target=_ipc_stage, args=(1, b, a, res))]
    for pr in ps:
        pr.start()
    got = {}
    for _ in range(2):
        s, mk, fl = res.get(timeout=240)
        got[s] = (mk, fl)
    for pr in ps:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got[1][1][0] == [2, 2] and got[0][1][1] == [2, 2] and got[1][1][2][0] == 2


def _dist_stage(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2409_06941_b200 import distributed, gpu
    gpu.glib()
    out = distributed.linked_harvest(
        lambda: gpu.ImageTask(sw=1920, sh=1080, dw=960, dh=540, batch=2, images_per_step=1),
        dict(layers=1, hidden=512, tokens=1024, profile_reps=1), num_micro_batches=2,
        epochs=2, warmup=1)
    q.put((rank, out["with"]["steps_completed"], out["with"]["makespan_s"], out["base"]["makespan_s"]))
    dist.destroy_process_group()


def test_linked_harvest_two_ranks(g):
    """bench.py's multi-GPU linked path (distributed.linked_harvest) with two
    ranks sharing this GPU: IPC handle exchange over the process group,
    lockstep runs, side tasks on both stages."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dist_stage, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for pr in ps:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(mk > 0 and base > 0 for _, _, mk, base in got)
