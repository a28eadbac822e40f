"""Multi-GPU plumbing: one process per GPU (torch.distributed), one pipeline
stage and one side-task worker per GPU.

* Side tasks shard as replicas: no collective on their data path.
* Alg. 1 placement is the only cross-rank decision: every rank all-gathers
  the workers' (GPUMem, task count), rebuilds the same WorkerStates and runs
  the product's deterministic `select_worker` -- identical answer on every
  rank, no broadcast needed; only the chosen rank submits the task to its
  local harness.
* The pipeline's exchange (activations forward, gradients backward) follows
  `pipeline_p2p_plan`: at each op boundary the stage posts op g-1's send and
  op g's receive as one group (NCCL group / batch_isend_irecv), which keeps
  1F1B deadlock-free (tests/test_p2p_plan.py).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .bubblesim import BubbleSim, OpKind, TaskProfile


def gather_workers(gpu_mem: float, task_count: int, group=None) -> List[Tuple[float, int]]:
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (float(gpu_mem), int(task_count)), group=group)
    return out


def select_worker_global(api: BubbleSim, task_memory: float,
                         workers: Sequence[Tuple[float, int]]) -> Optional[int]:
    """Alg. 1 (manager.cpp:5-19 semantics) over gathered worker states."""
    ws = api.workers([m for m, _ in workers])
    for w, (_, count) in enumerate(workers):
        for i in range(count):
            ws.push_task(w, f"~{w}.{i}")
    return api.select_worker(task_memory, ws)


def submit_collective(api: BubbleSim, profile: TaskProfile, local_gpu_mem: float,
                      local_task_count: int, group=None) -> Optional[int]:
    """Collective Alg. 1: returns the chosen rank (same on all ranks) or None."""
    return select_worker_global(api, profile.est_memory,
                                gather_workers(local_gpu_mem, local_task_count, group))


def run_p2p_plan(api: BubbleSim, m: int, compute: Callable[[OpKind, int, Optional[torch.Tensor]], torch.Tensor],
                 make_buffer: Callable[[], torch.Tensor], group=None) -> List[Tuple[OpKind, int]]:
    """Executes this rank's stage of a 1F1B pipeline with the product's P2P
    plan: for each op g (issue order) post group g (send op g-1's output,
    receive op g's input) and wait, then run `compute(kind, mb, input)`.
    Returns the executed op order."""
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    plan = api.pipeline_p2p_plan(rank, p, m)
    order = api.stage_issue_order(rank, p, m)
    outputs = {}
    done = []
    for g in range(len(order) + 1):
        ops, recv_buf = [], None
        for (grp, is_send, peer, kind, mb) in plan:
            if grp != g:
                continue
            if is_send:
                ops.append(dist.P2POp(dist.isend, outputs.pop((kind, mb)), peer, group))
            else:
                recv_buf = make_buffer()
                ops.append(dist.P2POp(dist.irecv, recv_buf, peer, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if g < len(order):
            kind, mb = order[g]
            out = compute(kind, mb, recv_buf)
            sends_out = (kind == OpKind.FP and rank + 1 < p) or (kind == OpKind.BP and rank > 0)
            if sends_out:
                outputs[(kind, mb)] = out
            done.append((kind, mb))
    assert not outputs, "every produced tensor must have been sent"
    return done


def link_pipeline(h, group=None) -> List[int]:
    """Peer-linked pipeline (transport="linked"): rank s is stage s.  Every
    rank publishes its mailbox's CUDA IPC handle (all-gather over the process
    group), opens its neighbours' mailboxes (NVLink peer mappings across GPUs,
    plain device memory on a shared GPU) and links them.  Returns the opened
    peer pointers (close them with gpu.ipc_close after the last run)."""
    from . import gpu
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    handles = [None] * p
    dist.all_gather_object(handles, gpu.ipc_handle(h.mailbox()), group=group)
    prev = gpu.ipc_open(handles[rank - 1]) if rank > 0 else None
    nxt = gpu.ipc_open(handles[rank + 1]) if rank < p - 1 else None
    h.link(prev, nxt)
    return [x for x in (prev, nxt) if x]


def linked_harvest(make_task, stage_shape: dict, num_micro_batches: int, epochs: int,
                   warmup: int, group=None, task_name: str = "side", step_group: int = 1,
                   side_sms: int = 0, dt_budget: float = 0.0) -> dict:
    """One stage of a real p-stage pipeline (p = world size) with a side task
    harvesting its bubbles: link, dry-run + bubble profiler, submit (Alg. 1
    on this stage's worker), warm-up, ΔT baseline, harvest.  Every rank must
    call it (the epochs run in lockstep through the mailboxes)."""
    from . import gpu
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    h = gpu.Harness(num_stages=p, num_micro_batches=num_micro_batches, stage=rank,
                    transport="linked", step_group=step_group, side_sms=side_sms,
                    dt_budget=dt_budget, **stage_shape)
    opened = link_pipeline(h, group)
    dist.barrier(group)
    h.run(2, False)
    h.reprofile_bubbles()
    task = make_task()
    ok, _ = h.submit(task_name, task, profile_steps=16)
    oks = [None] * p
    dist.all_gather_object(oks, bool(ok), group=group)  # every stage gives up together
    if not all(oks):
        h.close()
        for x in opened:
            gpu.ipc_close(x)
        raise RuntimeError(f"stages {[i for i, o in enumerate(oks) if not o]}: side task rejected by Alg. 1")
    h.run(max(1, warmup), True)
    base = h.run(epochs, False)
    r = h.run(epochs, True)
    prof = h.profile()
    dist.barrier(group)
    h.close()
    for x in opened:
        gpu.ipc_close(x)
    return {"stage": rank, "base": base, "with": r, "profile": prof}
