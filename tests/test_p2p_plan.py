"""Multi-GPU host logic on CPU: the 1F1B point-to-point plan (deadlock-free
under strict rendezvous for every small (p, m); the naive order is not),
and world_size > 1 gloo runs of the exchange and of collective Alg. 1."""
import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_06941_b200.bubblesim import OpKind, TaskProfile


def groups_of(plan):
    gs = {}
    for (g, is_send, peer, kind, mb) in plan:
        gs.setdefault(g, []).append((is_send, peer, kind, mb))
    n = max(gs) + 1 if gs else 0
    return [gs.get(g, []) for g in range(n)]


def rendezvous_completes(stage_groups):
    """Strictest rendezvous (no buffering): a stage posts the ops of its
    current group; an op completes only when the peer has posted the matching
    op; a stage leaves its group when all of the group's ops completed
    (ops inside one group progress independently, as in an NCCL group)."""
    p = len(stage_groups)
    cur = [0] * p
    done = set()  # (stage, group, index)

    def posted(s):
        if cur[s] >= len(stage_groups[s]):
            return []
        g = cur[s]
        return [((s, g, j), op) for j, op in enumerate(stage_groups[s][g]) if (s, g, j) not in done]

    while not all(cur[s] >= len(stage_groups[s]) for s in range(p)):
        progressed = False
        for s in range(p):
            for key, (is_send, peer, kind, mb) in posted(s):
                for pkey, (p_send, p_peer, p_kind, p_mb) in posted(peer):
                    if p_send != is_send and p_peer == s and (p_kind, p_mb) == (kind, mb):
                        done.update((key, pkey))
                        progressed = True
                        break
        for s in range(p):
            while cur[s] < len(stage_groups[s]) and all(
                    (s, cur[s], j) in done for j in range(len(stage_groups[s][cur[s]]))):
                cur[s] += 1
                progressed = True
        if not progressed:
            return False
    return True


def naive_groups(api, s, p, m):
    """send after op i and recv before op i+1 as *separate* blocking calls."""
    order = api.stage_issue_order(s, p, m)
    gs = []
    for i, (k, mb) in enumerate(order):
        if k == OpKind.FP and s > 0:
            gs.append([(False, s - 1, OpKind.FP, mb)])
        if k == OpKind.BP and s < p - 1:
            gs.append([(False, s + 1, OpKind.BP, mb)])
        if k == OpKind.FP and s < p - 1:
            gs.append([(True, s + 1, OpKind.FP, mb)])
        if k == OpKind.BP and s > 0:
            gs.append([(True, s - 1, OpKind.BP, mb)])
    return gs


def test_plan_is_consistent_and_deadlock_free(product):
    for p in range(1, 9):
        for m in range(1, 13):
            plans = [product.pipeline_p2p_plan(s, p, m) for s in range(p)]
            sends = {(s, peer, k, mb) for s in range(p) for (g, snd, peer, k, mb) in plans[s] if snd}
            recvs = {(peer, s, k, mb) for s in range(p) for (g, snd, peer, k, mb) in plans[s] if not snd}
            assert sends == recvs                       # every send has exactly its receive
            assert len(sends) == 2 * m * (p - 1)        # an activation and a gradient per mb and link
            assert rendezvous_completes([groups_of(pl) for pl in plans]), (p, m)


def test_naive_order_deadlocks(product):
    stuck = [(p, m) for p in range(2, 6) for m in range(2, 6)
             if not rendezvous_completes([naive_groups(product, s, p, m) for s in range(p)])]
    assert stuck  # why the plan pairs a send with the next receive


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_06941_b200 import api
        from paper_2409_06941_b200.distributed import run_p2p_plan, submit_collective
        a = api()

        # 1F1B exchange with data: FP adds the stage to the activation, BP
        # carries the activation back; stage 0 checks every gradient.
        got = {}

        def compute(kind, mb, x):
            if kind == OpKind.FP:
                v = torch.full((4,), float(mb * 100)) if x is None else x.clone()
                return v + rank
            if x is None:   # last stage: gradient starts from its own FP output
                return torch.full((4,), float(mb * 100 + sum(range(world))))
            if rank == 0:
                got[mb] = x[0].item()
            return x.clone()

        order = run_p2p_plan(a, m, compute, lambda: torch.zeros(4))
        ok_order = order == list(a.stage_issue_order(rank, world, m))
        ok_data = rank != 0 or all(got[mb] == mb * 100 + sum(range(world)) for mb in range(1, m + 1))

        # collective Alg. 1: every rank computes the same placement
        mem = [10.0, 20.0, 30.0, 40.0][rank]
        count = [2, 0, 1, 0][rank]
        picks = [submit_collective(a, TaskProfile(f"t{i}", 0.1, 0.1, est, 32), mem, count)
                 for i, est in enumerate([5.0, 15.0, 25.0, 35.0, 45.0])]
        all_picks = [None] * world
        dist.all_gather_object(all_picks, picks)
        q.put((rank, ok_order, ok_data, picks, all(p == picks for p in all_picks)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [1, 4, 6])
def test_gloo_world4_pipeline_exchange_and_collective_alg1(m):
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok_order, ok_data, picks, same in res:
        assert ok_order and ok_data and same
        # workers (mem, count): (10,2) (20,0) (30,1) (40,0): Alg. 1 (strict mem,
        # fewest tasks, lowest id); 25 GiB fits ranks 2 (1 task) and 3 (0 tasks)
        assert picks == [1, 1, 3, 3, None]
