"""ORACLE / TEST INFRASTRUCTURE ONLY -- tick-stepped restatement of the
reference's missing event loop (`run_experiment`, engine.hpp:94-98; semantics
SPEC.md:466-517, 316-322, 158-190, 365-373, 502 and SURVEY.md Appendix B; the
ambiguities are fixed as written in DESIGN.md §6).

It walks *every* tick and, inside a tick, runs the phases P1..P6 by scanning
all state.  The product engine (csrc/host/engine.cpp) jumps between
interesting ticks with an event agenda; parity tests require identical traces.
Decision functions (gate, Alg. 1/2, transitions, enforce, memory, profiling,
jitter) come from the host API bound to any library -- tests pass the
reference's own compiled sources (oracle/_ref) so those decisions are the
reference's.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

# enum values (freeride.h)
FP, BP = 0, 1
SUBMITTED, CREATED, PAUSED, RUNNING, STOPPED = range(5)
CREATE, INIT, START, RUN, PAUSE, STOP = range(6)
ITERATIVE, IMPERATIVE = 0, 1
MB_NONE, MB_IGNORES_PAUSE, MB_LEAK = 0, 1, 2
A_INIT, A_STEP, A_KERNEL, A_CHECK = 0, 1, 2, 3
K_OOM, K_PAUSE, K_INIT = 0, 1, 2
D_REJECTED, D_COMPLETED, D_KOOM, D_KPAUSE, D_KINIT, D_ACTIVE = range(6)
ISSUE_INIT, ISSUE_START, ISSUE_PAUSE, ARM_INIT_GUARD = range(4)


@dataclass
class Opts:
    check_overhead: int = 1
    rpc_latency: int = 0
    step_jitter: float = 0.0
    profile_steps: int = 32
    gate_max: bool = False
    grace: int = 100
    headroom: float = 0.0


@dataclass
class TaskRt:
    spec: object
    prof: object = None
    state: int = SUBMITTED
    worker: int = -1
    steps: int = 0
    mem: float = 0.0
    last_paused: Optional[int] = None
    initializing: bool = False
    want_init: bool = False
    pause_pending: bool = False
    gate_closed: bool = False
    bubble_end: int = 0
    busy: int = 0                  # step/kernel ticks executed (leak accrual)
    rng: int = 0
    limit: float = 0.0
    disp: Optional[int] = None


def run(api, cfg, tasks, opts: Opts, seed: int, with_tasks: bool):
    """Returns a dict of record lists (the RunTrace, engine.hpp:75-92)."""
    from paper_2409_06941_b200.bubblesim import (Bubble, BubbleType, PipelineConfig, ProfileOptions,
                                                 SideTaskRuntime, SideTaskSpec, SideTaskState,
                                                 TaskView)
    p, m, E = cfg.num_stages, cfg.num_micro_batches, cfg.num_epochs
    dur = lambda s, k: cfg.fp_ticks(s) if k == FP else cfg.bp_ticks(s)  # noqa: E731

    # profiled bubbles (one undelayed epoch), keyed per stage by their neighbours
    one = PipelineConfig(p, m, list(cfg.fp_duration), list(cfg.bp_duration), 1,
                         cfg.gpu_memory_total, list(cfg.stage_memory), cfg.tick_seconds)
    prof_tr = api.build_schedule(one)
    prof_b = []   # (stage, prev (k,mb)|None, next (k,mb)|None, duration, btype)
    for lb in api.extract_bubbles_linked(prof_tr):
        pv = prof_tr.ops[lb.prev_op] if lb.prev_op is not None else None
        nx = prof_tr.ops[lb.next_op] if lb.next_op is not None else None
        prof_b.append((lb.bubble.stage, None if pv is None else (int(pv.kind), pv.micro_batch),
                       None if nx is None else (int(nx.kind), nx.micro_batch),
                       lb.bubble.duration, lb.bubble.btype))

    # op DAG over all epochs
    order = {s: api.stage_issue_order(s, p, m) for s in range(p)}
    ops = {}
    for e in range(E):
        for s in range(p):
            for i, (k, mb) in enumerate(order[s]):
                deps = []
                if i > 0:
                    deps.append((e, s, int(order[s][i - 1][0]), order[s][i - 1][1]))
                elif e > 0:
                    deps.append((e - 1, s, int(order[s][-1][0]), order[s][-1][1]))
                if k == FP and s > 0:
                    deps.append((e, s - 1, FP, mb))
                if k == BP:
                    if s < p - 1:
                        deps.append((e, s + 1, BP, mb))
                    deps.append((e, s, FP, mb))
                ops[(e, s, int(k), mb)] = {"deps": deps, "ready": None, "start": None, "end": None}

    out = {k: [] for k in ("ops", "bubbles", "submits", "assigns", "rejects", "rpcs", "transitions",
                           "activities", "kills", "dispositions")}
    workers = api.workers([cfg.available_memory(s) for s in range(p)])
    rts: Dict[str, TaskRt] = {}
    gpu = [None] * p            # None | ("op", key, end) | ("act", kind, task, start, end)
    rpcs_pending: List[Tuple[int, int, int, str, int]] = []   # (land, seq, kind, task, bubble_end)
    timers: List[Tuple[int, int, str, int, int]] = []         # (due, seq, kind, task, issued)
    held = [None] * p           # deferred BubbleStarted (Bubble) per worker
    open_b = {}                 # (e, stage, j) -> start tick
    seq = [0]

    def nseq():
        seq[0] += 1
        return seq[0]

    def lookup(tid):
        t = rts[tid]
        return TaskView(SideTaskState(t.state), t.initializing)

    def rt_api(t):
        r = SideTaskRuntime(SideTaskSpec(t.spec.id, memory_demand=t.spec.memory_demand),
                            state=SideTaskState(t.state), steps_completed=t.steps,
                            memory_allocated=t.mem, last_paused=t.last_paused)
        return r

    def transition(t, kind, now):
        r = rt_api(t)
        api.apply_transition(r, kind, now)
        t.state, t.mem, t.last_paused = int(r.state), r.memory_allocated, r.last_paused
        out["transitions"].append((now, t.spec.id, kind, t.worker))

    def clear_current(w, tid):
        info = workers.info(w)
        if info["current_task"] == tid:
            workers.set_current_task(w, None)

    def finish(t, now, disp):
        t.disp = disp
        clear_current(t.worker, t.spec.id)

    def kill(t, now, reason):
        w = t.worker
        g = gpu[w]
        if g is not None and g[0] == "act" and g[2] == t.spec.id:
            out["activities"].append((g[3], now, t.spec.id, w, g[1], True))
            gpu[w] = None
        if t.state != STOPPED:
            transition(t, STOP, now)
        t.initializing = t.want_init = t.pause_pending = False
        out["kills"].append((now, t.spec.id, w, reason))
        finish(t, now, {K_OOM: D_KOOM, K_PAUSE: D_KPAUSE, K_INIT: D_KINIT}[reason])

    def land(kind, tid, bend, now):
        t = rts[tid]
        if t.state == STOPPED:
            return
        if kind == INIT:
            if t.state == CREATED and not t.initializing:
                t.initializing = True
                t.want_init = True
        elif kind == START:
            if t.state == PAUSED:
                transition(t, START, now)
                t.bubble_end = bend
                t.gate_closed = False
        elif kind == PAUSE:
            if t.state == RUNNING and t.spec.misbehavior != MB_IGNORES_PAUSE:  # ignored: keeps running
                g = gpu[t.worker]
                busy = g is not None and g[0] == "act" and g[2] == tid
                if busy:
                    t.pause_pending = True
                else:
                    pause_now(t, now)

    def pause_now(t, now):
        transition(t, PAUSE, now)
        t.pause_pending = False
        w = t.worker
        if held[w] is not None:
            b = held[w]
            held[w] = None
            bubble_started(w, b, now)

    def issue(kind, tid, now, bend=0):
        t = rts[tid]
        out["rpcs"].append((now, tid, kind, t.worker))
        if opts.rpc_latency == 0:
            land(kind, tid, bend, now)
        else:
            rpcs_pending.append((now + opts.rpc_latency, nseq(), kind, tid, bend))

    def current_pause_pending(w):
        cur = workers.info(w)["current_task"]
        return cur is not None and rts[cur].pause_pending

    def bubble_started(w, b, now):
        if current_pause_pending(w):
            held[w] = b
            return
        for act in api.on_bubble_started(workers, w, b, lookup):
            if act.kind == ISSUE_INIT:
                issue(INIT, act.task_id, now)
            elif act.kind == ISSUE_START:
                issue(START, act.task_id, now, b.start + b.duration)

    def bubble_ended(w, now):
        if held[w] is not None:
            held[w] = None
        for act in api.on_bubble_ended(workers, w, now, lookup):
            if act.kind == ISSUE_PAUSE:
                issue(PAUSE, act.task_id, now)
                timers.append((now + opts.grace, nseq(), K_PAUSE, act.task_id, now))
            elif act.kind == ARM_INIT_GUARD:
                timers.append((now + opts.grace, nseq(), K_INIT, act.task_id, now))

    def est(t):
        return t.prof.max_per_step_duration if opts.gate_max else t.prof.est_per_step_duration

    def draw(t):
        box = [t.rng]
        d = api.jittered_step_ticks(t.spec.per_step_duration, opts.step_jitter, box)
        t.rng = box[0]
        return d

    def leak_alloc(t, busy):
        return t.spec.memory_demand + t.spec.leak_rate_gib_per_s * (busy * cfg.tick_seconds)

    specs = sorted(tasks, key=lambda sp: sp.submit_time) if with_tasks else []
    subq = list(specs)
    epoch_done = [False] * E
    done_ops = 0
    total_ops = len(ops)
    tick = 0
    makespan = 0
    while done_ops < total_ops:
        now = tick
        # ---- P1: completions
        for s in range(p):
            g = gpu[s]
            if g is not None and g[0] == "op" and g[2] == now:
                ops[g[1]]["end"] = now
                done_ops += 1
                gpu[s] = None
        if done_ops == total_ops:
            makespan = now
        for s in range(p):
            g = gpu[s]
            if g is not None and g[0] == "act" and g[4] == now:
                kind, tid = g[1], g[2]
                t = rts[tid]
                gpu[s] = None
                out["activities"].append((g[3], now, tid, s, kind, False))
                if kind == A_INIT:
                    t.initializing = False
                    transition(t, INIT, now)
                    if api.check_memory(t.mem, t.limit) == 1:
                        kill(t, now, K_OOM)
                elif kind in (A_STEP, A_KERNEL):
                    t.busy += now - g[3]
                    t.steps += 1
                    if t.spec.total_steps is not None and t.steps >= t.spec.total_steps:
                        transition(t, STOP, now)
                        t.pause_pending = False
                        finish(t, now, D_COMPLETED)
                    elif t.pause_pending:
                        pause_now(t, now)
                elif kind == A_CHECK:
                    if t.pause_pending:
                        pause_now(t, now)
                    else:
                        t.check_done = now
        last_tick = done_ops == total_ops
        # ---- P2: readiness and bubble signals
        ends, starts = [], []
        for key, o in ops.items():
            if o["ready"] is None and all(ops[d]["end"] is not None and ops[d]["end"] <= now for d in o["deps"]):
                o["ready"] = now
        for e in range(E):
            if not epoch_done[e] and all(o["end"] is not None for k, o in ops.items() if k[0] == e):
                epoch_done[e] = True
                epoch_done_at = now
                ops_e_end = now
                for j, (s, pv, nx, d, bt) in enumerate(prof_b):
                    if nx is None:
                        ends.append((e, s, j))
                    if pv is None and e + 1 < E:
                        starts.append((e + 1, s, j))
        if now == 0:
            for j, (s, pv, nx, d, bt) in enumerate(prof_b):
                if pv is None:
                    starts.append((0, s, j))
        for e in range(E):
            for j, (s, pv, nx, d, bt) in enumerate(prof_b):
                if pv is not None:
                    o = ops[(e, s) + pv]
                    if o["end"] == now:
                        starts.append((e, s, j))
                if nx is not None:
                    o = ops[(e, s) + nx]
                    if o["ready"] == now:
                        ends.append((e, s, j))
        both = set(starts) & set(ends)
        fire_end = []
        for key in ends:
            if key in both:
                continue
            if key in open_b:
                st = open_b.pop(key)
                e, s, j = key
                out["bubbles"].append((s, e, st, now - st, cfg.available_memory(s), int(prof_b[j][4])))
                fire_end.append(key)
        fire_start = []
        for key in starts:
            if key in both:
                continue
            open_b[key] = now
            fire_start.append(key)
        if last_tick:   # run ends: the last epoch's trailing bubbles closed above
            break
        # ---- P3: manager events: BubbleEnded < TaskFinished < TaskSubmitted < BubbleStarted
        if with_tasks:
            for key in sorted(fire_end, key=lambda k: (k[1], k[0], k[2])):
                bubble_ended(key[1], now)
            while subq and subq[0].submit_time == now:
                sp = subq.pop(0)
                prof = api.profile_task(sp, ProfileOptions(opts.profile_steps, opts.step_jitter, cfg.tick_seconds), seed)
                t = TaskRt(spec=sp, prof=prof)
                t.rng = api.stream_seed(seed, sp.id, "run")
                t.limit = sp.memory_limit if sp.memory_limit is not None else prof.est_memory + opts.headroom
                rts[sp.id] = t
                out["submits"].append((now, sp.id, -1))
                o = api.submit_task(prof, workers)
                if o.assigned:
                    t.worker = o.worker_id
                    out["assigns"].append((now, sp.id, o.worker_id))
                    transition(t, CREATE, now)
                else:
                    out["rejects"].append((now, sp.id, -1))
                    t.disp = D_REJECTED
            for key in sorted(fire_start, key=lambda k: (k[1], k[0], k[2])):
                e, s, j = key
                bubble_started(s, Bubble(s, e, now, prof_b[j][3], cfg.available_memory(s), BubbleType(prof_b[j][4])), now)
            # ---- P4: RPC landings in issue order
            due = sorted([r for r in rpcs_pending if r[0] == now], key=lambda r: r[1])
            rpcs_pending[:] = [r for r in rpcs_pending if r[0] != now]
            for _, _, kind, tid, bend in due:
                land(kind, tid, bend, now)
            # ---- P5: limit timers in arming order
            dt = sorted([x for x in timers if x[0] == now], key=lambda x: x[1])
            timers[:] = [x for x in timers if x[0] != now]
            for _, _, kind, tid, issued in dt:
                t = rts[tid]
                if t.state == STOPPED:
                    continue
                if kind == K_PAUSE:
                    if api.framework_enforce(t.last_paused, issued, now, opts.grace) == 1:
                        kill(t, now, K_PAUSE)
                elif t.initializing:
                    kill(t, now, K_INIT)
            # memory-leak OOM: first tick the allocation exceeds the limit
            for s in range(p):
                g = gpu[s]
                if g is not None and g[0] == "act" and g[1] in (A_STEP, A_KERNEL):
                    t = rts[g[2]]
                    if t.spec.misbehavior == MB_LEAK and now > g[3]:
                        if api.check_memory(leak_alloc(t, t.busy + now - g[3]), t.limit) == 1:
                            t.mem = leak_alloc(t, t.busy + now - g[3])
                            kill(t, now, K_OOM)
        # ---- P6: GPU scheduling
        for s in range(p):
            if gpu[s] is not None:
                continue
            ready = sorted([k for k, o in ops.items() if k[1] == s and o["ready"] is not None and o["start"] is None],
                           key=lambda k: (k[0], order[s].index((k[2], k[3]))))
            if ready:
                k = ready[0]
                ops[k]["start"] = now
                gpu[s] = ("op", k, now + dur(s, k[2]))
                continue
            if not with_tasks:
                continue
            cur = workers.info(s)["current_task"]
            if cur is None:
                continue
            t = rts[cur]
            if t.state == STOPPED:
                continue
            if t.want_init:
                t.want_init = False
                gpu[s] = ("act", A_INIT, cur, now, now + t.spec.init_duration)
                if t.spec.init_duration == 0:
                    gpu[s] = None
                    out["activities"].append((now, now, cur, s, A_INIT, False))
                    t.initializing = False
                    transition(t, INIT, now)
                    if api.check_memory(t.mem, t.limit) == 1:
                        kill(t, now, K_OOM)
                continue
            if t.state != RUNNING or t.pause_pending or t.gate_closed:
                continue
            if t.spec.interface_kind == IMPERATIVE:
                gpu[s] = ("act", A_KERNEL, cur, now, now + draw(t))
                continue
            # iterative: Check then gate then Step (check_overhead 0: gate now)
            if getattr(t, "check_done", None) != now and opts.check_overhead > 0:
                gpu[s] = ("act", A_CHECK, cur, now, now + opts.check_overhead)
                continue
            t.check_done = None
            d = api.iterative_run(rt_api(t), t.bubble_end, now, est(t), cfg.tick_seconds, 0)
            if not d.run:
                t.gate_closed = True
                continue
            gpu[s] = ("act", A_STEP, cur, now, now + draw(t))
        tick += 1

    # ---- end of run: clip in-flight activities, dispositions
    for s in range(p):
        g = gpu[s]
        if g is not None and g[0] == "act":
            out["activities"].append((g[3], makespan, g[2], s, g[1], True))
    for key in sorted(ops, key=lambda k: (ops[k]["start"], k[1], ops[k]["end"], k[3])):
        o = ops[key]
        out["ops"].append((key[1], key[2], key[3], key[0], o["start"], o["end"]))
    for sp in specs:
        t = rts.get(sp.id)
        if t is None:
            continue
        disp = t.disp if t.disp is not None else D_ACTIVE
        out["dispositions"].append((sp.id, disp, t.steps, t.worker if t.worker >= 0 else None))
    out["makespan"] = makespan
    return out

