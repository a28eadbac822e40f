"""Host-side mirror of the reference's `bubblesim` C++ API over the C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/bubblesim/*.hpp (file:line cited per function);
every call goes through include/freeride.h.  `BubbleSim(lib)` binds any
library that exports the header -- the product by default, the reference's
own sources (oracle/_ref) in parity tests -- so both are driven by identical
Python code.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

from . import _abi as A
from ._abi import (CapacityError, FreeRideError, IllegalTransition,  # noqa: F401
                   InvariantError, SchemaError, ValidationError)


class OpKind(enum.IntEnum):           # pipeline.hpp:38
    FP = 0
    BP = 1


class BubbleType(enum.IntEnum):       # pipeline.hpp:55
    A = 0
    B = 1
    C = 2


class SideTaskState(enum.IntEnum):    # task.hpp:12
    Submitted = 0
    Created = 1
    Paused = 2
    Running = 3
    Stopped = 4


class TransitionKind(enum.IntEnum):   # task.hpp:15-22
    CreateSideTask = 0
    InitSideTask = 1
    StartSideTask = 2
    RunNextStep = 3
    PauseSideTask = 4
    StopSideTask = 5


class TaskInterface(enum.IntEnum):    # task.hpp:24
    Iterative = 0
    Imperative = 1


class MisbehaviorKind(enum.IntEnum):  # task.hpp:26
    None_ = 0
    IgnoresPause = 1
    MemoryLeak = 2


class Disposition(enum.IntEnum):      # task.hpp:97-104
    Rejected = 0
    Completed = 1
    KilledOom = 2
    KilledPauseTimeout = 3
    KilledInitTimeout = 4
    Active = 5


class Gate(enum.IntEnum):             # limits.hpp:22
    Run = 0
    Yield = 1


class MemCheck(enum.IntEnum):         # limits.hpp:17
    Ok = 0
    OomKill = 1


class Enforce(enum.IntEnum):          # limits.hpp:28
    Ok = 0
    Kill = 1


class ManagerActionKind(enum.IntEnum):  # manager.hpp:54-59
    IssueInit = 0
    IssueStart = 1
    IssuePause = 2
    ArmInitGuard = 3


class ActivityKind(enum.IntEnum):     # engine.hpp:15
    Init = 0
    Step = 1
    Kernel = 2
    Check = 3


class KillReason(enum.IntEnum):       # engine.hpp:16
    Oom = 0
    PauseTimeout = 1
    InitTimeout = 2


@dataclass
class PipelineConfig:                 # pipeline.hpp:13-36
    num_stages: int = 1
    num_micro_batches: int = 1
    fp_duration: List[int] = field(default_factory=list)
    bp_duration: List[int] = field(default_factory=list)
    num_epochs: int = 1
    gpu_memory_total: float = 0.0
    stage_memory: List[float] = field(default_factory=list)
    tick_seconds: float = 0.001

    def fp_ticks(self, stage: int) -> int:
        return self.fp_duration[0] if len(self.fp_duration) == 1 else self.fp_duration[stage]

    def bp_ticks(self, stage: int) -> int:
        return self.bp_duration[0] if len(self.bp_duration) == 1 else self.bp_duration[stage]

    def available_memory(self, stage: int) -> float:
        return self.gpu_memory_total - self.stage_memory[stage]


@dataclass(frozen=True)
class OpEvent:                        # pipeline.hpp:40-47
    stage: int
    kind: OpKind
    micro_batch: int
    epoch: int
    start: int
    end: int


@dataclass
class ScheduleTrace:                  # pipeline.hpp:49-53
    ops: List[OpEvent]
    epoch_spans: List[Tuple[int, int]]
    config: PipelineConfig


@dataclass(frozen=True)
class Bubble:                         # pipeline.hpp:58-67
    stage: int
    epoch: int
    start: int
    duration: int
    available_memory: float
    btype: BubbleType

    def end(self) -> int:
        return self.start + self.duration


@dataclass(frozen=True)
class LinkedBubble:                   # pipeline.hpp:102-106
    bubble: Bubble
    prev_op: Optional[int]
    next_op: Optional[int]


@dataclass
class SideTaskSpec:                   # task.hpp:33-50
    id: str
    interface_kind: TaskInterface = TaskInterface.Iterative
    per_step_duration: int = 1
    total_steps: Optional[int] = None
    init_duration: int = 0
    memory_demand: float = 0.0
    misbehavior: MisbehaviorKind = MisbehaviorKind.None_
    leak_rate_gib_per_s: float = 0.0
    submit_time: int = 0
    memory_limit: Optional[float] = None
    reference_throughput: Optional[float] = None


@dataclass
class SideTaskRuntime:                # task.hpp:52-60
    spec: SideTaskSpec
    state: SideTaskState = SideTaskState.Submitted
    steps_completed: int = 0
    memory_allocated: float = 0.0
    last_paused: Optional[int] = None
    assigned_worker: Optional[int] = None
    busy_until: Optional[int] = None


@dataclass(frozen=True)
class IterativeDecision:              # task.hpp:79-82
    run: bool
    step_end: int


@dataclass
class LimitConfig:                    # limits.hpp:9-15
    grace_period: int = 100
    memory_headroom: float = 0.0
    reclamation_delay: int = 0


@dataclass
class ProfileOptions:                 # profiler.hpp:33-37
    n_steps: int = 32
    step_jitter: float = 0.0
    tick_seconds: float = 0.001


@dataclass
class TaskProfile:                    # profiler.hpp:15-21
    task_id: str
    est_per_step_duration: Optional[float] = None
    max_per_step_duration: Optional[float] = None
    est_memory: float = 0.0
    profiled_steps: int = 0


@dataclass
class StageBubbleProfile:             # profiler.hpp:23-26
    durations: List[int]
    available_memory: float


@dataclass
class BubbleProfile:                  # profiler.hpp:28-31
    stages: List[StageBubbleProfile]
    rate: float


@dataclass(frozen=True)
class TaskView:                       # manager.hpp:47-50
    state: SideTaskState
    initializing: bool = False


@dataclass(frozen=True)
class ManagerAction:                  # manager.hpp:61-64
    kind: ManagerActionKind
    task_id: str


@dataclass
class SubmitOutcome:                  # manager.hpp:36-39
    assigned: bool = False
    worker_id: int = -1


@dataclass
class PriceConfig:                    # metrics.hpp:16-21
    price_server_1: float = 3.96
    price_server_2: float = 0.18


@dataclass
class TaskWork:                       # metrics.hpp:27-31
    id: str
    work: float = 0.0
    throughput_per_hour: Optional[float] = None


@dataclass(frozen=True)
class CostBreakdown:                  # metrics.hpp:33-38
    c_no_side: float
    c_extra: float
    c_side_tasks: float
    s: float


@dataclass(frozen=True)
class StageBreakdown:                 # metrics.hpp:51-62
    stage: int
    used_by_side_tasks: int
    runtime_overhead: int
    idle_oom: int
    idle_insufficient_time: int

    def total(self) -> int:
        return (self.used_by_side_tasks + self.runtime_overhead + self.idle_oom
                + self.idle_insufficient_time)


# RunTrace records (engine.hpp:18-65), the slice bubble_breakdown reads.
@dataclass(frozen=True)
class TransitionRecord:
    t: int
    task: str
    kind: TransitionKind
    worker: int = -1


@dataclass(frozen=True)
class ActivityRecord:
    start: int
    end: int
    task: str
    worker: int
    kind: ActivityKind
    clipped: bool = False


@dataclass(frozen=True)
class AssignRecord:
    t: int
    task: str
    worker: int = -1


def _id(s: str) -> bytes:
    b = s.encode()
    if len(b) >= A.TASK_ID_MAX:
        raise ValidationError("id", f"task id longer than {A.TASK_ID_MAX - 1} bytes")
    return b


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


class _Cfg:
    """Keeps the C arrays a fr_pipeline_config points into alive."""

    def __init__(self, cfg: PipelineConfig):
        self.fp = _arr(A.tick, cfg.fp_duration)
        self.bp = _arr(A.tick, cfg.bp_duration)
        self.mem = _arr(C.c_double, cfg.stage_memory)
        self.c = A.PipelineConfigC(
            num_stages=cfg.num_stages, num_micro_batches=cfg.num_micro_batches,
            num_epochs=cfg.num_epochs, n_fp=len(cfg.fp_duration), fp_duration=self.fp,
            n_bp=len(cfg.bp_duration), n_stage_memory=len(cfg.stage_memory),
            bp_duration=self.bp, stage_memory=self.mem,
            gpu_memory_total=cfg.gpu_memory_total, tick_seconds=cfg.tick_seconds)
        if not cfg.fp_duration:
            self.c.fp_duration = C.POINTER(A.tick)()
        if not cfg.bp_duration:
            self.c.bp_duration = C.POINTER(A.tick)()
        if not cfg.stage_memory:
            self.c.stage_memory = C.POINTER(C.c_double)()


def _spec_c(spec: SideTaskSpec) -> A.SideTaskSpecC:
    return A.SideTaskSpecC(
        id=_id(spec.id), interface_kind=int(spec.interface_kind),
        misbehavior=int(spec.misbehavior), has_total_steps=spec.total_steps is not None,
        has_memory_limit=spec.memory_limit is not None,
        has_reference_throughput=spec.reference_throughput is not None,
        per_step_duration=spec.per_step_duration, total_steps=spec.total_steps or 0,
        init_duration=spec.init_duration, memory_demand=spec.memory_demand,
        leak_rate_gib_per_s=spec.leak_rate_gib_per_s, submit_time=spec.submit_time,
        memory_limit=spec.memory_limit or 0.0,
        reference_throughput=spec.reference_throughput or 0.0)


def _rt_c(rt: SideTaskRuntime) -> A.TaskRuntimeC:
    return A.TaskRuntimeC(
        state=int(rt.state), has_last_paused=rt.last_paused is not None,
        has_assigned_worker=rt.assigned_worker is not None,
        assigned_worker=rt.assigned_worker or 0, has_busy_until=rt.busy_until is not None,
        steps_completed=rt.steps_completed, memory_allocated=rt.memory_allocated,
        last_paused=rt.last_paused or 0, busy_until=rt.busy_until or 0,
        memory_demand=rt.spec.memory_demand)


def _op_py(o) -> OpEvent:
    return OpEvent(o.stage, OpKind(o.kind), o.micro_batch, o.epoch, o.start, o.end)


def _bubble_py(b) -> Bubble:
    return Bubble(b.stage, b.epoch, b.start, b.duration, b.available_memory, BubbleType(b.btype))


def _bubble_c(b: Bubble, prev=-1, nxt=-1) -> A.BubbleC:
    return A.BubbleC(stage=b.stage, epoch=b.epoch, start=b.start, duration=b.duration,
                     available_memory=b.available_memory, btype=int(b.btype),
                     prev_op=prev, next_op=nxt)


def _profile_c(p: TaskProfile) -> A.TaskProfileC:
    return A.TaskProfileC(
        task_id=_id(p.task_id), has_est_per_step=p.est_per_step_duration is not None,
        profiled_steps=p.profiled_steps, est_per_step_duration=p.est_per_step_duration or 0.0,
        max_per_step_duration=p.max_per_step_duration or 0.0, est_memory=p.est_memory)


class WorkerStates:
    """The reference's caller-owned std::vector<WorkerState> (manager.hpp:17-28),
    held behind an opaque fr_manager handle."""

    def __init__(self, api: "BubbleSim", gpu_mem: Sequence[float]):
        self._api = api
        self._lib = api.lib
        h = C.c_void_p()
        api._check(self._lib.fr_manager_create(len(gpu_mem), _arr(C.c_double, gpu_mem),
                                               C.byref(h)))
        self._h = h
        self.n = len(gpu_mem)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.fr_manager_destroy(h)
            self._h = None

    def info(self, w: int) -> dict:
        out = A.WorkerInfoC()
        self._api._check(self._lib.fr_manager_worker_info(self._h, w, C.byref(out)))
        return {
            "worker_id": out.worker_id,
            "gpu_mem": out.gpu_mem,
            "task_queue": [self.queue_at(w, i) for i in range(out.queue_len)],
            "current_task": out.current_task.decode() if out.has_current_task else None,
            "current_bubble": _bubble_py(out.current_bubble) if out.has_current_bubble else None,
        }

    def queue_at(self, w: int, i: int) -> str:
        buf = C.create_string_buffer(A.TASK_ID_MAX)
        self._api._check(self._lib.fr_manager_queue_at(self._h, w, i, buf, A.TASK_ID_MAX))
        return buf.value.decode()

    def task_count(self, w: int) -> int:           # manager.hpp:25-27
        i = self.info(w)
        return len(i["task_queue"]) + (1 if i["current_task"] is not None else 0)

    def push_task(self, w: int, task_id: str):
        """Mirror a (remote) worker's queued task (distributed Alg. 1)."""
        self._api._check(self._lib.fr_manager_push_task(self._h, w, _id(task_id)))

    def set_current_task(self, w: int, task_id: Optional[str]):
        self._api._check(self._lib.fr_manager_set_current_task(
            self._h, w, None if task_id is None else _id(task_id)))


class BubbleSim:
    """The reference API (bubblesim::*) over one library exporting freeride.h."""

    def __init__(self, lib: C.CDLL):
        self.lib = A.bind(lib, A.HOST_PROTOTYPES)
        self.has_engine = hasattr(lib, "fr_run_experiment")
        if self.has_engine:
            A.bind(lib, A.ENGINE_PROTOTYPES)

    def pipeline_p2p_plan(self, stage: int, num_stages: int, m: int):
        """[(group, is_send, peer, kind, micro_batch)] of one stage's 1F1B loop."""
        cap = 4 * max(m, 1) + 4
        buf = (A.P2POpC * cap)()
        n = C.c_int64()
        self._check(self.lib.fr_pipeline_p2p_plan(stage, num_stages, m, buf, cap, C.byref(n)))
        return [(b.group, bool(b.is_send), b.peer, OpKind(b.kind), b.micro_batch)
                for b in buf[:n.value]]

    # ----------------------------------------------------------- engine.hpp
    def run_experiment(self, cfg: PipelineConfig, tasks: Sequence[SideTaskSpec], seed: int,
                       with_tasks: bool = True, check_overhead: int = 1, rpc_latency: int = 0,
                       step_jitter: float = 0.0, profile_steps: int = 32, gate_max: bool = False,
                       limits: LimitConfig = LimitConfig(), check: bool = False,
                       trace_path: Optional[str] = None) -> dict:  # engine.hpp:97-98
        """RunTrace as plain tuples: ops (stage, kind, mb, epoch, start, end);
        bubbles (stage, epoch, start, duration, avail, btype); submits/assigns/
        rejects (t, task, worker); rpcs/transitions (t, task, kind, worker);
        activities (start, end, task, worker, kind, clipped); kills
        (t, task, worker, reason); dispositions (task, disposition, steps, worker).
        check: also run replay_check (engine.hpp:104) -> out["violations"];
        trace_path: also write the JSONL trace stream (trace.hpp:19)."""
        if not self.has_engine:
            raise FreeRideError("library has no engine (the reference declares run_experiment only)")
        c = _Cfg(cfg)
        arr = (A.SideTaskSpecC * max(1, len(tasks)))(*[_spec_c(t) for t in tasks])
        ec = A.ExperimentConfigC(pipeline=c.c, tasks=arr, n_tasks=len(tasks),
                                 limits=A.LimitConfigC(limits.grace_period, limits.memory_headroom,
                                                       limits.reclamation_delay),
                                 runtime=A.RuntimeOptionsC(check_overhead, rpc_latency, step_jitter,
                                                           profile_steps, int(gate_max)))
        h = C.c_void_p()
        self._check(self.lib.fr_run_experiment(C.byref(ec), int(with_tasks), seed, C.byref(h)))
        return self.trace_dict(h, check, trace_path)

    def trace_dict(self, h, check: bool = False, trace_path: Optional[str] = None) -> dict:
        """An fr_run_trace handle (simulated, or recorded on the GPU by
        fr_harness_run_trace) as run_experiment's dict; destroys the handle."""
        try:
            n = A.RunTraceCountsC()
            self._check(self.lib.fr_run_trace_get_counts(h, C.byref(n)))

            def get(fn, ctype, count, *pre):
                buf = (ctype * max(1, count))()
                self._check(fn(h, *pre, buf, count))
                return [buf[i] for i in range(count)]

            out = {"makespan": n.makespan}
            out["ops"] = [(o.stage, o.kind, o.micro_batch, o.epoch, o.start, o.end)
                          for o in get(self.lib.fr_run_trace_ops, A.OpEventC, n.ops)]
            out["bubbles"] = [(b.stage, b.epoch, b.start, b.duration, b.available_memory, b.btype)
                              for b in get(self.lib.fr_run_trace_bubbles, A.BubbleC, n.bubbles)]
            for name, which, cnt in (("submits", 0, n.submits), ("assigns", 1, n.assigns),
                                     ("rejects", 2, n.rejects)):
                out[name] = [(r.t, r.task.decode(), r.worker)
                             for r in get(self.lib.fr_run_trace_assigns, A.AssignRecordC, cnt, which)]
            for name, which, cnt in (("transitions", 0, n.transitions), ("rpcs", 1, n.rpcs)):
                out[name] = [(r.t, r.task.decode(), r.kind, r.worker)
                             for r in get(self.lib.fr_run_trace_transitions, A.TransitionRecordC, cnt, which)]
            out["activities"] = [(a.start, a.end, a.task.decode(), a.worker, a.kind, bool(a.clipped))
                                 for a in get(self.lib.fr_run_trace_activities, A.ActivityRecordC, n.activities)]
            out["kills"] = [(k.t, k.task.decode(), k.worker, k.reason)
                            for k in get(self.lib.fr_run_trace_kills, A.KillRecordC, n.kills)]
            out["dispositions"] = [(d.task.decode(), d.disposition, d.steps_completed,
                                    d.worker if d.has_worker else None)
                                   for d in get(self.lib.fr_run_trace_dispositions, A.DispositionRecordC,
                                                n.dispositions)]
            if check:
                out["violations"] = self._trace_check(h)
            if trace_path is not None:
                self._check(self.lib.fr_run_trace_write_jsonl(h, trace_path.encode()))
            return out
        finally:
            self.lib.fr_run_trace_destroy(h)

    def _trace_check(self, h) -> List[str]:
        n = C.c_int32()
        buf = C.create_string_buffer(1 << 16)
        self._check(self.lib.fr_run_trace_check(h, buf, len(buf), C.byref(n)))
        return [x for x in buf.value.decode().split("\n") if x][: n.value] if n.value else []

    def replay_check_file(self, path: str) -> List[str]:
        """read_trace_file + replay_check (trace.hpp:20, engine.hpp:104)."""
        h = C.c_void_p()
        self._check(self.lib.fr_run_trace_read_jsonl(path.encode(), C.byref(h)))
        try:
            return self._trace_check(h)
        finally:
            self.lib.fr_run_trace_destroy(h)

    def _check(self, rc: int):
        A.raise_for(self.lib, rc)

    # -------------------------------------------------------- pipeline.hpp
    def validate(self, cfg: PipelineConfig):                         # :35
        c = _Cfg(cfg)
        self._check(self.lib.fr_pipeline_validate(C.byref(c.c)))

    def stage_issue_order(self, stage: int, num_stages: int, m: int):  # :72
        cap = max(0, 2 * m)
        buf = (A.Issue * max(1, cap))()
        n = C.c_int64()
        self._check(self.lib.fr_stage_issue_order(stage, num_stages, m, buf, cap, C.byref(n)))
        return [(OpKind(buf[i].kind), buf[i].micro_batch) for i in range(n.value)]

    def build_schedule_raw(self, cfg: PipelineConfig):
        c = _Cfg(cfg)
        cap = 2 * max(cfg.num_stages, 0) * max(cfg.num_micro_batches, 0) * max(cfg.num_epochs, 0)
        ops = (A.OpEventC * max(1, cap))()
        spans = (A.tick * max(2, 2 * max(cfg.num_epochs, 0)))()
        n = C.c_int64()
        self._check(self.lib.fr_build_schedule(C.byref(c.c), ops, cap, C.byref(n), spans))
        return ops, n.value, spans

    def build_schedule(self, cfg: PipelineConfig) -> ScheduleTrace:  # :78
        ops, n, spans = self.build_schedule_raw(cfg)
        return ScheduleTrace([_op_py(ops[i]) for i in range(n)],
                             [(spans[2 * e], spans[2 * e + 1]) for e in range(cfg.num_epochs)],
                             cfg)

    def extract_bubbles_linked(self, trace: ScheduleTrace) -> List[LinkedBubble]:  # :108
        cfg = trace.config
        c = _Cfg(cfg)
        ops = (A.OpEventC * max(1, len(trace.ops)))()
        for i, o in enumerate(trace.ops):
            ops[i] = A.OpEventC(o.stage, int(o.kind), o.micro_batch, o.epoch, o.start, o.end)
        spans = _arr(A.tick, [x for s in trace.epoch_spans for x in s])
        cap = cfg.num_epochs * cfg.num_stages * (2 * cfg.num_micro_batches + 1)
        out = (A.BubbleC * max(1, cap))()
        n = C.c_int64()
        self._check(self.lib.fr_extract_bubbles(C.byref(c.c), ops, len(trace.ops), spans, out,
                                                cap, C.byref(n)))
        res = []
        for i in range(n.value):
            b = out[i]
            res.append(LinkedBubble(_bubble_py(b), None if b.prev_op < 0 else b.prev_op,
                                    None if b.next_op < 0 else b.next_op))
        return res

    def extract_bubbles(self, trace: ScheduleTrace) -> List[Bubble]:  # :84
        return [lb.bubble for lb in self.extract_bubbles_linked(trace)]

    def bubble_rate(self, trace: ScheduleTrace, bubbles: Sequence[Bubble]) -> float:  # :87
        ops = (A.OpEventC * max(1, len(trace.ops)))()
        for i, o in enumerate(trace.ops):
            ops[i] = A.OpEventC(o.stage, int(o.kind), o.micro_batch, o.epoch, o.start, o.end)
        bs = (A.BubbleC * max(1, len(bubbles)))()
        for i, b in enumerate(bubbles):
            bs[i] = _bubble_c(b)
        r = C.c_double()
        self._check(self.lib.fr_bubble_rate(trace.config.num_stages, ops, len(trace.ops), bs,
                                            len(bubbles), C.byref(r)))
        return r.value

    def default_stage_memory(self, num_stages, gpu_memory_total, weight_mem,
                             activation_mem_per_microbatch) -> List[float]:  # :91
        out = (C.c_double * max(1, num_stages))()
        self._check(self.lib.fr_default_stage_memory(num_stages, gpu_memory_total, weight_mem,
                                                     activation_mem_per_microbatch, out))
        return [out[i] for i in range(num_stages)]

    # ------------------------------------------------------------ task.hpp
    def validate_spec(self, spec: SideTaskSpec, path: str = "tasks[0]"):  # :49
        s = _spec_c(spec)
        self._check(self.lib.fr_side_task_validate(C.byref(s), path.encode()))

    def transition_legal(self, frm: SideTaskState, kind: TransitionKind) -> bool:  # :69
        out = C.c_int32()
        self._check(self.lib.fr_transition_legal(int(frm), int(kind), C.byref(out)))
        return bool(out.value)

    def transition_target(self, frm, kind) -> SideTaskState:  # :70
        out = C.c_int32()
        self._check(self.lib.fr_transition_target(int(frm), int(kind), C.byref(out)))
        return SideTaskState(out.value)

    def apply_transition(self, rt: SideTaskRuntime, kind: TransitionKind, now: int):  # :75
        c = _rt_c(rt)
        self._check(self.lib.fr_apply_transition(C.byref(c), int(kind), now))
        rt.state = SideTaskState(c.state)
        rt.steps_completed = c.steps_completed
        rt.memory_allocated = c.memory_allocated
        rt.last_paused = c.last_paused if c.has_last_paused else None
        rt.assigned_worker = c.assigned_worker if c.has_assigned_worker else None
        rt.busy_until = c.busy_until if c.has_busy_until else None
        return rt

    def iterative_run(self, rt, bubble_end, now, est_step_seconds, tick_seconds,
                      actual_step_ticks) -> IterativeDecision:  # :87-89
        c = _rt_c(rt)
        out = A.IterativeDecisionC()
        self._check(self.lib.fr_iterative_run(C.byref(c), bubble_end, now, est_step_seconds,
                                              tick_seconds, actual_step_ticks, C.byref(out)))
        return IterativeDecision(bool(out.run), out.step_end)

    def imperative_run(self, rt, now, actual_kernel_ticks) -> int:  # :93
        c = _rt_c(rt)
        out = A.tick()
        self._check(self.lib.fr_imperative_run(C.byref(c), now, actual_kernel_ticks, C.byref(out)))
        return out.value

    # ---------------------------------------------------------- limits.hpp
    def validate_limits(self, lc: LimitConfig):  # :14
        c = A.LimitConfigC(lc.grace_period, lc.memory_headroom, lc.reclamation_delay)
        self._check(self.lib.fr_limit_config_validate(C.byref(c)))

    def check_memory(self, memory_allocated: float, limit: float) -> MemCheck:  # :20
        out = C.c_int32()
        self._check(self.lib.fr_check_memory(memory_allocated, limit, C.byref(out)))
        return MemCheck(out.value)

    def program_directed_gate(self, remaining: float, est: float) -> Gate:  # :26
        out = C.c_int32()
        self._check(self.lib.fr_program_directed_gate(remaining, est, C.byref(out)))
        return Gate(out.value)

    def framework_enforce(self, last_paused: Optional[int], pause_issued_at: int, now: int,
                          grace_period: int) -> Enforce:  # :34
        out = C.c_int32()
        self._check(self.lib.fr_framework_enforce(last_paused is not None, last_paused or 0,
                                                  pause_issued_at, now, grace_period,
                                                  C.byref(out)))
        return Enforce(out.value)

    # -------------------------------------------------------- profiler.hpp
    def stream_seed(self, seed: int, task_id: str, salt: str) -> int:  # :48
        return self.lib.fr_stream_seed(seed, task_id.encode(), salt.encode())

    def jittered_step_ticks(self, base: int, jitter: float, rng_state: List[int]) -> int:  # :53
        s = C.c_uint64(rng_state[0])
        t = self.lib.fr_jittered_step_ticks(base, jitter, C.byref(s))
        rng_state[0] = s.value
        return t

    def profile_task(self, spec: SideTaskSpec, opts: ProfileOptions, seed: int) -> TaskProfile:
        s = _spec_c(spec)                                                # :41
        o = A.ProfileOptionsC(n_steps=opts.n_steps, step_jitter=opts.step_jitter,
                              tick_seconds=opts.tick_seconds)
        out = A.TaskProfileC()
        self._check(self.lib.fr_profile_task(C.byref(s), C.byref(o), seed, C.byref(out)))
        has = bool(out.has_est_per_step)
        return TaskProfile(out.task_id.decode(), out.est_per_step_duration if has else None,
                           out.max_per_step_duration if has else None, out.est_memory,
                           out.profiled_steps)

    def profile_bubbles(self, cfg: PipelineConfig) -> BubbleProfile:  # :45
        c = _Cfg(cfg)
        p = max(cfg.num_stages, 1)
        cap = p * (2 * max(cfg.num_micro_batches, 1) + 1)
        d = (A.tick * cap)()
        offs = (C.c_int64 * (p + 1))()
        avail = (C.c_double * p)()
        rate = C.c_double()
        self._check(self.lib.fr_profile_bubbles(C.byref(c.c), d, cap, offs, avail,
                                                C.byref(rate)))
        stages = [StageBubbleProfile([d[k] for k in range(offs[s], offs[s + 1])], avail[s])
                  for s in range(cfg.num_stages)]
        return BubbleProfile(stages, rate.value)

    # --------------------------------------------------------- manager.hpp
    def workers(self, gpu_mem: Sequence[float]) -> WorkerStates:
        return WorkerStates(self, gpu_mem)

    def select_worker(self, task_memory: float, workers: WorkerStates) -> Optional[int]:  # :33
        out = C.c_int32()
        self._check(self.lib.fr_select_worker(workers._h, task_memory, C.byref(out)))
        return None if out.value < 0 else out.value

    def submit_task(self, profile: TaskProfile, workers: WorkerStates) -> SubmitOutcome:  # :43
        p = _profile_c(profile)
        a, w = C.c_int32(), C.c_int32()
        self._check(self.lib.fr_submit_task(workers._h, C.byref(p), C.byref(a), C.byref(w)))
        return SubmitOutcome(bool(a.value), w.value)

    def _lookup(self, lookup: Callable[[str], TaskView]):
        def cb(ctx, task_id, out):
            try:
                v = lookup(task_id.decode())
                out[0].state = int(v.state)
                out[0].initializing = int(bool(v.initializing))
                return A.FR_OK
            except Exception:  # noqa: BLE001 -- surfaced as a status code
                return A.FR_ERR_NOT_FOUND
        return A.LOOKUP_FN(cb)

    def _actions(self, fn, *args) -> List[ManagerAction]:
        out = (A.ManagerActionC * 8)()
        n = C.c_int32()
        self._check(fn(*args, out, 8, C.byref(n)))
        return [ManagerAction(ManagerActionKind(out[i].kind), out[i].task_id.decode())
                for i in range(n.value)]

    def on_bubble_started(self, workers: WorkerStates, worker: int, bubble: Bubble,
                          lookup: Callable[[str], TaskView]) -> List[ManagerAction]:  # :69
        cb = self._lookup(lookup)
        b = _bubble_c(bubble)
        return self._actions(self.lib.fr_on_bubble_started, workers._h, worker, C.byref(b), cb,
                             None)

    def on_bubble_ended(self, workers: WorkerStates, worker: int, now: int,
                        lookup: Callable[[str], TaskView]) -> List[ManagerAction]:  # :76
        cb = self._lookup(lookup)
        return self._actions(self.lib.fr_on_bubble_ended, workers._h, worker, now, cb, None)

    # --------------------------------------------------------- metrics.hpp
    def time_increase(self, t_no: float, t_with: float) -> float:  # :25
        out = C.c_double()
        self._check(self.lib.fr_time_increase(t_no, t_with, C.byref(out)))
        return out.value

    def cost_savings(self, t_no: float, delta_t: float, work: Sequence[TaskWork],
                     prices: PriceConfig = PriceConfig()) -> CostBreakdown:  # :45
        arr = (A.TaskWorkC * max(1, len(work)))()
        for i, w in enumerate(work):
            arr[i] = A.TaskWorkC(id=_id(w.id), work=w.work,
                                 has_throughput=w.throughput_per_hour is not None,
                                 throughput_per_hour=w.throughput_per_hour or 0.0)
        pc = A.PriceConfigC(prices.price_server_1, prices.price_server_2)
        out = A.CostBreakdownC()
        self._check(self.lib.fr_cost_savings(t_no, delta_t, arr, len(work), C.byref(pc),
                                             C.byref(out)))
        return CostBreakdown(out.c_no_side, out.c_extra, out.c_side_tasks, out.s)

    def bubble_breakdown(self, num_stages: int, profiles: Sequence[TaskProfile],
                         bubbles: Sequence[Bubble], assigns: Sequence[AssignRecord],
                         transitions: Sequence[TransitionRecord],
                         activities: Sequence[ActivityRecord]) -> List[StageBreakdown]:  # :64
        pr = (A.TaskProfileC * max(1, len(profiles)))(*[_profile_c(p) for p in profiles])
        bs = (A.BubbleC * max(1, len(bubbles)))(*[_bubble_c(b) for b in bubbles])
        asg = (A.AssignRecordC * max(1, len(assigns)))(
            *[A.AssignRecordC(t=a.t, worker=a.worker, task=_id(a.task)) for a in assigns])
        tr = (A.TransitionRecordC * max(1, len(transitions)))(
            *[A.TransitionRecordC(t=r.t, kind=int(r.kind), worker=r.worker, task=_id(r.task))
              for r in transitions])
        ac = (A.ActivityRecordC * max(1, len(activities)))(
            *[A.ActivityRecordC(start=a.start, end=a.end, worker=a.worker, kind=int(a.kind),
                                clipped=int(a.clipped), task=_id(a.task)) for a in activities])
        inp = A.BreakdownInputC(num_stages=num_stages, n_profiles=len(profiles), profiles=pr,
                                n_bubbles=len(bubbles), bubbles=bs, n_assigns=len(assigns),
                                assigns=asg, n_transitions=len(transitions), transitions=tr,
                                n_activities=len(activities), activities=ac)
        out = (A.StageBreakdownC * max(1, num_stages))()
        self._check(self.lib.fr_bubble_breakdown(C.byref(inp), out))
        return [StageBreakdown(out[s].stage, out[s].used_by_side_tasks, out[s].runtime_overhead,
                               out[s].idle_oom, out[s].idle_insufficient_time)
                for s in range(num_stages)]
