"""ctypes mirror of include/freeride.h.

One binding serves every library that exports the header: the product
(`_lib/libfreeride.so`) and, in tests only, the reference's own sources behind
the oracle shim (`oracle/_ref/libbubblesim_ref.so`).  Status codes are mapped
back onto the reference's exception types (types.hpp:22-42, task.hpp:62,
pipeline.cpp:155) so callers see the reference's error behaviour.
"""
from __future__ import annotations

import ctypes as C

TASK_ID_MAX = 64

FR_OK = 0
FR_ERR_VALIDATION = 1
FR_ERR_SCHEMA = 2
FR_ERR_INVARIANT = 3
FR_ERR_ILLEGAL_TRANSITION = 4
FR_ERR_CAPACITY = 5
FR_ERR_ARGUMENT = 6
FR_ERR_NOT_FOUND = 7
FR_ERR_UNSUPPORTED = 8
FR_ERR_CUDA_BASE = 100

tick = C.c_int64


class FreeRideError(RuntimeError):
    code = -1


class ValidationError(FreeRideError):
    """bubblesim::ValidationError (types.hpp:22): `.field` names the config field."""
    code = FR_ERR_VALIDATION

    def __init__(self, field, message):
        super().__init__(message)
        self.field = field


class SchemaError(FreeRideError):
    """bubblesim::SchemaError (types.hpp:34): `.path` names the document path."""
    code = FR_ERR_SCHEMA

    def __init__(self, path, message):
        super().__init__(message)
        self.path = path


class IllegalTransition(FreeRideError):
    """bubblesim::IllegalTransition (task.hpp:62)."""
    code = FR_ERR_ILLEGAL_TRANSITION


class InvariantError(FreeRideError):
    """std::logic_error raised by the reference (e.g. pipeline.cpp:155)."""
    code = FR_ERR_INVARIANT


class CapacityError(FreeRideError):
    code = FR_ERR_CAPACITY


class CudaError(FreeRideError):
    code = FR_ERR_CUDA_BASE


class Struct(C.Structure):
    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if isinstance(v, bytes):
                v = v.decode()
            out[name] = v
        return out


class PipelineConfigC(Struct):
    _fields_ = [
        ("num_stages", C.c_int32),
        ("num_micro_batches", C.c_int32),
        ("num_epochs", C.c_int32),
        ("n_fp", C.c_int32),
        ("fp_duration", C.POINTER(tick)),
        ("n_bp", C.c_int32),
        ("n_stage_memory", C.c_int32),
        ("bp_duration", C.POINTER(tick)),
        ("stage_memory", C.POINTER(C.c_double)),
        ("gpu_memory_total", C.c_double),
        ("tick_seconds", C.c_double),
    ]


class Issue(Struct):
    _fields_ = [("kind", C.c_int32), ("micro_batch", C.c_int32)]


class OpEventC(Struct):
    _fields_ = [
        ("stage", C.c_int32),
        ("kind", C.c_int32),
        ("micro_batch", C.c_int32),
        ("epoch", C.c_int32),
        ("start", tick),
        ("end", tick),
    ]


class BubbleC(Struct):
    _fields_ = [
        ("stage", C.c_int32),
        ("epoch", C.c_int32),
        ("start", tick),
        ("duration", tick),
        ("available_memory", C.c_double),
        ("btype", C.c_int32),
        ("reserved", C.c_int32),
        ("prev_op", C.c_int64),
        ("next_op", C.c_int64),
    ]


class SideTaskSpecC(Struct):
    _fields_ = [
        ("id", C.c_char * TASK_ID_MAX),
        ("interface_kind", C.c_int32),
        ("misbehavior", C.c_int32),
        ("has_total_steps", C.c_int32),
        ("has_memory_limit", C.c_int32),
        ("has_reference_throughput", C.c_int32),
        ("reserved", C.c_int32),
        ("per_step_duration", tick),
        ("total_steps", C.c_int64),
        ("init_duration", tick),
        ("memory_demand", C.c_double),
        ("leak_rate_gib_per_s", C.c_double),
        ("submit_time", tick),
        ("memory_limit", C.c_double),
        ("reference_throughput", C.c_double),
    ]


class TaskRuntimeC(Struct):
    _fields_ = [
        ("state", C.c_int32),
        ("has_last_paused", C.c_int32),
        ("has_assigned_worker", C.c_int32),
        ("assigned_worker", C.c_int32),
        ("has_busy_until", C.c_int32),
        ("reserved", C.c_int32),
        ("steps_completed", C.c_int64),
        ("memory_allocated", C.c_double),
        ("last_paused", tick),
        ("busy_until", tick),
        ("memory_demand", C.c_double),
    ]


class IterativeDecisionC(Struct):
    _fields_ = [("run", C.c_int32), ("reserved", C.c_int32), ("step_end", tick)]


class LimitConfigC(Struct):
    _fields_ = [
        ("grace_period", tick),
        ("memory_headroom", C.c_double),
        ("reclamation_delay", tick),
    ]


class ProfileOptionsC(Struct):
    _fields_ = [
        ("n_steps", C.c_int32),
        ("reserved", C.c_int32),
        ("step_jitter", C.c_double),
        ("tick_seconds", C.c_double),
    ]


class TaskProfileC(Struct):
    _fields_ = [
        ("task_id", C.c_char * TASK_ID_MAX),
        ("has_est_per_step", C.c_int32),
        ("profiled_steps", C.c_int32),
        ("est_per_step_duration", C.c_double),
        ("max_per_step_duration", C.c_double),
        ("est_memory", C.c_double),
    ]


class TaskViewC(Struct):
    _fields_ = [("state", C.c_int32), ("initializing", C.c_int32)]


class ManagerActionC(Struct):
    _fields_ = [("kind", C.c_int32), ("task_id", C.c_char * TASK_ID_MAX)]


class WorkerInfoC(Struct):
    _fields_ = [
        ("worker_id", C.c_int32),
        ("queue_len", C.c_int32),
        ("has_current_task", C.c_int32),
        ("has_current_bubble", C.c_int32),
        ("gpu_mem", C.c_double),
        ("current_task", C.c_char * TASK_ID_MAX),
        ("current_bubble", BubbleC),
    ]


class PriceConfigC(Struct):
    _fields_ = [("price_server_1", C.c_double), ("price_server_2", C.c_double)]


class TaskWorkC(Struct):
    _fields_ = [
        ("id", C.c_char * TASK_ID_MAX),
        ("work", C.c_double),
        ("has_throughput", C.c_int32),
        ("reserved", C.c_int32),
        ("throughput_per_hour", C.c_double),
    ]


class CostBreakdownC(Struct):
    _fields_ = [
        ("c_no_side", C.c_double),
        ("c_extra", C.c_double),
        ("c_side_tasks", C.c_double),
        ("s", C.c_double),
    ]


class StageBreakdownC(Struct):
    _fields_ = [
        ("stage", C.c_int32),
        ("reserved", C.c_int32),
        ("used_by_side_tasks", tick),
        ("runtime_overhead", tick),
        ("idle_oom", tick),
        ("idle_insufficient_time", tick),
    ]


class TransitionRecordC(Struct):
    _fields_ = [
        ("t", tick),
        ("kind", C.c_int32),
        ("worker", C.c_int32),
        ("task", C.c_char * TASK_ID_MAX),
    ]


class ActivityRecordC(Struct):
    _fields_ = [
        ("start", tick),
        ("end", tick),
        ("worker", C.c_int32),
        ("kind", C.c_int32),
        ("clipped", C.c_int32),
        ("reserved", C.c_int32),
        ("task", C.c_char * TASK_ID_MAX),
    ]


class KillRecordC(Struct):
    _fields_ = [
        ("t", tick),
        ("worker", C.c_int32),
        ("reason", C.c_int32),
        ("task", C.c_char * TASK_ID_MAX),
    ]


class AssignRecordC(Struct):
    _fields_ = [
        ("t", tick),
        ("worker", C.c_int32),
        ("reserved", C.c_int32),
        ("task", C.c_char * TASK_ID_MAX),
    ]


class DispositionRecordC(Struct):
    _fields_ = [
        ("disposition", C.c_int32),
        ("has_worker", C.c_int32),
        ("worker", C.c_int32),
        ("reserved", C.c_int32),
        ("steps_completed", C.c_int64),
        ("task", C.c_char * TASK_ID_MAX),
    ]


class BreakdownInputC(Struct):
    _fields_ = [
        ("num_stages", C.c_int32),
        ("n_profiles", C.c_int32),
        ("profiles", C.POINTER(TaskProfileC)),
        ("n_bubbles", C.c_int64),
        ("bubbles", C.POINTER(BubbleC)),
        ("n_assigns", C.c_int64),
        ("assigns", C.POINTER(AssignRecordC)),
        ("n_transitions", C.c_int64),
        ("transitions", C.POINTER(TransitionRecordC)),
        ("n_activities", C.c_int64),
        ("activities", C.POINTER(ActivityRecordC)),
    ]


class RuntimeOptionsC(Struct):
    _fields_ = [("check_overhead", tick), ("rpc_latency", tick), ("step_jitter", C.c_double),
                ("profile_steps", C.c_int32), ("gate_estimate", C.c_int32)]


class ExperimentConfigC(Struct):
    _fields_ = [("pipeline", PipelineConfigC), ("tasks", C.POINTER(SideTaskSpecC)),
                ("n_tasks", C.c_int32), ("reserved", C.c_int32), ("limits", LimitConfigC),
                ("runtime", RuntimeOptionsC)]


class RunTraceCountsC(Struct):
    _fields_ = [(n, C.c_int64) for n in ("ops", "bubbles", "submits", "assigns", "rejects", "rpcs",
                                         "transitions", "activities", "kills", "dispositions")] + \
               [("makespan", tick)]


LOOKUP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_char_p, C.POINTER(TaskViewC))

P = C.POINTER
i32, i64, u64, dbl, vp, cp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p, C.c_char_p

# name -> (restype, argtypes); every library exporting freeride.h host rows
HOST_PROTOTYPES = {
    "fr_abi_version": (C.c_int, []),
    "fr_last_error": (cp, []),
    "fr_last_error_field": (cp, []),
    "fr_pipeline_validate": (C.c_int, [P(PipelineConfigC)]),
    "fr_stage_issue_order": (C.c_int, [i32, i32, i32, P(Issue), i64, P(i64)]),
    "fr_build_schedule": (C.c_int, [P(PipelineConfigC), P(OpEventC), i64, P(i64), P(tick)]),
    "fr_extract_bubbles": (C.c_int, [P(PipelineConfigC), P(OpEventC), i64, P(tick), P(BubbleC), i64, P(i64)]),
    "fr_bubble_rate": (C.c_int, [i32, P(OpEventC), i64, P(BubbleC), i64, P(dbl)]),
    "fr_default_stage_memory": (C.c_int, [i32, dbl, dbl, dbl, P(dbl)]),
    "fr_side_task_validate": (C.c_int, [P(SideTaskSpecC), cp]),
    "fr_transition_legal": (C.c_int, [i32, i32, P(i32)]),
    "fr_transition_target": (C.c_int, [i32, i32, P(i32)]),
    "fr_apply_transition": (C.c_int, [P(TaskRuntimeC), i32, tick]),
    "fr_iterative_run": (C.c_int, [P(TaskRuntimeC), tick, tick, dbl, dbl, tick, P(IterativeDecisionC)]),
    "fr_imperative_run": (C.c_int, [P(TaskRuntimeC), tick, tick, P(tick)]),
    "fr_limit_config_validate": (C.c_int, [P(LimitConfigC)]),
    "fr_check_memory": (C.c_int, [dbl, dbl, P(i32)]),
    "fr_program_directed_gate": (C.c_int, [dbl, dbl, P(i32)]),
    "fr_framework_enforce": (C.c_int, [i32, tick, tick, tick, tick, P(i32)]),
    "fr_stream_seed": (u64, [u64, cp, cp]),
    "fr_jittered_step_ticks": (tick, [tick, dbl, P(u64)]),
    "fr_profile_task": (C.c_int, [P(SideTaskSpecC), P(ProfileOptionsC), u64, P(TaskProfileC)]),
    "fr_profile_bubbles": (C.c_int, [P(PipelineConfigC), P(tick), i64, P(i64), P(dbl), P(dbl)]),
    "fr_manager_create": (C.c_int, [i32, P(dbl), P(vp)]),
    "fr_manager_destroy": (None, [vp]),
    "fr_manager_worker_info": (C.c_int, [vp, i32, P(WorkerInfoC)]),
    "fr_manager_queue_at": (C.c_int, [vp, i32, i32, C.c_char_p, i32]),
    "fr_manager_set_current_task": (C.c_int, [vp, i32, cp]),
    "fr_select_worker": (C.c_int, [vp, dbl, P(i32)]),
    "fr_submit_task": (C.c_int, [vp, P(TaskProfileC), P(i32), P(i32)]),
    "fr_on_bubble_started": (C.c_int, [vp, i32, P(BubbleC), LOOKUP_FN, vp, P(ManagerActionC), i32, P(i32)]),
    "fr_on_bubble_ended": (C.c_int, [vp, i32, tick, LOOKUP_FN, vp, P(ManagerActionC), i32, P(i32)]),
    "fr_time_increase": (C.c_int, [dbl, dbl, P(dbl)]),
    "fr_cost_savings": (C.c_int, [dbl, dbl, P(TaskWorkC), i32, P(PriceConfigC), P(CostBreakdownC)]),
    "fr_bubble_breakdown": (C.c_int, [P(BreakdownInputC), P(StageBreakdownC)]),
}


class P2POpC(Struct):
    _fields_ = [("group", i32), ("is_send", i32), ("peer", i32), ("kind", i32), ("micro_batch", i32)]


# the engine rows (the reference declares run_experiment but has no .cpp)
ENGINE_PROTOTYPES = {
    "fr_pipeline_p2p_plan": (C.c_int, [i32, i32, i32, P(P2POpC), i64, P(i64)]),
    "fr_manager_push_task": (C.c_int, [vp, i32, cp]),
    "fr_run_experiment": (C.c_int, [P(ExperimentConfigC), i32, u64, P(vp)]),
    "fr_run_trace_destroy": (None, [vp]),
    "fr_run_trace_check": (C.c_int, [vp, C.c_char_p, i64, P(i32)]),
    "fr_run_trace_write_jsonl": (C.c_int, [vp, C.c_char_p]),
    "fr_run_trace_read_jsonl": (C.c_int, [C.c_char_p, P(vp)]),
    "fr_run_trace_get_counts": (C.c_int, [vp, P(RunTraceCountsC)]),
    "fr_run_trace_ops": (C.c_int, [vp, P(OpEventC), i64]),
    "fr_run_trace_bubbles": (C.c_int, [vp, P(BubbleC), i64]),
    "fr_run_trace_assigns": (C.c_int, [vp, i32, P(AssignRecordC), i64]),
    "fr_run_trace_transitions": (C.c_int, [vp, i32, P(TransitionRecordC), i64]),
    "fr_run_trace_activities": (C.c_int, [vp, P(ActivityRecordC), i64]),
    "fr_run_trace_kills": (C.c_int, [vp, P(KillRecordC), i64]),
    "fr_run_trace_dispositions": (C.c_int, [vp, P(DispositionRecordC), i64]),
}


def bind(lib: C.CDLL, prototypes: dict) -> C.CDLL:
    for name, (res, args) in prototypes.items():
        fn = getattr(lib, name)  # AttributeError: symbol missing -> loud
        fn.restype = res
        fn.argtypes = args
    return lib


def raise_for(lib: C.CDLL, rc: int):
    if rc == FR_OK:
        return
    msg = (lib.fr_last_error() or b"").decode(errors="replace")
    field = (lib.fr_last_error_field() or b"").decode(errors="replace")
    if rc == FR_ERR_VALIDATION:
        raise ValidationError(field, msg)
    if rc == FR_ERR_SCHEMA:
        raise SchemaError(field, msg)
    if rc == FR_ERR_ILLEGAL_TRANSITION:
        raise IllegalTransition(msg)
    if rc == FR_ERR_INVARIANT:
        raise InvariantError(msg)
    if rc == FR_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc >= FR_ERR_CUDA_BASE:
        e = CudaError(f"CUDA error {rc - FR_ERR_CUDA_BASE}: {msg}")
        raise e
    e = FreeRideError(f"status {rc}: {msg}")
    e.code = rc
    raise e


# ---------------------------------------------------------------- freeride_gpu.h
GPU_PROTOTYPES = {
    "fr_stream_create": (C.c_int, [i32, P(vp)]),
    "fr_stream_destroy": (C.c_int, [vp]),
    "fr_stream_synchronize": (C.c_int, [vp]),
    "fr_device_sm_count": (C.c_int, [P(i32)]),
    "fr_set_device": (C.c_int, [i32]),
    "fr_get_device": (C.c_int, [P(i32)]),
    "fr_clock_probe": (C.c_int, [vp, i64, vp]),
    "fr_memcpy": (C.c_int, [vp, vp, i64]),
    "fr_img_plan_create": (C.c_int, [i32, i32, i32, i32, P(vp)]),
    "fr_img_plan_set_overlap": (C.c_int, [vp, i32]),
    "fr_img_plan_destroy": (C.c_int, [vp]),
    "fr_img_plan_path": (C.c_int, [vp, P(i32)]),
    "fr_img_resize_watermark": (C.c_int, [vp, vp, vp, vp, i32, vp]),
    "fr_img_prepared_bytes": (C.c_int, [vp, P(i64)]),
    "fr_img_prepare_watermark": (C.c_int, [vp, vp, vp, vp]),
    "fr_img_resize_watermark_prepared": (C.c_int, [vp, vp, vp, vp, i32, vp]),
    "fr_img_resize_watermark_preemptible": (C.c_int, [vp, vp, vp, vp, i32, vp, i64, vp, vp]),
    "fr_img_preemptible_unit_rows": (C.c_int, [vp, i32, P(i32)]),
    "fr_img_generate": (C.c_int, [vp, i32, i32, i32, i32, u64, i32, vp]),
    "fr_img_generate_watermark": (C.c_int, [vp, i32, i32, u64, vp]),
}


class SideTaskVTableC(Struct):
    _fields_ = [
        ("create", C.CFUNCTYPE(C.c_int, vp)),
        ("init", C.CFUNCTYPE(C.c_int, vp, vp)),
        ("start", C.CFUNCTYPE(C.c_int, vp)),
        ("run_next_step", C.CFUNCTYPE(C.c_int, vp, vp)),
        ("pause", C.CFUNCTYPE(C.c_int, vp)),
        ("stop", C.CFUNCTYPE(C.c_int, vp)),
        ("finished", C.CFUNCTYPE(C.c_int, vp, C.c_int64, P(i32))),
        ("destroy", C.CFUNCTYPE(None, vp)),
        ("work_units_per_step", C.c_double),
        ("interface_kind", i32),
        ("carveout_hint", i32),
        ("run_gpu_workload", C.CFUNCTYPE(C.c_int, vp, vp, vp)),
        ("work_done", C.CFUNCTYPE(C.c_int, vp, vp, P(C.c_double))),
        ("cancel", C.CFUNCTYPE(C.c_int, vp)),
        ("set_sm_budget", C.CFUNCTYPE(C.c_int, vp, i32)),
    ]


class SyntheticTaskConfigC(Struct):
    _fields_ = [("step_ns", i64), ("profile_step_ns", i64), ("memory_demand_gib", C.c_double),
                ("leak_gib_per_step", C.c_double), ("total_steps", i64), ("cooperative", i32),
                ("reserved", i32), ("init_ns", i64)]


class PreemptC(Struct):
    _fields_ = [("stop_word", vp), ("token", C.c_uint32), ("reserved", C.c_uint32)]


class ImageTaskConfigC(Struct):
    _fields_ = [
        ("sw", i32), ("sh", i32), ("dw", i32), ("dh", i32),
        ("batch", i32), ("images_per_step", i32), ("host_io", i32), ("interface_kind", i32),
        ("seed", u64), ("total_steps", i64), ("host_ring", i32),
    ]


class PageRankTaskConfigC(Struct):
    _fields_ = [("scale", i32), ("edge_factor", i32), ("seed", u64), ("iters_per_step", i32),
                ("damping", C.c_float), ("total_steps", i64)]


GPU_PROTOTYPES.update({
    "fr_pr_graph_rmat": (C.c_int, [i32, i32, u64, vp, P(vp)]),
    "fr_pr_graph_from_edges": (C.c_int, [i32, i64, vp, vp, vp, P(vp)]),
    "fr_pr_graph_destroy": (C.c_int, [vp]),
    "fr_pr_graph_info": (C.c_int, [vp, P(i32), P(i64), P(i32)]),
    "fr_pr_graph_csr": (C.c_int, [vp, P(vp), P(vp), P(vp)]),
    "fr_pr_state_create": (C.c_int, [vp, P(vp)]),
    "fr_pr_state_destroy": (C.c_int, [vp]),
    "fr_pr_reset": (C.c_int, [vp, vp]),
    "fr_pr_step": (C.c_int, [vp, i32, C.c_float, vp]),
    "fr_pr_ranks": (C.c_int, [vp, P(vp), P(i64)]),
    "fr_pagerank_task_create": (C.c_int, [P(PageRankTaskConfigC), P(SideTaskVTableC), P(vp)]),
    "fr_pagerank_task_create_from_graph": (C.c_int, [P(PageRankTaskConfigC), vp, P(SideTaskVTableC), P(vp)]),
    "fr_pagerank_task_info": (C.c_int, [vp, P(i32), P(i64), P(dbl), P(vp), P(i64)]),
})


class SgdTaskConfigC(Struct):
    _fields_ = [("V", i32), ("k", i32), ("E", i64), ("edge_seed", u64), ("init_seed", u64),
                ("edges_per_step", i64), ("eta", C.c_float), ("lambda_", C.c_float),
                ("total_steps", i64), ("layout", i32), ("total_epochs", i32)]


SGD_LAYOUT_COO, SGD_LAYOUT_BY_USER = 0, 1

GPU_PROTOTYPES.update({
    "fr_sgd_problem_generate": (C.c_int, [i32, i64, i32, u64, u64, vp, P(vp)]),
    "fr_sgd_problem_from_edges": (C.c_int, [i32, i64, i32, vp, vp, vp, u64, vp, P(vp)]),
    "fr_sgd_problem_destroy": (C.c_int, [vp]),
    "fr_sgd_reinit": (C.c_int, [vp, u64, vp]),
    "fr_sgd_step": (C.c_int, [vp, i64, i64, C.c_float, C.c_float, vp]),
    "fr_sgd_group_by_user": (C.c_int, [vp, i64, vp]),
    "fr_sgd_problem_set_kernel": (C.c_int, [vp, i32]),
    "fr_sgd_problem_set_overlap": (C.c_int, [vp, i32]),
    "fr_sgd_sqerr": (C.c_int, [vp, i64, i64, vp, vp]),
    "fr_sgd_rmse": (C.c_int, [vp, vp, P(dbl)]),
    "fr_sgd_buffers": (C.c_int, [vp, P(vp), P(vp), P(vp), P(vp), P(i32), P(i64), P(i32)]),
    "fr_sgd_task_create": (C.c_int, [P(SgdTaskConfigC), P(SideTaskVTableC), P(vp)]),
    "fr_sgd_task_create_from_problem": (C.c_int, [P(SgdTaskConfigC), vp, P(SideTaskVTableC), P(vp)]),
    "fr_sgd_task_problem": (C.c_int, [vp, P(vp), P(i64)]),
})


class HarnessConfigC(Struct):
    _fields_ = [
        ("num_stages", i32), ("num_micro_batches", i32), ("stage", i32), ("layers", i32),
        ("hidden", i32), ("tokens", i32), ("ffn_mult", i32), ("profile_reps", i32),
        ("max_inflight_steps", i32), ("gate_estimate", i32),
        ("gpu_memory_total", dbl), ("weight_mem", dbl), ("activation_mem", dbl),
        ("fp_ticks_override", i64), ("bp_ticks_override", i64),
        ("profile_epochs", i32), ("transport", i32),
        ("memory_headroom_gib", dbl), ("grace_ns", i64), ("step_group", i32),
        ("harvest_fraction", dbl), ("reclamation_delay_ns", i64), ("side_sms", i32),
        ("min_side_sms", i32), ("dt_budget", dbl),
    ]


class HarnessProfileC(Struct):
    _fields_ = [
        ("fp_ticks", tick), ("bp_ticks", tick), ("epoch_span", tick), ("stage_bubble_ticks", tick),
        ("bubble_rate", dbl), ("available_memory", dbl), ("fp_tflops", dbl), ("bp_tflops", dbl),
        ("n_bubbles", i32), ("reserved", i32), ("clock_offset_err_ns", dbl),
    ]


class GateRecordC(Struct):
    _fields_ = [("now", tick), ("bubble_end", tick), ("est_seconds", dbl), ("step_ticks", tick),
                ("run", i32), ("signal", i32), ("step_end", tick), ("task", C.c_char * 64)]


class SignalRecordC(Struct):
    _fields_ = [("t", tick), ("kind", i32), ("epoch", i32), ("bubble", i32), ("looked_up", i32),
                ("duration", tick), ("view_state", i32), ("view_initializing", i32), ("n_actions", i32),
                ("actions", i32 * 4), ("deferred", i32), ("task", C.c_char * 64)]


class RunReportC(Struct):
    _fields_ = [
        ("epochs", i32), ("with_tasks", i32),
        ("makespan_s", dbl), ("bubble_s", dbl), ("used_s", dbl), ("overrun_s", dbl),
        ("work_units", dbl), ("steps_launched", i64), ("steps_completed", i64),
        ("dispatch_host_us", dbl), ("max_step_overrun_s", dbl),
        ("breakdown", StageBreakdownC), ("pauses", i64), ("kills", i64),
        ("kills_oom", i64), ("kills_pause_timeout", i64), ("kills_init_timeout", i64),
        ("op_growth", dbl), ("side_sms_mean", dbl), ("side_sms_final", i32), ("reserved2", i32),
        ("exchange_messages", i64), ("exchange_us", dbl), ("exchange_gbps", dbl),
    ]


GPU_PROTOTYPES.update({
    "fr_image_task_create": (C.c_int, [P(ImageTaskConfigC), P(SideTaskVTableC), P(vp)]),
    "fr_image_task_memory": (C.c_int, [P(ImageTaskConfigC), P(dbl)]),
    "fr_image_task_buffers": (C.c_int, [vp, P(vp), P(vp), P(vp), P(i64)]),
    "fr_image_task_host_output": (C.c_int, [vp, P(vp)]),
    "fr_harness_create": (C.c_int, [P(HarnessConfigC), P(vp)]),
    "fr_synthetic_task_create": (C.c_int, [P(SyntheticTaskConfigC), P(SideTaskVTableC), P(vp)]),
    "fr_harness_task_status": (C.c_int, [vp, C.c_char_p, P(i32), P(i32), P(dbl)]),
    "fr_harness_destroy": (C.c_int, [vp]),
    "fr_harness_set_harvest_fraction": (C.c_int, [vp, dbl]),
    "fr_harness_set_side_sms": (C.c_int, [vp, i32]),
    "fr_harness_set_dt_budget": (C.c_int, [vp, dbl]),
    "fr_harness_task_memory": (C.c_int, [vp, cp, P(dbl), P(dbl)]),
    "fr_harness_run_trace": (C.c_int, [vp, P(vp)]),
    "fr_harness_gate_log": (C.c_int, [vp, P(GateRecordC), i64, P(i64)]),
    "fr_harness_signal_log": (C.c_int, [vp, P(SignalRecordC), i64, P(i64)]),
    "fr_img_plan_set_max_sms": (C.c_int, [vp, i32]),
    "fr_sgd_problem_set_max_sms": (C.c_int, [vp, i32]),
    "fr_pr_state_set_max_sms": (C.c_int, [vp, i32]),
    "fr_l2_read_probe": (C.c_int, [vp, i64, i32, vp, vp]),
    "fr_harness_get_profile": (C.c_int, [vp, P(HarnessProfileC)]),
    "fr_harness_stage_bubbles": (C.c_int, [vp, P(BubbleC), i32, P(i32)]),
    "fr_harness_submit": (C.c_int, [vp, cp, P(SideTaskVTableC), vp, dbl, i32, P(TaskProfileC), P(i32)]),
    "fr_harness_run": (C.c_int, [vp, i32, i32, P(RunReportC)]),
    "fr_harness_reprofile": (C.c_int, [vp, cp, P(TaskProfileC)]),
    "fr_harness_stop_task": (C.c_int, [vp, cp]),
    "fr_harness_reprofile_bubbles": (C.c_int, [vp]),
    "fr_harness_timeline": (C.c_int, [vp, i32, P(dbl), i64, P(i64)]),
    "fr_harness_launches": (C.c_int, [vp, P(i64), P(i64)]),
    "fr_harness_mailbox": (C.c_int, [vp, P(vp), P(i64)]),
    "fr_harness_link": (C.c_int, [vp, vp, vp]),
    "fr_ipc_handle": (C.c_int, [vp, vp]),
    "fr_ipc_open": (C.c_int, [vp, P(vp)]),
    "fr_ipc_close": (C.c_int, [vp]),
})
