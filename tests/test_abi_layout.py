"""CPU-only: every ctypes mirror in paper_2409_06941_b200/_abi.py has the size
and field offsets of the C struct it stands for in include/*.h (compiled here
with gcc), so a header change cannot silently shift a field the Python side
writes (e.g. the configs that gained `layout` / `host_ring`)."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

from paper_2409_06941_b200 import _abi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MIRRORS = {
    "PipelineConfigC": "fr_pipeline_config", "Issue": "fr_issue", "OpEventC": "fr_op_event",
    "BubbleC": "fr_bubble", "SideTaskSpecC": "fr_side_task_spec", "TaskRuntimeC": "fr_task_runtime",
    "IterativeDecisionC": "fr_iterative_decision", "LimitConfigC": "fr_limit_config",
    "ProfileOptionsC": "fr_profile_options", "TaskProfileC": "fr_task_profile", "TaskViewC": "fr_task_view",
    "ManagerActionC": "fr_manager_action", "WorkerInfoC": "fr_worker_info", "PriceConfigC": "fr_price_config",
    "TaskWorkC": "fr_task_work", "CostBreakdownC": "fr_cost_breakdown", "StageBreakdownC": "fr_stage_breakdown",
    "TransitionRecordC": "fr_transition_record", "SideTaskVTableC": "fr_side_task_vtable",
    "SyntheticTaskConfigC": "fr_synthetic_task_config", "PreemptC": "fr_preempt",
    "ImageTaskConfigC": "fr_image_task_config", "PageRankTaskConfigC": "fr_pagerank_task_config",
    "SgdTaskConfigC": "fr_sgd_task_config", "HarnessConfigC": "fr_harness_config",
    "HarnessProfileC": "fr_harness_profile", "RunReportC": "fr_run_report",
    "GateRecordC": "fr_gate_record", "SignalRecordC": "fr_signal_record",
}


def _c_layouts():
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "freeride_gpu.h"', "int main(void) {"]
    for py, cname in MIRRORS.items():
        cls = getattr(A, py)
        lines.append(f'  printf("{py} size %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            cf = f[0].rstrip("_")
            lines.append(f'  printf("{py} {f[0]} %zu\\n", offsetof({cname}, {cf}));')
    lines.append("  return 0;\n}")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
        open(src, "w").write("\n".join(lines))
        r = subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = {}
    for line in out.splitlines():
        py, field, val = line.split()
        got[(py, field)] = int(val)
    return got


@pytest.fixture(scope="module")
def c_layouts():
    return _c_layouts()


@pytest.mark.parametrize("py", sorted(MIRRORS))
def test_ctypes_mirror_matches_header(c_layouts, py):
    cls = getattr(A, py)
    assert C.sizeof(cls) == c_layouts[(py, "size")], (py, C.sizeof(cls), c_layouts[(py, "size")])
    for f in cls._fields_:
        assert getattr(cls, f[0]).offset == c_layouts[(py, f[0])], (py, f[0])


def _gpu_lib():
    from paper_2409_06941_b200 import LIB_PATH
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in A.GPU_PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    lib.fr_last_error_field.restype = C.c_char_p
    return lib


def test_gpu_entry_points_validate_before_touching_cuda():
    """argument checks of the GPU rows run on the host and return the
    documented codes (and the offending field) on a machine with no GPU"""
    lib = _gpu_lib()
    out = C.c_void_p()
    assert lib.fr_sgd_step(None, 0, 1, 0.01, 0.05, None) == A.FR_ERR_ARGUMENT
    assert lib.fr_sgd_group_by_user(None, 1, None) == A.FR_ERR_ARGUMENT
    assert lib.fr_sgd_problem_generate(0, 10, 16, 1, 1, None, C.byref(out)) == A.FR_ERR_VALIDATION
    assert lib.fr_sgd_problem_generate(10, 10, 12, 1, 1, None, C.byref(out)) == A.FR_ERR_UNSUPPORTED
    assert lib.fr_sgd_problem_from_edges(0, 1, 16, None, None, None, 1, None, C.byref(out)) == A.FR_ERR_VALIDATION
    assert lib.fr_sgd_problem_from_edges(4, 1, 16, None, None, None, 1, None, C.byref(out)) == A.FR_ERR_ARGUMENT
    assert lib.fr_pr_graph_rmat(0, 16, 1, None, C.byref(out)) == A.FR_ERR_VALIDATION
    assert lib.fr_pr_graph_rmat(30, 4, 1, None, C.byref(out)) == A.FR_ERR_VALIDATION   # 2^32 edges
    assert lib.fr_pr_graph_from_edges(0, 0, None, None, None, C.byref(out)) == A.FR_ERR_VALIDATION
    assert lib.fr_pr_graph_from_edges(5, 3, None, None, None, C.byref(out)) == A.FR_ERR_ARGUMENT
    assert lib.fr_pr_step(None, 1, 0.85, None) == A.FR_ERR_ARGUMENT
    vt, user = A.SideTaskVTableC(), C.c_void_p()
    bad = A.ImageTaskConfigC(sw=3840, sh=2160, dw=1920, dh=1080, batch=10, images_per_step=3, host_io=0,
                             interface_kind=0, seed=1, total_steps=0, host_ring=0)
    assert lib.fr_image_task_create(C.byref(bad), C.byref(vt), C.byref(user)) == A.FR_ERR_VALIDATION
    assert lib.fr_last_error_field() == b"images_per_step"
    bad.images_per_step, bad.host_ring = 2, -1
    assert lib.fr_image_task_create(C.byref(bad), C.byref(vt), C.byref(user)) == A.FR_ERR_VALIDATION
    assert lib.fr_last_error_field() == b"host_ring"
    sgd = A.SgdTaskConfigC(V=100, k=16, E=1000, edge_seed=1, init_seed=1, edges_per_step=100, eta=0.01,
                           lambda_=0.05, total_steps=0, layout=7)
    assert lib.fr_sgd_task_create(C.byref(sgd), C.byref(vt), C.byref(user)) == A.FR_ERR_VALIDATION
    assert lib.fr_last_error_field() == b"layout"
