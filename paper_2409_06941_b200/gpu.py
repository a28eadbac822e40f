"""Python front end of include/freeride_gpu.h (side-task steps on sm_100a).

Device buffers are torch tensors (plumbing only); every computation runs in
the product library's kernels.  Calls are asynchronous on the given stream
(default: torch's current stream).  There is no CPU fallback: a missing
library or a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _abi as A
from . import lib as _load_lib

_glib = None


def glib() -> C.CDLL:
    global _glib
    if _glib is None:
        lib = _load_lib()
        A.bind(lib, A.HOST_PROTOTYPES)
        _glib = A.bind(lib, A.GPU_PROTOTYPES)
        if torch.cuda.is_available():  # start on torch's current device (this thread)
            A.raise_for(_glib, _glib.fr_set_device(torch.cuda.current_device()))
    return _glib


def set_device(device: int):
    """The library links its own CUDA runtime: select its device for the
    calling thread (glib() does it once for torch's current device)."""
    check(glib().fr_set_device(device))


def check(rc: int):
    A.raise_for(glib(), rc)


def _ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("side-task buffers must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("side-task buffers must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def l2_read_gbps(mbytes: int = 48, passes: int = 20) -> float:
    """Measured L2 read bandwidth (GB/s): an L2-resident buffer swept
    `passes` times (fr_l2_read_probe), CUDA events around the sweeps after a
    warm-up pass that brings the buffer into L2."""
    buf = torch.ones(mbytes << 18, dtype=torch.int32, device="cuda")
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    check(glib().fr_l2_read_probe(_ptr(buf), buf.numel() * 4, 1, _ptr(sink), s.cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        a.record(s)
        check(glib().fr_l2_read_probe(_ptr(buf), buf.numel() * 4, passes, _ptr(sink), s.cuda_stream))
        b.record(s)
        b.synchronize()
        best = max(best, buf.numel() * 4 * passes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def low_priority_stream(device=None) -> torch.cuda.Stream:
    """The stream class side-task steps run in (lowest CUDA priority)."""
    lo, _hi = torch.cuda.Stream.priority_range()
    return torch.cuda.Stream(device=device, priority=lo)


# ------------------------------------------------------------------ K5 image
class ImagePlan:
    """fr_img_plan: one (src -> dst) resize shape."""

    GENERAL, TMA_2X = 0, 1

    def __init__(self, sw: int, sh: int, dw: int, dh: int):
        self.sw, self.sh, self.dw, self.dh = sw, sh, dw, dh
        h = C.c_void_p()
        check(glib().fr_img_plan_create(sw, sh, dw, dh, C.byref(h)))
        self._h = h

    def set_overlap(self, on: bool = True):
        """consecutive exact-2x launches may overlap (fr_img_plan_set_overlap)"""
        check(glib().fr_img_plan_set_overlap(self._h, int(bool(on))))

    def set_max_sms(self, sms: int):
        """launches occupy at most `sms` SMs (0 = all; fr_img_plan_set_max_sms)"""
        check(glib().fr_img_plan_set_max_sms(self._h, int(sms)))

    @property
    def path(self) -> int:
        out = C.c_int32()
        check(glib().fr_img_plan_path(self._h, C.byref(out)))
        return out.value

    def run(self, src: torch.Tensor, dst: torch.Tensor, wm: torch.Tensor, stream=None):
        """dst[n,dh,dw,3] = blend(resize(src[n,sh,sw,3]), wm[dh,dw,4])."""
        n = src.shape[0]
        if tuple(src.shape[1:]) != (self.sh, self.sw, 3) or tuple(dst.shape) != (n, self.dh, self.dw, 3):
            raise ValueError("image shapes do not match the plan")
        if tuple(wm.shape) != (self.dh, self.dw, 4):
            raise ValueError("watermark must be [dh, dw, 4] RGBA")
        for t in (src, dst, wm):
            if t.dtype != torch.uint8:
                raise ValueError("images are uint8")
        check(glib().fr_img_resize_watermark(self._h, _ptr(src), _ptr(dst), _ptr(wm), n,
                                             _stream(stream)))
        return dst

    def prepare(self, wm: torch.Tensor, stream=None) -> torch.Tensor:
        """Prepared (premultiplied, plan-layout) copy of an RGBA watermark."""
        n = C.c_int64()
        check(glib().fr_img_prepared_bytes(self._h, C.byref(n)))
        out = torch.empty(n.value, dtype=torch.uint8, device=wm.device)
        check(glib().fr_img_prepare_watermark(self._h, _ptr(wm), _ptr(out), _stream(stream)))
        return out

    def run_prepared(self, src: torch.Tensor, dst: torch.Tensor, prepared: torch.Tensor, stream=None):
        n = src.shape[0]
        if tuple(src.shape[1:]) != (self.sh, self.sw, 3) or tuple(dst.shape) != (n, self.dh, self.dw, 3):
            raise ValueError("image shapes do not match the plan")
        check(glib().fr_img_resize_watermark_prepared(self._h, _ptr(src), _ptr(dst), _ptr(prepared), n,
                                                      _stream(stream)))
        return dst

    def run_preemptible(self, src, dst, prepared, counters, stop_word=None, token=0, max_rows=None,
                        stream=None):
        """Preemptible K5 (imperative interface): takes up to max_rows rows
        (default: one pass) in units of preemptible_unit_rows(n) rows,
        starting at unit counters[0] (mod n*dh / unit), stops taking units
        once stop_word[0] >= token; counters is a zeroed int32 tensor of 8
        (counters[2:4] = rows completed, uint64)."""
        n = src.shape[0]
        if tuple(src.shape[1:]) != (self.sh, self.sw, 3) or tuple(dst.shape) != (n, self.dh, self.dw, 3):
            raise ValueError("image shapes do not match the plan")
        pre = None
        if stop_word is not None:
            pre = A.PreemptC(stop_word=stop_word.data_ptr(), token=token)
        if max_rows is None:
            max_rows = n * self.dh
        check(glib().fr_img_resize_watermark_preemptible(
            self._h, _ptr(src), _ptr(dst), _ptr(prepared), n, _ptr(counters), max_rows,
            C.byref(pre) if pre is not None else None, _stream(stream)))
        return dst

    def preemptible_unit_rows(self, n: int) -> int:
        """rows per claimed unit of a preemptible launch over n frames"""
        out = C.c_int32()
        check(glib().fr_img_preemptible_unit_rows(self._h, n, C.byref(out)))
        return out.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _glib is not None:
            _glib.fr_img_plan_destroy(h)
            self._h = None


def img_generate(n, w, h, channels=3, seed=1, first_index=0, device="cuda", stream=None):
    out = torch.empty((n, h, w, channels), dtype=torch.uint8, device=device)
    check(glib().fr_img_generate(_ptr(out), n, w, h, channels, seed, first_index, _stream(stream)))
    return out


class ImageTask:
    """Built-in image side task (fr_image_task_create) -- a vtable + handle
    whose ownership passes to the Harness on submit."""

    def __init__(self, sw=3840, sh=2160, dw=1920, dh=1080, batch=64, images_per_step=8,
                 host_io=False, seed=1, total_steps=0, imperative=False, host_ring=0):
        """host_ring (host_io only): device staging slots in steps; the copy
        engines prefetch that many steps ahead, also while the pipeline computes"""
        self.cfg = A.ImageTaskConfigC(sw=sw, sh=sh, dw=dw, dh=dh, batch=batch,
                                      images_per_step=images_per_step, host_io=int(host_io),
                                      interface_kind=int(bool(imperative)), seed=seed,
                                      total_steps=total_steps, host_ring=host_ring)
        self.imperative = bool(imperative)
        self.batch, self.dw, self.dh = batch, dw, dh
        self.vt = A.SideTaskVTableC()
        self.user = C.c_void_p()
        check(glib().fr_image_task_create(C.byref(self.cfg), C.byref(self.vt), C.byref(self.user)))
        gib = C.c_double()
        check(glib().fr_image_task_memory(C.byref(self.cfg), C.byref(gib)))
        self.memory_gib = gib.value
        self.units_per_step = self.vt.work_units_per_step
        # per-step algorithmic HBM bytes (src + dst per image; the watermark
        # is read once per step and stays L2-resident across its images)
        # frames in + frames out + the prepared watermark once (L2-resident: 10 B/px
        # on the exact-2x path, read by every launch; the raw RGBA 4 B/px otherwise)
        exact2x = sw == 2 * dw and sh == 2 * dh and dw % 16 == 0
        self.bytes_per_step = images_per_step * (sw * sh * 3 + dw * dh * 3) + dw * dh * (10 if exact2x else 4)
        self.h2d_per_step = images_per_step * sw * sh * 3 if host_io else 0
        self.d2h_per_step = images_per_step * dw * dh * 3 if host_io else 0

    def host_outputs(self):
        """host_io tasks: copy of the pinned host output batch (numpy)."""
        import numpy as np
        p = C.c_void_p()
        check(glib().fr_image_task_host_output(self.user, C.byref(p)))
        if not p.value:
            return None
        torch.cuda.synchronize()
        n = self.batch * self.dh * self.dw * 3
        return np.ctypeslib.as_array((C.c_uint8 * n).from_address(p.value)).copy().reshape(
            self.batch, self.dh, self.dw, 3)

    def outputs(self):
        """Copy of the task's resident output batch [batch, dh, dw, 3] (None
        when the task holds no GPU state)."""
        src, dst, wm, steps = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
        check(glib().fr_image_task_buffers(self.user, C.byref(src), C.byref(dst), C.byref(wm),
                                           C.byref(steps)))
        if not dst.value:
            return None
        torch.cuda.synchronize()
        return _dev_copy(dst.value, self.batch * self.dh * self.dw * 3, torch.uint8).view(
            self.batch, self.dh, self.dw, 3)


def _dev_copy(ptr: int, n: int, dtype) -> torch.Tensor:
    """Copy n elements from a raw device pointer owned by the library."""
    out = torch.empty(n, dtype=dtype, device="cuda")
    if n:
        check(glib().fr_memcpy(out.data_ptr(), ptr, n * out.element_size()))
    return out


class SyntheticTask:
    """The reference's synthetic SideTaskSpec made real (fr_synthetic_task_create):
    steps are spin kernels on every SM, Init allocates memory_demand_gib,
    leak_gib_per_step reproduces MemoryLeak, step_ns >> profile_step_ns a task
    that overruns its bubbles (Fig. 9 scenarios)."""

    def __init__(self, step_ns=200_000, profile_step_ns=0, memory_demand_gib=0.25,
                 leak_gib_per_step=0.0, total_steps=0, cooperative=True, init_ns=0):
        self.cfg = A.SyntheticTaskConfigC(step_ns=step_ns, profile_step_ns=profile_step_ns,
                                          memory_demand_gib=memory_demand_gib,
                                          leak_gib_per_step=leak_gib_per_step,
                                          total_steps=total_steps, cooperative=int(cooperative),
                                          init_ns=init_ns)
        self.vt = A.SideTaskVTableC()
        self.user = C.c_void_p()
        check(glib().fr_synthetic_task_create(C.byref(self.cfg), C.byref(self.vt), C.byref(self.user)))
        self.memory_gib = memory_demand_gib
        self.units_per_step = 1.0
        self.bytes_per_step = 0
        self.h2d_per_step = self.d2h_per_step = 0


class PageRankGraph:
    """fr_pr_graph: an incoming CSR on the device -- RMAT-generated, or the
    caller's edge list via PageRankGraph.from_edges."""

    def __init__(self, scale=20, edge_factor=16, seed=1, stream=None, _handle=None):
        h = _handle
        if h is None:
            h = C.c_void_p()
            check(glib().fr_pr_graph_rmat(scale, edge_factor, seed, _stream(stream), C.byref(h)))
        self._h = h
        V, E, nb = C.c_int32(), C.c_int64(), C.c_int32()
        check(glib().fr_pr_graph_info(h, C.byref(V), C.byref(E), C.byref(nb)))
        self.V, self.E, self.n_blocks = V.value, E.value, nb.value

    @classmethod
    def from_edges(cls, V: int, src, dst, stream=None) -> "PageRankGraph":
        """edges src[e] -> dst[e] (int32 torch tensors, copied to the device if needed)"""
        glib()
        s = torch.as_tensor(src, dtype=torch.int32).cuda().contiguous()
        d = torch.as_tensor(dst, dtype=torch.int32).cuda().contiguous()
        if s.numel() != d.numel():
            raise ValueError("src and dst must have the same length")
        torch.cuda.synchronize()
        h = C.c_void_p()
        check(glib().fr_pr_graph_from_edges(V, s.numel(), s.data_ptr() if s.numel() else None,
                                            d.data_ptr() if d.numel() else None, _stream(stream), C.byref(h)))
        return cls(_handle=h)

    def csr(self):
        o, c, d = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(glib().fr_pr_graph_csr(self._h, C.byref(o), C.byref(c), C.byref(d)))
        torch.cuda.synchronize()
        return (_dev_copy(o.value, self.V + 1, torch.int32), _dev_copy(c.value, self.E, torch.int32),
                _dev_copy(d.value, self.V, torch.int32))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _glib is not None:
            _glib.fr_pr_graph_destroy(h)
            self._h = None


class PageRankState:
    def __init__(self, graph: PageRankGraph):
        self.graph = graph
        h = C.c_void_p()
        check(glib().fr_pr_state_create(graph._h, C.byref(h)))
        self._h = h

    def set_max_sms(self, sms: int):
        """iterations occupy at most `sms` SMs (0 = all; fr_pr_state_set_max_sms)"""
        check(glib().fr_pr_state_set_max_sms(self._h, int(sms)))

    def reset(self, stream=None):
        check(glib().fr_pr_reset(self._h, _stream(stream)))

    def step(self, iters=1, damping=0.85, stream=None):
        check(glib().fr_pr_step(self._h, iters, damping, _stream(stream)))

    def ranks(self) -> torch.Tensor:
        p, it = C.c_void_p(), C.c_int64()
        check(glib().fr_pr_ranks(self._h, C.byref(p), C.byref(it)))
        torch.cuda.synchronize()
        return _dev_copy(p.value, self.graph.V, torch.float32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _glib is not None:
            _glib.fr_pr_state_destroy(h)
            self._h = None


class PageRankTask:
    """Built-in PageRank side task (fr_pagerank_task_create); graph= runs it
    over the caller's PageRankGraph (fr_pagerank_task_create_from_graph)."""

    def __init__(self, scale=20, edge_factor=16, seed=1, iters_per_step=1, damping=0.85,
                 total_steps=0, graph: "PageRankGraph | None" = None):
        self.cfg = A.PageRankTaskConfigC(scale=scale, edge_factor=edge_factor, seed=seed,
                                         iters_per_step=iters_per_step, damping=damping,
                                         total_steps=total_steps)
        self.vt = A.SideTaskVTableC()
        self.user = C.c_void_p()
        if graph is None:
            check(glib().fr_pagerank_task_create(C.byref(self.cfg), C.byref(self.vt), C.byref(self.user)))
        else:
            check(glib().fr_pagerank_task_create_from_graph(C.byref(self.cfg), graph._h, C.byref(self.vt),
                                                            C.byref(self.user)))
        V, E, gib = C.c_int32(), C.c_int64(), C.c_double()
        check(glib().fr_pagerank_task_info(self.user, C.byref(V), C.byref(E), C.byref(gib), None, None))
        self.V, self.E, self.memory_gib = V.value, E.value, gib.value
        self.units_per_step = self.vt.work_units_per_step
        # compulsory bytes per pull iteration: offsets + col_idx + c gather
        # source (read once) + inv_outdeg + r' and c' writes
        # offsets, a column id and a source value per edge, r/c reads
        # and writes -- the standard pull-SpMV byte count
        self.bytes_per_step = iters_per_step * (4 * (self.V + 1) + 8 * self.E + 16 * self.V)
        self.h2d_per_step = self.d2h_per_step = 0

    def ranks(self):
        p, it = C.c_void_p(), C.c_int64()
        check(glib().fr_pagerank_task_info(self.user, None, None, None, C.byref(p), C.byref(it)))
        if not p.value:
            return None, it.value
        torch.cuda.synchronize()
        return _dev_copy(p.value, self.V, torch.float32), it.value


class SgdProblem:
    """fr_sgd_problem: rating graph + fp32 latent matrix on the device."""

    def __init__(self, V=3072441, E=117185083, k=16, edge_seed=2, init_seed=3, stream=None,
                 handle=None, by_user=False, window=1 << 21):
        """by_user: lay the edges out by user (fr_sgd_group_by_user, rounds of
        `window` edges) -> the user-grouped step kernel."""
        self._owned = handle is None
        if handle is None:
            handle = C.c_void_p()
            check(glib().fr_sgd_problem_generate(V, E, k, edge_seed, init_seed, _stream(stream),
                                                 C.byref(handle)))
            if by_user:
                check(glib().fr_sgd_group_by_user(handle, window, _stream(stream)))
        self._h = handle
        u, v, r, L = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        Vc, Ec, kc = C.c_int32(), C.c_int64(), C.c_int32()
        check(glib().fr_sgd_buffers(self._h, C.byref(u), C.byref(v), C.byref(r), C.byref(L),
                                    C.byref(Vc), C.byref(Ec), C.byref(kc)))
        self.V, self.E, self.k = Vc.value, Ec.value, kc.value
        self._ptr = dict(u=u.value, v=v.value, r=r.value, L=L.value)

    @classmethod
    def from_edges(cls, V, u, v, r, k=16, init_seed=3, by_user=False, window=1 << 21, stream=None):
        """the caller's ratings (u, v, r); by_user re-lays them out like the task"""
        glib()
        tu = torch.as_tensor(u, dtype=torch.int32).cuda().contiguous()
        tv = torch.as_tensor(v, dtype=torch.int32).cuda().contiguous()
        tr = torch.as_tensor(r, dtype=torch.float32).cuda().contiguous()
        if not (tu.numel() == tv.numel() == tr.numel()):
            raise ValueError("u, v, r must have the same length")
        torch.cuda.synchronize()
        h = C.c_void_p()
        n = tu.numel()
        check(glib().fr_sgd_problem_from_edges(V, n, k, tu.data_ptr() if n else None, tv.data_ptr() if n else None,
                                               tr.data_ptr() if n else None, init_seed, _stream(stream),
                                               C.byref(h)))
        if by_user:
            check(glib().fr_sgd_group_by_user(h, window, _stream(stream)))
        p = cls(handle=h)
        p._owned = True
        return p

    def reinit(self, seed=3, stream=None):
        check(glib().fr_sgd_reinit(self._h, seed, _stream(stream)))

    def set_max_sms(self, sms: int):
        """steps occupy at most `sms` SMs (0 = all; fr_sgd_problem_set_max_sms)"""
        check(glib().fr_sgd_problem_set_max_sms(self._h, int(sms)))

    def set_overlap(self, on: bool = True):
        """consecutive user-grouped steps on one stream may overlap
        (fr_sgd_problem_set_overlap; the built-in task's setting)"""
        check(glib().fr_sgd_problem_set_overlap(self._h, int(bool(on))))

    def step(self, e_begin, e_end, eta=0.01, lam=0.05, stream=None):
        check(glib().fr_sgd_step(self._h, e_begin, e_end, eta, lam, _stream(stream)))

    def epoch(self, eta=0.01, lam=0.05, stream=None):
        self.step(0, self.E, eta, lam, stream)

    def rmse(self, stream=None) -> float:
        out = C.c_double()
        check(glib().fr_sgd_rmse(self._h, _stream(stream), C.byref(out)))
        return out.value

    def edges(self):
        torch.cuda.synchronize()
        return (_dev_copy(self._ptr["u"], self.E, torch.int32), _dev_copy(self._ptr["v"], self.E, torch.int32),
                _dev_copy(self._ptr["r"], self.E, torch.float32))

    def latent(self):
        torch.cuda.synchronize()
        return _dev_copy(self._ptr["L"], self.V * self.k, torch.float32).view(self.V, self.k)

    def __del__(self):
        h = getattr(self, "_h", None)
        if self._owned and h is not None and h.value and _glib is not None:
            _glib.fr_sgd_problem_destroy(h)
            self._h = None


class SgdTask:
    """Built-in Graph-SGD side task (fr_sgd_task_create)."""

    def __init__(self, V=3072441, E=117185083, k=16, edge_seed=2, init_seed=3,
                 edges_per_step=1 << 21, eta=0.01, lam=0.05, total_steps=0, by_user=True,
                 problem: "SgdProblem | None" = None, total_epochs=0):
        """problem=: harvest over the caller's ratings (SgdProblem.from_edges); the
        task takes the problem over (fr_sgd_task_create_from_problem)"""
        if problem is not None:
            V, E, k = problem.V, problem.E, problem.k
        self.cfg = A.SgdTaskConfigC(V=V, k=k, E=E, edge_seed=edge_seed, init_seed=init_seed,
                                    edges_per_step=edges_per_step, eta=eta, lambda_=lam,
                                    total_steps=total_steps,
                                    layout=A.SGD_LAYOUT_BY_USER if by_user else A.SGD_LAYOUT_COO,
                                    total_epochs=total_epochs)
        self.vt = A.SideTaskVTableC()
        self.user = C.c_void_p()
        if problem is None:
            check(glib().fr_sgd_task_create(C.byref(self.cfg), C.byref(self.vt), C.byref(self.user)))
        else:
            if not problem._owned:
                raise ValueError("the problem already belongs to a task")
            check(glib().fr_sgd_task_create_from_problem(C.byref(self.cfg), problem._h, C.byref(self.vt),
                                                         C.byref(self.user)))
            problem._owned = False   # freed with the task now
        self.memory_gib = (E * 12 + V * k * 4) / 2 ** 30
        self.units_per_step = self.vt.work_units_per_step
        # algorithmic bytes: 12 B of edge + L_u and L_v read + written (268 B/edge at
        # k = 16); by user, L_v per edge (12 + 8k) and L_u once per held block
        # (a run of equal u, re-read every SGD_REFRESH = 16 edges): + 8k each
        self.by_user = by_user and k >= 16
        self.u_loads_per_edge = self._u_loads_per_edge() if self.by_user else 1.0
        self.bytes_per_step = edges_per_step * (12 + 8 * k + 8 * k * self.u_loads_per_edge)
        self.h2d_per_step = self.d2h_per_step = 0

    def problem(self):
        p, ep = C.c_void_p(), C.c_int64()
        check(glib().fr_sgd_task_problem(self.user, C.byref(p), C.byref(ep)))
        return SgdProblem(handle=p), ep.value

    REFRESH = 16   # sgd.cu SGD_REFRESH

    def _u_loads_per_edge(self) -> float:
        """L_u row loads per edge of the by-user kernel: one per run of equal u
        and one every REFRESH edges within it (segment cuts ignored: ~1 %)."""
        u = self.problem()[0].edges()[0]
        n = u.numel()
        if n == 0:
            return 0.0
        start = torch.ones(n, dtype=torch.bool, device=u.device)
        start[1:] = u[1:] != u[:-1]
        idx = torch.arange(n, device=u.device, dtype=torch.int64)
        run_start = torch.cummax(torch.where(start, idx, torch.zeros_like(idx)), 0).values
        loads = int((((idx - run_start) % self.REFRESH) == 0).sum())
        return loads / n


class PythonTask:
    """A side task written in Python (the paper's Python interface,
    PAPER.md:484-499): override the transition hooks; `run_next_step`
    must enqueue one bounded step on the given (low-priority) stream and
    return.  Hooks run on the harness worker thread (they take the GIL, so
    keep them short)."""

    work_units_per_step = 0.0
    memory_gib = 0.0
    carveout_hint = -1  # L1/shared split the task's kernels want (-1: none, 0: max L1)

    def create(self): pass
    def init(self, stream: int): pass
    def start(self): pass
    def run_next_step(self, stream: int): raise NotImplementedError
    def pause(self): pass
    def stop(self): pass
    def finished(self, steps_completed: int) -> bool: return False

    def __init__(self):
        def wrap(fn):
            def cb(*args):
                try:
                    fn(*args)
                    return A.FR_OK
                except Exception as e:  # noqa: BLE001 -- surfaced as a status
                    self.error = e
                    return A.FR_ERR_INVARIANT
            return cb

        def fin(user, steps, out):
            try:
                out[0] = int(bool(self.finished(steps)))
                return A.FR_OK
            except Exception as e:  # noqa: BLE001
                self.error = e
                return A.FR_ERR_INVARIANT

        f = A.SideTaskVTableC._fields_
        ty = dict(f)
        self._cbs = [
            ty["create"](wrap(lambda u: self.create())),
            ty["init"](wrap(lambda u, s: self.init(s))),
            ty["start"](wrap(lambda u: self.start())),
            ty["run_next_step"](wrap(lambda u, s: self.run_next_step(s))),
            ty["pause"](wrap(lambda u: self.pause())),
            ty["stop"](wrap(lambda u: self.stop())),
            ty["finished"](fin),
            ty["destroy"](lambda u: None),
        ]
        self.vt = A.SideTaskVTableC(*self._cbs, float(self.work_units_per_step))
        self.vt.carveout_hint = int(self.carveout_hint)
        self.user = C.c_void_p(0)
        self.units_per_step = float(self.work_units_per_step)
        self.error = None


class Harness:
    """fr_harness: one GPU replaying stage `stage` of a p-stage 1F1B pipeline
    of bf16 GEMM stand-ins, with a side-task worker harvesting its bubbles."""

    def __init__(self, num_stages=4, num_micro_batches=4, stage=0, layers=6, hidden=2048,
                 tokens=8192, ffn_mult=4, profile_reps=5, max_inflight_steps=2, gate_estimate=0,
                 gpu_memory_total=178.0, weight_mem=-1.0, activation_mem=-1.0,
                 fp_ticks=0, bp_ticks=0, profile_epochs=3, transport="replica",
                 memory_headroom_gib=0.0, grace_ns=0, step_group=1, harvest_fraction=1.0,
                 reclamation_delay_ns=0, side_sms=0, dt_budget=0.0, min_side_sms=0):
        """transport="replica": this GPU replays stage `stage` against the
        device clock (one GPU); "linked": a real pipeline stage whose
        neighbours are linked through mailboxes (see link())."""
        tp = {"replica": 0, "linked": 1}[transport]
        self.cfg = A.HarnessConfigC(
            num_stages=num_stages, num_micro_batches=num_micro_batches, stage=stage, layers=layers,
            hidden=hidden, tokens=tokens, ffn_mult=ffn_mult, profile_reps=profile_reps,
            max_inflight_steps=max_inflight_steps, gate_estimate=gate_estimate,
            gpu_memory_total=gpu_memory_total, weight_mem=weight_mem,
            activation_mem=activation_mem, fp_ticks_override=fp_ticks, bp_ticks_override=bp_ticks,
            profile_epochs=profile_epochs if tp == 0 else 0, transport=tp,
            memory_headroom_gib=memory_headroom_gib, grace_ns=grace_ns, step_group=step_group,
            harvest_fraction=harvest_fraction, reclamation_delay_ns=reclamation_delay_ns,
            side_sms=side_sms, dt_budget=dt_budget, min_side_sms=min_side_sms)
        h = C.c_void_p()
        check(glib().fr_harness_create(C.byref(self.cfg), C.byref(h)))
        self._h = h
        self._tasks = []

    def profile(self) -> dict:
        p = A.HarnessProfileC()
        check(glib().fr_harness_get_profile(self._h, C.byref(p)))
        return p.as_dict()

    def mailbox(self) -> int:
        """Device pointer of this stage's mailbox (transport="linked")."""
        p, n = C.c_void_p(), C.c_int64()
        check(glib().fr_harness_mailbox(self._h, C.byref(p), C.byref(n)))
        self.mailbox_bytes = n.value
        return p.value

    def link(self, prev_mailbox=None, next_mailbox=None):
        """Neighbours' mailbox pointers valid in this process (same process,
        or opened with ipc_open); None at the pipeline's ends."""
        check(glib().fr_harness_link(self._h, prev_mailbox, next_mailbox))

    DISPOSITIONS = ("rejected", "completed", "killed_oom", "killed_pause_timeout",
                    "killed_init_timeout", "active")
    STATES = ("submitted", "created", "paused", "running", "stopped")

    def task_status(self, task_id: str) -> dict:
        st, disp, gib = C.c_int32(), C.c_int32(), C.c_double()
        check(glib().fr_harness_task_status(self._h, task_id.encode(), C.byref(st), C.byref(disp),
                                            C.byref(gib)))
        return {"state": self.STATES[st.value], "disposition": self.DISPOSITIONS[disp.value],
                "memory_used_gib": gib.value}

    def stage_bubbles(self):
        out = (A.BubbleC * 1024)()
        n = C.c_int32()
        check(glib().fr_harness_stage_bubbles(self._h, out, 1024, C.byref(n)))
        return [out[i].as_dict() for i in range(n.value)]

    def submit(self, task_id: str, task, profile_steps=32):
        prof = A.TaskProfileC()
        assigned = C.c_int32()
        check(glib().fr_harness_submit(self._h, task_id.encode(), C.byref(task.vt), task.user,
                                       task.memory_gib, profile_steps, C.byref(prof),
                                       C.byref(assigned)))
        self._tasks.append(task)  # keep the ctypes vtable alive
        return bool(assigned.value), prof.as_dict()

    def reprofile(self, task_id: str) -> dict:
        """Re-estimate a task's per-step duration from its steps in the last run."""
        prof = A.TaskProfileC()
        check(glib().fr_harness_reprofile(self._h, task_id.encode(), C.byref(prof)))
        return prof.as_dict()

    def reprofile_bubbles(self):
        """Bubble durations := medians of the last run's measured bubbles."""
        check(glib().fr_harness_reprofile_bubbles(self._h))

    def set_harvest_fraction(self, fraction: float):
        """the gate sees only the first `fraction` of every bubble (1 = all)"""
        check(glib().fr_harness_set_harvest_fraction(self._h, float(fraction)))

    def stop_task(self, task_id: str):
        check(glib().fr_harness_stop_task(self._h, task_id.encode()))

    def run(self, epochs: int, with_tasks: bool = True) -> dict:
        r = A.RunReportC()
        check(glib().fr_harness_run(self._h, epochs, int(with_tasks), C.byref(r)))
        d = r.as_dict()
        d["breakdown"] = r.breakdown.as_dict()
        return d

    def set_side_sms(self, sms: int):
        """SM budget of the side tasks' kernels (0 = all); re-profile after a run"""
        check(glib().fr_harness_set_side_sms(self._h, int(sms)))

    def set_dt_budget(self, budget: float):
        """ΔT-budgeted harvesting for the next runs (0 = off): the worker sizes
        the side tasks' SM budget so the stage's ops run <= budget slower"""
        check(glib().fr_harness_set_dt_budget(self._h, float(budget)))

    def task_memory(self, task_id: str) -> dict:
        used, reserved = C.c_double(), C.c_double()
        check(glib().fr_harness_task_memory(self._h, task_id.encode(), C.byref(used), C.byref(reserved)))
        return {"used_gib": used.value, "reserved_gib": reserved.value}

    def run_trace(self, check_trace: bool = True, trace_path=None) -> dict:
        """The last run with tasks as a RunTrace (fr_harness_run_trace): the
        simulated engine's dict layout, plus "violations" (fr_run_trace_check)"""
        from . import api
        h = C.c_void_p()
        check(glib().fr_harness_run_trace(self._h, C.byref(h)))
        return api().trace_dict(h, check_trace, trace_path)

    def gate_log(self):
        n = C.c_int64()
        glib().fr_harness_gate_log(self._h, None, 0, C.byref(n))
        buf = (A.GateRecordC * max(1, n.value))()
        check(glib().fr_harness_gate_log(self._h, buf, n.value, C.byref(n)))
        return [buf[i].as_dict() for i in range(n.value)]

    def signal_log(self):
        n = C.c_int64()
        glib().fr_harness_signal_log(self._h, None, 0, C.byref(n))
        buf = (A.SignalRecordC * max(1, n.value))()
        check(glib().fr_harness_signal_log(self._h, buf, n.value, C.byref(n)))
        out = []
        for i in range(n.value):
            d = buf[i].as_dict()
            d["actions"] = [buf[i].actions[k] for k in range(buf[i].n_actions)]
            out.append(d)
        return out

    def timeline(self, which: int):
        n = C.c_int64()
        cap = 1 << 20
        buf = (C.c_double * (2 * cap))()
        check(glib().fr_harness_timeline(self._h, which, buf, cap, C.byref(n)))
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]

    def launches(self):
        a, b = C.c_int64(), C.c_int64()
        check(glib().fr_harness_launches(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            glib().fr_harness_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def ipc_handle(dev_ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (e.g. a mailbox)."""
    buf = C.create_string_buffer(64)
    check(glib().fr_ipc_handle(dev_ptr, buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    check(glib().fr_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)))
    return p.value


def ipc_close(dev_ptr: int):
    check(glib().fr_ipc_close(dev_ptr))


def img_generate_watermark(w, h, seed=7, device="cuda", stream=None):
    out = torch.empty((h, w, 4), dtype=torch.uint8, device=device)
    check(glib().fr_img_generate_watermark(_ptr(out), w, h, seed, _stream(stream)))
    return out
