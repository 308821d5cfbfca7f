"""Python binding of libms2g.so (include/ms2g.h): argument marshalling only.

Every step of the PnP-MS2G hot path runs in the hand-written sm_100a kernels of
libms2g; PyTorch supplies device memory, the current stream and (for the
multi-GPU view sharding) the process group used to broadcast the NCCL id or
gather the NVLink peer handles (NEXT-3).
There is no CPU fallback: without the built library or a CUDA device every
call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import torch

__all__ = [
    "MS2GError", "DivergedError", "Plan", "plan_geometry", "forward_project", "back_project", "sketch_down",
    "sketch_up", "sketched_grad", "power_iteration", "denoise", "schedule", "schedule_views", "pnp_ms2g_solve",
    "pnp_ms2g_solve_async", "solve_status", "attach_nccl", "attach_peers", "view_shard", "set_kernel_timing",
    "kernel_time", "launch_count", "lib_path", "load", "register_subset", "release_subset", "RegisteredSubset",
    "attach_multicast",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libms2g.so")

MS2G_OK, MS2G_ERR_CONFIG, MS2G_ERR_DIVERGED, MS2G_ERR_CUDA, MS2G_ERR_NCCL, MS2G_ERR_INPUT = 0, 2, 3, 5, 6, 7


class MS2GError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libms2g error {code}: {msg}")
        self.code = code


class DivergedError(MS2GError):
    pass


class GeomDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("fov", C.c_double), ("n_views", C.c_int32), ("arc_rad", C.c_double),
                ("n_bins", C.c_int32), ("sod", C.c_double), ("sdd", C.c_double), ("bin_pitch", C.c_double),
                ("view_begin", C.c_int32), ("view_end", C.c_int32), ("batch", C.c_int32)]


class Denoiser(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sigma", C.c_float), ("lambda_", C.c_float), ("tau", C.c_float),
                ("inner_iters", C.c_int32)]


class Stage(C.Structure):
    _fields_ = [("factor", C.c_int32), ("n_iters", C.c_int32), ("n_epochs", C.c_int32)]


class SolveDesc(C.Structure):
    _fields_ = [("stages", C.POINTER(Stage)), ("n_stages", C.c_int32), ("option", C.c_int32),
                ("n_subsets", C.c_int32), ("seed", C.c_uint64), ("den", Denoiser), ("alpha", C.c_float),
                ("power_iters", C.c_int32), ("check_every", C.c_int32), ("resampler", C.c_int32)]


class SchedEntry(C.Structure):
    _fields_ = [("i", C.c_int32), ("stage", C.c_int32), ("factor", C.c_int32), ("subset", C.c_int32),
                ("eta", C.c_double), ("a", C.c_double)]

    def as_tuple(self):
        return (self.i, self.stage, self.factor, self.subset, self.eta, self.a)


_lib = None


def lib_path() -> str:
    return _LIBPATH


def load():
    """Load libms2g.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIBPATH):
        raise RuntimeError(f"{_LIBPATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(_LIBPATH)
    p, i, f, d = C.c_void_p, C.c_int32, C.c_float, C.c_double
    L.ms2g_plan_geometry.argtypes = [C.POINTER(GeomDesc), C.POINTER(C.c_int32), i, C.POINTER(p)]
    L.ms2g_plan_destroy.argtypes = [p]
    L.ms2g_plan_destroy.restype = None
    L.ms2g_nccl_unique_id.argtypes = [p]
    L.ms2g_attach_nccl.argtypes = [p, p, i, i]
    L.ms2g_set_kernel_timing.argtypes = [p, i]
    L.ms2g_kernel_time.argtypes = [p, i, i, C.POINTER(d), C.POINTER(i)]
    L.ms2g_peer_export.argtypes = [p, p]
    L.ms2g_attach_peers.argtypes = [p, p, i, i]
    L.ms2g_forward_project.argtypes = [p, i, p, p, p, C.POINTER(C.c_int32), i, p]
    L.ms2g_back_project.argtypes = [p, i, p, p, f, i, C.POINTER(C.c_int32), i, i, p]
    L.ms2g_sketch_down.argtypes = [p, i, i, p, p, p]
    L.ms2g_sketch_up.argtypes = [p, i, i, p, p, f, p, p]
    L.ms2g_sketched_grad.argtypes = [p, i, i, p, p, p, C.POINTER(C.c_int32), i, p]
    L.ms2g_power_iteration.argtypes = [p, i, i, C.POINTER(d), p]
    L.ms2g_denoise.argtypes = [p, C.POINTER(Denoiser), p, p, p]
    L.ms2g_schedule.argtypes = [p, C.POINTER(SolveDesc), C.POINTER(SchedEntry), i, C.POINTER(C.c_int32)]
    L.ms2g_pnp_ms2g_solve.argtypes = [p, C.POINTER(SolveDesc), p, p, p, C.POINTER(SchedEntry), p]
    L.ms2g_schedule_views.argtypes = [p, C.POINTER(SolveDesc), i, C.POINTER(C.c_int32), i, C.POINTER(C.c_int32)]
    L.ms2g_pnp_ms2g_solve_async.argtypes = [p, C.POINTER(SolveDesc), p, p, p, p]
    L.ms2g_solve_status.argtypes = [p, p]
    L.ms2g_last_error.restype = C.c_char_p
    L.ms2g_launch_count.restype = C.c_uint64
    L.ms2g_plan_info.argtypes = [p, i, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i)]
    L.ms2g_mc_create.argtypes = [p, i, p]
    L.ms2g_attach_multicast.argtypes = [p, p, i, i, i]
    L.ms2g_register_subset.argtypes = [p, C.POINTER(C.c_int32), i, C.POINTER(i)]
    L.ms2g_release_subset.argtypes = [p, i]
    L.ms2g_forward_project_registered.argtypes = [p, i, p, p, p, i, p]
    L.ms2g_back_project_registered.argtypes = [p, i, p, p, f, i, i, i, p]
    L.ms2g_sketched_grad_registered.argtypes = [p, i, i, p, p, p, i, p]
    _lib = L
    return L


def _check(rc: int):
    if rc != MS2G_OK:
        msg = load().ms2g_last_error().decode(errors="replace")
        if rc == MS2G_ERR_DIVERGED:
            raise DivergedError(rc, msg)
        raise MS2GError(rc, msg)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor | None, name: str):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise MS2GError(MS2G_ERR_INPUT, f"{name} must be a contiguous float32 CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _subset(subset):
    if subset is None:
        return None, 0
    vals = [int(v) for v in (subset.tolist() if hasattr(subset, "tolist") else subset)]
    arr = (C.c_int32 * max(1, len(vals)))(*vals)
    return arr, len(vals)


class Plan:
    """Owns an ms2g_plan (device geometry tables + workspaces)."""

    def __init__(self, handle, n, n_views, n_bins, factors, view_begin, view_end, batch, device):
        self._h = handle
        self.n, self.n_views, self.n_bins = n, n_views, n_bins
        self.factors = tuple(factors)
        self.view_begin, self.view_end, self.batch = view_begin, view_end, batch
        self.device = device
        self.rank, self.nranks = 0, 1

    @property
    def handle(self):
        if self._h is None:
            raise MS2GError(MS2G_ERR_INPUT, "plan was destroyed")
        return self._h

    @property
    def n_local_views(self):
        return self.view_end - self.view_begin

    def nc(self, factor: int) -> int:
        return self.n // factor

    def destroy(self):
        if self._h is not None:
            load().ms2g_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()


def plan_geometry(n, n_views, n_bins, factors=(1,), fov=2.0, arc=2 * math.pi, sod=None, sdd=None,
                  bin_pitch=0.0, view_begin=0, view_end=None, batch=1) -> Plan:
    """ms2g_plan_geometry: fan-beam geometry O1 with per-factor tables."""
    if not torch.cuda.is_available():
        raise MS2GError(MS2G_ERR_CUDA, "no CUDA device: libms2g has no CPU path")
    L = load()
    sod = 2.0 * fov if sod is None else sod
    sdd = 4.0 * fov if sdd is None else sdd
    view_end = n_views if view_end is None else view_end
    desc = GeomDesc(n, fov, n_views, arc, n_bins, sod, sdd, bin_pitch, view_begin, view_end, batch)
    fs = (C.c_int32 * len(factors))(*factors)
    h = C.c_void_p()
    torch.cuda.current_device()
    _check(L.ms2g_plan_geometry(C.byref(desc), fs, len(factors), C.byref(h)))
    plan = Plan(h, n, n_views, n_bins, factors, view_begin, view_end, batch, torch.device("cuda"))
    plan.arc, plan.fov = arc, fov
    return plan


class RegisteredSubset:
    """A view subset uploaded once (ms2g_register_subset); pass it as `subset`."""

    def __init__(self, plan: Plan, sid: int, views):
        self.plan, self.id = plan, sid
        self.views = tuple(views)
        self.n_sel = sum(1 for v in self.views if plan.view_begin <= v < plan.view_end)

    def release(self):
        if self.id is not None and self.plan._h is not None:
            _check(load().ms2g_release_subset(self.plan.handle, self.id))
        self.id = None


def register_subset(plan: Plan, subset) -> RegisteredSubset:
    """Upload an ascending global view list once (+ its block orders); the
    projector / gradient calls then take it without a per-call copy."""
    sel, m = _subset(subset)
    sid = C.c_int32(-1)
    _check(load().ms2g_register_subset(plan.handle, sel, m, C.byref(sid)))
    return RegisteredSubset(plan, sid.value, [sel[k] for k in range(m)])


def release_subset(rs: RegisteredSubset):
    rs.release()


def _reg(subset):
    if isinstance(subset, RegisteredSubset):
        if subset.id is None:
            raise MS2GError(MS2G_ERR_INPUT, "subset was released")
        return subset.id
    return None


def _n_sel(plan: Plan, subset) -> int:
    if subset is None:
        return plan.n_local_views
    if isinstance(subset, RegisteredSubset):
        return subset.n_sel
    return sum(1 for v in subset if plan.view_begin <= int(v) < plan.view_end)


def forward_project(plan: Plan, factor: int, x, b=None, subset=None, out=None):
    """r = A_s x - b on the selected views, compacted [batch][n_sel][B]."""
    if out is None:
        out = torch.empty((plan.batch, _n_sel(plan, subset), plan.n_bins), device=x.device, dtype=torch.float32)
    rid = _reg(subset)
    if rid is not None:
        _check(load().ms2g_forward_project_registered(plan.handle, factor, _dev(x, "x"), _dev(b, "b"),
                                                      _dev(out, "out"), rid, _stream()))
        return out
    sel, m = _subset(subset)
    _check(load().ms2g_forward_project(plan.handle, factor, _dev(x, "x"), _dev(b, "b"), _dev(out, "out"), sel, m,
                                       _stream()))
    return out


def back_project(plan: Plan, factor: int, sino, img=None, scale=1.0, accumulate=False, subset=None,
                 allreduce=False):
    """img = scale A_s^T sino (+img if accumulate); allreduce: sum over the
    ranks attached by attach_nccl / attach_peers."""
    nc = plan.nc(factor)
    if img is None:
        img = torch.empty((plan.batch, nc, nc), device=sino.device, dtype=torch.float32)
    rid = _reg(subset)
    if rid is not None:
        _check(load().ms2g_back_project_registered(plan.handle, factor, _dev(sino, "sino"), _dev(img, "img"),
                                                   float(scale), int(bool(accumulate)), rid, int(bool(allreduce)),
                                                   _stream()))
        return img
    sel, m = _subset(subset)
    _check(load().ms2g_back_project(plan.handle, factor, _dev(sino, "sino"), _dev(img, "img"), float(scale),
                                    int(bool(accumulate)), sel, m, int(bool(allreduce)), _stream()))
    return img


RESAMPLERS = {"mean": 0, "bicubic": 1}


def _kind(resampler) -> int:
    return RESAMPLERS[resampler] if isinstance(resampler, str) else int(resampler)


def sketch_down(plan: Plan, factor: int, x, v=None, resampler="mean"):
    """S: s x s average pool ("mean", configs) or bicubic ("bicubic")."""
    nc = plan.nc(factor)
    if v is None:
        v = torch.empty((plan.batch, nc, nc), device=x.device, dtype=torch.float32)
    _check(load().ms2g_sketch_down(plan.handle, factor, _kind(resampler), _dev(x, "x"), _dev(v, "v"), _stream()))
    return v


def sketch_up(plan: Plan, factor: int, g, y=None, eta=0.0, z=None, resampler="mean"):
    """z = y - eta U g  (z = U g when y is None); U replication or bicubic."""
    if z is None:
        z = torch.empty((plan.batch, plan.n, plan.n), device=g.device, dtype=torch.float32)
    _check(load().ms2g_sketch_up(plan.handle, factor, _kind(resampler), _dev(g, "g"), _dev(y, "y"), float(eta),
                                 _dev(z, "z"), _stream()))
    return z


def sketched_grad(plan: Plan, factor: int, x, b, g=None, subset=None, resampler="mean"):
    """g = (V/|M|) U A_s^T (A_s S x - b_M)."""
    if g is None:
        g = torch.empty((plan.batch, plan.n, plan.n), device=x.device, dtype=torch.float32)
    rid = _reg(subset)
    if rid is not None:
        _check(load().ms2g_sketched_grad_registered(plan.handle, factor, _kind(resampler), _dev(x, "x"), _dev(b, "b"),
                                                    _dev(g, "g"), rid, _stream()))
        return g
    sel, m = _subset(subset)
    _check(load().ms2g_sketched_grad(plan.handle, factor, _kind(resampler), _dev(x, "x"), _dev(b, "b"), _dev(g, "g"),
                                     sel, m, _stream()))
    return g


def power_iteration(plan: Plan, factor: int, iters: int = 20) -> float:
    """L = <v, A_s^T A_s v> after `iters` normalised steps from 1/||1|| (P:156,
    reading Z5/Z6); also refreshes the plan's cached step for the factor."""
    L = C.c_double(0.0)
    _check(load().ms2g_power_iteration(plan.handle, factor, iters, C.byref(L), _stream()))
    return L.value


def _den(den) -> Denoiser:
    kind = den[0]
    if kind == "identity":
        return Denoiser(0, 0.0, 0.0, 0.125, 1)
    if kind == "gauss":
        return Denoiser(1, float(den[1]), 0.0, 0.125, 1)
    if kind == "tv":
        tau = float(den[3]) if len(den) > 3 else 0.125
        return Denoiser(2, 0.0, float(den[1]), tau, int(den[2]))
    raise MS2GError(MS2G_ERR_CONFIG, f"unknown denoiser {kind!r}")


def denoise(plan: Plan, den, z, out=None):
    """D(z): ("identity",) | ("gauss", sigma) | ("tv", lambda, iters[, tau])."""
    if out is None:
        out = torch.empty_like(z)
    d = _den(den)
    _check(load().ms2g_denoise(plan.handle, C.byref(d), _dev(z, "z"), _dev(out, "out"), _stream()))
    return out


def _solve_desc(stages, option, n_subsets, seed, den, alpha, power_iters, resampler="mean"):
    st = (Stage * len(stages))(*[Stage(*s) for s in stages])
    desc = SolveDesc(st, len(stages), option, n_subsets, seed, _den(den), alpha, power_iters, 1, _kind(resampler))
    return desc, st


def schedule(plan: Plan | None, stages, option=1, n_subsets=1, seed=0):
    """ms2g_schedule: bit-exact host schedule (plan may be None: no device needed)."""
    desc, keep = _solve_desc(stages, option, n_subsets, seed, ("identity",), 1.0, 20)
    n = C.c_int32(0)
    h = plan.handle if plan is not None else None
    _check(load().ms2g_schedule(h, C.byref(desc), None, 0, C.byref(n)))
    buf = (SchedEntry * max(1, n.value))()
    _check(load().ms2g_schedule(h, C.byref(desc), buf, n.value, C.byref(n)))
    return [buf[k].as_tuple() for k in range(n.value)]


def schedule_views(plan: Plan, stages, step: int, option=1, n_subsets=1, seed=0):
    """Global view indices used by schedule step `step` (host only)."""
    desc, keep = _solve_desc(stages, option, n_subsets, seed, ("identity",), 1.0, 20)
    n = C.c_int32(0)
    _check(load().ms2g_schedule_views(plan.handle, C.byref(desc), step, None, 0, C.byref(n)))
    buf = (C.c_int32 * max(1, n.value))()
    _check(load().ms2g_schedule_views(plan.handle, C.byref(desc), step, buf, n.value, C.byref(n)))
    return [buf[k] for k in range(n.value)]


def pnp_ms2g_solve(plan: Plan, stages, b, x0=None, option=1, n_subsets=1, seed=0, den=("gauss", 0.8),
                   alpha=0.5, power_iters=20, x_out=None, trace=False, resampler="mean"):
    """Algorithm 1 as one CUDA graph.  b: [batch][V_r][B].

    Device tensors in -> device tensor out.  Host (CPU) tensors are copied to
    the device (pinned, async) and the result is copied back: the end-to-end
    path a user of host buffers takes."""
    host = not b.is_cuda
    if host:
        dev = torch.device("cuda")
        b_d = b.pin_memory().to(dev, non_blocking=True) if not b.is_pinned() else b.to(dev, non_blocking=True)
        x0_d = None if x0 is None else x0.to(dev, non_blocking=True)
    else:
        b_d, x0_d = b, x0
    if x0_d is None:
        x0_d = torch.zeros((plan.batch, plan.n, plan.n), device=b_d.device, dtype=torch.float32)
    out_d = x_out if (x_out is not None and x_out.is_cuda) else torch.empty_like(x0_d)
    desc, keep = _solve_desc(stages, option, n_subsets, seed, den, alpha, power_iters, resampler)
    n_steps = len(schedule(plan, stages, option, n_subsets, seed))
    tr = (SchedEntry * max(1, n_steps))() if trace else None
    _check(load().ms2g_pnp_ms2g_solve(plan.handle, C.byref(desc), _dev(b_d, "b"), _dev(x0_d, "x0"),
                                      _dev(out_d, "x_out"), tr, _stream()))
    result = out_d
    if x_out is not None and not x_out.is_cuda:      # a host x_out is always written (either branch)
        x_out.copy_(out_d, non_blocking=x_out.is_pinned())
        torch.cuda.current_stream().synchronize()
        result = x_out
    elif host:
        result = torch.empty(out_d.shape, dtype=torch.float32).pin_memory()
        result.copy_(out_d, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    if trace:
        return result, [tr[k].as_tuple() for k in range(n_steps)]
    return result


def pnp_ms2g_solve_async(plan: Plan, stages, b, x0, x_out, option=1, n_subsets=1, seed=0, den=("gauss", 0.8),
                         alpha=0.5, power_iters=20, resampler="mean"):
    """Launch the cached solve graph on the current stream and return."""
    desc, keep = _solve_desc(stages, option, n_subsets, seed, den, alpha, power_iters, resampler)
    _check(load().ms2g_pnp_ms2g_solve_async(plan.handle, C.byref(desc), _dev(b, "b"), _dev(x0, "x0"),
                                            _dev(x_out, "x_out"), _stream()))


def solve_status(plan: Plan):
    _check(load().ms2g_solve_status(plan.handle, _stream()))


def broadcast_unique_id(uid: bytes | None, rank: int, nranks: int, group=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id over the torch process group."""
    import torch.distributed as dist
    obj = [uid if rank == 0 else None]
    if nranks > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise MS2GError(MS2G_ERR_NCCL, "bad NCCL unique id broadcast")
    return bytes(obj[0])


def attach_nccl(plan: Plan, rank: int, nranks: int, group=None):
    """Rank 0 makes the ncclUniqueId, torch.distributed broadcasts it, every
    rank attaches the plan (view-sharded allreduce of partial images)."""
    L = load()
    uid = None
    if rank == 0:
        buf = (C.c_uint8 * 128)()
        _check(L.ms2g_nccl_unique_id(buf))
        uid = bytes(buf)
    uid = broadcast_unique_id(uid, rank, nranks, group)
    _check(L.ms2g_attach_nccl(plan.handle, (C.c_uint8 * 128).from_buffer_copy(uid), rank, nranks))
    plan.rank, plan.nranks = rank, nranks
    return plan


def set_kernel_timing(plan: Plan, enable: bool = True):
    """Record CUDA events around every projector launch of the captured solve
    graph (measurement support; the graph is re-captured)."""
    _check(load().ms2g_set_kernel_timing(plan.handle, 1 if enable else 0))


def kernel_time(plan: Plan, kind: str, factor: int):
    """(total device ms, launches) of the 'forward' or 'backward' launches at
    `factor` in the last replayed solve (needs set_kernel_timing)."""
    t, n = C.c_double(), C.c_int32()
    _check(load().ms2g_kernel_time(plan.handle, {"forward": 0, "backward": 1}[kind], factor, C.byref(t), C.byref(n)))
    return t.value, n.value


def gather_blobs(blob: bytes, rank: int, nranks: int, group=None) -> bytes:
    """All-gather one fixed-size byte blob per rank (torch.distributed, any
    backend; plumbing only) and return them concatenated in rank order."""
    if nranks == 1:
        return blob
    import torch.distributed as dist
    out = [None] * nranks
    dist.all_gather_object(out, blob, group=group)
    if any(not isinstance(b, (bytes, bytearray)) or len(b) != len(blob) for b in out):
        raise MS2GError(MS2G_ERR_CONFIG, "peer blob exchange: blobs of different sizes")
    return b"".join(bytes(b) for b in out)


def attach_peers(plan: Plan, rank: int, nranks: int, group=None):
    """NEXT-3: sum backprojections over NVLink peer memory (fused, fixed rank
    order) instead of NCCL.  Every rank of the group must call it."""
    L = load()
    size = L.ms2g_peer_blob_size()
    mine = C.create_string_buffer(size)
    _check(L.ms2g_peer_export(plan.handle, mine))
    allb = gather_blobs(mine.raw, rank, nranks, group)
    buf = C.create_string_buffer(allb, len(allb))
    _check(L.ms2g_attach_peers(plan.handle, buf, rank, nranks))


def view_shard(n_views: int, rank: int, nranks: int):
    """Contiguous view shard of rank r: [r V / P, (r+1) V / P) (view sharding)."""
    return (n_views * rank) // nranks, (n_views * (rank + 1)) // nranks


def launch_count() -> int:
    return int(load().ms2g_launch_count())


def attach_multicast(plan: Plan, rank: int, nranks: int, group=None):
    """NEXT-3, NVLS form: rank 0 creates the NVSwitch multicast object, the
    process group broadcasts its blob, every rank imports it and adds its
    device, a barrier, then every rank binds and maps its buffer.  Raises
    MS2GError (code 5, naming the driver call) where multicast is unavailable;
    the plan then keeps its NCCL / peer paths."""
    import torch.distributed as dist
    L = load()
    size = L.ms2g_mc_blob_size()
    blob = None
    err = None
    if rank == 0:
        buf = C.create_string_buffer(size)
        rc = L.ms2g_mc_create(plan.handle, nranks, buf)
        blob = buf.raw if rc == MS2G_OK else None
        err = None if rc == MS2G_OK else (rc, L.ms2g_last_error().decode(errors="replace"))
    if nranks > 1:
        obj = [(blob, err)]
        dist.broadcast_object_list(obj, src=0, group=group)
        blob, err = obj[0]
    if err is not None:
        raise MS2GError(*err)
    b = C.create_string_buffer(blob, len(blob))
    _check(L.ms2g_attach_multicast(plan.handle, b, rank, nranks, 0))
    if nranks > 1:
        dist.barrier(group=group)
    _check(L.ms2g_attach_multicast(plan.handle, b, rank, nranks, 1))
    plan.rank, plan.nranks = rank, nranks
