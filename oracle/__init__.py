"""fp64 CPU oracle of the PnP-MS2G hot path (ctypes wrapper over ms2g_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with ``paper_2203_07308_b200`` (the CUDA product
path) and neither side imports the other; the only common module is
``ms2g_synth`` (seeded input generators, none of the method's arithmetic).

Every function cites the passage it follows (P:NN = PAPER.md line NN, S:NN =
SPEC.md line NN, O1..O13 = the SURVEY §8(c) readings recorded in DESIGN.md).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ms2g_oracle.c")
_LIB = os.path.join(_HERE, "libms2g_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, no FMA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-fPIC", "-shared", "-ffp-contract=off",
               _SRC, "-o", _LIB + ".tmp", "-lpthread", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Geom(C.Structure):
    _fields_ = [("n", C.c_int32), ("fov", C.c_double), ("n_views", C.c_int32), ("arc", C.c_double),
                ("n_bins", C.c_int32), ("sod", C.c_double), ("sdd", C.c_double),
                ("bin_pitch", C.c_double)]


class _Stage(C.Structure):
    _fields_ = [("factor", C.c_int32), ("n_iters", C.c_int32), ("n_epochs", C.c_int32)]


class SchedEntry(C.Structure):
    _fields_ = [("i", C.c_int32), ("stage", C.c_int32), ("factor", C.c_int32), ("subset", C.c_int32),
                ("eta", C.c_double), ("a", C.c_double)]

    def as_tuple(self):
        return (self.i, self.stage, self.factor, self.subset, self.eta, self.a)


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i, p = C.c_double, C.c_int, C.c_void_p
        G = C.POINTER(_Geom)
        _lib.orc_ray_endpoints.argtypes = [G, i, i, p, p]
        _lib.orc_ray_segments.argtypes = [G, i, i, i, p, p, i]
        _lib.orc_ray_segments.restype = i
        _lib.orc_ray_sum.argtypes = [G, i, p, i, i]
        _lib.orc_ray_sum.restype = d
        _lib.orc_forward.argtypes = [G, i, p, p, p, p, i, i]
        _lib.orc_forward.restype = C.c_longlong
        _lib.orc_backward.argtypes = [G, i, p, p, d, p, i, i]
        _lib.orc_backward_pixel.argtypes = [G, i, p, p, i, i, i]
        _lib.orc_backward_pixel.restype = d
        _lib.orc_sketch_down.argtypes = [i, i, p, p]
        _lib.orc_sketch_up.argtypes = [i, i, p, p]
        _lib.orc_sketched_grad.argtypes = [G, i, p, p, p, p, i, i]
        _lib.orc_sketched_grad_kind.argtypes = [G, i, i, p, p, p, p, i, i]
        _lib.orc_keys.argtypes = [d]
        _lib.orc_keys.restype = d
        _lib.orc_bicubic_down.argtypes = [i, i, p, p]
        _lib.orc_bicubic_up.argtypes = [i, i, p, p]
        _lib.orc_set_resampler.argtypes = [i]
        _lib.orc_power_iteration.argtypes = [G, i, i, i]
        _lib.orc_power_iteration.restype = d
        _lib.orc_gauss3_weights.argtypes = [d, p]
        _lib.orc_gauss3.argtypes = [i, d, p, p]
        _lib.orc_grad.argtypes = [i, p, p, p]
        _lib.orc_div.argtypes = [i, p, p, p]
        _lib.orc_tv_chambolle.argtypes = [i, d, d, i, p, p, p]
        _lib.orc_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        _lib.orc_splitmix64.restype = C.c_uint64
        _lib.orc_momentum.argtypes = [i]
        _lib.orc_momentum.restype = d
        _lib.orc_schedule.argtypes = [C.POINTER(_Stage), i, i, i, C.c_uint64, C.POINTER(SchedEntry), i]
        _lib.orc_schedule.restype = i
        _lib.orc_minibatch_views.argtypes = [i, i, C.c_uint64, i, p]
        _lib.orc_minibatch_views.restype = i
        _lib.orc_subset_views.argtypes = [i, i, i, p]
        _lib.orc_subset_views.restype = i
        _lib.orc_pnp_ms2g.argtypes = [G, C.POINTER(_Stage), i, i, i, C.c_uint64, i, d, d, d, i, d, i,
                                      p, p, p, C.POINTER(SchedEntry), p, i, C.POINTER(C.c_int)]
        _lib.orc_pnp_ms2g.restype = i
    return _lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


@dataclass(frozen=True)
class Geometry:
    """O1 fan-beam geometry."""
    n: int
    n_views: int
    n_bins: int
    fov: float = 2.0
    arc: float = 2 * np.pi
    sod: float | None = None        # default 2 W  (BASELINE configs[0])
    sdd: float | None = None        # default 4 W
    bin_pitch: float = 0.0          # <= 0 -> (sdd/sod) * W/N

    def c(self) -> _Geom:
        sod = self.sod if self.sod is not None else 2.0 * self.fov
        sdd = self.sdd if self.sdd is not None else 4.0 * self.fov
        return _Geom(self.n, self.fov, self.n_views, self.arc, self.n_bins, sod, sdd, self.bin_pitch)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _views(views, n_views):
    if views is None:
        return None, n_views
    v = np.ascontiguousarray(views, dtype=np.int32)
    return v, len(v)


def ray_endpoints(g: Geometry, v: int, t: int):
    s = np.zeros(2); d = np.zeros(2)
    lib().orc_ray_endpoints(C.byref(g.c()), v, t, _ptr(s), _ptr(d))
    return s, d


def ray_segments(g: Geometry, factor: int, v: int, t: int):
    """O2 Siddon segments of ray (v,t): (pixel indices i*n_c+j, lengths)."""
    cap = 2 * (g.n // factor) + 8
    pix = np.zeros(cap, dtype=np.int32); ln = np.zeros(cap)
    m = lib().orc_ray_segments(C.byref(g.c()), factor, v, t, _ptr(pix), _ptr(ln), cap)
    return pix[:m].copy(), ln[:m].copy()


def ray_sum(g: Geometry, factor: int, x, v: int, t: int) -> float:
    x = _f64(x)
    return lib().orc_ray_sum(C.byref(g.c()), factor, _ptr(x), v, t)


def forward(g: Geometry, factor: int, x, b=None, views=None, nthreads: int | None = None):
    """O2: r[k,t] = (A_s x)[views[k],t] - b[views[k],t]  (Eq. 7)."""
    x = _f64(x)
    vv, n_sel = _views(views, g.n_views)
    out = np.zeros((n_sel, g.n_bins))
    bb = _f64(b) if b is not None else None
    lib().orc_forward(C.byref(g.c()), factor, _ptr(x), _ptr(bb) if bb is not None else None, _ptr(out),
                      _ptr(vv) if vv is not None else None, n_sel, nthreads or default_threads())
    return out


def count_nnz(g: Geometry, factor: int, views=None, nthreads: int | None = None) -> int:
    """Exact number of positive-length ray-pixel segments of A_s on the views."""
    nc = g.n // factor
    x = np.zeros(nc * nc)
    vv, n_sel = _views(views, g.n_views)
    return int(lib().orc_forward(C.byref(g.c()), factor, _ptr(x), None, None,
                                 _ptr(vv) if vv is not None else None, n_sel, nthreads or default_threads()))


def backward(g: Geometry, factor: int, sino, scale: float = 1.0, views=None, nthreads: int | None = None):
    """O3: img = scale * A_s^T sino, sino compacted [n_sel][B]."""
    vv, n_sel = _views(views, g.n_views)
    s = _f64(sino).reshape(n_sel, g.n_bins)
    nc = g.n // factor
    img = np.zeros(nc * nc)
    lib().orc_backward(C.byref(g.c()), factor, _ptr(s), _ptr(img), float(scale),
                       _ptr(vv) if vv is not None else None, n_sel, nthreads or default_threads())
    return img.reshape(nc, nc)


def backward_pixel(g: Geometry, factor: int, sino, i: int, j: int, views=None) -> float:
    """(A_s^T r) at pixel (i,j) by the plain definition sum_rays len(R cap pixel) r."""
    vv, n_sel = _views(views, g.n_views)
    s = _f64(sino).reshape(n_sel, g.n_bins)
    return lib().orc_backward_pixel(C.byref(g.c()), factor, _ptr(s), _ptr(vv) if vv is not None else None,
                                    n_sel, i, j)


def sketch_down(x, s: int):
    """O4 S_s: s x s average pool."""
    x = _f64(x); n = x.shape[-1]
    v = np.zeros((n // s, n // s))
    lib().orc_sketch_down(n, s, _ptr(x), _ptr(v))
    return v


def sketch_up(gc, s: int):
    """O5 U_s: nearest replication (= s^2 S_s^T)."""
    gc = _f64(gc); nc = gc.shape[-1]
    out = np.zeros((nc * s, nc * s))
    lib().orc_sketch_up(nc * s, s, _ptr(gc), _ptr(out))
    return out


def sketched_grad(g: Geometry, factor: int, x, b, views=None, nthreads: int | None = None, resampler: int = 0):
    """O6/O7: g = (V/|M|) U A_s^T (A_s S x - b_M)  (Eqs. 6-7).
    b is the full [V][B] sinogram, indexed by view (b_M = its rows `views`).
    resampler 0: average pool + replication (O4/O5); 1: bicubic (NEXT-1)."""
    x = _f64(x); b = _f64(b)
    vv, n_sel = _views(views, g.n_views)
    out = np.zeros((g.n, g.n))
    lib().orc_sketched_grad_kind(C.byref(g.c()), factor, resampler, _ptr(x), _ptr(b), _ptr(out),
                                 _ptr(vv) if vv is not None else None, n_sel, nthreads or default_threads())
    return out


def keys(x: float) -> float:
    """Keys cubic convolution kernel, a = -0.5 (NEXT-1)."""
    return lib().orc_keys(float(x))


def bicubic_down(x, s: int):
    """NEXT-1 S: bicubic antialiased downscale by s (P:156 imresize)."""
    x = _f64(x); n = x.shape[-1]
    v = np.zeros((n // s, n // s))
    lib().orc_bicubic_down(n, s, _ptr(x), _ptr(v))
    return v


def bicubic_up(gc, s: int):
    """NEXT-1 U: bicubic upscale by s (P:156 imresize)."""
    gc = _f64(gc); nc = gc.shape[-1]
    out = np.zeros((nc * s, nc * s))
    lib().orc_bicubic_up(nc * s, s, _ptr(gc), _ptr(out))
    return out


def power_iteration(g: Geometry, factor: int, iters: int = 20, nthreads: int | None = None) -> float:
    """O8: L_iters of A_s^T A_s from v0 = 1/||1|| (configs[0])."""
    return lib().orc_power_iteration(C.byref(g.c()), factor, iters, nthreads or default_threads())


def gauss3_weights(sigma: float = 0.8):
    w = np.zeros(3)
    lib().orc_gauss3_weights(sigma, _ptr(w))
    return w


def gauss3(z, sigma: float = 0.8):
    """O9 Gaussian 3x3 denoiser, replicate boundary, rows then columns."""
    z = _f64(z); n = z.shape[-1]
    out = np.zeros_like(z)
    lib().orc_gauss3(n, sigma, _ptr(z), _ptr(out))
    return out


def grad(u):
    u = _f64(u); n = u.shape[-1]
    gx = np.zeros_like(u); gy = np.zeros_like(u)
    lib().orc_grad(n, _ptr(u), _ptr(gx), _ptr(gy))
    return gx, gy


def div(px, py):
    px = _f64(px); py = _f64(py); n = px.shape[-1]
    d = np.zeros_like(px)
    lib().orc_div(n, _ptr(px), _ptr(py), _ptr(d))
    return d


def tv_chambolle(f, lam: float, iters: int = 10, tau: float = 0.125, return_dual: bool = False):
    """O9 TV-prox by Chambolle's dual fixed point (Z18)."""
    f = _f64(f); n = f.shape[-1]
    u = np.zeros_like(f); p = np.zeros((2, n, n))
    lib().orc_tv_chambolle(n, lam, tau, iters, _ptr(f), _ptr(u), _ptr(p))
    return (u, p) if return_dual else u


def splitmix64_stream(seed: int, count: int):
    st = C.c_uint64(seed)
    return [lib().orc_splitmix64(C.byref(st)) for _ in range(count)]


def momentum(i: int) -> float:
    """a_i = (i-1)/(i+3)."""
    return lib().orc_momentum(i)


def schedule(stages, option: int = 1, n_subsets: int = 1, seed: int = 0):
    """O13 bit-exact schedule: list of (i, stage, factor, subset, eta=0, a)."""
    st = (_Stage * len(stages))(*[_Stage(*s) for s in stages])
    n = lib().orc_schedule(st, len(stages), option, n_subsets, seed, None, 0)
    if n < 0:
        raise ValueError("bad schedule description")
    buf = (SchedEntry * max(n, 1))()
    lib().orc_schedule(st, len(stages), option, n_subsets, seed, buf, n)
    return [buf[k].as_tuple() for k in range(n)]


def minibatch_views(n_views: int, m: int, seed: int, n_steps: int):
    """Option 4: per step m distinct views, uniform without replacement (partial
    Fisher-Yates on one SplitMix64 stream), ascending.  Shape (n_steps, m)."""
    out = np.zeros((max(n_steps, 1), m), dtype=np.int32)
    if lib().orc_minibatch_views(n_views, m, seed, n_steps, _ptr(out)) != 0:
        raise ValueError("bad minibatch size")
    return out[:n_steps].copy()


def subset_views(n_views: int, n_subsets: int, k: int):
    out = np.zeros(n_views, dtype=np.int32)
    m = lib().orc_subset_views(n_views, n_subsets, k, _ptr(out))
    return out[:m].copy()


class DivergedError(RuntimeError):
    pass


def pnp_ms2g(g: Geometry, stages, b, x0=None, option: int = 1, n_subsets: int = 1, seed: int = 0,
             den: tuple = ("identity",), alpha: float = 1.0, power_iters: int = 20,
             nthreads: int | None = None, resampler: int = 0):
    """O11 Algorithm 1.  den = ("identity",) | ("gauss", sigma) |
    ("tv", lambda, iters[, tau]).  Returns (x, trace, etas)."""
    n = g.n
    b = _f64(b)
    x0 = np.zeros((n, n)) if x0 is None else _f64(x0)
    out = np.zeros((n, n))
    kind, sigma, lam, tau, diters = 0, 0.8, 0.0, 0.125, 0
    if den[0] == "gauss":
        kind, sigma = 1, float(den[1])
    elif den[0] == "tv":
        kind, lam, diters = 2, float(den[1]), int(den[2])
        if len(den) > 3:
            tau = float(den[3])
    st = (_Stage * len(stages))(*[_Stage(*s) for s in stages])
    total = lib().orc_schedule(st, len(stages), option, n_subsets, seed, None, 0)
    trace = (SchedEntry * max(total, 1))()
    etas = np.zeros(len(stages))
    bad = C.c_int(0)
    lib().orc_set_resampler(resampler)
    rc = lib().orc_pnp_ms2g(C.byref(g.c()), st, len(stages), option, n_subsets, seed, kind, sigma, lam, tau,
                            diters, alpha, power_iters, _ptr(b), _ptr(x0), _ptr(out), trace, _ptr(etas),
                            nthreads or default_threads(), C.byref(bad))
    lib().orc_set_resampler(0)
    if rc == 3:
        raise DivergedError(f"non-finite iterate at iteration {bad.value}")
    if rc != 0:
        raise ValueError(f"oracle pnp_ms2g failed with code {rc}")
    return out, [trace[k].as_tuple() for k in range(total)], etas
