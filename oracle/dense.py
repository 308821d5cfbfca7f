"""Brute-force dense system matrix for tiny grids (TEST INFRASTRUCTURE ONLY).

An algorithm independent of the Siddon traversal in ms2g_oracle.c: every ray
segment [source, detector bin] is clipped against every closed pixel square
with the slab method, and the entry is the clipped Euclidean length.  This is
the plain definition of the ray-driven line-integral operator (
north star "Siddon exact intersection-length") and pins the oracle's O2/O3.
Geometry O1 is written out again here in numpy.
"""
from __future__ import annotations

import numpy as np


def endpoints(n_views, n_bins, n, fov=2.0, arc=2 * np.pi, sod=None, sdd=None, bin_pitch=0.0):
    sod = 2.0 * fov if sod is None else sod
    sdd = 4.0 * fov if sdd is None else sdd
    pitch = bin_pitch if bin_pitch > 0 else (sdd / sod) * fov / n
    th = arc * np.arange(n_views) / n_views
    c, s = np.cos(th), np.sin(th)
    u = (np.arange(n_bins) - 0.5 * (n_bins - 1)) * pitch
    src = np.stack([sod * c, sod * s], -1)[:, None, :].repeat(n_bins, 1)
    det = np.stack([-(sdd - sod) * c[:, None] - u[None, :] * s[:, None],
                    -(sdd - sod) * s[:, None] + u[None, :] * c[:, None]], -1)
    return src.reshape(-1, 2), det.reshape(-1, 2)


def clip_lengths(src, det, box_lo, box_hi):
    """Length of segment(s) src->det inside axis-aligned closed boxes (broadcast)."""
    d = det - src
    amin = np.zeros(np.broadcast_shapes(src.shape[:-1], box_lo.shape[:-1]))
    amax = np.ones_like(amin)
    miss = np.zeros(amin.shape, dtype=bool)
    for a in range(2):
        da = d[..., a]
        with np.errstate(divide="ignore", invalid="ignore"):
            a1 = (box_lo[..., a] - src[..., a]) / da
            a2 = (box_hi[..., a] - src[..., a]) / da
        zero = (da == 0)
        inside = (src[..., a] >= box_lo[..., a]) & (src[..., a] <= box_hi[..., a])
        miss |= zero & ~inside
        lo_ = np.where(zero, -np.inf, np.minimum(a1, a2))
        hi_ = np.where(zero, np.inf, np.maximum(a1, a2))
        amin = np.maximum(amin, lo_)
        amax = np.minimum(amax, hi_)
    ln = np.where(miss | (amax <= amin), 0.0, (amax - amin) * np.linalg.norm(d, axis=-1))
    return ln


def dense_A(n, n_views, n_bins, factor=1, **geo):
    """Dense A_s of shape (V*B, n_c^2); rows (v,t) row-major, cols i*n_c+j."""
    fov = geo.get("fov", 2.0)
    src, det = endpoints(n_views, n_bins, n, **geo)
    nc = n // factor
    h = fov / nc
    lo = -0.5 * fov
    ii, jj = np.meshgrid(np.arange(nc), np.arange(nc), indexing="ij")
    box_lo = np.stack([lo + jj * h, lo + ii * h], -1).reshape(-1, 2)
    box_hi = box_lo + h
    A = clip_lengths(src[:, None, :], det[:, None, :], box_lo[None], box_hi[None])
    return A
