"""Seeded synthetic inputs and the C1..C5 workload presets.

This module is the ONLY code shared by the oracle side (tests, cpu baseline)
and the CUDA product side (binding, bench).  It holds none of the method's
arithmetic: no projector, no sketch, no gradient, no denoiser.  It draws
phantoms (BASELINE.json configs: "seeded ellipses"), noise for given
projections (Gaussian; Poisson transmission data of P:122-126 Eq. 8), random
test sinograms, and the preset tables the configs name.

Seeds: seed = 220307308 + 1000*cfg + image (cfg 1-based), numpy
Generator(PCG64([seed, stream])), stream 0 = phantom, 1 = noise, 2.. = test.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 220307308


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), int(stream)]))


def config_seed(cfg: int, image: int = 0) -> int:
    return SEED_BASE + 1000 * cfg + image


def phantom(n: int, n_ellipses: int, seed: int, texture: float = 0.0, fov: float = 2.0) -> np.ndarray:
    """Additive ellipse phantom sampled at pixel centres (reading Z19).

    Per ellipse, draw order: u1, u2 (centre uniform in a disk of radius 0.5:
    rho = 0.5 sqrt(u1), psi = 2 pi u2), semi-axes a, b ~ U[0.05, 0.4],
    angle phi ~ U[0, pi), intensity ~ U[0, 1].  Boundary inclusive.  Optional
    i.i.d. U[-texture, texture] texture added to every pixel (C3).
    Pixel (i, j) centre: (-W/2 + (j+1/2) h, -W/2 + (i+1/2) h), row i along +y.
    """
    g = rng(seed, 0)
    h = fov / n
    c = -0.5 * fov + (np.arange(n) + 0.5) * h
    X, Y = np.meshgrid(c, c, indexing="xy")       # X[i,j] = x_j, Y[i,j] = y_i
    img = np.zeros((n, n))
    for _ in range(n_ellipses):
        u1, u2 = g.random(), g.random()
        rho, psi = 0.5 * np.sqrt(u1), 2 * np.pi * u2
        cx, cy = rho * np.cos(psi), rho * np.sin(psi)
        a, b = g.uniform(0.05, 0.4), g.uniform(0.05, 0.4)
        phi = g.uniform(0.0, np.pi)
        inten = g.random()
        dx, dy = X - cx, Y - cy
        xr = dx * np.cos(phi) + dy * np.sin(phi)
        yr = -dx * np.sin(phi) + dy * np.cos(phi)
        img += inten * ((xr / a) ** 2 + (yr / b) ** 2 <= 1.0)
    if texture > 0:
        img += g.uniform(-texture, texture, size=(n, n))
    return img.astype(np.float32)


def gaussian_data(p: np.ndarray, pct: float, seed: int) -> np.ndarray:
    """b = p + sigma N(0,1), sigma = pct * max(p)  (reading Z20; p given)."""
    g = rng(seed, 1)
    sigma = pct * float(np.max(p))
    return (np.asarray(p, np.float64) + sigma * g.standard_normal(p.shape)).astype(np.float32)


def poisson_data(p: np.ndarray, i0: float, seed: int) -> np.ndarray:
    """Transmission data of P:122-126 (Eq. 8): c ~ Poisson(I0 e^{-p}),
    c <- max(c, 1), b = -ln(c / I0)."""
    g = rng(seed, 1)
    c = g.poisson(i0 * np.exp(-np.asarray(p, np.float64)))
    c = np.maximum(c, 1)
    return (-np.log(c / i0)).astype(np.float32)


def random_sinogram(shape, seed: int, stream: int = 2, zero_mean: bool = True) -> np.ndarray:
    g = rng(seed, stream)
    if zero_mean:
        return g.standard_normal(shape).astype(np.float32)
    return g.random(shape).astype(np.float32)


def random_image(n: int, seed: int, stream: int = 3) -> np.ndarray:
    return rng(seed, stream).random((n, n)).astype(np.float32)


def split_epochs(total_epochs: int, n_stages: int):
    """np.array_split-style split: the first E mod K stages get ceil(E/K) (Z9)."""
    q, r = divmod(total_epochs, n_stages)
    return [q + (1 if k < r else 0) for k in range(n_stages)]


@dataclass
class Preset:
    """One of BASELINE.json configs[0..4] (C1..C5) with the SURVEY O12/Z10 readings."""
    cfg: int
    n: int
    n_views: int
    n_bins: int
    n_ellipses: int
    stages: list              # [(factor, n_iters, n_epochs)]
    option: int = 1
    n_subsets: int = 1
    den: tuple = ("gauss", 0.8)
    alpha: float = 0.5
    noise: tuple = ("gauss", 0.01)
    texture: float = 0.0
    batch: int = 1
    power_iters: int = 20
    extra: dict = field(default_factory=dict)

    @property
    def n_steps(self) -> int:
        if self.option == 1:
            return sum(s[1] for s in self.stages)
        return sum(s[2] for s in self.stages) * self.n_subsets


def _c3_stages():
    ep = split_epochs(8, 3)
    return [(4, 8 * ep[0], ep[0]), (2, 8 * ep[1], ep[1]), (1, 8 * ep[2], ep[2])]


PRESETS = {
    1: Preset(1, 64, 90, 96, 10, [(2, 10, 0), (1, 10, 0)], den=("gauss", 0.8), alpha=0.5,
              noise=("gauss", 0.01)),
    2: Preset(2, 256, 360, 384, 20, [(4, 15, 0), (2, 15, 0), (1, 20, 0)], den=("tv", 0.02, 10), alpha=1.0,
              noise=("gauss", 0.02)),
    3: Preset(3, 512, 720, 768, 30, _c3_stages(), option=2, n_subsets=8, den=("tv", 0.01, 10), alpha=1.0,
              noise=("gauss", 0.01), texture=0.05),
    4: Preset(4, 1024, 1440, 1536, 40, [(2, 30, 0), (1, 20, 0)], den=("gauss", 0.8), alpha=0.5,
              noise=("gauss", 0.01)),
    5: Preset(5, 512, 720, 768, 30, [(2, 20, 0), (1, 20, 0)], den=("tv", 0.02, 10), alpha=1.0,
              noise=("poisson", 1e5), batch=8, extra={"total_images": 64}),
}
