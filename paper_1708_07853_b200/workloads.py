"""Seeded synthetic inputs for the five BASELINE.json configs.

This module holds NO arithmetic of the method (no lifting, no filter): it only
draws pixels.  It is the one module shared by the CUDA path's callers (bench,
tests) and the oracle's callers, as DESIGN.md section 4 states.

The paper measures no public dataset and never states pixel content: it uses
"tiles ... comprising single-precision floating-point values"
and image edges up to 8192 (L340-345).  These generators stand in for that,
with the shapes of BASELINE.json ``configs``:

* ``uniform``: integer-valued pixels drawn uniformly from {0..255}, stored as
  fp32 (configs 1, 3, 5; reading C-A15 of DESIGN.md).
* ``smooth``: a sum of 8 random plane waves sin(2 pi (x cos t + y sin t)/T + p)
  with T log-uniform in [16, 512] px, t ~ U[0, pi), p ~ U[0, 2 pi), scaled
  affinely to [0, 255], plus N(0, 4^2) noise, clipped to [0, 255], cast to
  fp32 (configs 2, 4; reading C-A16).
* ``uniform_real``: continuous U[0, 255) fp32 (extra parity variant).

Every generator is a pure function of (width, height, seed) via numpy PCG64.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


def uniform_int(width: int, height: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 256, size=(height, width), dtype=np.uint8).astype(np.float32)


def uniform_real(width: int, height: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random(size=(height, width), dtype=np.float32) * np.float32(255.0)).astype(np.float32)


def smooth_noise(width: int, height: int, seed: int, waves: int = 8, sigma: float = 4.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    period = np.exp(rng.uniform(math.log(16.0), math.log(512.0), size=waves))
    theta = rng.uniform(0.0, math.pi, size=waves)
    phase = rng.uniform(0.0, 2.0 * math.pi, size=waves)
    x = np.arange(width, dtype=np.float64)
    y = np.arange(height, dtype=np.float64)
    field = np.zeros((height, width), dtype=np.float64)
    for T, t, p in zip(period, theta, phase):
        # sin(u + v) = sin u cos v + cos u sin v with u = kx x, v = ky y + p:
        # two outer products instead of a full-size sin per wave.
        kx = 2.0 * math.pi * math.cos(t) / T
        ky = 2.0 * math.pi * math.sin(t) / T
        u = kx * x
        v = ky * y + p
        field += np.outer(np.cos(v), np.sin(u))
        field += np.outer(np.sin(v), np.cos(u))
    lo, hi = field.min(), field.max()
    field -= lo
    field *= 255.0 / (hi - lo)
    field += rng.normal(0.0, sigma, size=(height, width))
    np.clip(field, 0.0, 255.0, out=field)
    return field.astype(np.float32)


GENERATORS = {"uniform": uniform_int, "smooth": smooth_noise, "uniform_real": uniform_real}


@dataclasses.dataclass(frozen=True)
class ImageGroup:
    width: int
    height: int
    count: int
    kind: str
    seed0: int          # image i uses seed seed0 + i

    def image(self, i: int) -> np.ndarray:
        return GENERATORS[self.kind](self.width, self.height, self.seed0 + i)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    levels: int
    groups: tuple       # of ImageGroup
    description: str

    @property
    def pixels(self) -> int:
        return sum(g.width * g.height * g.count for g in self.groups)


# BASELINE.json configs (1-based as in SURVEY.md section 8d), plus the 8193^2
# parity companion of config 4 (reading C-A14).
CONFIGS = {
    "1": Config("1", 1, (ImageGroup(512, 512, 1, "uniform", 1),),
                "512x512 integer-valued U{0..255}, 1 level"),
    "2": Config("2", 1, (ImageGroup(4096, 4096, 1, "smooth", 2),),
                "4096x4096 smooth+noise, 1 level"),
    "3": Config("3", 1, (ImageGroup(16384, 16384, 1, "uniform", 3),),
                "16384x16384 integer-valued U{0..255}, 1 level, row strips over G GPUs"),
    "4": Config("4", 8, (ImageGroup(8192, 8192, 1, "smooth", 4),),
                "8192x8192 smooth+noise, 8 levels"),
    "4b": Config("4b", 8, (ImageGroup(8193, 8193, 1, "smooth", 4),),
                 "8193x8193 smooth+noise, 8 levels (odd at every level; parity companion)"),
    "5": Config("5", 3, (ImageGroup(2048, 2048, 256, "uniform", 5000),
                         ImageGroup(4095, 3001, 32, "uniform", 6000)),
                "256 x 2048^2 + 32 x 4095x3001 integer-valued, 3 levels, images sharded"),
}


def level_pixels(width: int, height: int, levels: int) -> int:
    """Sum over levels of the level-input pixel count (W_{k+1} = ceil(W_k/2))."""
    total, w, h = 0, width, height
    for _ in range(levels):
        total += w * h
        w, h = (w + 1) // 2, (h + 1) // 2
    return total
