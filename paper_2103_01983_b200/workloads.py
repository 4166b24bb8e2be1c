"""Seeded synthetic inputs for the BASELINE.json configs.

No public dataset is involved: the reference's own studies are synthetic
(experiment.cpp:194-253). Generators are self-specified so that the oracle
and the device consume identical bytes on any machine:

* SplitMix64 stream per config seed; u = (z >> 11) * 2^-53 with 0 -> 2^-53.
* Gaussians by Box–Muller on consecutive uniform pairs:
  sqrt(-2 ln u1) cos(2 pi u2), sqrt(-2 ln u1) sin(2 pi u2).
* Reference ``delta`` is the square of BASELINE.json's delta
  (kernel.hpp:37 adds ``delta`` to d^2 directly).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class SplitMix64:
    def __init__(self, seed: int):
        self.state = np.uint64(seed)
        self.count = 0

    def next_u64(self, m: int) -> np.ndarray:
        k = np.arange(self.count + 1, self.count + m + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = self.state + k * _GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.count += m
        return z

    def uniform(self, m: int) -> np.ndarray:
        u = (self.next_u64(m) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        u[u == 0.0] = 2.0 ** -53
        return u

    def normal(self, m: int) -> np.ndarray:
        h = (m + 1) // 2
        u = self.uniform(2 * h)
        u1, u2 = u[0::2], u[1::2]
        rad = np.sqrt(-2.0 * np.log(u1))
        z = np.empty(2 * h)
        z[0::2] = rad * np.cos(2.0 * np.pi * u2)
        z[1::2] = rad * np.sin(2.0 * np.pi * u2)
        return z[:m]


@dataclass
class Workload:
    name: str
    n: int
    x0: np.ndarray        # SoA [chi..., psi...]
    gamma: np.ndarray
    delta: float          # reference delta (= BASELINE delta squared)
    dt: float = 1e-3
    n_steps: int = 0
    inflow: Optional[np.ndarray] = None


def config1(n: int = 4096, seed: int = 1) -> Workload:
    """BASELINE configs[0]: uniform unit disk, Γ ~ N(0,1)/N, δ = 0.01, 100 steps at dt = 1e-3."""
    rng = SplitMix64(seed)
    r = np.sqrt(rng.uniform(n))
    phi = 2.0 * np.pi * rng.uniform(n)
    g = rng.normal(n) / n
    x0 = np.concatenate([r * np.cos(phi), r * np.sin(phi)])
    return Workload("config1_fom_n4096", n, x0, g, 0.01 ** 2, 1e-3, 100)


def config2(n: int = 65536, seed: int = 2) -> Workload:
    """BASELINE configs[1]: Gaussian patch N(0, 0.25² I), Γ ∝ exp(-r²/0.1), ΣΓ = 1, δ = 0.005."""
    rng = SplitMix64(seed)
    z = rng.normal(2 * n) * 0.25
    x, y = z[:n], z[n:]
    w = np.exp(-(x * x + y * y) / 0.1)
    g = w / w.sum()
    return Workload("config2_velocity_n65536", n, np.concatenate([x, y]), g, 0.005 ** 2)


def config3(n: int = 1 << 20, seed: int = 3) -> Workload:
    """BASELINE configs[2]: two Gaussian patches σ = 0.15 at (∓0.5, 0), Γ = 2/N (each patch totals 1).
    δ unspecified in BASELINE.json → δ = 0.005."""
    rng = SplitMix64(seed)
    z = rng.normal(2 * n) * 0.15
    x, y = z[:n].copy(), z[n:].copy()
    half = n // 2
    x[:half] -= 0.5
    x[half:] += 0.5
    g = np.full(n, 2.0 / n)
    return Workload("config3_bh_n1048576", n, np.concatenate([x, y]), g, 0.005 ** 2)


def config5(n: int = 1 << 22, seed: int = 5) -> Workload:
    """BASELINE configs[4]: uniform [0,1]², Γ ~ N(0,1)/N, δ = 1e-3, 20 steps."""
    rng = SplitMix64(seed)
    x = rng.uniform(n)
    y = rng.uniform(n)
    g = rng.normal(n) / n
    return Workload("config5_sharded_fom_n4194304", n, np.concatenate([x, y]), g, 1e-3 ** 2, 1e-3, 20)
