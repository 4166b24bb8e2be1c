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


@dataclass
class PtromWorkload:
    """BASELINE configs[3] inputs."""
    name: str
    n: int
    x0: np.ndarray         # reference state x_ref (SoA)
    gamma_a: np.ndarray    # Γ(μ) = gamma_a + μ·gamma_b  (patch A fixed, patch B scaled by μ)
    gamma_b: np.ndarray
    phi: np.ndarray        # 2N x M POD basis (column-major / Fortran order)
    sv: np.ndarray         # M singular values (weighted POD space, reduction.hpp:74-77)
    phi_r: np.ndarray      # 2N x M_r residual basis
    mu: np.ndarray         # instance parameters
    delta: float
    dt: float
    n_steps: int
    n_samples: int


def _orthonormal(a: np.ndarray) -> np.ndarray:
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))[None, :]
    return np.asfortranarray(q)


N_FIELDS = 24      # smooth Fourier displacement fields in the snapshot family
N_SNAPSHOTS = 200


def pod_of_snapshots(x0: np.ndarray, fields: np.ndarray, amps: np.ndarray, modes: int):
    """build_pod (reduction.hpp:32-66) of the snapshot matrix
    S = x0·1ᵀ + 1e-2·F·Aᵀ (columns s = x0 + 1e-2·Σ_k a_ks F_k), computed
    without forming the 2N x n_s matrix: S = B Cᵀ with B = [x0, F] and
    C = [1, 1e-2·A], so with B = Q_B R_B, S = Q_B (R_B Cᵀ) and the thin SVD of
    the small (K+1) x n_s factor gives U = Q_B Û and σ. The numerical-rank
    check and the sign rule (largest-magnitude entry positive, first on ties)
    are the reference's."""
    b = np.concatenate([x0[:, None], fields], axis=1)
    c = np.concatenate([np.ones((amps.shape[0], 1)), 1e-2 * amps], axis=1)
    qb, rb = np.linalg.qr(b)
    uh, sv, _ = np.linalg.svd(rb @ c.T, full_matrices=False)
    cutoff = max(x0.shape[0], amps.shape[0]) * np.finfo(np.float64).eps * sv[0]
    rank = int(np.sum(sv > cutoff))
    if modes > rank:
        raise ValueError(f"build_pod: requested {modes} modes but snapshots have numerical rank {rank}")
    phi = qb @ uh[:, :modes]
    for c_ in range(modes):
        arg = int(np.argmax(np.abs(phi[:, c_])))
        if phi[arg, c_] < 0:
            phi[:, c_] = -phi[:, c_]
    return np.asfortranarray(phi), sv[:modes].copy()


def config4(n: int = 1 << 20, n_inst: int = 4096, modes: int = 16, modes_r: int = 32, n_steps: int = 50,
            seed: int = 4) -> PtromWorkload:
    """Two patches as config 3; Γ(μ) = 2/N on patch A and μ·2/N on patch B, μ ~ U[0.5, 2] (seeded).

    Φ: the M-mode POD (build_pod, reduction.hpp:32-66)
    of 200 seeded snapshots x0 + 1e-2·Σ_k a_ks·F_k over 24 smooth Fourier
    displacement fields F_k = (cos(a·x + b·y + φ), sin(c·x + e·y + ψ)) with
    seeded wavenumbers in [-3π, 3π] and seeded phases, amplitudes
    a_ks ~ N(0, 1)/k (a decaying spectrum); σ are the snapshot matrix's own
    singular values (they weight the POD space W = Φσ the surrogate tree is
    built on, reduction.hpp:74-77). Φ_r: seeded random orthonormal 2N x M_r
    (as test_rom.cpp:50-58). Samples n = ceil(0.02 N)."""
    base = config3(n, seed=3)
    rng = SplitMix64(seed)
    x, y = base.x0[:n], base.x0[n:]
    half = n // 2
    ga = np.zeros(n)
    gb = np.zeros(n)
    ga[:half] = 2.0 / n
    gb[half:] = 2.0 / n
    nf = max(N_FIELDS, modes + 8)
    waves = rng.uniform(4 * nf) * 6.0 - 3.0
    phases = rng.uniform(2 * nf) * 2.0 * np.pi
    fields = np.empty((2 * n, nf))
    for k in range(nf):
        a, b, c, e = waves[4 * k:4 * k + 4] * np.pi
        fields[:n, k] = np.cos(a * x + b * y + phases[2 * k])
        fields[n:, k] = np.sin(c * x + e * y + phases[2 * k + 1])
    amps = rng.normal(N_SNAPSHOTS * nf).reshape(N_SNAPSHOTS, nf) / np.arange(1, nf + 1)[None, :]
    phi, sv = pod_of_snapshots(base.x0, fields, amps, modes)
    phi_r = _orthonormal(rng.normal(2 * n * modes_r).reshape(modes_r, 2 * n).T)
    mu = 0.5 + 1.5 * rng.uniform(n_inst)
    return PtromWorkload("config4_ptrom_n%d" % n, n, base.x0.copy(), ga, gb, phi, sv, phi_r, mu, 0.005 ** 2, 1e-3,
                         n_steps, int(np.ceil(0.02 * n)))
