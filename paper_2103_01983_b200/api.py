"""Host-side mirror of the reference's FOM interface over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/ptrom/{types,kernel,integrators}.hpp, so code and
tests written against the reference read the same here:

    ParticleSystem        kernel.hpp:77-94
    pairwise_velocity     kernel.hpp:107-129
    inexact_kernel_jacobian / BlockDiagonalJacobian  kernel.hpp:134-170
    NewtonConfig / TimeGrid  integrators.hpp:15-23, 55-66
    PairwiseModel         integrators.hpp:69-79  (velocity / jacobian seam)
    fom_simulate          integrators.hpp:243-272 (whole trajectory on device)
    config_error / numerical_error  types.hpp:23-32

Every call runs on the B200 through libptrom_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib


class ConfigError(ValueError):
    """types.hpp:23-26 config_error (CLI exit code 2)."""


class NumericalError(ArithmeticError):
    """types.hpp:28-32 numerical_error (CLI exit code 3)."""


class CudaError(RuntimeError):
    """Device/driver failure (status 4)."""


# ptrom_b200.h status codes
OK, CONFIG, NUMERICAL, CUDA = 0, 2, 3, 4


class KernelForm:  # kernel.hpp:16
    standard = 0
    denominator_scaled = 1


# thread-local in the reference (kernel.hpp:18-25); process-wide here.
_kernel_eval_counter = 0


def kernel_eval_count() -> int:
    return _kernel_eval_counter


def reset_kernel_eval_count() -> None:
    global _kernel_eval_counter
    _kernel_eval_counter = 0


def _bump(n: int) -> None:
    global _kernel_eval_counter
    _kernel_eval_counter += int(n)


class Context:
    """One ptrom_ctx per (device, host thread); bound to a CUDA stream."""

    def __init__(self, device: int = 0, stream: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        rc = lib.ptrom_create(int(device), C.c_void_p(stream or None), C.byref(h))
        if rc != OK:
            raise CudaError(f"ptrom_create(device={device}) failed with status {rc} "
                            "(libptrom_b200 needs an sm_100a B200 GPU)")
        self._h = h
        self.device = device
        self.lib = lib

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream: int) -> None:
        self.check(self.lib.ptrom_set_stream(self._h, C.c_void_p(stream or None)))

    def synchronize(self) -> None:
        self.check(self.lib.ptrom_synchronize(self._h))

    def check(self, rc: int) -> None:
        if rc == OK:
            return
        msg = self.lib.ptrom_last_error(self._h).decode()
        if rc == CONFIG:
            raise ConfigError(msg)
        if rc == NUMERICAL:
            raise NumericalError(msg)
        raise CudaError(msg)

    def set_tuning(self, key: str, value: int) -> None:
        """Engine knobs (ptrom_set_tuning); results do not depend on them."""
        self.check(self.lib.ptrom_set_tuning(self._h, key.encode(), int(value)))

    def close(self) -> None:
        if self._h:
            self.lib.ptrom_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    ctx = _default_ctx.get(device)
    if ctx is None:
        ctx = Context(device)
        _default_ctx[device] = ctx
    return ctx


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


@dataclass
class ParticleSystem:  # kernel.hpp:77-94
    circulation: np.ndarray
    delta: float = 0.0
    inflow: Optional[np.ndarray] = None
    kernel_form: int = KernelForm.standard

    def size(self) -> int:
        return int(np.asarray(self.circulation).shape[0])


@dataclass
class BlockDiagonalJacobian:  # kernel.hpp:134-152
    dfx_dx: np.ndarray
    dfx_dy: np.ndarray
    dfy_dx: np.ndarray
    dfy_dy: np.ndarray

    def block(self, i: int) -> np.ndarray:
        return np.array([[self.dfx_dx[i], self.dfx_dy[i]], [self.dfy_dx[i], self.dfy_dy[i]]])


def _as(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def pairwise_velocity(state, sys: ParticleSystem, ctx: Optional[Context] = None) -> np.ndarray:
    """kernel.hpp:107-129 — all-pairs velocity, SoA [chi..., psi...] in and out."""
    ctx = ctx or default_context()
    dtype = np.float32 if np.asarray(state).dtype == np.float32 else np.float64
    x = _as(state, dtype)
    g = _as(sys.circulation, dtype)
    inflow = _as(sys.inflow, dtype)
    n = g.shape[0]
    if x.shape[0] != 2 * n:
        raise ConfigError(f"pairwise_velocity: state dimension {x.shape[0]} does not match particle count {n}")
    if inflow is not None and inflow.shape[0] != 2 * n:
        raise ConfigError("inflow size must be twice the particle count")
    f = np.empty(2 * n, dtype=dtype)
    cnt = C.c_uint64()
    fn = ctx.lib.ptrom_pairwise_velocity_f32 if dtype == np.float32 else ctx.lib.ptrom_pairwise_velocity_f64
    ctx.check(fn(ctx.handle, n, _p(x), _p(g), float(sys.delta), int(sys.kernel_form), _p(inflow), _p(f),
                 C.byref(cnt)))
    _bump(cnt.value)
    return f


def inexact_kernel_jacobian(state, sys: ParticleSystem, ctx: Optional[Context] = None) -> BlockDiagonalJacobian:
    """kernel.hpp:154-170 — per-particle 2x2 self blocks."""
    ctx = ctx or default_context()
    x = _as(state, np.float64)
    g = _as(sys.circulation, np.float64)
    n = g.shape[0]
    if x.shape[0] != 2 * n:
        raise ConfigError(f"inexact_kernel_jacobian: state dimension {x.shape[0]} does not match particle count {n}")
    out = [np.empty(n) for _ in range(4)]
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_inexact_kernel_jacobian_f64(ctx.handle, n, _p(x), _p(g), float(sys.delta),
                                                        int(sys.kernel_form), *(_p(o) for o in out), C.byref(cnt)))
    return BlockDiagonalJacobian(*out)


def hamiltonian(state, sys: ParticleSystem, ctx: Optional[Context] = None) -> float:
    """kernel.hpp:174-191 — Kirchhoff–Routh energy Σ_{i<j} Γi Γj log|r_ij| / 2π."""
    ctx = ctx or default_context()
    x = _as(state, np.float64)
    g = _as(sys.circulation, np.float64)
    n = g.shape[0]
    if x.shape[0] != 2 * n:
        raise ConfigError(f"hamiltonian: state dimension {x.shape[0]} does not match particle count {n}")
    out = C.c_double()
    ctx.check(ctx.lib.ptrom_hamiltonian_f64(ctx.handle, n, _p(x), _p(g), C.byref(out)))
    return out.value


@dataclass
class LatticeSpec:  # kernel.hpp:194-208
    x_min: float
    x_max: float
    nx: int
    y_min: float
    y_max: float
    ny: int

    def x_at(self, i: int) -> float:
        return self.x_min + (self.x_max - self.x_min) * float(i) / float(self.nx - 1)

    def y_at(self, j: int) -> float:
        return self.y_min + (self.y_max - self.y_min) * float(j) / float(self.ny - 1)


def velocity_field_grid(state, sys: ParticleSystem, lattice: LatticeSpec, c_g: float, l: float, gamma_bar: float,
                        ctx: Optional[Context] = None) -> np.ndarray:
    """kernel.hpp:213-238 — (ny, nx) array, entry (j, i) = |f(x_i, y_j)|·c_g·l/Γ̄."""
    ctx = ctx or default_context()
    x = _as(state, np.float64)
    g = _as(sys.circulation, np.float64)
    n = g.shape[0]
    if x.shape[0] != 2 * n:
        raise ConfigError(f"velocity_field_grid: state dimension {x.shape[0]} does not match particle count {n}")
    nx, ny = int(lattice.nx), int(lattice.ny)
    grid = np.empty(max(nx, 0) * max(ny, 0), dtype=np.float64)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_velocity_field_grid_f64(
        ctx.handle, n, _p(x), _p(g), float(sys.delta), int(sys.kernel_form), float(lattice.x_min),
        float(lattice.x_max), nx, float(lattice.y_min), float(lattice.y_max), ny, float(c_g), float(l),
        float(gamma_bar), _p(grid) if grid.size else None, C.byref(cnt)))
    _bump(cnt.value)
    return grid.reshape(nx, ny).T  # column-major (ny x nx) → [j, i]


@dataclass
class TimeGrid:  # integrators.hpp:15-23
    dt: float
    n_steps: int
    t0: float = 0.0


@dataclass
class NewtonConfig:  # integrators.hpp:55-66
    tol: float = 1e-10
    max_iters: int = 100
    jacobian_refresh_period: int = 1


@dataclass
class SimulateResult:  # integrators.hpp:226-241
    snapshots: np.ndarray  # (2N, n_steps), column s = state after step s
    iterations: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    relative_residual: list = field(default_factory=list)
    dt: float = 0.0
    t0: float = 0.0

    def all_converged(self) -> bool:
        return all(bool(c) for c in self.converged)


@dataclass
class PairwiseModel:  # integrators.hpp:69-79
    sys: ParticleSystem

    def velocity(self, x):
        return pairwise_velocity(x, self.sys)

    def jacobian(self, x):
        return inexact_kernel_jacobian(x, self.sys)


def fom_simulate(x0, model_or_sys, grid: TimeGrid, cfg: NewtonConfig = NewtonConfig(),
                 ctx: Optional[Context] = None) -> SimulateResult:
    """integrators.hpp:243-272 for the PairwiseModel: the whole implicit-
    trapezoidal / inexact-Newton march runs on the device."""
    ctx = ctx or default_context()
    sys = model_or_sys.sys if isinstance(model_or_sys, PairwiseModel) else model_or_sys
    x = _as(x0, np.float64)
    g = _as(sys.circulation, np.float64)
    inflow = _as(sys.inflow, np.float64)
    n = g.shape[0]
    if x.shape[0] != 2 * n:
        raise ConfigError(f"pairwise_velocity: state dimension {x.shape[0]} does not match particle count {n}")
    steps = int(grid.n_steps)
    snaps = np.empty((max(steps, 0), 2 * n), dtype=np.float64)  # row s = column s of the reference matrix
    iters = np.zeros(max(steps, 0), dtype=np.int32)
    conv = np.zeros(max(steps, 0), dtype=np.uint8)
    rel = np.zeros(max(steps, 0), dtype=np.float64)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_fom_simulate_f64(ctx.handle, n, _p(x), _p(g), float(sys.delta), int(sys.kernel_form),
                                             _p(inflow), float(grid.dt), steps, float(cfg.tol), int(cfg.max_iters),
                                             int(cfg.jacobian_refresh_period), _p(snaps), _p(iters), _p(conv),
                                             _p(rel), C.byref(cnt)))
    _bump(cnt.value)
    return SimulateResult(snaps.T, iters.tolist(), conv.tolist(), rel.tolist(), grid.dt, grid.t0)
