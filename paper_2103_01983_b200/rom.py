"""Host mirror of the reference's PTROM online interface over the C ABI
(reduction.hpp:18-431, rom.hpp:17-412); every computation runs on the B200.

    PODBasis(phi, singular_values, x_ref)          reduction.hpp:18-26
    GnatOperator(basis, sample_ids, A)             reduction.hpp:173-180
    SurrogateSourceBasis.from_tables(...)          reduction.hpp:280-302
      .reassign_cluster_circulation(gamma, basis)  reduction.hpp:400-431
    hyperpair(surrogate, target_positions, x_hat, sys)          rom.hpp:101-155
    RomConfig / RomTrajectory                                    rom.hpp:17-41
    ptrom_simulate(basis, op, surrogate, sys, grid, cfg)        rom.hpp:404-412
    ptrom_simulate_batch(basis, op, surrogate, gamma_a, gamma_b, mu, sys, grid, cfg)
        batched online queries for Γ(μ) = gamma_a + μ·gamma_b
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .api import BlockDiagonalJacobian, ConfigError, Context, ParticleSystem, TimeGrid, _bump, default_context


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _fortran(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class PODBasis:  # reduction.hpp:18-26
    def __init__(self, phi, singular_values, x_ref, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.phi = _fortran(phi)
        self.singular_values = _f64(singular_values)
        self.x_ref = _f64(x_ref)
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ptrom_basis_create(self.ctx.handle, self.phi.shape[0], self.phi.shape[1],
                                                       _p(self.phi), _p(self.singular_values), _p(self.x_ref),
                                                       C.byref(h)))
        self._h = h
        self._shape = self.phi.shape

    @classmethod
    def adopt(cls, ctx: Context, handle, n_dofs: int, modes: int) -> "PODBasis":
        """Wraps a device basis the library built (ptrom_bundle_to_device); no host copy."""
        b = cls.__new__(cls)
        b.ctx, b._h, b._shape = ctx, handle, (int(n_dofs), int(modes))
        b.phi = b.singular_values = b.x_ref = None
        return b

    def dim(self):
        return self._shape[0]

    def modes(self):
        return self._shape[1]

    def reconstruct_output(self, x_hat, dofs=None) -> np.ndarray:
        """rom.hpp:45-58 (dofs given) / rom.hpp:60-64 reconstruct_full (dofs None), on the device."""
        xh = _fortran(x_hat)
        if xh.ndim == 1:
            xh = xh.reshape(-1, 1, order="F")
        if xh.shape[0] != self.modes():
            raise ConfigError("reconstruct_output: coordinate dimension mismatch")
        d = None if dofs is None else _i64(dofs)
        n_out = self.dim() if d is None else d.shape[0]
        out = np.zeros((n_out, xh.shape[1]), order="F")
        self.ctx.check(self.ctx.lib.ptrom_reconstruct_output_f64(self.ctx.handle, self._h, xh.shape[1], _p(xh),
                                                                 0 if d is None else d.shape[0], _p(d), _p(out)))
        return out

    def reconstruct_full(self, x_hat) -> np.ndarray:
        return self.reconstruct_output(x_hat, None)

    def __del__(self):
        try:
            self.ctx.lib.ptrom_basis_free(self._h)
        except Exception:
            pass


class GnatOperator:  # reduction.hpp:173-180
    def __init__(self, basis: PODBasis, sample_ids, A):
        self.ctx = basis.ctx
        self.sample_ids = _i64(sample_ids)
        self.A = _fortran(A)
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ptrom_gnat_op_create(self.ctx.handle, basis._h, self.sample_ids.shape[0],
                                                         _p(self.sample_ids), self.A.shape[0], _p(self.A),
                                                         C.byref(h)))
        self._h = h

    @classmethod
    def adopt(cls, ctx: Context, handle, sample_ids) -> "GnatOperator":
        """Wraps a device operator the library built (ptrom_bundle_to_device)."""
        g = cls.__new__(cls)
        g.ctx, g._h, g.sample_ids, g.A = ctx, handle, _i64(sample_ids), None
        return g

    def __del__(self):
        try:
            self.ctx.lib.ptrom_gnat_op_free(self._h)
        except Exception:
            pass


class SurrogateSourceBasis:  # reduction.hpp:280-302
    def __init__(self, ctx, h, modes, n_clusters, n_direct, n_targets, target_ids):
        self.ctx, self._h = ctx, h
        self.m, self.n_clusters, self.n_direct, self.n_targets = modes, n_clusters, n_direct, n_targets
        self.target_ids = target_ids

    @staticmethod
    def from_tables(phi_tilde, gamma_tilde, x0_tilde, zero_gamma, mem_off, mem_ids, target_ids, cl_off, cl_list,
                    direct_ids, direct_phi, direct_x0, direct_gamma, d_off, d_list,
                    ctx: Optional[Context] = None) -> "SurrogateSourceBasis":
        ctx = ctx or default_context()
        pt_, dp = _fortran(phi_tilde), _fortran(direct_phi)
        arrs = [pt_, _f64(gamma_tilde), _f64(x0_tilde), np.ascontiguousarray(zero_gamma, dtype=np.uint8),
                _i64(mem_off), _i64(mem_ids), _i64(target_ids), _i64(cl_off), _i64(cl_list), _i64(direct_ids), dp,
                _f64(direct_x0), _f64(direct_gamma), _i64(d_off), _i64(d_list)]
        m = pt_.shape[1] if pt_.ndim == 2 else dp.shape[1]
        nc = arrs[1].shape[0]
        nt = arrs[6].shape[0]
        u = arrs[9].shape[0]
        h = C.c_void_p()
        ctx.check(ctx.lib.ptrom_surrogate_create(ctx.handle, m, nc, _p(arrs[0]), _p(arrs[1]), _p(arrs[2]),
                                                 _p(arrs[3]), _p(arrs[4]), _p(arrs[5]), nt, _p(arrs[6]), _p(arrs[7]),
                                                 _p(arrs[8]), u, _p(arrs[9]), _p(arrs[10]), _p(arrs[11]),
                                                 _p(arrs[12]), _p(arrs[13]), _p(arrs[14]), C.byref(h)))
        return SurrogateSourceBasis(ctx, h, m, nc, u, nt, arrs[6])

    @staticmethod
    def cluster_pod(basis: PODBasis, gamma, target_ids, criterion, leaf_capacity: int = 1) -> "SurrogateSourceBasis":
        """reduction.hpp:388-395: weighted POD tree + cluster_pod, on the device."""
        ctx = basis.ctx
        g, t = _f64(gamma), _i64(target_ids)
        h = C.c_void_p()
        ctx.check(ctx.lib.ptrom_cluster_pod_f64(ctx.handle, basis._h, _p(g), int(leaf_capacity), criterion.kind,
                                                criterion.value, t.shape[0], _p(t), C.byref(h)))
        sz = np.zeros(6, np.int64)
        ctx.check(ctx.lib.ptrom_surrogate_sizes(h, _p(sz)))
        return SurrogateSourceBasis(ctx, h, basis.modes(), int(sz[0]), int(sz[1]), int(sz[2]), t)

    def export_lists(self) -> dict:
        sz = np.zeros(6, np.int64)
        self.ctx.check(self.ctx.lib.ptrom_surrogate_sizes(self._h, _p(sz)))
        nc, u, nt, nm, ncl, ndl = (int(v) for v in sz)
        out = dict(cluster_node_ids=np.zeros(nc, np.int32), mem_off=np.zeros(nc + 1, np.int64),
                   mem_ids=np.zeros(max(nm, 1), np.int64), cl_off=np.zeros(nt + 1, np.int64),
                   cl_list=np.zeros(max(ncl, 1), np.int64), direct_ids=np.zeros(max(u, 1), np.int64),
                   d_off=np.zeros(nt + 1, np.int64), d_list=np.zeros(max(ndl, 1), np.int64),
                   direct_phi=np.zeros((2 * u, self.m), order="F"), direct_x0=np.zeros(2 * u))
        self.ctx.check(self.ctx.lib.ptrom_surrogate_export_lists(self.ctx.handle, self._h, *(_p(out[k]) for k in (
            "cluster_node_ids", "mem_off", "mem_ids", "cl_off", "cl_list", "direct_ids", "d_off", "d_list",
            "direct_phi", "direct_x0"))))
        out["mem_ids"], out["cl_list"], out["d_list"] = out["mem_ids"][:nm], out["cl_list"][:ncl], out["d_list"][:ndl]
        out["direct_ids"] = out["direct_ids"][:u]
        return out

    def export(self) -> dict:
        nc, u, m = self.n_clusters, self.n_direct, self.m
        out = dict(phi_tilde=np.zeros((2 * nc, m), order="F"), gamma_tilde=np.zeros(nc), x0_tilde=np.zeros(2 * nc),
                   zero_gamma=np.zeros(nc, np.uint8), direct_gamma=np.zeros(u))
        self.ctx.check(self.ctx.lib.ptrom_surrogate_export(self.ctx.handle, self._h, *(_p(out[k]) for k in (
            "phi_tilde", "gamma_tilde", "x0_tilde", "zero_gamma", "direct_gamma"))))
        return out

    def reassign_cluster_circulation(self, gamma, basis: PODBasis) -> None:
        g = _f64(gamma)
        self.ctx.check(self.ctx.lib.ptrom_reassign_cluster_circulation_f64(self.ctx.handle, self._h, g.shape[0],
                                                                            _p(g), basis._h))

    def __del__(self):
        try:
            self.ctx.lib.ptrom_surrogate_free(self._h)
        except Exception:
            pass


@dataclass
class HyperpairResult:  # rom.hpp:94-99
    f: np.ndarray
    jac: BlockDiagonalJacobian
    cluster_positions: np.ndarray
    direct_positions: np.ndarray


def greedy_sample(phi_r, n_target: int, preseed=(), ctx: Optional[Context] = None) -> np.ndarray:
    """reduction.hpp:93-168 (device scoring and selection)."""
    ctx = ctx or default_context()
    pr = _fortran(phi_r)
    pre = _i64(list(preseed))
    out = np.zeros(int(n_target), np.int64)
    ctx.check(ctx.lib.ptrom_greedy_sample_f64(ctx.handle, pr.shape[0], pr.shape[1], _p(pr), int(n_target),
                                              pre.shape[0], _p(pre), _p(out)))
    return out


def build_gnat_operator(phi_r, sample_ids, ctx: Optional[Context] = None) -> np.ndarray:
    """reduction.hpp:182-220 → A = pinv(P Φ_r) (m_r x 2 n_s)."""
    ctx = ctx or default_context()
    pr = _fortran(phi_r)
    ids = _i64(sample_ids)
    A = np.zeros((pr.shape[1], 2 * ids.shape[0]), order="F")
    ctx.check(ctx.lib.ptrom_build_gnat_operator_f64(ctx.handle, pr.shape[0], pr.shape[1], _p(pr), ids.shape[0],
                                                    _p(ids), _p(A)))
    return A


def hyperpair(sur: SurrogateSourceBasis, target_positions, x_hat, sys: ParticleSystem) -> HyperpairResult:
    tp, xh, inflow = _f64(target_positions), _f64(x_hat), _f64(sys.inflow)
    nt = sur.n_targets
    if tp.shape[0] != 2 * nt:
        raise ConfigError("hyperpair: target position vector has wrong length")
    f = np.zeros(2 * nt)
    jac = np.zeros((4, nt))
    cpos = np.zeros(2 * sur.n_clusters)
    dpos = np.zeros(2 * sur.n_direct)
    cnt = C.c_uint64()
    n = sys.size()
    sur.ctx.check(sur.ctx.lib.ptrom_hyperpair_f64(sur.ctx.handle, sur._h, _p(tp), _p(xh), float(sys.delta),
                                                  int(sys.kernel_form), n, _p(inflow), _p(f), _p(jac), _p(cpos),
                                                  _p(dpos), C.byref(cnt)))
    _bump(cnt.value)
    return HyperpairResult(f, BlockDiagonalJacobian(*jac), cpos, dpos)


@dataclass
class RomConfig:  # rom.hpp:17-27
    tol: float = 1e-4
    max_iters: int = 100
    step_length: float = 1.0


@dataclass
class RomTrajectory:  # rom.hpp:29-41
    x_hat: np.ndarray  # M x n_steps (single) or n_inst x n_steps x M (batch)
    iterations: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    converged: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    def all_converged(self) -> bool:
        return bool(np.all(self.converged))


def ptrom_simulate(basis: PODBasis, op: GnatOperator, sur: SurrogateSourceBasis, sys: ParticleSystem,
                   grid: TimeGrid, cfg: RomConfig = RomConfig()) -> RomTrajectory:
    """rom.hpp:404-412 — reassigns the surrogate in place, then marches on the device."""
    ctx = sur.ctx
    g, inflow = _f64(sys.circulation), _f64(sys.inflow)
    m, steps = basis.modes(), int(grid.n_steps)
    x_hat = np.zeros((m, steps), order="F")
    iters = np.zeros(steps, np.int32)
    conv = np.zeros(steps, np.uint8)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_ptrom_simulate_f64(ctx.handle, basis._h, op._h, sur._h, g.shape[0], _p(g),
                                               float(sys.delta), int(sys.kernel_form), _p(inflow), float(grid.dt),
                                               steps, float(cfg.tol), int(cfg.max_iters), float(cfg.step_length),
                                               _p(x_hat), _p(iters), _p(conv), C.byref(cnt)))
    _bump(cnt.value)
    return RomTrajectory(x_hat, iters, conv)


def ptrom_simulate_batch(basis: PODBasis, op: GnatOperator, sur: SurrogateSourceBasis, gamma_a, gamma_b, mu,
                         sys: ParticleSystem, grid: TimeGrid, cfg: RomConfig = RomConfig(),
                         batch: int = 0) -> RomTrajectory:
    """Online queries for Γ(μ) = gamma_a + μ·gamma_b, all instances on the device."""
    ctx = sur.ctx
    ga, gb, mu_, inflow = _f64(gamma_a), _f64(gamma_b), _f64(mu), _f64(sys.inflow)
    m, steps, ni = basis.modes(), int(grid.n_steps), mu_.shape[0]
    x_hat = np.zeros((ni, steps, m))
    iters = np.zeros((ni, steps), np.int32)
    conv = np.zeros((ni, steps), np.uint8)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_ptrom_simulate_batch_f64(ctx.handle, basis._h, op._h, sur._h, ga.shape[0], _p(ga), _p(gb),
                                                     ni, _p(mu_), int(batch), float(sys.delta), int(sys.kernel_form),
                                                     _p(inflow), float(grid.dt), steps, float(cfg.tol),
                                                     int(cfg.max_iters), float(cfg.step_length), _p(x_hat),
                                                     _p(iters), _p(conv), C.byref(cnt)))
    _bump(cnt.value)
    return RomTrajectory(x_hat, iters, conv)
