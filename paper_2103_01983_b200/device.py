"""Device-buffer entry points over torch CUDA tensors (stream-ordered).

Thin wrappers of the ``ptrom_dev_*`` C ABI: tensors must be contiguous CUDA
tensors on the context's device; the call is enqueued on torch's current
stream and does not synchronize. A numerical failure detected on the device
(coincident pair with delta == 0, singular Newton block) is latched and
raised by :func:`synchronize`.
"""
from __future__ import annotations

from typing import Optional

import torch

from .api import Context, default_context


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("device entry points take contiguous CUDA tensors")
    return t.data_ptr()


def _ctx(ctx: Optional[Context], t: torch.Tensor) -> Context:
    ctx = ctx or default_context(t.device.index or 0)
    ctx.set_stream(torch.cuda.current_stream(t.device).cuda_stream)
    return ctx


def pairwise_velocity(x: torch.Tensor, gamma: torch.Tensor, delta: float, form: int = 0,
                      inflow: Optional[torch.Tensor] = None, t_begin: int = 0, t_end: Optional[int] = None,
                      out: Optional[torch.Tensor] = None, ctx: Optional[Context] = None) -> torch.Tensor:
    """kernel.hpp:107-129 for target rows [t_begin, t_end): out is (2, m) so
    row k holds chi/psi velocity of particle t_begin + k (ld = m)."""
    n = gamma.shape[0]
    t_end = n if t_end is None else t_end
    m = t_end - t_begin
    if out is None:
        out = torch.empty(2 * m, dtype=x.dtype, device=x.device)
    ctx = _ctx(ctx, x)
    if x.dtype == torch.float32:
        fn = ctx.lib.ptrom_dev_pairwise_velocity_f32
    elif x.dtype == torch.float64:
        fn = ctx.lib.ptrom_dev_pairwise_velocity_f64
    else:
        raise ValueError("pairwise_velocity: float32 or float64 state expected")
    ctx.check(fn(ctx.handle, n, _ptr(x), _ptr(gamma), float(delta), int(form), _ptr(inflow), t_begin, t_end,
                 _ptr(out), m))
    return out


def fom_simulate(x0: torch.Tensor, gamma: torch.Tensor, delta: float, dt: float, n_steps: int, form: int = 0,
                 inflow: Optional[torch.Tensor] = None, tol: float = 1e-10, max_iters: int = 100, refresh: int = 1,
                 snapshots: Optional[torch.Tensor] = None, ctx: Optional[Context] = None):
    """integrators.hpp:243-272 on device-resident state (ptrom_dev_fom_simulate_f64):
    returns (snapshots (n_steps, 2n) on the device, iterations, converged,
    relative_residual, velocity evaluations, Jacobian evaluations). Synchronizes."""
    import ctypes as C

    import numpy as np
    n = gamma.shape[0]
    if snapshots is None:
        snapshots = torch.empty(max(n_steps, 1), 2 * n, dtype=torch.float64, device=x0.device)
    it = np.zeros(max(n_steps, 1), np.int32)
    cv = np.zeros(max(n_steps, 1), np.uint8)
    rr = np.zeros(max(n_steps, 1), np.float64)
    nv, nj = C.c_uint64(), C.c_uint64()
    ctx = _ctx(ctx, x0)
    ctx.check(ctx.lib.ptrom_dev_fom_simulate_f64(ctx.handle, n, _ptr(x0), _ptr(gamma), float(delta), int(form),
                                                 _ptr(inflow), float(dt), int(n_steps), float(tol), int(max_iters),
                                                 int(refresh), _ptr(snapshots), it.ctypes.data, cv.ctypes.data,
                                                 rr.ctypes.data, C.byref(nv), C.byref(nj)))
    return snapshots[:n_steps], it[:n_steps], cv[:n_steps], rr[:n_steps], nv.value, nj.value


def inexact_kernel_jacobian(x: torch.Tensor, gamma: torch.Tensor, delta: float, form: int = 0, t_begin: int = 0,
                            t_end: Optional[int] = None, ctx: Optional[Context] = None) -> torch.Tensor:
    """kernel.hpp:154-170 rows [t_begin, t_end) → (4, m): dfx_dx, dfx_dy, dfy_dx, dfy_dy."""
    n = gamma.shape[0]
    t_end = n if t_end is None else t_end
    m = t_end - t_begin
    out = torch.empty(4, m, dtype=torch.float64, device=x.device)
    ctx = _ctx(ctx, x)
    ctx.check(ctx.lib.ptrom_dev_inexact_kernel_jacobian_f64(ctx.handle, n, _ptr(x), _ptr(gamma), float(delta),
                                                            int(form), t_begin, t_end, out[0].data_ptr(),
                                                            out[1].data_ptr(), out[2].data_ptr(),
                                                            out[3].data_ptr()))
    return out


def newton_blocks(x: torch.Tensor, gamma: torch.Tensor, delta: float, form: int, dt: float, t_begin: int,
                  t_end: int, out: torch.Tensor, ctx: Optional[Context] = None) -> torch.Tensor:
    """integrators.hpp:181-194 refactor for rows [t_begin, t_end): out (m, 4)."""
    n = gamma.shape[0]
    ctx = _ctx(ctx, x)
    ctx.check(ctx.lib.ptrom_dev_newton_blocks_f64(ctx.handle, n, _ptr(x), _ptr(gamma), float(delta), int(form),
                                                  float(dt), t_begin, t_end, _ptr(out)))
    return out


def residual(xi, fxi, xprev, fprev, dt: float, r: torch.Tensor, norm2: torch.Tensor, m: int, ld: int,
             ctx: Optional[Context] = None) -> None:
    """integrators.hpp:47-53 on m local rows (k, k+ld); norm2 gets Σ r² (fixed order)."""
    ctx = _ctx(ctx, xi)
    ctx.check(ctx.lib.ptrom_dev_residual_f64(ctx.handle, m, ld, _ptr(xi), _ptr(fxi), _ptr(xprev), _ptr(fprev),
                                             float(dt), _ptr(r), _ptr(norm2)))


def newton_update(inv: torch.Tensor, r: torch.Tensor, x: torch.Tensor, m: int, ld: int,
                  ctx: Optional[Context] = None) -> None:
    """integrators.hpp:161-167 on m local rows."""
    ctx = _ctx(ctx, x)
    ctx.check(ctx.lib.ptrom_dev_newton_update_f64(ctx.handle, m, ld, _ptr(inv), _ptr(r), _ptr(x)))


def hamiltonian(x: torch.Tensor, gamma: torch.Tensor, out: Optional[torch.Tensor] = None,
                ctx: Optional[Context] = None) -> torch.Tensor:
    """kernel.hpp:174-191 on device; out is a 1-element float64 tensor."""
    n = gamma.shape[0]
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=x.device)
    ctx = _ctx(ctx, x)
    ctx.check(ctx.lib.ptrom_dev_hamiltonian_f64(ctx.handle, n, _ptr(x), _ptr(gamma), _ptr(out)))
    return out


def velocity_field_grid(x: torch.Tensor, gamma: torch.Tensor, delta: float, form: int, lattice, c_g: float,
                        l: float, gamma_bar: float, ctx: Optional[Context] = None) -> torch.Tensor:
    """kernel.hpp:213-238 on device → (ny, nx) tensor (a transposed view of the column-major grid)."""
    n = gamma.shape[0]
    nx, ny = int(lattice.nx), int(lattice.ny)
    grid = torch.empty(nx, ny, dtype=torch.float64, device=x.device)
    ctx = _ctx(ctx, x)
    ctx.check(ctx.lib.ptrom_dev_velocity_field_grid_f64(
        ctx.handle, n, _ptr(x), _ptr(gamma), float(delta), int(form), float(lattice.x_min), float(lattice.x_max),
        nx, float(lattice.y_min), float(lattice.y_max), ny, float(c_g), float(l), float(gamma_bar), _ptr(grid)))
    return grid.t()


def synchronize(ctx: Optional[Context] = None, device: int = 0) -> None:
    (ctx or default_context(device)).synchronize()
