"""Multi-GPU communicator and sharded drivers — a thin mirror of the C ABI
(include/ptrom_b200.h "multi-GPU", csrc/comm.cu, csrc/rom_capi.cu).

SURVEY.md §8b asks for ``ptrom_comm_init`` plus ``*_sharded`` variants of the
FOM and of the PTROM batch, so a C++ host can shard without Python. Here:

* :class:`Comm` wraps one ``ptrom_comm`` per rank:
  - ``Comm.nccl(ctx, group)``: rank 0's ``ptrom_comm_unique_id`` is shared
    through torch.distributed, then every rank calls ``ptrom_comm_init``
    (NCCL over NVLink / NVSwitch);
  - ``Comm.host(ctx, group)``: ``ptrom_comm_init_host`` with all-gather and
    broadcast callbacks over a torch.distributed group (gloo), for hosts that
    bring their own transport — and for the two-process tests on one GPU,
    where the collectives block on the host, never inside a kernel.
* :func:`fom_simulate_sharded` → ``ptrom_fom_simulate_sharded_f64``
  (integrators.hpp:243-272 with the targets split across ranks).
* :func:`ptrom_simulate_batch_sharded` → ``ptrom_ptrom_simulate_batch_sharded_f64``
  (rom.hpp:404-412 batched; instances split, shared tables broadcast once).
* :func:`barnes_hut_velocity_sharded` → ``ptrom_barnes_hut_velocity_sharded_f64``
  (BarnesHutModel velocity; replicated build, tree slots split, slot blocks
  all-gathered).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .api import Context, NewtonConfig, ParticleSystem, TimeGrid, _p, default_context


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)

ALL_GATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int)


class HostCollectives(C.Structure):
    _fields_ = [("all_gather", ALL_GATHER_FN), ("broadcast", BROADCAST_FN)]


def torch_host_collectives(group=None):
    """ptrom_host_collectives over a torch.distributed group (gloo): the C
    library calls these with raw host pointers. Returns (struct, keep-alive)."""
    import sys
    import traceback

    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def all_gather(_user, send, recv, nbytes):
        try:
            src = torch.zeros(nbytes, dtype=torch.uint8)
            if nbytes:
                C.memmove(src.data_ptr(), send, nbytes)
            outs = [torch.zeros(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            for r, o in enumerate(outs):
                if nbytes:
                    C.memmove(recv + r * nbytes, o.data_ptr(), nbytes)
            return 0
        except Exception:
            traceback.print_exc(file=sys.stderr)
            return 1

    def broadcast(_user, buf, nbytes, root):
        try:
            if not nbytes:
                return 0
            t = torch.zeros(nbytes, dtype=torch.uint8)
            C.memmove(t.data_ptr(), buf, nbytes)
            dist.broadcast(t, src=root, group=group)
            C.memmove(buf, t.data_ptr(), nbytes)
            return 0
        except Exception:
            traceback.print_exc(file=sys.stderr)
            return 1

    ag, bc = ALL_GATHER_FN(all_gather), BROADCAST_FN(broadcast)
    ops = HostCollectives(ag, bc)
    return ops, (ag, bc, ops)


class Comm:
    """One rank's ptrom_comm (see the module docstring)."""

    def __init__(self, ctx: Context, handle, rank: int, world: int, keep=()):
        self.ctx, self._h, self.rank, self.world = ctx, handle, rank, world
        self._keep = keep  # ctypes callbacks must outlive the communicator

    @property
    def handle(self):
        return self._h

    @property
    def transport(self) -> str:
        return "nccl" if self.ctx.lib.ptrom_comm_transport(self._h) == 1 else "host"

    @staticmethod
    def nccl(ctx: Optional[Context] = None, group=None, rank: Optional[int] = None,
             world: Optional[int] = None) -> "Comm":
        """NCCL communicator; without torch.distributed only world = 1 works."""
        ctx = ctx or default_context()
        uid = (C.c_uint8 * 128)()
        if rank is None:
            import torch.distributed as dist
            if dist.is_initialized():
                rank, world = dist.get_rank(group), dist.get_world_size(group)
            else:
                rank, world = 0, 1
        if rank == 0:
            ctx.check(ctx.lib.ptrom_comm_unique_id(uid))
        if world > 1:
            import torch.distributed as dist
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        ctx.check(ctx.lib.ptrom_comm_init(ctx.handle, int(rank), int(world), uid, C.byref(h)))
        return Comm(ctx, h, rank, world)

    @staticmethod
    def host(ctx: Optional[Context] = None, group=None) -> "Comm":
        """Host-transport communicator over a torch.distributed (gloo) group."""
        import torch.distributed as dist
        ctx = ctx or default_context()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        ops, keep = torch_host_collectives(group)
        h = C.c_void_p()
        ctx.check(ctx.lib.ptrom_comm_init_host(ctx.handle, rank, world, C.byref(ops), None, C.byref(h)))
        return Comm(ctx, h, rank, world, keep=keep)

    def bounds(self, count: int) -> tuple[int, int]:
        return count * self.rank // self.world, count * (self.rank + 1) // self.world

    def close(self) -> None:
        if self._h:
            self.ctx.lib.ptrom_comm_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ShardedFomResult:
    snapshots_local: np.ndarray  # (2m, n_steps): rows [x_lo..x_hi-1, y_lo..y_hi-1]
    iterations: np.ndarray
    converged: np.ndarray
    relative_residual: np.ndarray
    lo: int
    hi: int
    pair_evals: int


def fom_simulate_sharded(comm: Comm, x0, system: ParticleSystem, grid: TimeGrid,
                         newton: Optional[NewtonConfig] = None) -> ShardedFomResult:
    """ptrom_fom_simulate_sharded_f64: every rank passes the full x0 and gets its rows."""
    newton = newton or NewtonConfig()
    ctx = comm.ctx
    x = _f64(x0)
    g = _f64(system.circulation)
    n = g.shape[0]
    lo, hi = comm.bounds(n)
    m = hi - lo
    steps = int(grid.n_steps)
    snaps = np.zeros((max(steps, 1), 2 * m))
    it = np.zeros(max(steps, 1), np.int32)
    cv = np.zeros(max(steps, 1), np.uint8)
    rr = np.zeros(max(steps, 1))
    inflow = None if system.inflow is None else _f64(system.inflow)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_fom_simulate_sharded_f64(
        ctx.handle, comm.handle, n, _p(x), _p(g), float(system.delta), int(system.kernel_form), _p(inflow),
        float(grid.dt), steps, float(newton.tol), int(newton.max_iters), int(newton.jacobian_refresh_period),
        _p(snaps), _p(it), _p(cv), _p(rr), C.byref(cnt)))
    return ShardedFomResult(snaps[:steps].T.copy(), it[:steps], cv[:steps], rr[:steps], lo, hi, cnt.value)


def barnes_hut_velocity_sharded(comm: Comm, x, system: ParticleSystem, criterion, leaf_capacity: int = 32):
    """ptrom_barnes_hut_velocity_sharded_f64: every rank passes the full state
    and gets the full velocity (2n) and the summed pair count."""
    ctx = comm.ctx
    xs = _f64(x)
    g = _f64(system.circulation)
    n = g.shape[0]
    f = np.zeros(2 * n)
    inflow = None if system.inflow is None else _f64(system.inflow)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_barnes_hut_velocity_sharded_f64(
        ctx.handle, comm.handle, n, _p(xs), _p(g), float(system.delta), int(system.kernel_form),
        int(criterion.kind), float(criterion.value), int(leaf_capacity), _p(inflow), _p(f), C.byref(cnt)))
    return f, cnt.value


def ptrom_simulate_batch_sharded(comm: Comm, basis, op, sur, gamma_a, gamma_b, mu, system: ParticleSystem,
                                 grid: TimeGrid, cfg, batch: int = 0, root: int = 0):
    """ptrom_ptrom_simulate_batch_sharded_f64: basis/op/sur/Γ/μ needed on root
    only (None elsewhere); returns the gathered trajectory on every rank."""
    from .rom import RomTrajectory
    ctx = comm.ctx
    is_root = comm.rank == root
    ga = _f64(gamma_a) if is_root else None
    gb = _f64(gamma_b) if is_root else None
    mus = _f64(mu) if is_root else None
    inflow = None if (not is_root or system.inflow is None) else _f64(system.inflow)
    n = int(ga.shape[0]) if is_root else 0
    n_inst = int(mus.shape[0]) if is_root else 0
    box = np.array([n, n_inst, basis.modes() if is_root else 0], np.int64)
    if comm.world > 1:  # output sizes for the non-root ranks (the library broadcasts the rest)
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(box)
        dist.broadcast(t, src=root)
        box = t.numpy()
    n, n_inst, m = (int(v) for v in box)
    steps = int(grid.n_steps)
    xh = np.zeros((n_inst, max(steps, 1), m))
    it = np.zeros((n_inst, max(steps, 1)), np.int32)
    cv = np.zeros((n_inst, max(steps, 1)), np.uint8)
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_ptrom_simulate_batch_sharded_f64(
        ctx.handle, comm.handle, int(root), basis._h if is_root else None, op._h if is_root else None,
        sur._h if is_root else None, n, _p(ga), _p(gb), n_inst, _p(mus), int(batch), float(system.delta),
        int(system.kernel_form), _p(inflow), float(grid.dt), steps, float(cfg.tol), int(cfg.max_iters),
        float(cfg.step_length), _p(xh), _p(it), _p(cv), C.byref(cnt)))
    return RomTrajectory(xh[:, :steps], it[:, :steps], cv[:, :steps])
