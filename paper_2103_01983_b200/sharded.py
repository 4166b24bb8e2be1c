"""Multi-GPU drivers, one process per GPU over torch.distributed.

The product's sharded FOM and PTROM batch are C ABI entry points
(ptrom_fom_simulate_sharded_f64, ptrom_ptrom_simulate_batch_sharded_f64 over a
ptrom_comm; Python mirror in comm.py) so a C++ host shards without Python.
This module holds the torch.distributed restatements of the same control
flow with pluggable per-rank backends — exercised on CPU with gloo, where
the C ABI (CUDA-only) cannot run — plus the peer-memory FOM variant and the
Barnes–Hut target split.

ShardedFom — the implicit-trapezoidal FOM (integrators.hpp:117-272) with the
targets split evenly across ranks. Per Newton iteration:
  * residual on the rank's rows and its squared norm; the G partial norms are
    all-gathered and summed in rank order on every rank (NCCL's all-reduce is
    not order-deterministic across G), so every rank takes the same
    convergence decision (integrators.hpp:140-155);
  * the Newton update of the rank's rows (2x2 blocks are local: the Jacobian
    self-blocks need no exchange);
  * all-gather of the updated source positions (x then y, NVLink/NVSwitch),
    then the all-pairs velocity of the rank's targets against all sources.

With `exchange="peer"` (CUDA backend, one GPU per process) the per-iteration
all-gather is replaced by the peer-memory exchange (peer.py): each rank
publishes its updated rows in CUDA-IPC memory and the velocity kernel reads
the other ranks' blocks in place over NVLink; the Newton-block refresh (once
per refresh period) still gathers the positions.

PtromInstanceSplit — μ instances of the PTROM online path split evenly across
ranks (no communication during the march); reduced states gathered at the end.

ShardedBarnesHut — BarnesHutModel::velocity (integrators.hpp:83-102) with the
build replicated and the far field split by target: every rank
builds the identical tree from the replicated state (the build is
deterministic), evaluates the targets of its contiguous range of tree slots
(spatially coherent), and the slot-ordered shards are all-gathered and
scattered back to particle order through the tree permutation.

The compute backend is pluggable: CudaBackend (libptrom_b200.so through the
device C ABI) is the product; tests drive the same control logic with a CPU
backend over gloo.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Even contiguous split of n targets (rank r owns [lo, hi))."""
    return rank * n // world, (rank + 1) * n // world


class CudaBackend:
    """Per-rank device kernels through the C ABI (ptrom_dev_*)."""

    def __init__(self, gamma: torch.Tensor, delta: float, form: int = 0, inflow: Optional[torch.Tensor] = None):
        from . import device as dev
        from .api import default_context
        self.dev = dev
        self.gamma, self.delta, self.form, self.inflow = gamma, float(delta), int(form), inflow
        self.device = gamma.device
        self.ctx = default_context(gamma.device.index or 0)

    def velocity_rows(self, x_full, lo, hi, out):
        self.dev.pairwise_velocity(x_full, self.gamma, self.delta, self.form, self.inflow, lo, hi, out)

    def newton_blocks(self, x_full, lo, hi, dt, out):
        self.dev.newton_blocks(x_full, self.gamma, self.delta, self.form, dt, lo, hi, out)

    def residual(self, xi, fxi, xp, fp, dt, r, norm2, m):
        self.dev.residual(xi, fxi, xp, fp, dt, r, norm2, m, m)

    def newton_update(self, inv, r, x, m):
        self.dev.newton_update(inv, r, x, m, m)

    def check(self):
        self.dev.synchronize()


@dataclass
class ShardedResult:
    snapshots_local: torch.Tensor  # (n_steps, 2m): rank's rows [x_lo..x_hi, y_lo..y_hi] per step
    iterations: list
    converged: list
    relative_residual: list
    lo: int
    hi: int


class ShardedFom:
    def __init__(self, n: int, backend, group=None, exchange: str = "allgather"):
        self.n = n
        self.backend = backend
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.lo, self.hi = shard_bounds(n, self.rank, self.world)
        self.m = self.hi - self.lo
        if exchange not in ("allgather", "peer"):
            raise ValueError("exchange must be 'allgather' or 'peer'")
        self.exchange = exchange
        self._peer = None
        if exchange == "peer":
            from .peer import PeerExchange
            self._peer = PeerExchange(n, ctx=getattr(backend, "ctx", None), group=group)
            self._token = torch.zeros(1, dtype=torch.float32, device=backend.device)

    def _peer_velocity(self, xi, fxi):
        """Publish this rank's rows, order against the peers, evaluate in place."""
        self._peer.write_local(xi)
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                self._peer.barrier(self._token)
            else:  # gloo (tests): host barrier after the copy completed
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
        be = self.backend
        self._peer.velocity(be.gamma, be.delta, fxi, be.form, be.inflow)

    def _gather_positions(self, x_local, x_full):
        """Local SoA rows → full SoA state on every rank (the per-iteration exchange)."""
        n, m = self.n, self.m
        if self.world == 1:
            x_full.copy_(x_local)
            return
        counts = [shard_bounds(n, r, self.world)[1] - shard_bounds(n, r, self.world)[0] for r in range(self.world)]
        if len(set(counts)) == 1:
            dist.all_gather_into_tensor(x_full[:n], x_local[:m].contiguous(), group=self.group)
            dist.all_gather_into_tensor(x_full[n:], x_local[m:].contiguous(), group=self.group)
        else:  # uneven shards: pad every rank's block to the largest one
            mx = max(counts)
            buf = torch.zeros(2 * mx, dtype=x_local.dtype, device=x_local.device)
            buf[:m] = x_local[:m]
            buf[mx:mx + m] = x_local[m:]
            out = torch.empty(self.world * 2 * mx, dtype=x_local.dtype, device=x_local.device)
            dist.all_gather_into_tensor(out, buf, group=self.group)
            out = out.view(self.world, 2, mx)
            x_full[:n].copy_(torch.cat([out[r, 0, :counts[r]] for r in range(self.world)]))
            x_full[n:].copy_(torch.cat([out[r, 1, :counts[r]] for r in range(self.world)]))

    def _global_norm(self, norm2_local) -> float:
        """Fixed-order global ‖r‖: all-gather the partials, sum in rank order."""
        if self.world == 1:
            return math.sqrt(float(norm2_local.item()))
        parts = torch.empty(self.world, dtype=torch.float64, device=norm2_local.device)
        dist.all_gather_into_tensor(parts, norm2_local.reshape(1), group=self.group)
        total = 0.0
        for v in parts.cpu().tolist():
            total += v
        return math.sqrt(total)

    def simulate(self, x0_full: torch.Tensor, dt: float, n_steps: int, tol: float = 1e-10, max_iters: int = 100,
                 refresh: int = 1) -> ShardedResult:
        """integrators.hpp:243-272 over the rank's targets."""
        if not dt > 0:
            raise ValueError("time step must be positive")
        if tol <= 0 or max_iters < 1 or refresh < 1:
            raise ValueError("invalid Newton configuration")
        n, m, lo, hi, be = self.n, self.m, self.lo, self.hi, self.backend
        dev, dtp = x0_full.device, x0_full.dtype
        x_full = x0_full.clone()
        x_prev = torch.cat([x0_full[lo:hi], x0_full[n + lo:n + hi]]).contiguous()
        f_prev = torch.empty(2 * m, dtype=dtp, device=dev)
        be.velocity_rows(x_full, lo, hi, f_prev)
        xi = torch.empty_like(x_prev)
        fxi = torch.empty_like(f_prev)
        r = torch.empty_like(x_prev)
        inv = torch.empty((max(m, 1), 4), dtype=dtp, device=dev)
        norm2 = torch.zeros(1, dtype=torch.float64, device=dev)
        snaps = torch.empty((n_steps, 2 * m), dtype=dtp, device=dev)
        iters, conv, rels = [], [], []
        have_blocks = False
        x_prev_full = x_full.clone()
        for s in range(n_steps):
            xi.copy_(x_prev)
            fxi.copy_(f_prev)
            x_full.copy_(x_prev_full)
            refresh_due = (s % refresh) == 0 or not have_blocks
            refreshed = False
            x_stale = False  # peer mode: x_full lags the published rows
            updates, converged, r0, rel = 0, False, 0.0, 0.0
            while True:
                be.residual(xi, fxi, x_prev, f_prev, dt, r, norm2, m)
                nr = self._global_norm(norm2)
                if updates == 0:
                    r0 = nr
                    if r0 == 0.0:
                        converged, rel = True, 0.0
                        break
                rel = nr / r0
                if rel <= tol:
                    converged = True
                    break
                if updates >= max_iters:
                    break
                if refresh_due and not refreshed:
                    if x_stale:
                        self._gather_positions(xi, x_full)
                        x_stale = False
                    be.newton_blocks(x_full, lo, hi, dt, inv)
                    refreshed = have_blocks = True
                be.newton_update(inv, r, xi, m)
                updates += 1
                if self._peer is not None:
                    self._peer_velocity(xi, fxi)
                    x_stale = True
                else:
                    self._gather_positions(xi, x_full)
                    be.velocity_rows(x_full, lo, hi, fxi)
            if x_stale:  # the accepted state is the next step's Jacobian point
                self._gather_positions(xi, x_full)
            x_prev, xi = xi, x_prev
            f_prev, fxi = fxi, f_prev
            x_prev_full.copy_(x_full)
            snaps[s].copy_(x_prev)
            iters.append(updates)
            conv.append(int(converged))
            rels.append(rel)
        be.check()
        return ShardedResult(snaps, iters, conv, rels, lo, hi)

    def close(self):
        if self._peer is not None:
            self._peer.close()
            self._peer = None


class PtromInstanceSplit:
    """μ instances split evenly across ranks: the shared
    tables live on the root only and are broadcast once, every rank marches
    its block of instances with no communication, and the reduced states are
    gathered in instance order on every rank. The product path is the C ABI's
    ptrom_ptrom_simulate_batch_sharded_f64 (comm.py); this is the same
    control flow over torch.distributed with a pluggable per-rank `march`, so
    the split / broadcast / gather logic is tested on CPU with gloo."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def local_slice(self, n_inst: int) -> tuple[int, int]:
        return shard_bounds(n_inst, self.rank, self.world)

    def broadcast_tables(self, tables: Optional[dict], root: int = 0) -> dict:
        """One broadcast of the root's table dict (numpy arrays and scalars)."""
        if self.world == 1:
            return tables
        box = [tables if self.rank == root else None]
        dist.broadcast_object_list(box, src=root, group=self.group)
        return box[0]

    def run(self, tables: Optional[dict], march, root: int = 0):
        """tables (root only) must hold 'mu'; march(tables, mu_block) returns
        (x_hat [k][n_steps][M], iterations [k][n_steps]) for its k instances."""
        tables = self.broadcast_tables(tables, root)
        mu = np.asarray(tables["mu"])
        lo, hi = self.local_slice(mu.shape[0])
        xh, it = march(tables, mu[lo:hi])
        return (self.gather(torch.as_tensor(np.asarray(xh)), mu.shape[0]).numpy(),
                self.gather(torch.as_tensor(np.asarray(it)), mu.shape[0]).numpy())

    def gather(self, local: torch.Tensor, n_inst: int) -> torch.Tensor:
        """Concatenate per-rank instance blocks (leading dimension) in rank order."""
        if self.world == 1:
            return local
        counts = [shard_bounds(n_inst, r, self.world)[1] - shard_bounds(n_inst, r, self.world)[0]
                  for r in range(self.world)]
        tail = tuple(local.shape[1:])
        mx = max(counts)
        buf = torch.zeros((mx,) + tail, dtype=local.dtype, device=local.device)
        buf[:local.shape[0]] = local
        out = torch.empty((self.world * mx,) + tail, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        return torch.cat([out[r * mx:r * mx + counts[r]] for r in range(self.world)])


class CudaBhBackend:
    """Replicated build + slot-range far field through ptrom_dev_barnes_hut_velocity_slots_f64."""

    def __init__(self, device_index: int = 0):
        from .api import default_context
        self.ctx = default_context(device_index)
        self.pairs = 0

    def slots(self, x_full, gamma, delta, form, crit_kind, crit_value, leaf, inflow, lo, hi):
        import ctypes as C
        n = gamma.shape[0]
        out = torch.empty(2 * max(hi - lo, 0), dtype=torch.float64, device=x_full.device)
        perm = torch.empty(n, dtype=torch.int32, device=x_full.device)
        cnt = C.c_uint64()
        self.ctx.check(self.ctx.lib.ptrom_dev_barnes_hut_velocity_slots_f64(
            self.ctx.handle, n, x_full.data_ptr(), gamma.data_ptr(), float(delta), int(form), int(crit_kind),
            float(crit_value), int(leaf), inflow.data_ptr() if inflow is not None else None, lo, hi,
            out.data_ptr() if out.numel() else None, perm.data_ptr(), C.byref(cnt)))
        self.pairs = cnt.value
        return out, perm


class ShardedBarnesHut:
    """Target-sharded Barnes–Hut velocity (see the module docstring)."""

    def __init__(self, n: int, backend, group=None):
        self.n, self.be, self.group = n, backend, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.lo, self.hi = shard_bounds(n, self.rank, self.world)

    def velocity(self, x_full: torch.Tensor, gamma: torch.Tensor, delta: float, crit_kind: int = 0,
                 crit_value: float = 0.5, leaf: int = 32, form: int = 0,
                 inflow: Optional[torch.Tensor] = None) -> torch.Tensor:
        n, lo, hi = self.n, self.lo, self.hi
        f_loc, perm = self.be.slots(x_full, gamma, delta, form, crit_kind, crit_value, leaf, inflow, lo, hi)
        m = hi - lo
        if self.world == 1:
            fxs, fys = f_loc[:m], f_loc[m:]
        else:
            counts = [shard_bounds(n, r, self.world)[1] - shard_bounds(n, r, self.world)[0]
                      for r in range(self.world)]
            mx = max(counts)
            buf = torch.zeros(2 * mx, dtype=torch.float64, device=x_full.device)
            buf[:m] = f_loc[:m]
            buf[mx:mx + m] = f_loc[m:]
            outs = [torch.empty_like(buf) for _ in range(self.world)]
            dist.all_gather(outs, buf, group=self.group)
            fxs = torch.cat([outs[r][:counts[r]] for r in range(self.world)])
            fys = torch.cat([outs[r][mx:mx + counts[r]] for r in range(self.world)])
        idx = perm.long()
        f = torch.empty(2 * n, dtype=torch.float64, device=x_full.device)
        f[idx] = fxs
        f[n + idx] = fys
        return f
