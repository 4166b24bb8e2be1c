"""Peer-memory exchange for the target-sharded all-pairs evaluation (SURVEY.md
§8e) — one process per GPU, sources read in place over NVLink.

Each rank keeps its particles' positions (SoA block: x then y) in a CUDA-IPC
shareable buffer; the handles are exchanged once through torch.distributed
and every rank maps its peers' buffers. An evaluation is then one kernel
(`ptrom_dev_pairwise_velocity_peers_f64`) whose source tiles come from the
owning rank's HBM, so the position exchange overlaps the pair arithmetic tile
by tile instead of running as a separate all-gather. The only collective per
evaluation is the barrier that orders "every rank wrote its block" before
"every rank reads" (a one-element all-reduce on the compute stream).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import torch
import torch.distributed as dist

from .api import Context, default_context
from .sharded import shard_bounds


class PeerExchange:
    def __init__(self, n: int, ctx: Optional[Context] = None, group=None, counts: Optional[Sequence[int]] = None):
        self.n = n
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world > 8:
            raise ValueError("peer exchange supports at most 8 ranks")
        self.ctx = ctx or default_context(torch.cuda.current_device())
        lib = self.ctx.lib
        if counts is None:
            counts = [shard_bounds(n, r, self.world)[1] - shard_bounds(n, r, self.world)[0] for r in range(self.world)]
        self.counts = list(counts)
        self.offsets = [0]
        for c in self.counts:
            self.offsets.append(self.offsets[-1] + c)
        self.lo, self.hi = self.offsets[self.rank], self.offsets[self.rank + 1]
        self.m = self.hi - self.lo
        p = C.c_void_p()
        self.ctx.check(lib.ptrom_ipc_alloc(self.ctx.handle, 16 * max(self.m, 1), C.byref(p)))
        self.local_ptr = p.value
        self._opened = []
        handle = (C.c_uint8 * 64)()
        self.ctx.check(lib.ptrom_ipc_get_handle(self.ctx.handle, self.local_ptr, handle))
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, bytes(handle), group=group)
        else:
            handles = [bytes(handle)]
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(self.local_ptr)
                continue
            q = C.c_void_p()
            buf = (C.c_uint8 * 64).from_buffer_copy(handles[r])
            self.ctx.check(lib.ptrom_ipc_open_handle(self.ctx.handle, buf, C.byref(q)))
            self._opened.append(q.value)
            ptrs.append(q.value)
        self.peer_ptrs = (C.c_void_p * self.world)(*ptrs)
        self.peer_off = (C.c_int64 * (self.world + 1))(*self.offsets)

    def _stream(self):
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def write_local(self, x_local: torch.Tensor) -> None:
        """Publish this rank's positions (contiguous (2, m) or 2m float64)."""
        if x_local.numel() != 2 * self.m or not x_local.is_contiguous():
            raise ValueError("x_local must be a contiguous 2m tensor")
        self._stream()
        self.ctx.check(self.ctx.lib.ptrom_dev_memcpy(self.ctx.handle, self.local_ptr, x_local.data_ptr(),
                                                     16 * self.m))

    def barrier(self, token: torch.Tensor) -> None:
        """Orders every rank's write_local before any rank's read (stream-ordered)."""
        if self.world > 1:
            dist.all_reduce(token, group=self.group)

    def velocity(self, gamma: torch.Tensor, delta: float, out: torch.Tensor, form: int = 0,
                 inflow: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Velocity of this rank's rows against all n sources (out: 2m, ld m)."""
        self._stream()
        self.ctx.check(self.ctx.lib.ptrom_dev_pairwise_velocity_peers_f64(
            self.ctx.handle, self.n, self.world, self.peer_ptrs, self.peer_off, gamma.data_ptr(), float(delta),
            int(form), inflow.data_ptr() if inflow is not None else None, self.lo, self.hi, self.local_ptr,
            out.data_ptr(), self.m))
        return out

    def close(self) -> None:
        lib = self.ctx.lib
        for q in self._opened:
            lib.ptrom_ipc_close_handle(self.ctx.handle, q)
        self._opened = []
        if self.local_ptr:
            lib.ptrom_ipc_free(self.ctx.handle, self.local_ptr)
            self.local_ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
