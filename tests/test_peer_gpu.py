"""Peer-memory exchange (paper_2103_01983_b200/peer.py): the
target-sharded velocity kernel reading every rank's source block in place.
On one GPU the ranks are virtual (separate device buffers) or two processes
sharing the device through CUDA IPC; the kernel must equal the flat path
bit for bit and the oracle within 1e-12."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,G", [(6000, 1), (6000, 3), (65536, 8), (10007, 5)])
def test_peer_blocks_equal_flat_path_bitwise(pt, oracle, n, G):
    from paper_2103_01983_b200 import device as dev
    from paper_2103_01983_b200.sharded import shard_bounds
    w = workloads.config2(n=n) if n == 65536 else workloads.config1(n=n, seed=n)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    bounds = [shard_bounds(n, r, G) for r in range(G)]
    blocks = [torch.cat([x[lo:hi], x[n + lo:n + hi]]).contiguous() for lo, hi in bounds]
    ptrs = (C.c_void_p * G)(*[b.data_ptr() for b in blocks])
    offs = (C.c_int64 * (G + 1))(*([0] + [hi for _, hi in bounds]))
    ctx = pt.default_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    full = np.zeros(2 * n)
    for r, (lo, hi) in enumerate(bounds):
        m = hi - lo
        out = torch.empty(2 * m, dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.ptrom_dev_pairwise_velocity_peers_f64(ctx.handle, n, G, ptrs, offs, g.data_ptr(), w.delta, 0,
                                                                None, lo, hi, blocks[r].data_ptr(), out.data_ptr(), m))
        flat = dev.pairwise_velocity(x, g, w.delta, 0, None, lo, hi)
        dev.synchronize(ctx)
        np.testing.assert_array_equal(out.cpu().numpy(), flat.cpu().numpy())
        o = out.cpu().numpy()
        full[lo:hi], full[n + lo:n + hi] = o[:m], o[m:]
    rows = np.r_[0:min(n, 2048), n:n + min(n, 2048)]
    ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_end=min(n, 2048), threads=os.cpu_count() or 1)
    assert rel(full[rows], ref[rows]) <= 1e-12


def test_peer_validation(pt):
    ctx = pt.default_context(0)
    one = (C.c_void_p * 1)(None)
    bad = (C.c_int64 * 2)(0, 5)
    rc = ctx.lib.ptrom_dev_pairwise_velocity_peers_f64(ctx.handle, 10, 1, one, bad, None, 0.1, 0, None, 0, 10, None,
                                                       None, 10)
    assert rc == 2
    assert "span" in ctx.lib.ptrom_last_error(ctx.handle).decode()


def _ipc_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2103_01983_b200.peer import PeerExchange
        w = workloads.config1(n=n, seed=77)
        ex = PeerExchange(n)
        x = torch.tensor(w.x0, device="cuda")
        xl = torch.cat([x[ex.lo:ex.hi], x[n + ex.lo:n + ex.hi]]).contiguous()
        ex.write_local(xl)
        torch.cuda.synchronize()
        dist.barrier()
        g = torch.tensor(w.gamma, device="cuda")
        out = torch.empty(2 * ex.m, dtype=torch.float64, device="cuda")
        ex.velocity(g, w.delta, out)
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, (ex.lo, ex.hi, out.cpu().numpy()))
        dist.barrier()
        ex.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


def test_ipc_exchange_two_processes_one_gpu(oracle):
    """Two ranks (processes) share cuda:0 through CUDA IPC mappings: each reads
    the other's block in place; the stitched field equals the oracle."""
    import queue
    import torch.multiprocessing as mp
    n = 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = None
    for _ in range(240):
        try:
            parts = q.get(timeout=1.0)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert parts is not None, [p.exitcode for p in procs]
    w = workloads.config1(n=n, seed=77)
    full = np.zeros(2 * n)
    for lo, hi, o in parts:
        m = hi - lo
        full[lo:hi], full[n + lo:n + hi] = o[:m], o[m:]
    ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta)
    assert rel(full, ref) <= 1e-12


def _fom_peer_worker(rank, world, port, n, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2103_01983_b200.sharded import CudaBackend, ShardedFom
        w = workloads.config1(n=n, seed=5)
        g = torch.tensor(w.gamma, device="cuda")
        fom = ShardedFom(n, CudaBackend(g, w.delta), exchange="peer")
        res = fom.simulate(torch.tensor(w.x0, device="cuda"), w.dt, steps)
        parts = [None] * world
        dist.all_gather_object(parts, (res.lo, res.hi, res.snapshots_local.cpu().numpy(), res.iterations))
        dist.barrier()
        fom.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


def test_sharded_fom_peer_exchange_two_processes(oracle):
    """ShardedFom(exchange='peer'): velocity evaluations read the other rank's
    rows in place (CUDA IPC); trajectory equals the oracle's within 1e-12."""
    import queue
    import torch.multiprocessing as mp
    n, steps = 800, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_fom_peer_worker, args=(r, 2, port, n, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = None
    for _ in range(300):
        try:
            parts = q.get(timeout=1.0)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert parts is not None, [p.exitcode for p in procs]
    w = workloads.config1(n=n, seed=5)
    snaps, iters, _, _ = oracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, steps)
    full = np.zeros((steps, 2 * n))
    for lo, hi, loc, its in parts:
        m = hi - lo
        full[:, lo:hi], full[:, n + lo:n + hi] = loc[:, :m], loc[:, m:]
    for k in range(steps):
        assert rel(full[k], snaps[:, k]) <= 1e-12
