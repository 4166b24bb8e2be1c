"""Multi-rank control logic of the sharded drivers (paper_2103_01983_b200/
sharded.py) on CPU with gloo, world sizes 2 and 3 (uneven shards). The
per-rank compute is a CPU test backend over the oracle; on GPUs the same
driver runs CudaBackend (NCCL). The sharded trajectory must match the
single-process oracle FOM within 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _run(world, target, args, timeout=240):
    """Spawn `world` gloo ranks; return what rank 0 puts on the queue."""
    import queue
    import time
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    t0 = time.time()
    result = None
    while time.time() - t0 < timeout:
        try:
            result = q.get(timeout=1.0)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert result is not None, [p.exitcode for p in procs]
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return result


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleBackend:
    """CPU backend with the ShardedFom backend interface (test only)."""

    def __init__(self, oracle, gamma, delta, form=0, inflow=None):
        self.o, self.gamma, self.delta, self.form, self.inflow = oracle, gamma, delta, form, inflow
        self.n = len(gamma)

    def velocity_rows(self, x_full, lo, hi, out):
        n, m = self.n, hi - lo
        f = self.o.pairwise_velocity(x_full.numpy(), self.gamma, self.delta, self.form, self.inflow, lo, hi)
        out[:m] = torch.from_numpy(f[lo:hi])
        out[m:] = torch.from_numpy(f[n + lo:n + hi])

    def newton_blocks(self, x_full, lo, hi, dt, out):
        j = self.o.inexact_kernel_jacobian(x_full.numpy(), self.gamma, self.delta, self.form, lo, hi)[:, lo:hi]
        h = dt / 2.0
        b00, b01, b10, b11 = 1.0 - h * j[0], 0.0 - h * j[1], 0.0 - h * j[2], 1.0 - h * j[3]
        det = b00 * b11 - b01 * b10
        out[:, 0] = torch.from_numpy(b11 / det)
        out[:, 1] = torch.from_numpy(-b01 / det)
        out[:, 2] = torch.from_numpy(-b10 / det)
        out[:, 3] = torch.from_numpy(b00 / det)

    def residual(self, xi, fxi, xp, fp, dt, r, norm2, m):
        r.copy_((xi - xp) - (dt / 2.0) * (fxi + fp))
        norm2[0] = float(np.sum(r.numpy() ** 2))

    def newton_update(self, inv, r, x, m):
        r0, r1 = -r[:m], -r[m:]
        x[:m] += inv[:, 0] * r0 + inv[:, 1] * r1
        x[m:] += inv[:, 2] * r0 + inv[:, 3] * r1

    def check(self):
        pass


def _fom_worker(rank, world, port, n, steps, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_01983_b200 import workloads
        from paper_2103_01983_b200.sharded import ShardedFom
        w = workloads.config1(n=n)
        fom = ShardedFom(n, OracleBackend(pyoracle, w.gamma, w.delta))
        res = fom.simulate(torch.tensor(w.x0), w.dt, steps)
        parts = [None] * world
        dist.all_gather_object(parts, (res.lo, res.hi, res.snapshots_local.numpy(), res.iterations))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 64), (3, 50)])
def test_sharded_fom_matches_single_process_oracle(oracle, world, n):
    from paper_2103_01983_b200 import workloads
    steps = 4
    parts = _run(world, _fom_worker, (n, steps))
    w = workloads.config1(n=n)
    snaps, iters, _, _ = oracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, steps)
    full = np.zeros((steps, 2 * n))
    for lo, hi, loc, its in parts:
        m = hi - lo
        full[:, lo:hi] = loc[:, :m]
        full[:, n + lo:n + hi] = loc[:, m:]
        assert list(its) == list(iters)
    for s in range(steps):
        assert np.linalg.norm(full[s] - snaps[:, s]) / np.linalg.norm(snaps[:, s]) <= 1e-12


def _oracle_march(oracle):
    """Per-rank march of the CPU test: the oracle's ptrom_simulate
    (rom.hpp:404-412) for each instance of the block, from the broadcast tables."""
    def march(t, mu_block):
        xs, its = [], []
        for m in mu_block:
            sur = oracle.Surrogate(t["phi"], t["sv"], t["x0"], t["g1"], t["ids"], 1, 1.0, 1)
            xo, it, _ = oracle.ptrom_simulate(sur, t["phi"], t["sv"], t["x0"], t["ids"], t["A"],
                                              t["gamma_a"] + m * t["gamma_b"], t["delta"], t["dt"], t["steps"],
                                              1e-300, 5)
            xs.append(xo.T.copy())
            its.append(np.asarray(it, np.int32))
        m_ = t["phi"].shape[1]
        return (np.array(xs).reshape(len(mu_block), t["steps"], m_),
                np.array(its, np.int32).reshape(len(mu_block), t["steps"]))
    return march


def _ptrom_tables(oracle, n=512, n_inst=7, steps=3):
    from paper_2103_01983_b200 import workloads
    w = workloads.config4(n=n, n_inst=n_inst, modes=6, modes_r=12)
    ids = oracle.greedy_sample(w.phi_r, w.n_samples)
    A = oracle.build_gnat_operator(w.phi_r, ids)
    return {"phi": w.phi, "sv": w.sv, "x0": w.x0, "g1": w.gamma_a + w.gamma_b, "ids": ids, "A": A,
            "gamma_a": w.gamma_a, "gamma_b": w.gamma_b, "delta": w.delta, "dt": w.dt, "steps": steps, "mu": w.mu}


def _split_worker(rank, world, port, root, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_01983_b200.sharded import PtromInstanceSplit
        pyoracle.build()
        sp = PtromInstanceSplit()
        tables = _ptrom_tables(pyoracle) if rank == root else None  # the root alone holds the tables
        xh, it = sp.run(tables, _oracle_march(pyoracle), root=root)
        parts = [None] * world
        dist.all_gather_object(parts, (xh, it))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,root", [(2, 0), (3, 2)])
def test_ptrom_instance_split_march_matches_single_process_oracle(oracle, world, root):
    """μ split across gloo ranks: tables broadcast from the root once, each
    rank marches its block, x̂ gathered in instance order on every rank —
    identical to the single-process per-instance oracle."""
    parts = _run(world, _split_worker, (root,))
    t = _ptrom_tables(oracle)
    want_x, want_it = _oracle_march(oracle)(t, t["mu"])
    for xh, it in parts:
        np.testing.assert_array_equal(xh, want_x)
        np.testing.assert_array_equal(it, want_it)


def test_shard_bounds_cover_everything():
    from paper_2103_01983_b200.sharded import shard_bounds
    for n in (1, 7, 64, 4194304):
        for g in (1, 2, 3, 8):
            b = [shard_bounds(n, r, g) for r in range(g)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(g - 1))


class OracleBhBackend:
    """CPU backend with the ShardedBarnesHut interface: the oracle's build_tree and
    per-target bh_velocity (quadtree.hpp:124-162, 257-281), slots [lo, hi)."""

    def __init__(self, oracle):
        self.o = oracle

    def slots(self, x_full, gamma, delta, form, crit_kind, crit_value, leaf, inflow, lo, hi):
        x, g = x_full.numpy(), gamma.numpy()
        n = g.shape[0]
        tree = self.o.Tree(x[:n], x[n:], g, leaf)
        out = torch.zeros(2 * (hi - lo), dtype=torch.float64)
        for k in range(lo, hi):
            i = int(tree.perm[k])
            f = tree.bh_velocity(x, g, delta, crit_kind, crit_value, form=form, t_begin=i, t_end=i + 1)
            out[k - lo] = f[i]
            out[(hi - lo) + k - lo] = f[n + i]
        return out, torch.from_numpy(tree.perm.astype(np.int32))


def _bh_worker(rank, world, port, n, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_01983_b200 import workloads
        from paper_2103_01983_b200.sharded import ShardedBarnesHut
        w = workloads.config3(n=n)
        bh = ShardedBarnesHut(n, OracleBhBackend(pyoracle))
        f = bh.velocity(torch.tensor(w.x0), torch.tensor(w.gamma), w.delta, 0, 0.5, 4)
        if rank == 0:
            out_q.put(f.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 160), (3, 101)])
def test_sharded_barnes_hut_matches_single_process_oracle(oracle, world, n):
    """Replicated build, far field split by tree slot, shards gathered back to
    particle order: bit-identical to the oracle's single-process bh_velocity."""
    from paper_2103_01983_b200 import workloads
    f = _run(world, _bh_worker, (n,))
    w = workloads.config3(n=n)
    tree = oracle.Tree(w.x0[:n], w.x0[n:], w.gamma, 4)
    np.testing.assert_array_equal(f, tree.bh_velocity(w.x0, w.gamma, w.delta, 0, 0.5))


def _host_coll_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C
        from paper_2103_01983_b200.comm import torch_host_collectives
        ops, _keep = torch_host_collectives()
        # what the C library does: raw host pointers, rank-ordered all-gather,
        # broadcast from a root, zero-byte calls
        send = (C.c_double * 3)(rank, rank + 0.5, -rank)
        recv = (C.c_double * (3 * world))()
        assert ops.all_gather(None, C.addressof(send), C.addressof(recv), 24) == 0
        assert ops.all_gather(None, C.addressof(send), C.addressof(recv), 0) == 0
        buf = (C.c_int64 * 4)(*([7, 8, 9, 10] if rank == world - 1 else [0, 0, 0, 0]))
        assert ops.broadcast(None, C.addressof(buf), 32, world - 1) == 0
        parts = [None] * world
        dist.all_gather_object(parts, (list(recv), list(buf)))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_transport_callbacks_over_gloo(world):
    """The ptrom_host_collectives callbacks (comm.py) the C ABI's host
    transport calls: rank-ordered all-gather and broadcast on raw buffers."""
    parts = _run(world, _host_coll_worker, ())
    want = [v for r in range(world) for v in (r, r + 0.5, -r)]
    for recv, buf in parts:
        assert recv == want
        assert buf == [7, 8, 9, 10]
