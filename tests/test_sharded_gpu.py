"""Multi-GPU C ABI (include/ptrom_b200.h "multi-GPU"):
ptrom_comm_init / ptrom_comm_init_host and the *_sharded drivers.

On the one GPU a test box has:
  * NCCL communicators of world size 1 (the real ncclCommInitRank path);
  * two ranks as two processes sharing cuda:0 through the host transport
    (ptrom_comm_init_host over gloo): every collective blocks on the host,
    never inside a kernel, so the ranks' kernels never wait on each other.
The sharded results must equal the oracle within 1e-12 and the single-GPU
entry points bit for bit where the arithmetic is the same."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_nccl_world1_fom_sharded_equals_single_gpu(pt, oracle, monkeypatch):
    from paper_2103_01983_b200.comm import Comm, fom_simulate_sharded
    w = workloads.config1(n=1500)
    steps = 6
    comm = Comm.nccl()
    assert comm.transport == "nccl" and comm.world == 1
    sys_ = pt.ParticleSystem(w.gamma, w.delta)
    res = fom_simulate_sharded(comm, w.x0, sys_, pt.TimeGrid(w.dt, steps))
    # same kernels, same fixed-order norm: bit-identical to the single-GPU graph path
    monkeypatch.setenv("PTROM_FOM_PERSISTENT", "0")
    single = pt.fom_simulate(w.x0, sys_, pt.TimeGrid(w.dt, steps))
    monkeypatch.delenv("PTROM_FOM_PERSISTENT")
    assert np.array_equal(res.snapshots_local, single.snapshots)
    assert list(res.iterations) == list(single.iterations)
    # the persistent small-system kernel (the default at this size) evaluates the
    # step's last velocity together with the next Jacobian: same states to rounding
    small = pt.fom_simulate(w.x0, sys_, pt.TimeGrid(w.dt, steps))
    assert list(small.iterations) == list(single.iterations)
    assert max(rel(small.snapshots[:, s], single.snapshots[:, s]) for s in range(steps)) <= 1e-12
    snaps, iters, _, _ = oracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, steps)
    assert max(rel(res.snapshots_local[:, s], snaps[:, s]) for s in range(steps)) <= 1e-12
    assert res.pair_evals == (1 + int(np.sum(res.iterations))) * w.n * (w.n - 1)
    comm.close()


def test_nccl_world1_velocity_sharded_equals_flat(pt):
    import ctypes as C
    from paper_2103_01983_b200 import device as dev
    from paper_2103_01983_b200.comm import Comm
    w = workloads.config2(n=9000)
    comm = Comm.nccl()
    ctx = comm.ctx
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    x_full = torch.zeros_like(x)
    f = torch.empty_like(x)
    ctx.check(ctx.lib.ptrom_dev_pairwise_velocity_sharded_f64(ctx.handle, comm.handle, w.n, x.data_ptr(),
                                                              x_full.data_ptr(), g.data_ptr(), w.delta, 0, None,
                                                              f.data_ptr()))
    flat = dev.pairwise_velocity(x, g, w.delta)
    dev.synchronize(ctx)
    assert torch.equal(x_full, x) and torch.equal(f, flat)
    with pytest.raises(pt.ConfigError):
        ctx.check(ctx.lib.ptrom_dev_pairwise_velocity_sharded_f64(ctx.handle, None, w.n, x.data_ptr(),
                                                                  x_full.data_ptr(), g.data_ptr(), w.delta, 0, None,
                                                                  f.data_ptr()))
    comm.close()
    del C


def _ptrom_problem(oracle, n=4096, n_inst=5):
    from paper_2103_01983_b200 import rom
    w = workloads.config4(n=n, n_inst=n_inst)
    ids = oracle.greedy_sample(w.phi_r, w.n_samples)
    A = oracle.build_gnat_operator(w.phi_r, ids)
    g1 = w.gamma_a + w.gamma_b
    s = oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, ids, A)
    sur = rom.SurrogateSourceBasis.from_tables(
        s.phi_tilde, s.gamma_tilde, s.x0_tilde, s.zero_gamma, s.mem_off, s.mem_ids, s.targets, s.cl_off, s.cl_list,
        s.direct_ids, s.direct_phi, s.direct_x0, s.direct_gamma, s.d_off, s.d_list)
    return w, ids, A, g1, basis, op, sur


def test_nccl_world1_ptrom_batch_sharded_equals_single_gpu(pt, oracle):
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.comm import Comm, ptrom_simulate_batch_sharded
    w, ids, A, g1, basis, op, sur = _ptrom_problem(oracle)
    cfg = rom.RomConfig(1e-300, 5, 1.0)
    grid = pt.TimeGrid(w.dt, 4)
    sys_ = pt.ParticleSystem(g1, w.delta)
    comm = Comm.nccl()
    tb = ptrom_simulate_batch_sharded(comm, basis, op, sur, w.gamma_a, w.gamma_b, w.mu, sys_, grid, cfg, batch=2)
    ts = rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu, sys_, grid, cfg, batch=2)
    assert np.array_equal(tb.x_hat, ts.x_hat)
    assert np.array_equal(tb.iterations, ts.iterations)
    comm.close()


def _spawn(worker, world, args, timeout=300):
    import queue
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=worker, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    out = None
    for _ in range(timeout):
        try:
            out = q.get(timeout=1.0)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert out is not None, [p.exitcode for p in procs]
    return out


def _fom_worker(rank, world, port, n, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2103_01983_b200 as pt
        from paper_2103_01983_b200.comm import Comm, fom_simulate_sharded
        w = workloads.config1(n=n, seed=21)
        comm = Comm.host()
        inflow = np.linspace(-0.3, 0.2, 2 * n)
        res = fom_simulate_sharded(comm, w.x0, pt.ParticleSystem(w.gamma, w.delta, inflow), pt.TimeGrid(w.dt, steps))
        parts = [None] * world
        dist.all_gather_object(parts, (res.lo, res.hi, res.snapshots_local, list(res.iterations)))
        comm.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 900), (3, 701)])
def test_host_transport_fom_sharded_matches_oracle(pt, oracle, world, n):
    """ptrom_fom_simulate_sharded_f64 at world 2 and 3 (uneven shards, inflow):
    the stitched trajectory equals the single-process oracle within 1e-12,
    with the same Newton iteration counts on every rank."""
    steps = 5
    parts = _spawn(_fom_worker, world, (n, steps))
    w = workloads.config1(n=n, seed=21)
    inflow = np.linspace(-0.3, 0.2, 2 * n)
    snaps, iters, _, _ = oracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, steps, inflow=inflow)
    full = np.zeros((2 * n, steps))
    for lo, hi, loc, its in parts:
        m = hi - lo
        full[lo:hi], full[n + lo:n + hi] = loc[:m], loc[m:]
        assert its == list(iters)
    for s in range(steps):
        assert rel(full[:, s], snaps[:, s]) <= 1e-12


def _ptrom_worker(rank, world, port, root, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2103_01983_b200 as pt
        from oracle import pyoracle
        from paper_2103_01983_b200 import rom
        from paper_2103_01983_b200.comm import Comm, ptrom_simulate_batch_sharded
        pyoracle.build()
        comm = Comm.host()
        cfg = rom.RomConfig(1e-300, 5, 1.0)
        if rank == root:  # only the root holds the offline tables
            w, ids, A, g1, basis, op, sur = _ptrom_problem(pyoracle, n_inst=7)
            tr = ptrom_simulate_batch_sharded(comm, basis, op, sur, w.gamma_a, w.gamma_b, w.mu,
                                              pt.ParticleSystem(g1, w.delta), pt.TimeGrid(w.dt, 4), cfg, batch=2,
                                              root=root)
        else:
            tr = ptrom_simulate_batch_sharded(comm, None, None, None, None, None, None,
                                              pt.ParticleSystem(np.zeros(1), 2.5e-5), pt.TimeGrid(1e-3, 4), cfg,
                                              batch=2, root=root)
        parts = [None] * world
        dist.all_gather_object(parts, (tr.x_hat, tr.iterations))
        comm.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,root", [(2, 0), (3, 1)])
def test_host_transport_ptrom_batch_sharded(pt, oracle, world, root):
    """ptrom_ptrom_simulate_batch_sharded_f64: tables on the root only, one
    broadcast, the 7 instances split 7/world, x̂ gathered on every rank: each
    rank's gathered result equals the single-GPU batch bit for bit, and every
    instance the oracle's ptrom_simulate within 1e-12."""
    from paper_2103_01983_b200 import rom
    parts = _spawn(_ptrom_worker, world, (root,))
    w, ids, A, g1, basis, op, sur = _ptrom_problem(oracle, n_inst=7)
    cfg = rom.RomConfig(1e-300, 5, 1.0)
    ts = rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu, pt.ParticleSystem(g1, w.delta),
                                  pt.TimeGrid(w.dt, 4), cfg, batch=2)
    for xh, it in parts:
        assert np.array_equal(xh, ts.x_hat)
        assert np.array_equal(it, ts.iterations)
    for i, m in enumerate(w.mu):
        xo, it_o, _ = oracle.ptrom_simulate(oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1), w.phi, w.sv,
                                            w.x0, ids, A, w.gamma_a + m * w.gamma_b, w.delta, w.dt, 4, 1e-300, 5)
        assert max(rel(parts[0][0][i, s], xo[:, s]) for s in range(4)) <= 1e-12


def _sym_velocity_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2103_01983_b200.comm import Comm
        rng = np.random.default_rng(n)
        x = rng.uniform(-1, 1, 2 * n)
        g = rng.normal(0, 1, n) / n
        inflow = rng.uniform(-1, 1, 2 * n)
        comm = Comm.host()
        ctx = comm.ctx
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        lo, hi = comm.bounds(n)
        m = hi - lo
        xd = torch.tensor(x, device="cuda")
        x_local = torch.cat([xd[lo:hi], xd[n + lo:n + hi]]).contiguous()
        x_ws = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        gd = torch.tensor(g, device="cuda")
        infd = torch.tensor(inflow, device="cuda")
        f = torch.empty(2 * m, dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.ptrom_dev_pairwise_velocity_sharded_f64(ctx.handle, comm.handle, n, x_local.data_ptr(),
                                                                  x_ws.data_ptr(), gd.data_ptr(), 2.5e-5, 0,
                                                                  infd.data_ptr(), f.data_ptr()))
        ctx.check(ctx.lib.ptrom_synchronize(ctx.handle))
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, f.cpu().numpy()))
        comm.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 20480), (3, 20481)])
def test_host_transport_unordered_pair_sharded_velocity_bitwise(pt, world, n):
    """Sharded full evaluation over unordered pairs (allpairs_sym.cu): each
    rank computes its share of the block pairs, one reduce-scatter of the
    partial rows (a single non-zero contributor per element: exact) and the
    same fixed-order reduction — bit-identical to the single-GPU call."""
    parts = _spawn(_sym_velocity_worker, world, (n,))
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, 2 * n)
    g = rng.normal(0, 1, n) / n
    inflow = rng.uniform(-1, 1, 2 * n)
    single = pt.pairwise_velocity(x, pt.ParticleSystem(g, 2.5e-5, inflow))
    for lo, hi, f in parts:
        m = hi - lo
        assert np.array_equal(f[:m], single[lo:hi]) and np.array_equal(f[m:], single[n + lo:n + hi])


@pytest.mark.parametrize("world,n", [(2, 20480), (3, 20481)])
def test_host_transport_fom_sharded_unordered_pairs(pt, world, n):
    """ptrom_fom_simulate_sharded_f64 above the unordered-pair size (n ≥ 16,384,
    divisible by the world size): velocities and Newton-block Jacobians are
    sharded over the block pairs with one reduce-scatter each (bit-identical
    rows); the stitched trajectory equals the single-GPU fom_simulate within
    1e-12 with the same Newton iteration counts."""
    steps = 3
    parts = _spawn(_fom_worker, world, (n, steps))
    w = workloads.config1(n=n, seed=21)
    inflow = np.linspace(-0.3, 0.2, 2 * n)
    single = pt.fom_simulate(w.x0, pt.ParticleSystem(w.gamma, w.delta, inflow), pt.TimeGrid(w.dt, steps))
    full = np.zeros((2 * n, steps))
    for lo, hi, loc, its in parts:
        m = hi - lo
        full[lo:hi], full[n + lo:n + hi] = loc[:m], loc[m:]
        assert its == list(single.iterations)
    for s in range(steps):
        assert rel(full[:, s], single.snapshots[:, s]) <= 1e-12


def _bh_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2103_01983_b200 as pt
        from paper_2103_01983_b200.comm import Comm, barnes_hut_velocity_sharded
        from paper_2103_01983_b200.tree import ClusterCriterion
        w = workloads.config3(n=n)
        inflow = np.linspace(-0.1, 0.1, 2 * n)
        comm = Comm.host()
        f, cnt = barnes_hut_velocity_sharded(comm, w.x0, pt.ParticleSystem(w.gamma, w.delta, inflow),
                                             ClusterCriterion.barnes_hut(0.5), 32)
        comm.close()
        if rank == 0:
            q.put((f, cnt))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 20000), (3, 12345)])
def test_host_transport_barnes_hut_sharded_bitwise(pt, world, n):
    """ptrom_barnes_hut_velocity_sharded_f64: replicated
    deterministic build, tree slots split across ranks, slot blocks all-gathered
    and scattered back — the full velocity equals the single-GPU
    ptrom_barnes_hut_velocity_f64 bit for bit, with the same pair count."""
    import ctypes
    f, cnt = _spawn(_bh_worker, world, (n,))
    w = workloads.config3(n=n)
    inflow = np.linspace(-0.1, 0.1, 2 * n)
    ctx = pt.default_context()
    single = np.zeros(2 * n)
    c1 = ctypes.c_uint64()
    ctx.check(ctx.lib.ptrom_barnes_hut_velocity_f64(ctx.handle, n, w.x0.ctypes.data, w.gamma.ctypes.data, w.delta, 0,
                                                    0, 0.5, 32, inflow.ctypes.data, single.ctypes.data,
                                                    ctypes.byref(c1)))
    assert np.array_equal(f, single)
    assert cnt == c1.value
