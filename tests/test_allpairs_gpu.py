"""Parity of the sm_100a all-pairs kernels (through the C ABI) against the
CPU oracle. Tolerances are north_star's: 1e-12 relative (2-norm) in fp64,
1e-5 relative in fp32 (judged against the fp64 oracle)."""
import os

import numpy as np
import pytest

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
FP64_TOL = 1e-12
FP32_TOL = 1e-5


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def random_system(rng, n, box=5.0):
    x = rng.uniform(-box, box, 2 * n)
    g = rng.uniform(-2.0, 2.0, n)
    return x, g


@pytest.mark.parametrize("n", [1, 2, 3, 7, 33, 129, 1000, 4097])
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("delta", [0.0, 0.3])
def test_velocity_small_systems(pt, oracle, n, form, delta):
    rng = np.random.default_rng(1000 + n)
    x, g = random_system(rng, n)
    inflow = rng.uniform(-1, 1, 2 * n) if n % 2 else None
    f = pt.pairwise_velocity(x, pt.ParticleSystem(g, delta, inflow, form))
    ref = oracle.pairwise_velocity(x, g, delta, form, inflow)
    assert rel(f, ref) <= FP64_TOL


def test_velocity_config2_full_size_rows(pt, oracle):
    """BASELINE configs[1] at full N = 65,536 (fp64); the oracle checks 4,096
    target rows spread over the particle range against every source."""
    w = workloads.config2()
    f = pt.pairwise_velocity(w.x0, pt.ParticleSystem(w.gamma, w.delta))
    n = w.n
    for b in (0, 30000, n - 2048):
        ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=b, t_end=b + 2048, threads=THREADS)
        rows = np.r_[b:b + 2048, n + b:n + b + 2048]
        assert rel(f[rows], ref[rows]) <= FP64_TOL


def test_velocity_config5_full_size_rows(pt, oracle):
    """BASELINE configs[4] at its full size, N = 4,194,304 (δ = 1e-3): one
    evaluation through the host C ABI (17.6e12 pairs), then 3 x 512 target
    rows (start, middle, end) against every source on the oracle."""
    w = workloads.config5()
    n = w.n
    f = pt.pairwise_velocity(w.x0, pt.ParticleSystem(w.gamma, w.delta))
    assert np.all(np.isfinite(f))
    for b in (0, n // 2 - 256, n - 512):
        ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=b, t_end=b + 512, threads=THREADS)
        rows = np.r_[b:b + 512, n + b:n + b + 512]
        assert rel(f[rows], ref[rows]) <= FP64_TOL, b


def test_velocity_config2_fp32(pt, oracle):
    w = workloads.config2()
    x32 = w.x0.astype(np.float32)
    g32 = w.gamma.astype(np.float32)
    f32 = pt.pairwise_velocity(x32, pt.ParticleSystem(g32, np.float32(w.delta)))
    assert f32.dtype == np.float32
    n = w.n
    b = 12345
    ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=b, t_end=b + 4096, threads=THREADS)
    rows = np.r_[b:b + 4096, n + b:n + b + 4096]
    assert rel(f32[rows].astype(np.float64), ref[rows]) <= FP32_TOL


def test_velocity_fp32_small_against_fp32_oracle(pt, oracle):
    rng = np.random.default_rng(7)
    x, g = random_system(rng, 500)
    x, g = x.astype(np.float32), g.astype(np.float32)
    f = pt.pairwise_velocity(x, pt.ParticleSystem(g, np.float32(0.05)))
    ref64 = oracle.pairwise_velocity(x.astype(np.float64), g.astype(np.float64), float(np.float32(0.05)))
    assert rel(f.astype(np.float64), ref64) <= FP32_TOL


def test_kernel_pair_unit_distance_known_answer(pt):
    # test_kernel.cpp:73-85: target (0,0), source (1,0), Γ = 2π → (0, −1); δ = 1 → (0, −0.5)
    x = np.array([0.0, 1.0, 0.0, 0.0])
    g = np.array([0.0, 2.0 * np.pi])
    f0 = pt.pairwise_velocity(x, pt.ParticleSystem(g, 0.0))
    f1 = pt.pairwise_velocity(x, pt.ParticleSystem(g, 1.0))
    assert abs(f0[0]) < 1e-15 and abs(f0[2] + 1.0) < 1e-15
    assert abs(f1[0]) < 1e-15 and abs(f1[2] + 0.5) < 1e-15
    # test_kernel.cpp:103-113 denominator-scaled: −1/(2π+3)
    g2 = np.array([0.0, 1.0])
    f2 = pt.pairwise_velocity(x, pt.ParticleSystem(g2, 3.0, None, pt.KernelForm.denominator_scaled))
    assert abs(f2[2] + 1.0 / (2.0 * np.pi + 3.0)) < 1e-15


def test_zero_circulation_returns_inflow_exactly(pt):
    # test_kernel.cpp:141-151
    inflow = np.arange(1.0, 7.0)
    f = pt.pairwise_velocity(np.array([0, 1, 2, 0, 1, 2.0]), pt.ParticleSystem(np.zeros(3), 0.0, inflow))
    assert np.array_equal(f, inflow)


def test_coincident_points_raise_numerical_error(pt):
    # test_kernel.cpp:182-195 (delta = 0 coincident pair → numerical_error)
    with pytest.raises(pt.NumericalError):
        pt.pairwise_velocity(np.array([1.0, 1.0, 2.0, 2.0]), pt.ParticleSystem(np.ones(2), 0.0))
    # regularized: finite, and the context recovers for the next call
    f = pt.pairwise_velocity(np.array([1.0, 1.0, 2.0, 2.0]), pt.ParticleSystem(np.ones(2), 0.5))
    assert np.all(f == 0.0)


def test_input_validation_raises_config_error(pt):
    sys_ = pt.ParticleSystem(np.ones(2), 0.1)
    with pytest.raises(pt.ConfigError):
        pt.pairwise_velocity(np.array([1.0, 2.0, 3.0]), sys_)
    with pytest.raises(pt.ConfigError):
        pt.pairwise_velocity(np.array([0.0, 1.0, 0.0, np.nan]), sys_)
    with pytest.raises(pt.ConfigError):
        pt.pairwise_velocity(np.zeros(4), pt.ParticleSystem(np.ones(2), -1.0))
    with pytest.raises(pt.ConfigError):
        pt.pairwise_velocity(np.zeros(4), pt.ParticleSystem(np.array([1.0, np.inf]), 0.1))


def test_kernel_eval_counter_counts_ordered_pairs(pt):
    # test_kernel.cpp:312-321: N(N−1)
    pt.reset_kernel_eval_count()
    pt.pairwise_velocity(np.random.default_rng(5).uniform(-5, 5, 8), pt.ParticleSystem(np.ones(4), 0.1))
    assert pt.kernel_eval_count() == 12


@pytest.mark.parametrize("n,delta,form", [(2, 0.0, 0), (5, 0.2, 0), (300, 0.01, 1), (5000, 1e-4, 0)])
def test_jacobian_parity(pt, oracle, n, delta, form):
    rng = np.random.default_rng(17 + n)
    x, g = random_system(rng, n)
    jac = pt.inexact_kernel_jacobian(x, pt.ParticleSystem(g, delta, None, form))
    ref = oracle.inexact_kernel_jacobian(x, g, delta, form, threads=THREADS)
    got = np.stack([jac.dfx_dx, jac.dfx_dy, jac.dfy_dx, jac.dfy_dy])
    assert rel(got, ref) <= FP64_TOL


def test_jacobian_two_particle_known_answer(pt):
    # test_kernel.cpp:197-210 → [[0, −1], [−1, 0]]
    jac = pt.inexact_kernel_jacobian(np.array([0.0, 1.0, 0.0, 0.0]), pt.ParticleSystem(np.array([0.0, 2 * np.pi])))
    assert np.allclose(jac.block(0), [[0.0, -1.0], [-1.0, 0.0]], atol=1e-14, rtol=0)


def test_device_entry_points_rows_and_ld(pt, oracle):
    import torch
    from paper_2103_01983_b200 import device as dev
    w = workloads.config1(n=3000)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    out = dev.pairwise_velocity(x, g, w.delta, t_begin=1000, t_end=2100)
    dev.synchronize()
    ref = oracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=1000, t_end=2100)
    got = out.cpu().numpy()
    want = np.r_[ref[1000:2100], ref[3000 + 1000:3000 + 2100]]
    assert rel(got, want) <= FP64_TOL


def test_repeatable_bitwise(pt):
    """Fixed-order reductions: two evaluations are bit-identical."""
    w = workloads.config2(n=20000)
    s = pt.ParticleSystem(w.gamma, w.delta)
    a = pt.pairwise_velocity(w.x0, s)
    b = pt.pairwise_velocity(w.x0, s)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("scale,delta", [(1.0, 0.3), (2.0 ** 15, 1e3), (2.0 ** 30, 1e10), (1.0, 1e-300),
                                         (1e-3, 1e-9)])
def test_reciprocal_tiers_match_oracle(pt, oracle, scale, delta):
    """Exercises the 4-way (|x| < 2^14, δ' >= 2^-31), 2-way (|x| < 2^29) and
    safe (huge coordinates, tiny δ) reciprocal tiers, incl. the unmasked
    fast-path diagonal, on a size with ragged tiles."""
    rng = np.random.default_rng(int(scale) % 1000 + 17)
    n = 20000 + 37
    x = rng.uniform(-1.0, 1.0, 2 * n) * scale
    g = rng.uniform(-1.0, 1.0, n)
    f = pt.pairwise_velocity(x, pt.ParticleSystem(g, delta))
    ref = oracle.pairwise_velocity(x, g, delta, t_end=1500, threads=THREADS)
    rows = np.r_[0:1500, n:n + 1500]
    assert rel(f[rows], ref[rows]) <= FP64_TOL


@pytest.mark.parametrize("scale,delta", [(1.0, 1e9), (1.0, 5e9), (1.0, 1e10), (1e3, 1e12), (1.0, 1e20),
                                         (2.0 ** 13, 2.0 ** 29), (2.0 ** 13, 2.0 ** 29 * 1.0000001),
                                         (2.0 ** 28, 2.0 ** 60), (2.0 ** 28, 2.0 ** 61), (1.0, 1e200)])
def test_reciprocal_tiers_large_delta_small_coordinates(pt, oracle, scale, delta):
    """δ' above the fast tiers' product range: the 4-way tier needs δ' ≤ 2^29
    and the 2-way tier δ' ≤ 2^60 (the fp32 seed of P = Π q must stay inside
    [2^-126, 2^126)); beyond that the tile must take the safe per-pair tier
    and still match the reference (kernel.hpp:29-42)."""
    rng = np.random.default_rng(int(np.log2(delta)) + 3)
    n = 4096 + 19
    x = rng.uniform(-1.0, 1.0, 2 * n) * scale
    g = rng.uniform(-1.0, 1.0, n)
    for form in (0, 1):
        f = pt.pairwise_velocity(x, pt.ParticleSystem(g, delta, None, form))
        ref = oracle.pairwise_velocity(x, g, delta, form, t_end=700, threads=THREADS)
        rows = np.r_[0:700, n:n + 700]
        assert np.all(np.isfinite(f))
        assert rel(f[rows], ref[rows]) <= FP64_TOL, (form, delta)
    jac = pt.inexact_kernel_jacobian(x[np.r_[0:600, n:n + 600]], pt.ParticleSystem(g[:600], delta))
    refj = oracle.inexact_kernel_jacobian(x[np.r_[0:600, n:n + 600]], g[:600], delta, 0, threads=THREADS)
    got = np.stack([jac.dfx_dx, jac.dfx_dy, jac.dfy_dx, jac.dfy_dy])
    assert rel(got, refj) <= FP64_TOL


def test_empty_system_is_a_config_error(pt):
    with pytest.raises(pt.ConfigError, match="empty"):
        pt.pairwise_velocity(np.zeros(0), pt.ParticleSystem(np.zeros(0), 0.1))
    with pytest.raises(pt.ConfigError):
        pt.hamiltonian(np.zeros(0), pt.ParticleSystem(np.zeros(0), 0.1))
    with pytest.raises(pt.ConfigError):
        pt.fom_simulate(np.zeros(0), pt.ParticleSystem(np.zeros(0), 0.1), pt.TimeGrid(1e-3, 2))


def test_single_particle_has_only_inflow(pt):
    f = pt.pairwise_velocity(np.array([0.5, -0.25]), pt.ParticleSystem(np.array([3.0]), 0.0, np.array([0.1, -0.2])))
    assert f.tolist() == [0.1, -0.2]


def test_device_validation_order_and_messages(pt):
    """kernel.hpp:84-103 order on the uploaded copies: circulation, δ, inflow, state."""
    import ctypes as C
    ctx = pt.default_context()
    lib = ctx.lib
    n = 300
    rng = np.random.default_rng(9)
    x, g, inf_ = rng.uniform(-1, 1, 2 * n), np.ones(n), np.zeros(2 * n)
    f = np.empty(2 * n)

    def call(x, g, delta, inflow):
        p = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        rc = lib.ptrom_pairwise_velocity_f64(ctx.handle, n, p(x), p(g), delta, 0, p(inflow), p(f), None)
        return rc, lib.ptrom_last_error(ctx.handle).decode()

    bad_g, bad_x, bad_i = g.copy(), x.copy(), inf_.copy()
    bad_g[n - 1] = np.nan
    bad_x[2 * n - 1] = np.inf
    bad_i[7] = -np.inf
    rc, msg = call(x, bad_g, -1.0, bad_i)
    assert rc != 0 and "non-finite circulation" in msg
    rc, msg = call(bad_x, g, -1.0, bad_i)
    assert rc != 0 and "negative desingularization" in msg
    rc, msg = call(bad_x, g, 0.1, bad_i)
    assert rc != 0 and "non-finite inflow" in msg
    rc, msg = call(bad_x, g, 0.1, inf_)
    assert rc != 0 and "pairwise_velocity: non-finite state" in msg
    rc, msg = call(x, g, 0.1, inf_)
    assert rc == 0, msg


@pytest.mark.parametrize("n,scale,delta,form,inflow", [(16384, 1.0, 2.5e-5, 0, False), (20037, 1.0, 0.3, 1, True),
                                                       (40000, 2.0 ** 15, 1e3, 0, False), (33000, 1.0, 0.0, 0, True),
                                                       (65536, 0.25, 2.5e-5, 0, False)])
def test_unordered_pair_kernel_matches_one_sided_and_oracle(pt, oracle, monkeypatch, n, scale, delta, form, inflow):
    """Full self-evaluations (n ≥ 16,384) run over unordered pairs
    (allpairs_sym.cu: one reciprocal per pair (i, j) for both directions,
    rotating per-source accumulators, fixed-order block partials). Against the
    one-sided kernel (PTROM_ALLPAIRS_SYM=0) and the oracle, ragged blocks,
    inflow, both forms, the safe tier (|x| ≥ 2^14) and δ = 0; run to run
    bit-identical."""
    rng = np.random.default_rng(n)
    x = rng.uniform(-1.0, 1.0, 2 * n) * scale
    g = rng.normal(0.0, 1.0, n) / n
    infl = rng.uniform(-1, 1, 2 * n) if inflow else None
    sys_ = pt.ParticleSystem(g, delta, infl, form)
    f = pt.pairwise_velocity(x, sys_)
    f2 = pt.pairwise_velocity(x, sys_)
    assert np.array_equal(f, f2)
    monkeypatch.setenv("PTROM_ALLPAIRS_SYM", "0")
    one_sided = pt.pairwise_velocity(x, sys_)
    monkeypatch.delenv("PTROM_ALLPAIRS_SYM")
    assert rel(f, one_sided) <= FP64_TOL
    rows_b = [0, n // 2, n - 700]
    for b in rows_b:
        ref = oracle.pairwise_velocity(x, g, delta, form, infl, t_begin=b, t_end=b + 700, threads=THREADS)
        rows = np.r_[b:b + 700, n + b:n + b + 700]
        assert rel(f[rows], ref[rows]) <= FP64_TOL, b


def test_unordered_pair_kernel_flags_coincident_pair(pt):
    """δ = 0 and two coincident particles: the reference throws
    (kernel.hpp:38-39); the unordered-pair kernel must report it too."""
    n = 20000
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 2 * n)
    x[17], x[n + 17] = x[15000], x[n + 15000]
    with pytest.raises(pt.NumericalError):
        pt.pairwise_velocity(x, pt.ParticleSystem(np.ones(n), 0.0))


@pytest.mark.parametrize("n,scale,delta,form,inflow", [(16384, 1.0, 2.5e-5, 0, False), (20037, 1.0, 0.3, 1, True),
                                                       (40000, 2.0 ** 14, 1e3, 0, False), (33000, 1.0, 0.0, 0, True),
                                                       (65536, 0.25, 0.005, 0, False)])
def test_unordered_pair_kernel_fp32(pt, oracle, monkeypatch, n, scale, delta, form, inflow):
    """fp32 full self-evaluations over unordered pairs (allpairs_sym.cu,
    allpairs_sym_f32_kernel): against the one-sided fp32 kernel
    (PTROM_ALLPAIRS_SYM=0) and the fp64 oracle at the fp32 tolerance, ragged
    blocks, inflow, both forms, the safe tier (|x| ≥ 2^13) and δ = 0; run to
    run bit-identical."""
    rng = np.random.default_rng(n + 1)
    x = (rng.uniform(-1.0, 1.0, 2 * n) * scale).astype(np.float32)
    g = (rng.normal(0.0, 1.0, n) / n).astype(np.float32)
    infl = rng.uniform(-1, 1, 2 * n).astype(np.float32) if inflow else None
    sys_ = pt.ParticleSystem(g, np.float32(delta), infl, form)
    f = pt.pairwise_velocity(x, sys_)
    assert f.dtype == np.float32
    assert np.array_equal(f, pt.pairwise_velocity(x, sys_))
    monkeypatch.setenv("PTROM_ALLPAIRS_SYM", "0")
    one_sided = pt.pairwise_velocity(x, sys_)
    monkeypatch.delenv("PTROM_ALLPAIRS_SYM")
    assert rel(f.astype(np.float64), one_sided.astype(np.float64)) <= FP32_TOL
    x64, g64 = x.astype(np.float64), g.astype(np.float64)
    i64 = infl.astype(np.float64) if inflow else None
    d64 = float(np.float32(delta))
    for b in (0, n // 2, n - 700):
        ref = oracle.pairwise_velocity(x64, g64, d64, form, i64, t_begin=b, t_end=b + 700, threads=THREADS)
        rows = np.r_[b:b + 700, n + b:n + b + 700]
        assert rel(f[rows].astype(np.float64), ref[rows]) <= FP32_TOL, b


def test_unordered_pair_kernel_fp32_flags_coincident_pair(pt):
    n = 20000
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 2 * n).astype(np.float32)
    x[17], x[n + 17] = x[15000], x[n + 15000]
    with pytest.raises(pt.NumericalError):
        pt.pairwise_velocity(x, pt.ParticleSystem(np.ones(n, np.float32), np.float32(0.0)))


@pytest.mark.parametrize("n,scale,delta,form", [(16384, 1.0, 2.5e-5, 0), (20037, 1.0, 0.3, 1),
                                                (40000, 2.0 ** 15, 1e3, 0), (33000, 1.0, 0.004, 0)])
def test_unordered_pair_jacobian(pt, oracle, monkeypatch, n, scale, delta, form):
    """Full-set self-block Jacobians (n ≥ 16,384) over unordered pairs
    (allpairs_sym_jac_kernel: the even terms w·(rx ry, ry² − rx², 1) shared
    by (i, j) and (j, i)): against the one-sided kernel (PTROM_ALLPAIRS_SYM=0)
    and the oracle, ragged blocks, both forms, the safe tier (|x| ≥ 2^14);
    run to run bit-identical."""
    rng = np.random.default_rng(n + 7)
    x = rng.uniform(-1.0, 1.0, 2 * n) * scale
    g = rng.normal(0.0, 1.0, n) / n
    sys_ = pt.ParticleSystem(g, delta, None, form)

    def stack(j):
        return np.stack([j.dfx_dx, j.dfx_dy, j.dfy_dx, j.dfy_dy])

    got = stack(pt.inexact_kernel_jacobian(x, sys_))
    assert np.array_equal(got, stack(pt.inexact_kernel_jacobian(x, sys_)))
    monkeypatch.setenv("PTROM_ALLPAIRS_SYM", "0")
    one_sided = stack(pt.inexact_kernel_jacobian(x, sys_))
    monkeypatch.delenv("PTROM_ALLPAIRS_SYM")
    assert rel(got, one_sided) <= FP64_TOL
    for b in (0, n // 2, n - 600):
        ref = oracle.inexact_kernel_jacobian(x, g, delta, form, t_begin=b, t_end=b + 600, threads=THREADS)
        assert rel(got[:, b:b + 600], ref[:, b:b + 600]) <= FP64_TOL, b
