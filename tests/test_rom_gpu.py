"""PTROM online path on the B200 vs the oracle (reduction.hpp:400-431,
rom.hpp:71-412). Offline tables (greedy samples, A = pinv(PΦ_r), surrogate)
come from the oracle so the online kernels are checked in isolation;
reduced states within 1e-12 relative (north_star)."""
import numpy as np
import pytest

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def to_device(rom, s, ctx=None):
    return rom.SurrogateSourceBasis.from_tables(
        s.phi_tilde, s.gamma_tilde, s.x0_tilde, s.zero_gamma, s.mem_off, s.mem_ids, s.targets, s.cl_off, s.cl_list,
        s.direct_ids, s.direct_phi, s.direct_x0, s.direct_gamma, s.d_off, s.d_list, ctx=ctx)


class Problem:
    def __init__(self, oracle, n=4096, modes=16, modes_r=32, n_inst=6, seed=4):
        w = workloads.config4(n=n, n_inst=n_inst, modes=modes, modes_r=modes_r, seed=seed)
        self.w = w
        self.ids = oracle.greedy_sample(w.phi_r, w.n_samples)
        self.A = oracle.build_gnat_operator(w.phi_r, self.ids)
        self.g1 = w.gamma_a + w.gamma_b  # nominal μ = 1 (surrogate build)
        self.oracle = oracle

    def surrogate(self):
        w = self.w
        return self.oracle.Surrogate(w.phi, w.sv, w.x0, self.g1, self.ids, 1, 1.0, 1)


@pytest.fixture(scope="module")
def prob(oracle):
    return Problem(oracle)


def test_reassign_is_bit_exact(pt, prob):
    from paper_2103_01983_b200 import rom
    w = prob.w
    os_ = prob.surrogate()
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    ds = to_device(rom, os_)
    g = w.gamma_a + 1.37 * w.gamma_b
    os_.reassign(g)
    ds.reassign_cluster_circulation(g, basis)
    e = ds.export()
    np.testing.assert_array_equal(e["phi_tilde"], os_.phi_tilde)
    np.testing.assert_array_equal(e["x0_tilde"], os_.x0_tilde)
    np.testing.assert_array_equal(e["gamma_tilde"], os_.gamma_tilde)
    np.testing.assert_array_equal(e["direct_gamma"], os_.direct_gamma)


@pytest.mark.parametrize("modes,big", [(16, 32), (16, 100), (5, 64), (48, 32), (63, 40), (63, 4096)])
def test_reassign_big_cluster_path_bit_exact(pt, oracle, modes, big):
    """reduction.hpp:400-431 through the one-CTA-per-cluster path
    (reassign_big_kernel): the threshold is lowered so clusters of this
    N = 4,096 problem take it (config 4's largest cluster has ~2e5 members),
    and the mode count reaches the 63-mode limit, where the chunk of staged
    rows is sized from the opt-in shared memory. Tables bitwise."""
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.api import Context
    p = Problem(oracle, n=4096, modes=modes, modes_r=max(32, modes + 1), n_inst=2, seed=7)
    w = p.w
    ctx = Context(0)
    ctx.set_tuning("reassign_big_members", big)
    os_ = p.surrogate()
    sizes = np.diff(np.asarray(os_.mem_off))
    assert sizes.max() > big or big == 4096
    basis = rom.PODBasis(w.phi, w.sv, w.x0, ctx=ctx)
    # device-built surrogate (cluster_pod runs the same reassign at μ = 1;
    # the host-table constructor is limited to the online engine's 32 modes)
    from paper_2103_01983_b200.tree import ClusterCriterion
    ds = rom.SurrogateSourceBasis.cluster_pod(basis, p.g1, p.ids, ClusterCriterion.neighbor(1.0), 1)
    e = ds.export()
    np.testing.assert_array_equal(e["phi_tilde"], os_.phi_tilde)
    np.testing.assert_array_equal(e["x0_tilde"], os_.x0_tilde)
    for mu in (1.37, 0.0):  # μ = 0 zeroes patch B: zero-circulation clusters take the 1/|c| fallback
        g = w.gamma_a + mu * w.gamma_b
        os_.reassign(g)
        ds.reassign_cluster_circulation(g, basis)
        e = ds.export()
        np.testing.assert_array_equal(e["phi_tilde"], os_.phi_tilde)
        np.testing.assert_array_equal(e["x0_tilde"], os_.x0_tilde)
        np.testing.assert_array_equal(e["gamma_tilde"], os_.gamma_tilde)
        np.testing.assert_array_equal(e["direct_gamma"], os_.direct_gamma)
    del ds, basis
    with pytest.raises(pt.ConfigError):
        ctx.set_tuning("no_such_knob", 1)
    ctx.close()


@pytest.mark.parametrize("delta,form", [(2.5e-5, 0), (0.01, 1)])
def test_hyperpair_parity(pt, prob, delta, form):
    from paper_2103_01983_b200 import rom
    w = prob.w
    os_ = prob.surrogate()
    ds = to_device(rom, os_)
    rng = np.random.default_rng(48)
    xh = rng.uniform(-0.1, 0.1, w.phi.shape[1])
    nt = len(prob.ids)
    tp = np.r_[w.x0[prob.ids] + w.phi[prob.ids] @ xh, w.x0[prob.ids + w.n] + w.phi[prob.ids + w.n] @ xh]
    inflow = rng.uniform(-1, 1, 2 * w.n)
    f, jac, cpos, dpos = os_.hyperpair(tp, xh, prob.g1, delta, form, inflow)
    sys_ = pt.ParticleSystem(prob.g1, delta, inflow, form)
    pt.reset_kernel_eval_count()
    hp = rom.hyperpair(ds, tp, xh, sys_)
    assert pt.kernel_eval_count() == len(os_.cl_list) + len(os_.d_list)  # test_rom.cpp:401-433
    assert rel(hp.f, f) <= 1e-12
    got = np.stack([hp.jac.dfx_dx, hp.jac.dfx_dy, hp.jac.dfy_dx, hp.jac.dfy_dy])
    assert rel(got, jac) <= 1e-12
    assert rel(hp.cluster_positions, cpos) <= 1e-14
    assert rel(hp.direct_positions, dpos) <= 1e-14
    assert nt == hp.f.shape[0] // 2


def test_hyperpair_drops_coincident_cluster_and_flags_collision(pt):
    # test_rom.cpp:254-301
    from paper_2103_01983_b200 import rom
    sur = rom.SurrogateSourceBasis.from_tables(
        np.zeros((2, 3)), [0.7], [1.0, 2.0], [0], [0, 1], [0], [0], [0, 1], [0], [1], np.zeros((2, 3)), [3.0, 2.0],
        [0.5], [0, 1], [0])
    sys0 = pt.ParticleSystem(np.ones(2), 0.0)
    hp = rom.hyperpair(sur, [1.0, 2.0], np.zeros(3), sys0)
    d = pt.pairwise_velocity(np.array([1.0, 3.0, 2.0, 2.0]), pt.ParticleSystem(np.array([0.0, 0.5]), 0.0))
    assert abs(hp.f[0] - d[0]) <= 1e-15 and abs(hp.f[1] - d[2]) <= 1e-15
    col = rom.SurrogateSourceBasis.from_tables(
        np.zeros((2, 3)), [0.7], [1.0, 2.0], [0], [0, 1], [0], [0], [0, 1], [0], [1], np.zeros((2, 3)), [1.0, 2.0],
        [0.5], [0, 1], [0])
    with pytest.raises(pt.NumericalError):
        rom.hyperpair(col, [1.0, 2.0], np.zeros(3), sys0)


@pytest.mark.parametrize("tol,max_iters,steps", [(1e-300, 5, 20), (1e-6, 100, 15)])
def test_ptrom_simulate_parity(pt, prob, tol, max_iters, steps):
    """rom.hpp:404-412 single instance: reassign to Γ(μ = 1.6), march."""
    from paper_2103_01983_b200 import rom
    w = prob.w
    g = w.gamma_a + 1.6 * w.gamma_b
    os_ = prob.surrogate()
    xo, it_o, cv_o = prob.oracle.ptrom_simulate(os_, w.phi, w.sv, w.x0, prob.ids, prob.A, g, w.delta, w.dt, steps,
                                                tol, max_iters)
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, prob.ids, prob.A)
    ds = to_device(rom, prob.surrogate())
    tr = rom.ptrom_simulate(basis, op, ds, pt.ParticleSystem(g, w.delta), pt.TimeGrid(w.dt, steps),
                            rom.RomConfig(tol, max_iters, 1.0))
    np.testing.assert_array_equal(tr.iterations, it_o)
    np.testing.assert_array_equal(tr.converged, cv_o)
    worst = max(rel(tr.x_hat[:, s], xo[:, s]) for s in range(steps))
    assert worst <= 1e-12, worst


def test_batch_affine_matches_per_instance_oracle(pt, prob):
    """Batched online queries over μ: every instance equals the oracle's
    ptrom_simulate with Γ(μ) = Γa + μ Γb (fresh surrogate each)."""
    from paper_2103_01983_b200 import rom
    w = prob.w
    steps = 12
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, prob.ids, prob.A)
    ds = to_device(rom, prob.surrogate())
    mu = np.array([0.5, 0.8, 1.0, 1.3, 1.7, 2.0])
    cfg = rom.RomConfig(1e-300, 5, 1.0)
    tr = rom.ptrom_simulate_batch(basis, op, ds, w.gamma_a, w.gamma_b, mu, pt.ParticleSystem(prob.g1, w.delta),
                                  pt.TimeGrid(w.dt, steps), cfg, batch=4)
    for i, m in enumerate(mu):
        xo, it_o, _ = prob.oracle.ptrom_simulate(prob.surrogate(), w.phi, w.sv, w.x0, prob.ids, prob.A,
                                                 w.gamma_a + m * w.gamma_b, w.delta, w.dt, steps, 1e-300, 5)
        np.testing.assert_array_equal(tr.iterations[i], it_o)
        worst = max(rel(tr.x_hat[i, s], xo[:, s]) for s in range(steps))
        assert worst <= 1e-12, (m, worst)


def test_padded_modes(pt, oracle):
    """M = 6, M_r = 8 (DMMA tiles padded with zero columns/rows)."""
    from paper_2103_01983_b200 import rom
    p = Problem(oracle, n=2048, modes=6, modes_r=8, seed=9)
    w = p.w
    g = w.gamma_a + 0.9 * w.gamma_b
    xo, it_o, _ = oracle.ptrom_simulate(p.surrogate(), w.phi, w.sv, w.x0, p.ids, p.A, g, w.delta, w.dt, 10, 1e-300, 4)
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, p.ids, p.A)
    tr = rom.ptrom_simulate(basis, op, to_device(rom, p.surrogate()), pt.ParticleSystem(g, w.delta),
                            pt.TimeGrid(w.dt, 10), rom.RomConfig(1e-300, 4, 1.0))
    np.testing.assert_array_equal(tr.iterations, it_o)
    assert max(rel(tr.x_hat[:, s], xo[:, s]) for s in range(10)) <= 1e-12


def test_validation(pt, prob):
    from paper_2103_01983_b200 import rom
    w = prob.w
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    with pytest.raises(pt.ConfigError):
        rom.GnatOperator(basis, prob.ids[::-1], prob.A)  # unsorted ids
    op = rom.GnatOperator(basis, prob.ids, prob.A)
    ds = to_device(rom, prob.surrogate())
    with pytest.raises(pt.ConfigError):
        rom.ptrom_simulate(basis, op, ds, pt.ParticleSystem(prob.g1, w.delta), pt.TimeGrid(0.0, 3))
    with pytest.raises(pt.ConfigError):
        rom.ptrom_simulate(basis, op, ds, pt.ParticleSystem(prob.g1, w.delta), pt.TimeGrid(w.dt, 3),
                           rom.RomConfig(tol=0.0))


# ------------------------------------------------------- offline producers --
@pytest.mark.parametrize("n,nr,nt", [(30, 3, 4), (30, 7, 9), (30, 12, 15), (25, 20, 6), (12, 5, 12), (4000, 32, 80)])
def test_greedy_sample_ids_equal_oracle(pt, oracle, n, nr, nt):
    # test_reduction.cpp:238-250 shapes (numpy-seeded matrices)
    from paper_2103_01983_b200 import rom
    phi_r = np.random.default_rng(81 + n + nr).uniform(-1, 1, (2 * n, nr))
    np.testing.assert_array_equal(rom.greedy_sample(phi_r, nt), oracle.greedy_sample(phi_r, nt))


def test_greedy_sample_hand_cases(pt):
    # test_reduction.cpp:271-292: single column, lower index wins ties, preseeds
    from paper_2103_01983_b200 import rom
    phi_r = np.zeros((10, 1))
    phi_r[[0, 1, 2, 3, 4, 7], 0] = [0.1, 0.9, 0.5, 0.2, 0.3, 0.6]
    assert list(rom.greedy_sample(phi_r, 1)) == [1]
    assert list(rom.greedy_sample(phi_r, 2)) == [1, 2]
    tie = np.zeros((12, 1))
    tie[1, 0] = tie[4, 0] = 0.5
    assert list(rom.greedy_sample(tie, 1)) == [1]
    ids = rom.greedy_sample(np.random.default_rng(101).uniform(-1, 1, (40, 6)), 8, preseed=[17, 3])
    assert 17 in ids and 3 in ids and list(ids) == sorted(ids)
    with pytest.raises(pt.ConfigError):
        rom.greedy_sample(phi_r, 6)


def test_gnat_operator_matches_oracle_and_rank_check(pt, oracle, prob):
    from paper_2103_01983_b200 import rom
    A = rom.build_gnat_operator(prob.w.phi_r, prob.ids)
    assert rel(A, prob.A) <= 1e-12
    defi = np.zeros((8, 2))
    defi[0, :] = 1.0
    defi[4, :] = 2.0
    defi[1, 0] = 1.0
    defi[2, 1] = 1.0
    with pytest.raises(pt.NumericalError, match="rank 1"):
        rom.build_gnat_operator(defi, [0])


def test_device_cluster_pod_tables_equal_oracle(pt, prob):
    """build_weighted_pod_tree(leaf 1) + cluster_pod(neighbor 1) on the device:
    lists byte-equal, tables bit-equal (same member order and formula)."""
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.tree import ClusterCriterion
    w = prob.w
    os_ = prob.surrogate()
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    ds = rom.SurrogateSourceBasis.cluster_pod(basis, prob.g1, prob.ids, ClusterCriterion.neighbor(1.0), 1)
    L = ds.export_lists()
    np.testing.assert_array_equal(L["cluster_node_ids"], os_.cluster_node_ids)
    for k, ok in (("mem_off", os_.mem_off), ("mem_ids", os_.mem_ids), ("cl_off", os_.cl_off),
                  ("cl_list", os_.cl_list), ("direct_ids", os_.direct_ids), ("d_off", os_.d_off),
                  ("d_list", os_.d_list)):
        np.testing.assert_array_equal(L[k], ok, err_msg=k)
    np.testing.assert_array_equal(L["direct_phi"], os_.direct_phi)
    np.testing.assert_array_equal(L["direct_x0"], os_.direct_x0)
    e = ds.export()
    np.testing.assert_array_equal(e["phi_tilde"], os_.phi_tilde)
    np.testing.assert_array_equal(e["x0_tilde"], os_.x0_tilde)
    np.testing.assert_array_equal(e["gamma_tilde"], os_.gamma_tilde)
    np.testing.assert_array_equal(e["direct_gamma"], os_.direct_gamma)


def test_config4_pipeline_built_on_device(pt, oracle):
    """BASELINE configs[3] recipe at N = 65,536 end to end with product-built
    offline tables: sample ids, surrogate lists equal the oracle's and the
    batched x̂ match the oracle's per-instance ptrom_simulate."""
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.tree import ClusterCriterion
    w = workloads.config4(n=1 << 16, n_inst=4)
    ids = rom.greedy_sample(w.phi_r, w.n_samples)
    np.testing.assert_array_equal(ids, oracle.greedy_sample(w.phi_r, w.n_samples))
    A = rom.build_gnat_operator(w.phi_r, ids)
    g1 = w.gamma_a + w.gamma_b
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, ids, A)
    ds = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
    steps = 5
    tr = rom.ptrom_simulate_batch(basis, op, ds, w.gamma_a, w.gamma_b, w.mu, pt.ParticleSystem(g1, w.delta),
                                  pt.TimeGrid(w.dt, steps), rom.RomConfig(1e-300, 5, 1.0))
    A_o = oracle.build_gnat_operator(w.phi_r, ids)
    for i, m in enumerate(w.mu):
        os_ = oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
        xo, it_o, _ = oracle.ptrom_simulate(os_, w.phi, w.sv, w.x0, ids, A_o, w.gamma_a + m * w.gamma_b, w.delta,
                                            w.dt, steps, 1e-300, 5)
        assert max(rel(tr.x_hat[i, s], xo[:, s]) for s in range(steps)) <= 1e-12


@pytest.fixture(scope="module")
def config4_full(pt, oracle):
    """BASELINE configs[3] at its full size, N = 1,048,576:
    Φ the 16-mode POD of 200 seeded snapshots, M_r = 32, n_t = 20,972.
    Sample ids and A come from the product (the oracle's greedy scan at this
    N is ~2e10 score evaluations; ids are pinned byte-equal at smaller N), so
    both sides consume identical bytes."""
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.tree import ClusterCriterion
    w = workloads.config4(n_inst=4)
    ids = rom.greedy_sample(w.phi_r, w.n_samples)
    A = rom.build_gnat_operator(w.phi_r, ids)
    g1 = w.gamma_a + w.gamma_b
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, ids, A)
    ds = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
    os_ = oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
    return w, ids, A, g1, basis, op, ds, os_


def test_config4_full_size_surrogate_equals_oracle(pt, config4_full):
    """Full-N weighted POD tree (leaf 1) + cluster_pod(neighbor p_c = 1):
    every list byte-equal and every table bitwise (reduction.hpp:236-385),
    including the > 4,096-member clusters (reassign_big_kernel)."""
    w, ids, A, g1, basis, op, ds, os_ = config4_full
    L = ds.export_lists()
    sizes = np.diff(os_.mem_off)
    assert sizes.max() > 4096  # the one-CTA-per-cluster reassign path is exercised
    np.testing.assert_array_equal(L["cluster_node_ids"], os_.cluster_node_ids)
    for k, ok in (("mem_off", os_.mem_off), ("mem_ids", os_.mem_ids), ("cl_off", os_.cl_off),
                  ("cl_list", os_.cl_list), ("direct_ids", os_.direct_ids), ("d_off", os_.d_off),
                  ("d_list", os_.d_list)):
        np.testing.assert_array_equal(L[k], ok, err_msg=k)
    e = ds.export()
    for k in ("phi_tilde", "x0_tilde", "gamma_tilde", "direct_gamma"):
        np.testing.assert_array_equal(e[k], getattr(os_, k), err_msg=k)


def test_config4_full_size_reassign_bit_exact(pt, config4_full):
    """reduction.hpp:400-431 at N = 1M for μ = 1.37: the 203 clusters above
    4,096 members (largest ~2.4e5) go through reassign_big_kernel."""
    w, ids, A, g1, basis, op, ds, os_ = config4_full
    g = w.gamma_a + 1.37 * w.gamma_b
    from paper_2103_01983_b200 import rom
    from oracle import pyoracle
    o2 = pyoracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
    o2.reassign(g)
    d2 = rom.SurrogateSourceBasis.from_tables(
        os_.phi_tilde, os_.gamma_tilde, os_.x0_tilde, os_.zero_gamma, os_.mem_off, os_.mem_ids, os_.targets,
        os_.cl_off, os_.cl_list, os_.direct_ids, os_.direct_phi, os_.direct_x0, os_.direct_gamma, os_.d_off,
        os_.d_list)
    d2.reassign_cluster_circulation(g, basis)
    e = d2.export()
    for k in ("phi_tilde", "x0_tilde", "gamma_tilde", "direct_gamma"):
        np.testing.assert_array_equal(e[k], getattr(o2, k), err_msg=k)


def test_config4_full_size_ptrom_simulate(pt, oracle, config4_full):
    """rom.hpp:404-412 at N = 1M: the single-instance drop-in (exact
    reassign, 1 instance x 2 steps) and the batched affine path (2 instances
    x 2 steps), both against the oracle's ptrom_simulate; RomConfig{1e-300,
    5, 1} as the §8d config (5 GN updates, 6 hyperpair calls per step)."""
    from paper_2103_01983_b200 import rom
    w, ids, A, g1, basis, op, ds, os_ = config4_full
    steps = 2
    mu0 = float(w.mu[0])
    g = w.gamma_a + mu0 * w.gamma_b
    xo, it_o, cv_o = oracle.ptrom_simulate(oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1), w.phi, w.sv,
                                           w.x0, ids, A, g, w.delta, w.dt, steps, 1e-300, 5)
    d1 = rom.SurrogateSourceBasis.from_tables(
        os_.phi_tilde, os_.gamma_tilde, os_.x0_tilde, os_.zero_gamma, os_.mem_off, os_.mem_ids, os_.targets,
        os_.cl_off, os_.cl_list, os_.direct_ids, os_.direct_phi, os_.direct_x0, os_.direct_gamma, os_.d_off,
        os_.d_list)
    tr = rom.ptrom_simulate(basis, op, d1, pt.ParticleSystem(g, w.delta), pt.TimeGrid(w.dt, steps),
                            rom.RomConfig(1e-300, 5, 1.0))
    np.testing.assert_array_equal(tr.iterations, it_o)
    assert max(rel(tr.x_hat[:, s], xo[:, s]) for s in range(steps)) <= 1e-12
    mus = np.array([w.mu[1], w.mu[2]])
    tb = rom.ptrom_simulate_batch(basis, op, ds, w.gamma_a, w.gamma_b, mus, pt.ParticleSystem(g1, w.delta),
                                  pt.TimeGrid(w.dt, steps), rom.RomConfig(1e-300, 5, 1.0))
    for i, m in enumerate(mus):
        xo, it_o, _ = oracle.ptrom_simulate(oracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1), w.phi, w.sv,
                                            w.x0, ids, A, w.gamma_a + m * w.gamma_b, w.delta, w.dt, steps, 1e-300, 5)
        np.testing.assert_array_equal(tb.iterations[i], it_o)
        assert max(rel(tb.x_hat[i, s], xo[:, s]) for s in range(steps)) <= 1e-12, m


@pytest.mark.parametrize("delta", [None, 0.0])
def test_hyperpair_kernel_variants_bitwise(pt, prob, delta):
    """The batched march's hyperpair kernels (ptrom_set_tuning
    "hyperpair_variant": engine U = 3 default, U = 4, per-SM target ranges,
    and the generic kernel) give bit-identical x̂ — same per-target summation
    order — with a partial 32-instance chunk (B = 40), δ = 0 included (the
    coincident-centroid check path), and match the oracle."""
    from paper_2103_01983_b200 import rom
    w = prob.w
    d = w.delta if delta is None else delta
    steps = 4
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, prob.ids, prob.A)
    ds = to_device(rom, prob.surrogate())
    mu = np.linspace(0.5, 2.0, 40)
    ctx = ds.ctx
    out = {}
    try:
        for v in (1, 0, 2, 3):
            ctx.set_tuning("hyperpair_variant", v)
            tr = rom.ptrom_simulate_batch(basis, op, ds, w.gamma_a, w.gamma_b, mu, pt.ParticleSystem(prob.g1, d),
                                          pt.TimeGrid(w.dt, steps), rom.RomConfig(1e-300, 5, 1.0), batch=40)
            out[v] = np.asarray(tr.x_hat).copy()
    finally:
        ctx.set_tuning("hyperpair_variant", 0)
    for v in (0, 2, 3):
        np.testing.assert_array_equal(out[v], out[1])
    for i in (0, 17, 39):
        xo, _, _ = prob.oracle.ptrom_simulate(prob.surrogate(), w.phi, w.sv, w.x0, prob.ids, prob.A,
                                              w.gamma_a + mu[i] * w.gamma_b, d, w.dt, steps, 1e-300, 5)
        assert max(rel(out[0][i, s], xo[:, s]) for s in range(steps)) <= 1e-12


def test_batch_engine_inflow_scaled_form(pt, prob):
    """The batched march's engine kernels with an inflow field and the
    denominator-scaled kernel form (kernel.hpp:29-42): x̂ matches the oracle's
    per-instance ptrom_simulate and the generic kernel bit for bit."""
    from paper_2103_01983_b200 import rom
    w = prob.w
    rng = np.random.default_rng(11)
    inflow = rng.uniform(-0.05, 0.05, 2 * w.n)
    steps = 4
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, prob.ids, prob.A)
    ds = to_device(rom, prob.surrogate())
    mu = np.array([0.6, 1.1, 1.9])
    sys_ = pt.ParticleSystem(prob.g1, 0.02, inflow, 1)
    out = {}
    try:
        for v in (0, 1):
            ds.ctx.set_tuning("hyperpair_variant", v)
            tr = rom.ptrom_simulate_batch(basis, op, ds, w.gamma_a, w.gamma_b, mu, sys_, pt.TimeGrid(w.dt, steps),
                                          rom.RomConfig(1e-300, 5, 1.0))
            out[v] = np.asarray(tr.x_hat).copy()
    finally:
        ds.ctx.set_tuning("hyperpair_variant", 0)
    np.testing.assert_array_equal(out[0], out[1])
    for i, m in enumerate(mu):
        xo, _, _ = prob.oracle.ptrom_simulate(prob.surrogate(), w.phi, w.sv, w.x0, prob.ids, prob.A,
                                              w.gamma_a + m * w.gamma_b, 0.02, w.dt, steps, 1e-300, 5, 1.0, 1, inflow)
        assert max(rel(out[0][i, s], xo[:, s]) for s in range(steps)) <= 1e-12, m
