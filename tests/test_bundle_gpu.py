"""An OfflineBundle written in the reference layout drives the device online
path exactly like in-memory tables, and reconstruct_output/full
(rom.hpp:45-64) on the device match the oracle."""
import numpy as np
import pytest

from paper_2103_01983_b200 import bundle, workloads

pytestmark = pytest.mark.gpu


def test_bundle_to_device_simulate_equals_in_memory(pt, oracle, tmp_path):
    from paper_2103_01983_b200 import rom
    w = workloads.config4(n=2048, n_inst=2, modes=8, modes_r=16, seed=11)
    ids = oracle.greedy_sample(w.phi_r, w.n_samples)
    A = oracle.build_gnat_operator(w.phi_r, ids)
    g = w.gamma_a + w.gamma_b
    s = oracle.Surrogate(w.phi, w.sv, w.x0, g, ids, 1, 1.0, 1)
    b = bundle.OfflineBundle(
        config={"n": 2048}, basis_phi=w.phi, basis_sv=w.sv, basis_xref=w.x0, residual_phi=w.phi_r,
        residual_sv=np.ones(w.phi_r.shape[1]), gnat_a=A, sample_ids=ids, phi_tilde=s.phi_tilde, x0_tilde=s.x0_tilde,
        gamma_tilde=s.gamma_tilde, cluster_node_ids=s.cluster_node_ids, mem_off=s.mem_off, mem_ids=s.mem_ids,
        zero_gamma=s.zero_gamma, target_ids=s.targets, cl_off=s.cl_off, cl_list=s.cl_list, d_off=s.d_off,
        d_list=s.d_list, direct_ids=s.direct_ids, direct_phi=s.direct_phi, direct_x0=s.direct_x0,
        direct_gamma=s.direct_gamma)
    b.save(tmp_path / "b")
    basis, op, sur = bundle.OfflineBundle.load(tmp_path / "b").to_device()
    steps = 6
    gm = w.gamma_a + 1.3 * w.gamma_b
    tr = rom.ptrom_simulate(basis, op, sur, pt.ParticleSystem(gm, w.delta), pt.TimeGrid(w.dt, steps),
                            rom.RomConfig(1e-8, 20, 1.0))
    # the C loader (ptrom_bundle_open + ptrom_bundle_to_device) drives the same march bit for bit
    nb, no, ns = bundle.to_device_native(tmp_path / "b")
    tn = rom.ptrom_simulate(nb, no, ns, pt.ParticleSystem(gm, w.delta), pt.TimeGrid(w.dt, steps),
                            rom.RomConfig(1e-8, 20, 1.0))
    np.testing.assert_array_equal(tn.x_hat, tr.x_hat)
    np.testing.assert_array_equal(tn.iterations, tr.iterations)
    xo, it_o, _ = oracle.ptrom_simulate(oracle.Surrogate(w.phi, w.sv, w.x0, g, ids, 1, 1.0, 1), w.phi, w.sv, w.x0,
                                        ids, A, gm, w.delta, w.dt, steps, 1e-8, 20)
    np.testing.assert_array_equal(tr.iterations, it_o)
    for k in range(steps):
        assert np.linalg.norm(tr.x_hat[:, k] - xo[:, k]) <= 1e-12 * np.linalg.norm(xo[:, k])
    # the trajectory round-trips as a time series
    bundle.write_trajectory(tmp_path / "xhat.ptmx", tr.x_hat, w.dt)
    mf = bundle.read_matrix(tmp_path / "xhat.ptmx")
    np.testing.assert_array_equal(mf.data, tr.x_hat)
    assert mf.dt == w.dt
    # reconstruction of QoI dofs on device (rom.hpp:45-58)
    dofs = np.array([0, 5, 2047, 2048, 4095, 17])
    out = basis.reconstruct_output(tr.x_hat, dofs)
    ref = oracle.reconstruct_output(w.phi, w.x0, tr.x_hat, dofs)
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)
    full = basis.reconstruct_full(tr.x_hat)
    assert full.shape == (4096, steps)
    assert np.linalg.norm(full - oracle.reconstruct_output(w.phi, w.x0, tr.x_hat)) <= 1e-13 * np.linalg.norm(full)


def test_reconstruct_validation(pt):
    from paper_2103_01983_b200 import rom
    rng = np.random.default_rng(3)
    basis = rom.PODBasis(rng.standard_normal((40, 3)), np.ones(3), np.zeros(40))
    with pytest.raises(pt.ConfigError, match="coordinate dimension mismatch"):
        basis.reconstruct_output(np.zeros((4, 2)), [0])
    with pytest.raises(pt.ConfigError, match="dof out of range"):
        basis.reconstruct_output(np.zeros((3, 2)), [40])
    x = rng.standard_normal((3, 70))  # > one 32-step stage
    out = basis.reconstruct_output(x, [1, 39])
    np.testing.assert_allclose(out, basis.phi[[1, 39]] @ x, rtol=1e-13, atol=1e-14)
