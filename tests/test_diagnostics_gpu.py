"""hamiltonian (kernel.hpp:174-191) and velocity_field_grid (kernel.hpp:213-238)
— SURVEY.md §8f row 1 — through the C ABI, against the oracle and the
reference's known answers (test_kernel.cpp:248-310)."""
import numpy as np
import pytest

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu


def test_hamiltonian_two_particle_value(pt):
    # test_kernel.cpp:248-255
    e = np.exp(1.0)
    sys = pt.ParticleSystem(np.ones(2), 0.0)
    h = pt.hamiltonian(np.array([0.0, e, 0.0, 0.0]), sys)
    assert abs(h - 1.0 / (2 * np.pi)) <= 1e-14 * (1 + abs(h))


@pytest.mark.parametrize("n", [6, 1000, 8192])
def test_hamiltonian_matches_oracle_and_translation(pt, oracle, n):
    w = workloads.config1(n=n, seed=23)
    sys = pt.ParticleSystem(w.gamma, 0.0)
    h = pt.hamiltonian(w.x0, sys)
    ref = oracle.hamiltonian(w.x0, w.gamma)
    # Different summation order: bound the difference by the sum of |terms|.
    x, y = w.x0[:n], w.x0[n:]
    if n <= 1000:
        d = np.hypot(x[:, None] - x[None, :], y[:, None] - y[None, :])
        np.fill_diagonal(d, 1.0)
        mag = np.sum(np.abs(np.outer(w.gamma, w.gamma) * np.log(d))) / (4 * np.pi)
    else:
        mag = np.sum(np.abs(w.gamma)) ** 2 * 10.0
    assert abs(h - ref) <= 1e-13 * mag + 1e-12 * abs(ref), (h, ref)
    # bit-reproducible run to run
    assert pt.hamiltonian(w.x0, sys) == h
    shifted = w.x0.copy()
    shifted[:n] += 3.25
    shifted[n:] -= 1.5
    assert abs(pt.hamiltonian(shifted, sys) - h) <= 1e-12 * (abs(h) + mag)


def test_hamiltonian_coincident_pair_names_first_pair(pt):
    w = workloads.config1(n=300, seed=3)
    x = w.x0.copy()
    n = 300
    x[17], x[17 + n] = x[5], x[5 + n]
    x[250], x[250 + n] = x[40], x[40 + n]
    with pytest.raises(pt.NumericalError, match="coincident particles 5 and 17"):
        pt.hamiltonian(x, pt.ParticleSystem(w.gamma, 0.0))
    # the context stays usable
    assert np.isfinite(pt.hamiltonian(w.x0, pt.ParticleSystem(w.gamma, 0.0)))


def test_velocity_field_grid_single_vortex(pt):
    # test_kernel.cpp:287-310
    sys = pt.ParticleSystem(np.array([2 * np.pi]), 0.0)
    x = np.zeros(2)
    lat = pt.LatticeSpec(-1.0, 1.0, 2, 0.0, 1.0, 2)
    c_g, l, gb = 1.25, 2.0, 4.0
    g = pt.velocity_field_grid(x, sys, lat, c_g, l, gb)
    assert g.shape == (2, 2)
    tol = lambda a, b: abs(a - b) <= 1e-13 * (1 + max(abs(a), abs(b)))
    assert tol(g[0, 0], c_g * l / gb) and tol(g[0, 1], c_g * l / gb)
    assert tol(g[1, 0], c_g * l / gb / np.sqrt(2.0))
    with pytest.raises(pt.ConfigError):
        pt.velocity_field_grid(x, sys, lat, c_g, l, 0.0)
    with pytest.raises(pt.ConfigError):
        pt.velocity_field_grid(x, sys, pt.LatticeSpec(-1.0, 1.0, 1, 0.0, 1.0, 2), c_g, l, gb)
    with pytest.raises(pt.NumericalError):
        pt.velocity_field_grid(x, sys, pt.LatticeSpec(-1.0, 1.0, 3, -1.0, 1.0, 3), c_g, l, gb)


@pytest.mark.parametrize("nx,ny,form", [(33, 17, 0), (200, 150, 1)])
def test_velocity_field_grid_matches_oracle(pt, oracle, nx, ny, form):
    w = workloads.config1(n=4096, seed=7)
    sys = pt.ParticleSystem(w.gamma, w.delta, kernel_form=form)
    lat = pt.LatticeSpec(-1.2, 1.1, nx, -0.9, 1.3, ny)
    got = pt.velocity_field_grid(w.x0, sys, lat, 1.3, 0.7, 0.05)
    ref = oracle.velocity_field_grid(w.x0, w.gamma, w.delta, form, -1.2, 1.1, nx, -0.9, 1.3, ny, 1.3, 0.7, 0.05)
    assert got.shape == (ny, nx)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12


def test_device_entry_points(pt, oracle):
    import torch
    from paper_2103_01983_b200 import device as dev
    w = workloads.config1(n=2048, seed=9)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    h = dev.hamiltonian(x, g)
    lat = pt.LatticeSpec(-1.0, 1.0, 40, -1.0, 1.0, 30)
    grid = dev.velocity_field_grid(x, g, w.delta, 0, lat, 1.0, 1.0, 1.0)
    dev.synchronize()
    assert float(h.item()) == pt.hamiltonian(w.x0, pt.ParticleSystem(w.gamma, 0.0))
    ref = oracle.velocity_field_grid(w.x0, w.gamma, w.delta, 0, -1.0, 1.0, 40, -1.0, 1.0, 30, 1.0, 1.0, 1.0)
    assert np.linalg.norm(grid.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-12
