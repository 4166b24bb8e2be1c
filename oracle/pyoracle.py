"""ctypes wrapper of the CPU ORACLE (oracle/build/libptrom_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the checker or the
CPU baseline — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libptrom_oracle.so")
KAT = os.path.join(HERE, "build", "kat")


def build() -> None:
    subprocess.run(["make", "-C", HERE, "-j4"], check=True, stdout=subprocess.DEVNULL)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_kernel_eval_count.restype = C.c_uint64
        _lib.oracle_tree_num_nodes.restype = C.c_int64
        _lib.oracle_tree_build_f64.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                               C.POINTER(C.c_void_p)]
        _lib.oracle_tree_free.argtypes = [C.c_void_p]
        _lib.oracle_tree_num_nodes.argtypes = [C.c_void_p]
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().oracle_last_error().decode())


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def pairwise_velocity(x, gamma, delta, form=0, inflow=None, t_begin=0, t_end=None, threads=1):
    """kernel.hpp:107-129 over target rows [t_begin, t_end) (others zero)."""
    dtype = np.float32 if np.asarray(x).dtype == np.float32 else np.float64
    x = np.ascontiguousarray(x, dtype=dtype)
    g = np.ascontiguousarray(gamma, dtype=dtype)
    inf = None if inflow is None else np.ascontiguousarray(inflow, dtype=dtype)
    n = g.shape[0]
    t_end = n if t_end is None else t_end
    f = np.zeros(2 * n, dtype=dtype)
    if dtype == np.float32:
        _check(lib().oracle_pairwise_velocity_f32(C.c_int64(n), _p(x), _p(g), C.c_float(delta), C.c_int(form),
                                                  _p(inf), C.c_int64(t_begin), C.c_int64(t_end), C.c_int(threads),
                                                  _p(f)))
    else:
        _check(lib().oracle_pairwise_velocity_f64(C.c_int64(n), _p(x), _p(g), C.c_double(delta), C.c_int(form),
                                                  _p(inf), C.c_int64(t_begin), C.c_int64(t_end), C.c_int(threads),
                                                  _p(f)))
    return f


def inexact_kernel_jacobian(x, gamma, delta, form=0, t_begin=0, t_end=None, threads=1):
    """kernel.hpp:154-170 → (4, N) dfx_dx, dfx_dy, dfy_dx, dfy_dy."""
    x, g = _f64(x), _f64(gamma)
    n = g.shape[0]
    t_end = n if t_end is None else t_end
    out = np.zeros((4, n))
    _check(lib().oracle_inexact_kernel_jacobian_f64(C.c_int64(n), _p(x), _p(g), C.c_double(delta), C.c_int(form),
                                                    C.c_int64(t_begin), C.c_int64(t_end), C.c_int(threads),
                                                    _p(out[0]), _p(out[1]), _p(out[2]), _p(out[3])))
    return out


def hamiltonian(x, gamma):
    """kernel.hpp:174-191."""
    x, g = _f64(x), _f64(gamma)
    out = C.c_double()
    _check(lib().oracle_hamiltonian_f64(C.c_int64(g.shape[0]), _p(x), _p(g), C.byref(out)))
    return out.value


def velocity_field_grid(x, gamma, delta, form, x_min, x_max, nx, y_min, y_max, ny, c_g, l, gamma_bar):
    """kernel.hpp:213-238 → (ny, nx) array."""
    x, g = _f64(x), _f64(gamma)
    grid = np.zeros(nx * ny)
    d = C.c_double
    _check(lib().oracle_velocity_field_grid_f64(C.c_int64(g.shape[0]), _p(x), _p(g), d(delta), C.c_int(form),
                                                d(x_min), d(x_max), C.c_int64(nx), d(y_min), d(y_max),
                                                C.c_int64(ny), d(c_g), d(l), d(gamma_bar), _p(grid)))
    return grid.reshape(nx, ny).T


def reconstruct_output(phi, x_ref, x_hat, dofs=None):
    """rom.hpp:45-58 (rows dofs) / rom.hpp:60-64 (all rows): x_ref[d] + Φ[d,:]·x̂."""
    phi, x_ref, x_hat = np.asarray(phi, float), np.asarray(x_ref, float), np.asarray(x_hat, float)
    rows = np.arange(phi.shape[0]) if dofs is None else np.asarray(dofs, np.int64)
    return phi[rows, :] @ x_hat + x_ref[rows][:, None]


def fom_simulate(x0, gamma, delta, dt, n_steps, form=0, inflow=None, tol=1e-10, max_iters=100, refresh=1,
                 threads=1):
    """integrators.hpp:243-272 → (snapshots (2N, steps), iterations, converged, relative_residual)."""
    x0, g, inf = _f64(x0), _f64(gamma), _f64(inflow)
    n = g.shape[0]
    snaps = np.zeros((n_steps, 2 * n))
    iters = np.zeros(n_steps, dtype=np.int32)
    conv = np.zeros(n_steps, dtype=np.uint8)
    rel = np.zeros(n_steps)
    _check(lib().oracle_fom_simulate_f64(C.c_int64(n), _p(x0), _p(g), C.c_double(delta), C.c_int(form), _p(inf),
                                         C.c_double(dt), C.c_int64(n_steps), C.c_double(tol), C.c_int(max_iters),
                                         C.c_int(refresh), C.c_int(threads), _p(snaps), _p(iters), _p(conv),
                                         _p(rel)))
    return snaps.T, iters, conv, rel


class Tree:
    """quadtree.hpp:124-162 build_tree; arrays exported in SoA form."""

    def __init__(self, px, py, gamma, leaf_capacity):
        self.px, self.py, self.gamma = _f64(px), _f64(py), _f64(gamma)
        self.n = self.px.shape[0]
        h = C.c_void_p()
        _check(lib().oracle_tree_build_f64(self.n, _p(self.px), _p(self.py), _p(self.gamma), leaf_capacity,
                                           C.byref(h)))
        self.h = h
        nn = lib().oracle_tree_num_nodes(h)
        self.num_nodes = nn
        self.bounds = np.zeros((nn, 4))
        self.width = np.zeros(nn)
        self.centroid = np.zeros((nn, 2))
        self.gamma_sum = np.zeros(nn)
        self.children = np.zeros((nn, 4), dtype=np.int32)
        self.begin = np.zeros(nn, dtype=np.int64)
        self.end = np.zeros(nn, dtype=np.int64)
        self.depth = np.zeros(nn, dtype=np.int32)
        self.fallback = np.zeros(nn, dtype=np.uint8)
        self.perm = np.zeros(self.n, dtype=np.int64)
        self.slot = np.zeros(self.n, dtype=np.int64)
        self.leaf_node = np.zeros(self.n, dtype=np.int32)
        lib().oracle_tree_export(h, *(_p(a) for a in (self.bounds, self.width, self.centroid, self.gamma_sum,
                                                       self.children, self.begin, self.end, self.depth,
                                                       self.fallback, self.perm, self.slot, self.leaf_node)))

    def collect_clusters(self, target, crit_kind, crit_value):
        nn, nd = C.c_int64(), C.c_int64()
        _check(lib().oracle_collect_clusters(self.h, C.c_int64(target), C.c_int(crit_kind), C.c_double(crit_value),
                                             None, C.c_int64(0), None, C.c_int64(0), C.byref(nn), C.byref(nd)))
        nodes = np.zeros(nn.value, dtype=np.int32)
        direct = np.zeros(nd.value, dtype=np.int64)
        _check(lib().oracle_collect_clusters(self.h, C.c_int64(target), C.c_int(crit_kind), C.c_double(crit_value),
                                             _p(nodes), C.c_int64(nn.value), _p(direct), C.c_int64(nd.value),
                                             C.byref(nn), C.byref(nd)))
        return nodes, direct

    def bh_velocity(self, x, gamma, delta, crit_kind, crit_value, form=0, inflow=None, t_begin=0, t_end=None,
                    threads=1):
        x, g, inf = _f64(x), _f64(gamma), _f64(inflow)
        t_end = self.n if t_end is None else t_end
        f = np.zeros(2 * self.n)
        _check(lib().oracle_bh_velocity_f64(self.h, C.c_int64(self.n), _p(x), _p(g), C.c_double(delta),
                                            C.c_int(form), _p(inf), C.c_int(crit_kind), C.c_double(crit_value),
                                            C.c_int64(t_begin), C.c_int64(t_end), C.c_int(threads), _p(f)))
        return f

    def bh_jacobian(self, x, gamma, delta, crit_kind, crit_value, form=0):
        x, g = _f64(x), _f64(gamma)
        out = np.zeros((4, self.n))
        _check(lib().oracle_bh_jacobian_f64(self.h, C.c_int64(self.n), _p(x), _p(g), C.c_double(delta),
                                            C.c_int(form), C.c_int(crit_kind), C.c_double(crit_value),
                                            _p(out[0]), _p(out[1]), _p(out[2]), _p(out[3])))
        return out

    def __del__(self):
        try:
            lib().oracle_tree_free(self.h)
        except Exception:
            pass


# ------------------------------------------------------------------ rom ----
def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _fortran(m):
    """Column-major float64 buffer of a 2-D array (Eigen layout)."""
    return np.asfortranarray(np.asarray(m, dtype=np.float64))


def greedy_sample(phi_r, n_target, preseed=()):
    """reduction.hpp:93-168 → sorted sample ids."""
    pr = _fortran(phi_r)
    pre = _i64(list(preseed))
    out = np.zeros(n_target, np.int64)
    _check(lib().oracle_greedy_sample(C.c_int64(pr.shape[0]), C.c_int64(pr.shape[1]), _p(pr), C.c_int64(n_target),
                                      C.c_int64(pre.shape[0]), _p(pre), _p(out)))
    return out


def build_gnat_operator(phi_r, sample_ids):
    """reduction.hpp:182-220 → A (m_r x 2 n_s)."""
    pr = _fortran(phi_r)
    ids = _i64(sample_ids)
    A = np.zeros((pr.shape[1], 2 * ids.shape[0]), order="F")
    _check(lib().oracle_build_gnat_operator(C.c_int64(pr.shape[0]), C.c_int64(pr.shape[1]), _p(pr),
                                            C.c_int64(ids.shape[0]), _p(ids), _p(A)))
    return A


class Surrogate:
    """build_weighted_pod_tree + cluster_pod (reduction.hpp:236-385)."""

    def __init__(self, phi, sv, x_ref, gamma, targets, crit_kind=1, crit_value=1.0, leaf_capacity=1):
        self.phi, self.sv, self.x_ref = _fortran(phi), _f64(sv), _f64(x_ref)
        self.gamma = _f64(gamma)
        self.n = self.gamma.shape[0]
        self.m = self.phi.shape[1]
        t = _i64(targets)
        h = C.c_void_p()
        _check(lib().oracle_surrogate_build(C.c_int64(self.n), C.c_int64(self.m), _p(self.phi), _p(self.sv),
                                            _p(self.x_ref), _p(self.gamma), C.c_int64(leaf_capacity),
                                            C.c_int(crit_kind), C.c_double(crit_value), C.c_int64(t.shape[0]),
                                            _p(t), C.byref(h)))
        self.h = h
        self.targets = t
        self.refresh()

    def refresh(self):
        sz = np.zeros(6, np.int64)
        lib().oracle_surrogate_sizes(self.h, _p(sz))
        nc, u, nmem, ncl, nd, nt = (int(v) for v in sz)
        m = self.m
        self.n_clusters, self.n_direct = nc, u
        self.phi_tilde = np.zeros((2 * nc, m), order="F")
        self.gamma_tilde = np.zeros(nc)
        self.x0_tilde = np.zeros(2 * nc)
        self.zero_gamma = np.zeros(nc, np.uint8)
        self.mem_off = np.zeros(nc + 1, np.int64)
        self.mem_ids = np.zeros(max(nmem, 1), np.int64)
        self.cluster_node_ids = np.zeros(nc, np.int32)
        self.cl_off = np.zeros(nt + 1, np.int64)
        self.cl_list = np.zeros(max(ncl, 1), np.int64)
        self.direct_ids = np.zeros(u, np.int64)
        self.direct_phi = np.zeros((2 * u, m), order="F")
        self.direct_x0 = np.zeros(2 * u)
        self.direct_gamma = np.zeros(u)
        self.d_off = np.zeros(nt + 1, np.int64)
        self.d_list = np.zeros(max(nd, 1), np.int64)
        lib().oracle_surrogate_export(self.h, *(_p(a) for a in (
            self.phi_tilde, self.gamma_tilde, self.x0_tilde, self.zero_gamma, self.mem_off, self.mem_ids,
            self.cluster_node_ids, self.cl_off, self.cl_list, self.direct_ids, self.direct_phi, self.direct_x0,
            self.direct_gamma, self.d_off, self.d_list)))
        self.mem_ids = self.mem_ids[:nmem]
        self.cl_list = self.cl_list[:ncl]
        self.d_list = self.d_list[:nd]

    def reassign(self, gamma):
        g = _f64(gamma)
        _check(lib().oracle_surrogate_reassign(self.h, C.c_int64(g.shape[0]), _p(g)))
        self.refresh()

    def hyperpair(self, target_positions, x_hat, gamma, delta, form=0, inflow=None):
        nt = self.targets.shape[0]
        tp, xh, g, inf = _f64(target_positions), _f64(x_hat), _f64(gamma), _f64(inflow)
        f = np.zeros(2 * nt)
        jac = np.zeros((4, nt))
        cpos = np.zeros(2 * self.n_clusters)
        dpos = np.zeros(2 * self.n_direct)
        _check(lib().oracle_hyperpair(self.h, C.c_int64(g.shape[0]), _p(g), C.c_double(delta), C.c_int(form),
                                      _p(inf), _p(tp), _p(xh), _p(f), _p(jac), _p(cpos), _p(dpos)))
        return f, jac, cpos, dpos

    def __del__(self):
        try:
            lib().oracle_surrogate_free(self.h)
        except Exception:
            pass


def ptrom_simulate(surrogate, phi, sv, x_ref, sample_ids, A, gamma, delta, dt, n_steps, tol=1e-4, max_iters=100,
                   step_length=1.0, form=0, inflow=None):
    """rom.hpp:404-412 (surrogate=None: the gappy GnatSolver baseline)."""
    phi_f, sv_, xr = _fortran(phi), _f64(sv), _f64(x_ref)
    ids = _i64(sample_ids)
    A_ = _fortran(A)
    g, inf = _f64(gamma), _f64(inflow)
    m = phi_f.shape[1]
    x_hat = np.zeros((m, n_steps), order="F")
    iters = np.zeros(n_steps, np.int32)
    conv = np.zeros(n_steps, np.uint8)
    _check(lib().oracle_ptrom_simulate(surrogate.h if surrogate is not None else None, C.c_int64(g.shape[0]),
                                       C.c_int64(m), _p(phi_f), _p(sv_), _p(xr), C.c_int64(ids.shape[0]), _p(ids),
                                       C.c_int64(A_.shape[0]), _p(A_), _p(g), C.c_double(delta), C.c_int(form),
                                       _p(inf), C.c_double(dt), C.c_int64(n_steps), C.c_double(tol),
                                       C.c_int(max_iters), C.c_double(step_length), _p(x_hat), _p(iters),
                                       _p(conv)))
    if surrogate is not None:
        surrogate.refresh()
    return x_hat, iters, conv
