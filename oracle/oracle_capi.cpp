// oracle_capi.cpp — C entry points over the CPU ORACLE (test infrastructure
// only: called from tests/, __graft_entry__.smoke() and bench.py's CPU legs).
// Status codes mirror the product ABI: 0 ok, 2 config_error, 3 numerical_error.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ptrom_oracle.hpp"
#include "ptrom_oracle_rom.hpp"
#include "ptrom_oracle_tree.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const config_error& e) {
    g_err = e.what();
    return 2;
  } catch (const numerical_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

template <class S>
ParticleSystem<S> make_sys(std::int64_t n, const S* gamma, S delta, int form, const S* inflow) {
  ParticleSystem<S> sys;
  sys.circulation.assign(gamma, gamma + n);
  sys.delta = delta;
  sys.kernel_form = form ? KernelForm::denominator_scaled : KernelForm::standard;
  if (inflow) {
    sys.has_inflow = true;
    sys.inflow.assign(inflow, inflow + 2 * n);
  }
  return sys;
}

// Target-parallel pairwise model (OpenMP over targets; each target's sum is
// still the reference's sequential loop). n_threads == 1 is the reference's
// serial protocol.
template <class S>
struct ThreadedPairwiseModel {
  ParticleSystem<S> sys;
  int n_threads = 1;
  std::vector<S> velocity(const std::vector<S>& x) const {
    sys.validate();
    check_state<S>(x, sys, "pairwise_velocity");
    std::vector<S> f(x.size(), S(0));
    rows(x, f.data(), 0, sys.size());
    return f;
  }
  void rows(const std::vector<S>& x, S* f, Index b, Index e) const {
    if (n_threads <= 1) {
      pairwise_velocity_rows<S>(x, sys, b, e, f);
      return;
    }
    std::string err;
    int code = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(n_threads)
    for (Index i = b; i < e; ++i) {
      try {
        pairwise_velocity_rows<S>(x, sys, i, i + 1, f);
      } catch (const numerical_error& ex) {
#pragma omp critical
        {
          code = 3;
          err = ex.what();
        }
      }
    }
    if (code == 3) throw numerical_error(err);
  }
  BlockDiagonalJacobian<S> jacobian(const std::vector<S>& x) const {
    sys.validate();
    check_state<S>(x, sys, "inexact_kernel_jacobian");
    auto jac = BlockDiagonalJacobian<S>::Zero(sys.size());
    jac_rows(x, jac, 0, sys.size());
    return jac;
  }
  void jac_rows(const std::vector<S>& x, BlockDiagonalJacobian<S>& jac, Index b, Index e) const {
    if (n_threads <= 1) {
      inexact_kernel_jacobian_rows<S>(x, sys, b, e, jac);
      return;
    }
    std::string err;
    int code = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(n_threads)
    for (Index i = b; i < e; ++i) {
      try {
        inexact_kernel_jacobian_rows<S>(x, sys, i, i + 1, jac);
      } catch (const numerical_error& ex) {
#pragma omp critical
        {
          code = 3;
          err = ex.what();
        }
      }
    }
    if (code == 3) throw numerical_error(err);
  }
};

void check_range(std::int64_t n, std::int64_t b, std::int64_t e) {
  if (b < 0 || e > n || b > e) throw config_error("target range outside [0, n]");
}

}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
std::uint64_t oracle_kernel_eval_count() { return kernel_eval_counter; }
void oracle_reset_kernel_eval_count() { kernel_eval_counter = 0; }

int oracle_kernel_pair_f64(double tx, double ty, double sx, double sy, double gamma, double delta, int form,
                           double* out) {
  return guarded([&] {
    const V2<double> k = kernel_pair<double>({tx, ty}, {sx, sy}, gamma, delta,
                                             form ? KernelForm::denominator_scaled : KernelForm::standard);
    out[0] = k.x;
    out[1] = k.y;
  });
}

int oracle_kernel_pair_jacobian_f64(double tx, double ty, double sx, double sy, double gamma, double delta,
                                    int form, double* out) {
  return guarded([&] {
    const M2<double> j = kernel_pair_jacobian<double>({tx, ty}, {sx, sy}, gamma, delta,
                                                      form ? KernelForm::denominator_scaled : KernelForm::standard);
    out[0] = j.a00;
    out[1] = j.a01;
    out[2] = j.a10;
    out[3] = j.a11;
  });
}

// kernel.hpp:107-129 over targets [t_begin, t_end) (rows outside stay 0).
int oracle_pairwise_velocity_f64(std::int64_t n, const double* x, const double* gamma, double delta, int form,
                                 const double* inflow, std::int64_t t_begin, std::int64_t t_end, int n_threads,
                                 double* f) {
  return guarded([&] {
    ThreadedPairwiseModel<double> m{make_sys<double>(n, gamma, delta, form, inflow), n_threads};
    m.sys.validate();
    std::vector<double> xs(x, x + 2 * n);
    check_state<double>(xs, m.sys, "pairwise_velocity");
    check_range(n, t_begin, t_end);
    std::memset(f, 0, sizeof(double) * 2 * n);
    m.rows(xs, f, t_begin, t_end);
  });
}

int oracle_pairwise_velocity_f32(std::int64_t n, const float* x, const float* gamma, float delta, int form,
                                 const float* inflow, std::int64_t t_begin, std::int64_t t_end, int n_threads,
                                 float* f) {
  return guarded([&] {
    ThreadedPairwiseModel<float> m{make_sys<float>(n, gamma, delta, form, inflow), n_threads};
    m.sys.validate();
    std::vector<float> xs(x, x + 2 * n);
    check_state<float>(xs, m.sys, "pairwise_velocity");
    check_range(n, t_begin, t_end);
    std::memset(f, 0, sizeof(float) * 2 * n);
    m.rows(xs, f, t_begin, t_end);
  });
}

// kernel.hpp:154-170 over targets [t_begin, t_end).
int oracle_inexact_kernel_jacobian_f64(std::int64_t n, const double* x, const double* gamma, double delta,
                                       int form, std::int64_t t_begin, std::int64_t t_end, int n_threads,
                                       double* jxx, double* jxy, double* jyx, double* jyy) {
  return guarded([&] {
    ThreadedPairwiseModel<double> m{make_sys<double>(n, gamma, delta, form, nullptr), n_threads};
    m.sys.validate();
    std::vector<double> xs(x, x + 2 * n);
    check_state<double>(xs, m.sys, "inexact_kernel_jacobian");
    check_range(n, t_begin, t_end);
    auto jac = BlockDiagonalJacobian<double>::Zero(n);
    m.jac_rows(xs, jac, t_begin, t_end);
    std::memcpy(jxx, jac.dfx_dx.data(), sizeof(double) * n);
    std::memcpy(jxy, jac.dfx_dy.data(), sizeof(double) * n);
    std::memcpy(jyx, jac.dfy_dx.data(), sizeof(double) * n);
    std::memcpy(jyy, jac.dfy_dy.data(), sizeof(double) * n);
  });
}

int oracle_hamiltonian_f64(std::int64_t n, const double* x, const double* gamma, double* out) {
  return guarded([&] {
    auto sys = make_sys<double>(n, gamma, 0.0, 0, nullptr);
    std::vector<double> xs(x, x + 2 * n);
    *out = hamiltonian<double>(xs, sys);
  });
}

int oracle_velocity_field_grid_f64(std::int64_t n, const double* x, const double* gamma, double delta, int form,
                                   double x_min, double x_max, std::int64_t nx, double y_min, double y_max,
                                   std::int64_t ny, double c_g, double l, double gamma_bar, double* grid) {
  return guarded([&] {
    auto sys = make_sys<double>(n, gamma, delta, form, nullptr);
    std::vector<double> xs(x, x + 2 * n);
    const LatticeSpec<double> lat{x_min, x_max, nx, y_min, y_max, ny};
    const auto g = velocity_field_grid<double>(xs, sys, lat, c_g, l, gamma_bar);
    std::memcpy(grid, g.data(), sizeof(double) * g.size());
  });
}

// integrators.hpp:243-272 with the PairwiseModel (optionally target-threaded).
int oracle_fom_simulate_f64(std::int64_t n, const double* x0, const double* gamma, double delta, int form,
                            const double* inflow, double dt, std::int64_t n_steps, double tol, int max_iters,
                            int refresh, int n_threads, double* snapshots, int* iters, std::uint8_t* converged,
                            double* rel) {
  return guarded([&] {
    ThreadedPairwiseModel<double> m{make_sys<double>(n, gamma, delta, form, inflow), n_threads};
    NewtonConfig cfg{tol, max_iters, refresh};
    std::vector<double> xs(x0, x0 + 2 * n);
    auto res = fom_simulate<double>(xs, m, dt, n_steps, cfg);
    std::memcpy(snapshots, res.snapshots.data(), sizeof(double) * res.snapshots.size());
    for (std::int64_t s = 0; s < n_steps; ++s) {
      iters[s] = res.iterations[static_cast<size_t>(s)];
      converged[s] = static_cast<std::uint8_t>(res.converged[static_cast<size_t>(s)]);
      rel[s] = res.relative_residual[static_cast<size_t>(s)];
    }
  });
}

// ---------------------------------------------------------------- tree ----
struct oracle_tree {
  QuadTree<double> t;
};

int oracle_tree_build_f64(std::int64_t n, const double* px, const double* py, const double* gamma,
                          std::int64_t leaf_capacity, oracle_tree** out) {
  return guarded([&] {
    auto* h = new oracle_tree;
    try {
      h->t = build_tree<double>(std::vector<double>(px, px + n), std::vector<double>(py, py + n),
                                std::vector<double>(gamma, gamma + n), leaf_capacity);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void oracle_tree_free(oracle_tree* h) { delete h; }
std::int64_t oracle_tree_num_nodes(const oracle_tree* h) { return static_cast<std::int64_t>(h->t.nodes.size()); }

// Node table in structure-of-arrays form, matching the product's export.
void oracle_tree_export(const oracle_tree* h, double* bounds /*4*nn*/, double* width, double* centroid /*2*nn*/,
                        double* gamma_sum, std::int32_t* children /*4*nn*/, std::int64_t* begin, std::int64_t* end,
                        std::int32_t* depth, std::uint8_t* fallback, std::int64_t* perm, std::int64_t* slot,
                        std::int32_t* leaf_node) {
  const auto& t = h->t;
  for (size_t i = 0; i < t.nodes.size(); ++i) {
    const auto& nd = t.nodes[i];
    for (int k = 0; k < 4; ++k) {
      bounds[4 * i + k] = nd.bounds[static_cast<size_t>(k)];
      children[4 * i + k] = nd.children[static_cast<size_t>(k)];
    }
    width[i] = nd.width;
    centroid[2 * i] = nd.centroid.x;
    centroid[2 * i + 1] = nd.centroid.y;
    gamma_sum[i] = nd.gamma_sum;
    begin[i] = nd.begin;
    end[i] = nd.end;
    depth[i] = nd.depth;
    fallback[i] = nd.centroid_fallback ? 1 : 0;
  }
  for (size_t p = 0; p < t.perm.size(); ++p) {
    perm[p] = t.perm[p];
    slot[p] = t.slot[p];
    leaf_node[p] = t.leaf_node[p];
  }
}

// quadtree.hpp:213-252. Returns the list lengths; copies at most the given
// capacities.
int oracle_collect_clusters(const oracle_tree* h, std::int64_t target, int crit_kind, double crit_value,
                            std::int32_t* nodes, std::int64_t nodes_cap, std::int64_t* direct,
                            std::int64_t direct_cap, std::int64_t* n_nodes, std::int64_t* n_direct) {
  return guarded([&] {
    const auto crit = crit_kind ? ClusterCriterion<double>::neighbor(crit_value)
                                : ClusterCriterion<double>::barnes_hut(crit_value);
    const ClusterList cl = collect_clusters(h->t, target, crit);
    *n_nodes = static_cast<std::int64_t>(cl.cluster_nodes.size());
    *n_direct = static_cast<std::int64_t>(cl.direct_ids.size());
    for (size_t k = 0; k < cl.cluster_nodes.size() && static_cast<std::int64_t>(k) < nodes_cap; ++k)
      nodes[k] = cl.cluster_nodes[k];
    for (size_t k = 0; k < cl.direct_ids.size() && static_cast<std::int64_t>(k) < direct_cap; ++k)
      direct[k] = cl.direct_ids[k];
  });
}

// quadtree.hpp:257-281 over targets [t_begin, t_end).
int oracle_bh_velocity_f64(const oracle_tree* h, std::int64_t n, const double* x, const double* gamma,
                           double delta, int form, const double* inflow, int crit_kind, double crit_value,
                           std::int64_t t_begin, std::int64_t t_end, int n_threads, double* f) {
  return guarded([&] {
    auto sys = make_sys<double>(n, gamma, delta, form, inflow);
    sys.validate();
    std::vector<double> xs(x, x + 2 * n);
    check_state<double>(xs, sys, "bh_velocity");
    if (h->t.size() != n) throw config_error("bh_velocity: tree size mismatch");
    check_range(n, t_begin, t_end);
    const auto crit = crit_kind ? ClusterCriterion<double>::neighbor(crit_value)
                                : ClusterCriterion<double>::barnes_hut(crit_value);
    std::memset(f, 0, sizeof(double) * 2 * n);
    if (n_threads <= 1) {
      bh_velocity_rows<double>(h->t, xs, sys, crit, t_begin, t_end, f);
      return;
    }
    int code = 0;
    std::string err;
#pragma omp parallel for schedule(dynamic, 256) num_threads(n_threads)
    for (std::int64_t i = t_begin; i < t_end; ++i) {
      try {
        bh_velocity_rows<double>(h->t, xs, sys, crit, i, i + 1, f);
      } catch (const numerical_error& ex) {
#pragma omp critical
        {
          code = 3;
          err = ex.what();
        }
      }
    }
    if (code) throw numerical_error(err);
  });
}

int oracle_bh_jacobian_f64(const oracle_tree* h, std::int64_t n, const double* x, const double* gamma,
                           double delta, int form, int crit_kind, double crit_value, double* jxx, double* jxy,
                           double* jyx, double* jyy) {
  return guarded([&] {
    auto sys = make_sys<double>(n, gamma, delta, form, nullptr);
    std::vector<double> xs(x, x + 2 * n);
    const auto crit = crit_kind ? ClusterCriterion<double>::neighbor(crit_value)
                                : ClusterCriterion<double>::barnes_hut(crit_value);
    auto jac = bh_jacobian<double>(h->t, xs, sys, crit);
    std::memcpy(jxx, jac.dfx_dx.data(), sizeof(double) * n);
    std::memcpy(jxy, jac.dfx_dy.data(), sizeof(double) * n);
    std::memcpy(jyx, jac.dfy_dx.data(), sizeof(double) * n);
    std::memcpy(jyy, jac.dfy_dy.data(), sizeof(double) * n);
  });
}

// ----------------------------------------------------------------- rom ----
static Mat mat_from(Index rows, Index cols, const double* p) {
  Mat m(rows, cols);
  std::copy(p, p + rows * cols, m.a.begin());
  return m;
}

// reduction.hpp:93-168
int oracle_greedy_sample(std::int64_t n_dofs, std::int64_t n_r, const double* phi_r, std::int64_t n_target,
                         std::int64_t n_preseed, const std::int64_t* preseed, std::int64_t* out) {
  return guarded([&] {
    std::vector<Index> pre(preseed, preseed + n_preseed);
    const auto ids = greedy_sample(mat_from(n_dofs, n_r, phi_r), n_target, pre);
    std::copy(ids.begin(), ids.end(), out);
  });
}

// reduction.hpp:182-220 (A is m_r x 2 n_s, column-major)
int oracle_build_gnat_operator(std::int64_t n_dofs, std::int64_t m_r, const double* phi_r, std::int64_t n_s,
                               const std::int64_t* ids, double* A) {
  return guarded([&] {
    const auto op = build_gnat_operator(mat_from(n_dofs, m_r, phi_r), std::vector<Index>(ids, ids + n_s));
    std::copy(op.A.a.begin(), op.A.a.end(), A);
  });
}

struct oracle_surrogate {
  SurrogateSourceBasis s;
  PODBasis basis;
};

static PODBasis basis_from(std::int64_t n_dofs, std::int64_t m, const double* phi, const double* sv,
                           const double* x_ref) {
  PODBasis b;
  b.phi = mat_from(n_dofs, m, phi);
  b.singular_values.assign(sv, sv + m);
  b.x_ref.assign(x_ref, x_ref + n_dofs);
  return b;
}

// build_weighted_pod_tree (reduction.hpp:236-274) + cluster_pod (304-385)
int oracle_surrogate_build(std::int64_t n, std::int64_t m, const double* phi, const double* sv, const double* x_ref,
                           const double* gamma, std::int64_t leaf_cap, int crit_kind, double crit_value,
                           std::int64_t n_t, const std::int64_t* targets, oracle_surrogate** out) {
  return guarded([&] {
    auto* h = new oracle_surrogate;
    try {
      h->basis = basis_from(2 * n, m, phi, sv, x_ref);
      const auto crit = crit_kind ? ClusterCriterion<double>::neighbor(crit_value)
                                  : ClusterCriterion<double>::barnes_hut(crit_value);
      h->s = cluster_pod(h->basis, Vec(gamma, gamma + n), std::vector<Index>(targets, targets + n_t), crit, leaf_cap);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void oracle_surrogate_free(oracle_surrogate* h) { delete h; }

// sizes: [n_c, u, n_membership, n_cluster_list, n_direct_list, n_t]
void oracle_surrogate_sizes(const oracle_surrogate* h, std::int64_t* sz) {
  const auto& s = h->s;
  sz[0] = s.num_clusters();
  sz[1] = s.num_direct();
  std::int64_t a = 0, b = 0, c = 0;
  for (const auto& v : s.cluster_membership) a += static_cast<std::int64_t>(v.size());
  for (const auto& v : s.per_target_clusters) b += static_cast<std::int64_t>(v.size());
  for (const auto& v : s.per_target_direct) c += static_cast<std::int64_t>(v.size());
  sz[2] = a;
  sz[3] = b;
  sz[4] = c;
  sz[5] = static_cast<std::int64_t>(s.target_ids.size());
}

static void csr(const std::vector<std::vector<Index>>& v, std::int64_t* off, std::int64_t* ids) {
  off[0] = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    off[i + 1] = off[i] + static_cast<std::int64_t>(v[i].size());
    std::copy(v[i].begin(), v[i].end(), ids + off[i]);
  }
}

void oracle_surrogate_export(const oracle_surrogate* h, double* phi_tilde, double* gamma_tilde, double* x0_tilde,
                             std::uint8_t* zero_gamma, std::int64_t* mem_off, std::int64_t* mem_ids,
                             std::int32_t* cluster_node_ids, std::int64_t* cl_off, std::int64_t* cl_list,
                             std::int64_t* direct_ids, double* direct_phi, double* direct_x0, double* direct_gamma,
                             std::int64_t* d_off, std::int64_t* d_list) {
  const auto& s = h->s;
  std::copy(s.phi_tilde.a.begin(), s.phi_tilde.a.end(), phi_tilde);
  std::copy(s.gamma_tilde.begin(), s.gamma_tilde.end(), gamma_tilde);
  std::copy(s.x0_tilde.begin(), s.x0_tilde.end(), x0_tilde);
  for (size_t c = 0; c < s.zero_gamma.size(); ++c) zero_gamma[c] = static_cast<std::uint8_t>(s.zero_gamma[c]);
  csr(s.cluster_membership, mem_off, mem_ids);
  std::copy(s.cluster_node_ids.begin(), s.cluster_node_ids.end(), cluster_node_ids);
  csr(s.per_target_clusters, cl_off, cl_list);
  std::copy(s.direct_ids.begin(), s.direct_ids.end(), direct_ids);
  std::copy(s.direct_phi.a.begin(), s.direct_phi.a.end(), direct_phi);
  std::copy(s.direct_x0.begin(), s.direct_x0.end(), direct_x0);
  std::copy(s.direct_gamma.begin(), s.direct_gamma.end(), direct_gamma);
  csr(s.per_target_direct, d_off, d_list);
}

// reduction.hpp:400-431
int oracle_surrogate_reassign(oracle_surrogate* h, std::int64_t n, const double* gamma) {
  return guarded([&] { reassign_cluster_circulation(h->s, Vec(gamma, gamma + n), h->basis); });
}

// rom.hpp:101-155 (jac: 4 x n_t, rows dfx_dx, dfx_dy, dfy_dx, dfy_dy)
int oracle_hyperpair(const oracle_surrogate* h, std::int64_t n, const double* gamma, double delta, int form,
                     const double* inflow, const double* target_positions, const double* x_hat, double* f,
                     double* jac, double* cpos, double* dpos) {
  return guarded([&] {
    const auto sys = make_sys<double>(n, gamma, delta, form, inflow);
    const Index nt = static_cast<Index>(h->s.target_ids.size());
    const auto hp = hyperpair(h->s, Vec(target_positions, target_positions + 2 * nt),
                              Vec(x_hat, x_hat + h->basis.modes()), sys);
    std::copy(hp.f.begin(), hp.f.end(), f);
    std::copy(hp.jac.dfx_dx.begin(), hp.jac.dfx_dx.end(), jac);
    std::copy(hp.jac.dfx_dy.begin(), hp.jac.dfx_dy.end(), jac + nt);
    std::copy(hp.jac.dfy_dx.begin(), hp.jac.dfy_dx.end(), jac + 2 * nt);
    std::copy(hp.jac.dfy_dy.begin(), hp.jac.dfy_dy.end(), jac + 3 * nt);
    if (cpos) std::copy(hp.cluster_positions.begin(), hp.cluster_positions.end(), cpos);
    if (dpos) std::copy(hp.direct_positions.begin(), hp.direct_positions.end(), dpos);
  });
}

// rom.hpp:404-412 ptrom_simulate (surrogate mutated by the reassignment);
// with h == NULL the gappy GnatSolver baseline (rom.hpp:358-385) runs instead.
int oracle_ptrom_simulate(oracle_surrogate* h, std::int64_t n, std::int64_t m, const double* phi, const double* sv,
                          const double* x_ref, std::int64_t n_s, const std::int64_t* sample_ids, std::int64_t m_r,
                          const double* A, const double* gamma, double delta, int form, const double* inflow,
                          double dt, std::int64_t n_steps, double tol, int max_iters, double step_length,
                          double* x_hat, int* iters, std::uint8_t* conv) {
  return guarded([&] {
    const auto sys = make_sys<double>(n, gamma, delta, form, inflow);
    GnatOperator op;
    op.sample_ids.assign(sample_ids, sample_ids + n_s);
    for (Index k = 0; k < n_s; ++k) op.sampled_dofs.push_back(sample_ids[k]);
    for (Index k = 0; k < n_s; ++k) op.sampled_dofs.push_back(sample_ids[k] + n);
    op.A = mat_from(m_r, 2 * n_s, A);
    RomConfig cfg{tol, max_iters, step_length};
    RomTrajectory tr;
    if (h) {
      tr = ptrom_simulate(h->basis, op, h->s, sys, dt, n_steps, cfg);
    } else {
      const PODBasis b = basis_from(2 * n, m, phi, sv, x_ref);
      GnatSolver solver(b, op, sys, dt, cfg);
      tr = solver.simulate(n_steps);
    }
    std::copy(tr.x_hat.a.begin(), tr.x_hat.a.end(), x_hat);
    for (Index s = 0; s < n_steps; ++s) {
      iters[s] = tr.iterations[s];
      conv[s] = static_cast<std::uint8_t>(tr.converged[s]);
    }
  });
}

}  // extern "C"
