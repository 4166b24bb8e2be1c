// ptrom_b200.hpp — header-only C++ adapters over the C ABI (ptrom_b200.h)
// that satisfy the reference's duck-typed FOM `Model` concept
// (integrators.hpp:69-102: velocity(x), jacobian(x)) so that
// FomStepper / fom_simulate / metrics can run on the B200 unchanged.
//
//  * ptrom_b200::Context           RAII owner of a ptrom_ctx (one per device/thread)
//  * ptrom_b200::PairwiseModelVec  std::vector<double> flavour (no Eigen needed)
//  * ptrom_b200::CudaPairwiseModel Eigen flavour, a drop-in for
//                                  ptrom::PairwiseModel<double> (integrators.hpp:69-79);
//                                  only compiled when <Eigen/Dense> and the
//                                  reference headers are available.
//
// Errors map to the reference's exception types: status 2 → config_error,
// status 3 → numerical_error (types.hpp:23-32); other failures → runtime_error.
// Every velocity call adds N(N-1) to the reference's kernel_eval_counter
// (kernel.hpp:18-25) when the reference headers are present.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ptrom_b200.h"

namespace ptrom_b200 {

struct config_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct numerical_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    if (ptrom_create(device, stream, &ctx_) != PTROM_OK)
      throw std::runtime_error("ptrom_create failed: libptrom_b200 needs an sm_100a (B200) device");
  }
  ~Context() { ptrom_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ptrom_ctx* get() const { return ctx_; }

  // Throws the reference-equivalent exception for a non-zero status.
  template <class ConfigErr = config_error, class NumErr = numerical_error>
  void check(int rc) const {
    if (rc == PTROM_OK) return;
    const std::string msg = ptrom_last_error(ctx_);
    if (rc == PTROM_CONFIG_ERROR) throw ConfigErr(msg);
    if (rc == PTROM_NUMERICAL_ERROR) throw NumErr(msg);
    throw std::runtime_error(msg);
  }

 private:
  ptrom_ctx* ctx_ = nullptr;
};

struct BlockDiagonalJacobianVec {  // kernel.hpp:134-152
  std::vector<double> dfx_dx, dfx_dy, dfy_dx, dfy_dy;
};

// std::vector flavour of the Model concept.
class PairwiseModelVec {
 public:
  PairwiseModelVec(const Context& ctx, std::vector<double> circulation, double delta, int form = PTROM_FORM_STANDARD,
                   std::vector<double> inflow = {})
      : ctx_(ctx), gamma_(std::move(circulation)), delta_(delta), form_(form), inflow_(std::move(inflow)) {}

  std::vector<double> velocity(const std::vector<double>& x) const {  // kernel.hpp:107-129
    const int64_t n = static_cast<int64_t>(gamma_.size());
    if (static_cast<int64_t>(x.size()) != 2 * n)
      throw config_error("pairwise_velocity: state dimension " + std::to_string(x.size()) +
                         " does not match particle count " + std::to_string(n));
    std::vector<double> f(x.size());
    uint64_t pairs = 0;
    ctx_.check(ptrom_pairwise_velocity_f64(ctx_.get(), n, x.data(), gamma_.data(), delta_, form_,
                                           inflow_.empty() ? nullptr : inflow_.data(), f.data(), &pairs));
    pair_evals_ += pairs;
    return f;
  }
  BlockDiagonalJacobianVec jacobian(const std::vector<double>& x) const {  // kernel.hpp:154-170
    const int64_t n = static_cast<int64_t>(gamma_.size());
    BlockDiagonalJacobianVec j{std::vector<double>(n), std::vector<double>(n), std::vector<double>(n),
                               std::vector<double>(n)};
    ctx_.check(ptrom_inexact_kernel_jacobian_f64(ctx_.get(), n, x.data(), gamma_.data(), delta_, form_,
                                                 j.dfx_dx.data(), j.dfx_dy.data(), j.dfy_dx.data(),
                                                 j.dfy_dy.data(), nullptr));
    return j;
  }
  uint64_t pair_evals() const { return pair_evals_; }

 private:
  const Context& ctx_;
  std::vector<double> gamma_;
  double delta_;
  int form_;
  std::vector<double> inflow_;
  mutable uint64_t pair_evals_ = 0;
};

// std::vector flavour of BarnesHutModel (integrators.hpp:83-102): the tree is
// rebuilt from the evaluation state on every call, like the reference's.
class BarnesHutModelVec {
 public:
  BarnesHutModelVec(const Context& ctx, std::vector<double> circulation, double delta, int crit_kind,
                    double crit_value, int64_t leaf_capacity, int form = PTROM_FORM_STANDARD,
                    std::vector<double> inflow = {})
      : ctx_(ctx), gamma_(std::move(circulation)), delta_(delta), form_(form), kind_(crit_kind),
        value_(crit_value), leaf_(leaf_capacity), inflow_(std::move(inflow)) {}

  std::vector<double> velocity(const std::vector<double>& x) const {  // quadtree.hpp:257-281
    const int64_t n = static_cast<int64_t>(gamma_.size());
    if (static_cast<int64_t>(x.size()) != 2 * n) throw config_error("bh_velocity: state dimension mismatch");
    std::vector<double> f(x.size());
    uint64_t pairs = 0;
    ctx_.check(ptrom_barnes_hut_velocity_f64(ctx_.get(), n, x.data(), gamma_.data(), delta_, form_, kind_, value_,
                                             leaf_, inflow_.empty() ? nullptr : inflow_.data(), f.data(), &pairs));
    pair_evals_ += pairs;
    return f;
  }
  BlockDiagonalJacobianVec jacobian(const std::vector<double>& x) const {  // quadtree.hpp:285-308
    const int64_t n = static_cast<int64_t>(gamma_.size());
    if (static_cast<int64_t>(x.size()) != 2 * n) throw config_error("bh_jacobian: state dimension mismatch");
    BlockDiagonalJacobianVec j{std::vector<double>(n), std::vector<double>(n), std::vector<double>(n),
                               std::vector<double>(n)};
    ptrom_tree* tree = nullptr;
    ctx_.check(ptrom_tree_build_f64(ctx_.get(), n, x.data(), x.data() + n, gamma_.data(), leaf_, &tree));
    const int rc = ptrom_bh_jacobian_f64(ctx_.get(), tree, n, x.data(), gamma_.data(), delta_, form_, kind_, value_,
                                         j.dfx_dx.data(), j.dfx_dy.data(), j.dfy_dx.data(), j.dfy_dy.data());
    ptrom_tree_free(tree);
    ctx_.check(rc);
    return j;
  }
  uint64_t pair_evals() const { return pair_evals_; }

 private:
  const Context& ctx_;
  std::vector<double> gamma_;
  double delta_;
  int form_, kind_;
  double value_;
  int64_t leaf_;
  std::vector<double> inflow_;
  mutable uint64_t pair_evals_ = 0;
};

// ------------------------------------------------------ PTROM online path --
// Drop-in for ptrom::ptrom_simulate<double> (rom.hpp:404-412) on the
// reference's own offline types: PODBasis {phi, singular_values, x_ref},
// GnatOperator {sample_ids, A}, SurrogateSourceBasis {phi_tilde, gamma_tilde,
// x0_tilde, cluster_membership, zero_gamma, target_ids, per_target_clusters,
// per_target_direct, direct_ids, direct_phi, direct_x0, direct_gamma},
// ParticleSystem {circulation, delta, kernel_form, inflow}, RomConfig {tol,
// max_iters, step_length}, RomTrajectory {x_hat, iterations, converged}.
// Matrices may be Eigen (data(), rows(), cols(), resize()) or any column-major
// type with the fields {rows, cols, a}; nested index lists become the C ABI's
// CSR arrays here, so the caller writes no marshalling. As in the reference
// the surrogate is reassigned in place: its tables are written back.
namespace detail {
template <class M>
const double* mat_data(const M& m) {
  if constexpr (requires { m.data(); }) return m.data();
  else return m.a.data();
}
template <class M>
double* mat_data(M& m) {
  if constexpr (requires { m.data(); }) return m.data();
  else return m.a.data();
}
template <class M>
int64_t mat_rows(const M& m) {
  if constexpr (requires { m.rows(); }) return static_cast<int64_t>(m.rows());
  else return static_cast<int64_t>(m.rows);
}
template <class M>
int64_t mat_cols(const M& m) {
  if constexpr (requires { m.cols(); }) return static_cast<int64_t>(m.cols());
  else return static_cast<int64_t>(m.cols);
}
template <class M>
void mat_resize(M& m, int64_t r, int64_t c) {
  if constexpr (requires { m.resize(r, c); }) m.resize(r, c);
  else m = M(r, c);
}
template <class L>
void to_csr(const L& nested, std::vector<int64_t>& off, std::vector<int64_t>& flat) {
  off.assign(1, 0);
  flat.clear();
  for (const auto& l : nested) {
    for (const auto v : l) flat.push_back(static_cast<int64_t>(v));
    off.push_back(static_cast<int64_t>(flat.size()));
  }
}
template <class V>
std::vector<int64_t> to_i64(const V& v) {
  return std::vector<int64_t>(v.begin(), v.end());
}
template <class Sys>
const double* inflow_ptr(const Sys& sys) {
  if constexpr (requires { sys.has_inflow; }) return sys.has_inflow ? sys.inflow.data() : nullptr;
  else if constexpr (requires { sys.inflow->data(); }) return sys.inflow ? sys.inflow->data() : nullptr;
  else return sys.inflow.empty() ? nullptr : sys.inflow.data();
}
}  // namespace detail

// Device-resident copies of the offline products (basis, operator,
// surrogate) for repeated online queries; `simulate` is rom.hpp:404-412.
class DevicePtrom {
 public:
  template <class Basis, class Op, class Sur>
  DevicePtrom(const Context& ctx, const Basis& basis, const Op& op, const Sur& sur) : ctx_(ctx) {
    const int64_t nd = detail::mat_rows(basis.phi), m = detail::mat_cols(basis.phi);
    n_ = nd / 2;
    m_ = m;
    ctx_.check(ptrom_basis_create(ctx_.get(), nd, m, detail::mat_data(basis.phi), basis.singular_values.data(),
                                  basis.x_ref.data(), &basis_));
    const std::vector<int64_t> ids = detail::to_i64(op.sample_ids);
    check_or_free(ptrom_gnat_op_create(ctx_.get(), basis_, static_cast<int64_t>(ids.size()), ids.data(),
                                       detail::mat_rows(op.A), detail::mat_data(op.A), &op_));
    std::vector<int64_t> mem_off, mem_ids, cl_off, cl_list, d_off, d_list;
    detail::to_csr(sur.cluster_membership, mem_off, mem_ids);
    detail::to_csr(sur.per_target_clusters, cl_off, cl_list);
    detail::to_csr(sur.per_target_direct, d_off, d_list);
    const std::vector<int64_t> tid = detail::to_i64(sur.target_ids), did = detail::to_i64(sur.direct_ids);
    std::vector<uint8_t> zg(sur.zero_gamma.begin(), sur.zero_gamma.end());
    const int64_t nc = static_cast<int64_t>(sur.gamma_tilde.size());
    check_or_free(ptrom_surrogate_create(
        ctx_.get(), detail::mat_cols(sur.phi_tilde), nc, detail::mat_data(sur.phi_tilde), sur.gamma_tilde.data(),
        sur.x0_tilde.data(), zg.data(), mem_off.data(), mem_ids.data(), static_cast<int64_t>(tid.size()), tid.data(),
        cl_off.data(), cl_list.data(), static_cast<int64_t>(did.size()), did.data(), detail::mat_data(sur.direct_phi),
        sur.direct_x0.data(), sur.direct_gamma.data(), d_off.data(), d_list.data(), &sur_));
  }
  ~DevicePtrom() {
    ptrom_surrogate_free(sur_);
    ptrom_gnat_op_free(op_);
    ptrom_basis_free(basis_);
  }
  DevicePtrom(const DevicePtrom&) = delete;
  DevicePtrom& operator=(const DevicePtrom&) = delete;

  // rom.hpp:404-412: reassign the surrogate to sys.circulation (on the device
  // and in `sur`, the reference's in-place mutation) and march n_steps.
  template <class Sur, class Sys, class Cfg, class Traj>
  void simulate(Sur& sur, const Sys& sys, double dt, int64_t n_steps, const Cfg& cfg, Traj& out,
                uint64_t* pair_evals = nullptr) {
    detail::mat_resize(out.x_hat, m_, n_steps);
    out.iterations.assign(static_cast<size_t>(n_steps), 0);
    std::vector<uint8_t> conv(static_cast<size_t>(n_steps), 0);
    uint64_t pairs = 0;
    ctx_.check(ptrom_ptrom_simulate_f64(ctx_.get(), basis_, op_, sur_, n_, sys.circulation.data(), sys.delta,
                                        static_cast<int>(sys.kernel_form), detail::inflow_ptr(sys), dt, n_steps,
                                        cfg.tol, cfg.max_iters, cfg.step_length, detail::mat_data(out.x_hat),
                                        out.iterations.data(), conv.data(), &pairs));
    out.converged.assign(conv.begin(), conv.end());
    std::vector<uint8_t> zg(sur.zero_gamma.size());
    ctx_.check(ptrom_surrogate_export(ctx_.get(), sur_, detail::mat_data(sur.phi_tilde), sur.gamma_tilde.data(),
                                      sur.x0_tilde.data(), zg.data(), sur.direct_gamma.data()));
    for (size_t c = 0; c < zg.size(); ++c) sur.zero_gamma[c] = static_cast<char>(zg[c]);
    if (pair_evals) *pair_evals = pairs;
  }

  ptrom_basis* basis() const { return basis_; }
  ptrom_gnat_op* op() const { return op_; }
  ptrom_surrogate* surrogate() const { return sur_; }

 private:
  void check_or_free(int rc) {
    if (rc == PTROM_OK) return;
    const std::string msg = ptrom_last_error(ctx_.get());
    ptrom_gnat_op_free(op_);
    ptrom_basis_free(basis_);
    op_ = nullptr;
    basis_ = nullptr;
    if (rc == PTROM_CONFIG_ERROR) throw config_error(msg);
    if (rc == PTROM_NUMERICAL_ERROR) throw numerical_error(msg);
    throw std::runtime_error(msg);
  }
  const Context& ctx_;
  int64_t n_ = 0, m_ = 0;
  ptrom_basis* basis_ = nullptr;
  ptrom_gnat_op* op_ = nullptr;
  ptrom_surrogate* sur_ = nullptr;
};

// One-shot form with the reference's signature shape:
//   ptrom_simulate(basis, op, surrogate&, sys, grid.dt, grid.n_steps, cfg, traj)
template <class Basis, class Op, class Sur, class Sys, class Cfg, class Traj>
void ptrom_simulate(const Context& ctx, const Basis& basis, const Op& op, Sur& sur, const Sys& sys, double dt,
                    int64_t n_steps, const Cfg& cfg, Traj& out) {
  DevicePtrom d(ctx, basis, op, sur);
  d.simulate(sur, sys, dt, n_steps, cfg, out);
}

}  // namespace ptrom_b200

#if __has_include(<Eigen/Dense>) && __has_include("ptrom/kernel.hpp")
#include <Eigen/Dense>

#include "ptrom/kernel.hpp"
#include "ptrom/types.hpp"

namespace ptrom_b200 {

// Drop-in for ptrom::PairwiseModel<double> (integrators.hpp:69-79): same
// members, same exceptions, same counter semantics, computed on the B200.
struct CudaPairwiseModel {
  const Context* ctx;
  ptrom::ParticleSystem<double> sys;

  ptrom::VectorX<double> velocity(const Eigen::Ref<const ptrom::VectorX<double>>& x) const {
    sys.validate();
    ptrom::check_state<double>(x, sys, "pairwise_velocity");
    const Eigen::VectorXd xc = x;  // contiguous host copy (x may be a strided Ref)
    ptrom::VectorX<double> f(x.size());
    uint64_t pairs = 0;
    ctx->check<ptrom::config_error, ptrom::numerical_error>(ptrom_pairwise_velocity_f64(
        ctx->get(), sys.size(), xc.data(), sys.circulation.data(), sys.delta, static_cast<int>(sys.kernel_form),
        sys.inflow ? sys.inflow->data() : nullptr, f.data(), &pairs));
    ptrom::detail::kernel_eval_counter += pairs;
    return f;
  }
  ptrom::BlockDiagonalJacobian<double> jacobian(const Eigen::Ref<const ptrom::VectorX<double>>& x) const {
    sys.validate();
    ptrom::check_state<double>(x, sys, "inexact_kernel_jacobian");
    const Eigen::VectorXd xc = x;
    auto j = ptrom::BlockDiagonalJacobian<double>::Zero(sys.size());
    ctx->check<ptrom::config_error, ptrom::numerical_error>(ptrom_inexact_kernel_jacobian_f64(
        ctx->get(), sys.size(), xc.data(), sys.circulation.data(), sys.delta, static_cast<int>(sys.kernel_form),
        j.dfx_dx.data(), j.dfx_dy.data(), j.dfy_dx.data(), j.dfy_dy.data(), nullptr));
    return j;
  }
};

// Drop-in for ptrom::BarnesHutModel<double> (integrators.hpp:83-102): same
// members (sys, criterion, leaf_capacity); the tree is rebuilt on the B200
// from the evaluation state on every call, as the reference does.
struct CudaBarnesHutModel {
  const Context* ctx;
  ptrom::ParticleSystem<double> sys;
  ptrom::ClusterCriterion<double> criterion;
  ptrom::Index leaf_capacity;

  int kind() const { return criterion.kind == ptrom::ClusterCriterion<double>::Kind::barnes_hut ? 0 : 1; }
  ptrom::VectorX<double> velocity(const Eigen::Ref<const ptrom::VectorX<double>>& x) const {
    sys.validate();
    ptrom::check_state<double>(x, sys, "bh_velocity");
    const Eigen::VectorXd xc = x;
    ptrom::VectorX<double> f(x.size());
    uint64_t pairs = 0;
    ctx->check<ptrom::config_error, ptrom::numerical_error>(ptrom_barnes_hut_velocity_f64(
        ctx->get(), sys.size(), xc.data(), sys.circulation.data(), sys.delta, static_cast<int>(sys.kernel_form),
        kind(), criterion.value, leaf_capacity, sys.inflow ? sys.inflow->data() : nullptr, f.data(), &pairs));
    ptrom::detail::kernel_eval_counter += pairs;
    return f;
  }
  ptrom::BlockDiagonalJacobian<double> jacobian(const Eigen::Ref<const ptrom::VectorX<double>>& x) const {
    sys.validate();
    ptrom::check_state<double>(x, sys, "bh_jacobian");
    const Eigen::VectorXd xc = x;
    const ptrom::Index n = sys.size();
    auto j = ptrom::BlockDiagonalJacobian<double>::Zero(n);
    ptrom_tree* tree = nullptr;
    ctx->check<ptrom::config_error, ptrom::numerical_error>(
        ptrom_tree_build_f64(ctx->get(), n, xc.data(), xc.data() + n, sys.circulation.data(), leaf_capacity, &tree));
    const int rc = ptrom_bh_jacobian_f64(ctx->get(), tree, n, xc.data(), sys.circulation.data(), sys.delta,
                                         static_cast<int>(sys.kernel_form), kind(), criterion.value,
                                         j.dfx_dx.data(), j.dfx_dy.data(), j.dfy_dx.data(), j.dfy_dy.data());
    ptrom_tree_free(tree);
    ctx->check<ptrom::config_error, ptrom::numerical_error>(rc);
    return j;
  }
};

}  // namespace ptrom_b200
#endif
