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
