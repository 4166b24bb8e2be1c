// ptrom_oracle.hpp — CPU ORACLE (test infrastructure only).
//
// A plain-C++ restatement (no Eigen, no third-party code) of the reference
// hot path, used ONLY by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs as the checker and CPU baseline. The
// product (paper_2103_01983_b200/, libptrom_b200.so) never links or calls it.
//
// Every function cites the reference line it follows (paths are relative to
// /root/reference/proj). Summation orders, branch structure and the
// multiply-then-add rounding of the reference are kept: build with
// -ffp-contract=off so that no a*b+c is fused (the reference's Release build
// on x86-64 without -march emits mulsd+addsd).
//
// Where the reference calls Eigen for a reduction (VectorX::norm()) the
// restatement uses a plain ascending sum; Eigen's SIMD reduction order is not
// reproducible without Eigen, and no reference test pins it bitwise
// (SURVEY.md §8c "Third-party boundary").
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Index = std::int64_t;

// types.hpp:23-32
struct config_error : std::runtime_error {
  explicit config_error(const std::string& w) : std::runtime_error(w) {}
};
struct numerical_error : std::runtime_error {
  explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};

// kernel.hpp:16
enum class KernelForm : std::uint8_t { standard = 0, denominator_scaled = 1 };

// kernel.hpp:18-25 — thread-local pair-evaluation counter.
inline thread_local std::uint64_t kernel_eval_counter = 0;

// EIGEN_PI is a long double literal; S(EIGEN_PI) rounds it to S.
inline constexpr long double kPiL = 3.141592653589793238462643383279502884197169399375105820974944592307816406L;

template <class S>
struct V2 {
  S x, y;
};
template <class S>
struct M2 {  // row-major 2x2: a00 a01 / a10 a11
  S a00, a01, a10, a11;
};

// kernel.hpp:29-42
template <class S>
inline V2<S> kernel_pair(V2<S> target, V2<S> source, S gamma, S delta,
                         KernelForm form = KernelForm::standard) {
  ++kernel_eval_counter;
  const S rx = target.x - source.x;
  const S ry = target.y - source.y;
  const S d2 = rx * rx + ry * ry;
  const S two_pi = S(2) * S(kPiL);
  const S den = (form == KernelForm::standard) ? d2 + delta : two_pi * d2 + delta;
  if (den == S(0))
    throw numerical_error("kernel_pair: coincident target/source with zero desingularization");
  const S pre = (form == KernelForm::standard) ? gamma / (two_pi * den) : gamma / den;
  return {-ry * pre, rx * pre};
}

// kernel.hpp:45-73
template <class S>
inline M2<S> kernel_pair_jacobian(V2<S> target, V2<S> source, S gamma, S delta,
                                  KernelForm form = KernelForm::standard) {
  const S rx = target.x - source.x;
  const S ry = target.y - source.y;
  const S d2 = rx * rx + ry * ry;
  const S two_pi = S(2) * S(kPiL);
  M2<S> out;
  if (form == KernelForm::standard) {
    const S q = d2 + delta;
    if (q == S(0))
      throw numerical_error(
          "kernel_pair_jacobian: coincident target/source with zero desingularization");
    const S c = gamma / (two_pi * q * q);
    out.a00 = c * (S(2) * rx * ry);
    out.a01 = c * (ry * ry - rx * rx - delta);
    out.a10 = c * (ry * ry - rx * rx + delta);
    out.a11 = c * (-S(2) * rx * ry);
  } else {
    const S q = two_pi * d2 + delta;
    if (q == S(0))
      throw numerical_error(
          "kernel_pair_jacobian: coincident target/source with zero desingularization");
    const S c = gamma / (q * q);
    out.a00 = c * (S(2) * two_pi * rx * ry);
    out.a01 = c * (S(2) * two_pi * ry * ry - q);
    out.a10 = c * (q - S(2) * two_pi * rx * rx);
    out.a11 = c * (-S(2) * two_pi * rx * ry);
  }
  return out;
}

// kernel.hpp:77-94 — circulation, delta, optional inflow (2N), form.
template <class S>
struct ParticleSystem {
  std::vector<S> circulation;
  S delta = S(0);
  bool has_inflow = false;
  std::vector<S> inflow;
  KernelForm kernel_form = KernelForm::standard;

  Index size() const { return static_cast<Index>(circulation.size()); }

  void validate() const {  // kernel.hpp:84-93
    if (circulation.empty()) throw config_error("particle system is empty");
    for (S g : circulation)
      if (!std::isfinite(g)) throw config_error("non-finite circulation");
    if (!(delta >= S(0))) throw config_error("negative desingularization constant");
    if (has_inflow && static_cast<Index>(inflow.size()) != 2 * size())
      throw config_error("inflow size must be twice the particle count");
    if (has_inflow)
      for (S v : inflow)
        if (!std::isfinite(v)) throw config_error("non-finite inflow");
  }
};

// kernel.hpp:96-103
template <class S>
inline void check_state(const std::vector<S>& state, const ParticleSystem<S>& sys, const char* who) {
  if (static_cast<Index>(state.size()) != 2 * sys.size())
    throw config_error(std::string(who) + ": state dimension " + std::to_string(state.size()) +
                       " does not match particle count " + std::to_string(sys.size()));
  for (S v : state)
    if (!std::isfinite(v)) throw config_error(std::string(who) + ": non-finite state");
}

// kernel.hpp:107-129 — restricted to targets [t_begin, t_end) so that the CPU
// baseline can time a bounded sample; rows outside the range are left zero.
// The per-target loop body is exactly the reference's.
template <class S>
inline void pairwise_velocity_rows(const std::vector<S>& state, const ParticleSystem<S>& sys,
                                   Index t_begin, Index t_end, S* f /* 2N */) {
  const Index n = sys.size();
  for (Index i = t_begin; i < t_end; ++i) {
    const V2<S> xi{state[i], state[i + n]};
    S fx = S(0), fy = S(0);
    for (Index j = 0; j < n; ++j) {
      if (j == i) continue;
      const V2<S> k = kernel_pair<S>(xi, V2<S>{state[j], state[j + n]}, sys.circulation[j],
                                     sys.delta, sys.kernel_form);
      fx += k.x;
      fy += k.y;
    }
    f[i] = fx;
    f[i + n] = fy;
    if (sys.has_inflow) {  // kernel.hpp:127, f += inflow after the loop
      f[i] = f[i] + sys.inflow[i];
      f[i + n] = f[i + n] + sys.inflow[i + n];
    }
  }
}

template <class S>
inline std::vector<S> pairwise_velocity(const std::vector<S>& state, const ParticleSystem<S>& sys) {
  sys.validate();
  check_state<S>(state, sys, "pairwise_velocity");
  std::vector<S> f(state.size(), S(0));
  pairwise_velocity_rows<S>(state, sys, 0, sys.size(), f.data());
  return f;
}

// kernel.hpp:134-152
template <class S>
struct BlockDiagonalJacobian {
  std::vector<S> dfx_dx, dfx_dy, dfy_dx, dfy_dy;
  static BlockDiagonalJacobian Zero(Index n) {
    return {std::vector<S>(n, S(0)), std::vector<S>(n, S(0)), std::vector<S>(n, S(0)),
            std::vector<S>(n, S(0))};
  }
  M2<S> block(Index i) const { return {dfx_dx[i], dfx_dy[i], dfy_dx[i], dfy_dy[i]}; }
  void add_block(Index i, const M2<S>& b) {
    dfx_dx[i] += b.a00;
    dfx_dy[i] += b.a01;
    dfy_dx[i] += b.a10;
    dfy_dy[i] += b.a11;
  }
};

// kernel.hpp:154-170 (target range as for pairwise_velocity_rows)
template <class S>
inline void inexact_kernel_jacobian_rows(const std::vector<S>& state, const ParticleSystem<S>& sys,
                                         Index t_begin, Index t_end, BlockDiagonalJacobian<S>& jac) {
  const Index n = sys.size();
  for (Index i = t_begin; i < t_end; ++i) {
    const V2<S> xi{state[i], state[i + n]};
    for (Index j = 0; j < n; ++j) {
      if (j == i) continue;
      jac.add_block(i, kernel_pair_jacobian<S>(xi, V2<S>{state[j], state[j + n]},
                                               sys.circulation[j], sys.delta, sys.kernel_form));
    }
  }
}

template <class S>
inline BlockDiagonalJacobian<S> inexact_kernel_jacobian(const std::vector<S>& state,
                                                        const ParticleSystem<S>& sys) {
  sys.validate();
  check_state<S>(state, sys, "inexact_kernel_jacobian");
  auto jac = BlockDiagonalJacobian<S>::Zero(sys.size());
  inexact_kernel_jacobian_rows<S>(state, sys, 0, sys.size(), jac);
  return jac;
}

// kernel.hpp:174-192 (diagnostic; §8f "next")
template <class S>
inline S hamiltonian(const std::vector<S>& state, const ParticleSystem<S>& sys) {
  sys.validate();
  check_state<S>(state, sys, "hamiltonian");
  const Index n = sys.size();
  S acc = S(0);
  for (Index i = 0; i < n; ++i) {
    for (Index j = i + 1; j < n; ++j) {
      const S rx = state[i] - state[j];
      const S ry = state[i + n] - state[j + n];
      const S d2 = rx * rx + ry * ry;
      if (d2 == S(0))
        throw numerical_error("hamiltonian: coincident particles " + std::to_string(i) + " and " +
                              std::to_string(j));
      acc += sys.circulation[i] * sys.circulation[j] * std::log(std::sqrt(d2));
    }
  }
  return acc / (S(2) * S(kPiL));
}

// kernel.hpp:195-208 — rectangular evaluation lattice.
template <class S>
struct LatticeSpec {
  S x_min, x_max;
  Index nx;
  S y_min, y_max;
  Index ny;
  void validate() const {
    if (nx < 2 || ny < 2) throw config_error("lattice needs at least 2 points per axis");
    if (!(x_max > x_min) || !(y_max > y_min)) throw config_error("degenerate lattice extents");
  }
  S x_at(Index i) const { return x_min + (x_max - x_min) * S(i) / S(nx - 1); }
  S y_at(Index j) const { return y_min + (y_max - y_min) * S(j) / S(ny - 1); }
};

// kernel.hpp:213-238 — |f| * c_g * l / gamma_bar at every lattice vertex;
// grid is ny x nx column-major (entry (j, i) at j + i * ny).
template <class S>
inline std::vector<S> velocity_field_grid(const std::vector<S>& state, const ParticleSystem<S>& sys,
                                          const LatticeSpec<S>& lattice, S c_g, S l, S gamma_bar) {
  sys.validate();
  check_state<S>(state, sys, "velocity_field_grid");
  lattice.validate();
  if (!(gamma_bar > S(0))) throw config_error("velocity_field_grid: gamma_bar must be positive");
  if (!(c_g > S(0)) || !(l > S(0)))
    throw config_error("velocity_field_grid: characteristic length must be positive");
  const Index n = sys.size();
  const S scale = c_g * l / gamma_bar;
  std::vector<S> grid(static_cast<size_t>(lattice.ny * lattice.nx));
  for (Index j = 0; j < lattice.ny; ++j) {
    for (Index i = 0; i < lattice.nx; ++i) {
      const V2<S> vertex{lattice.x_at(i), lattice.y_at(j)};
      S fx = S(0), fy = S(0);
      for (Index p = 0; p < n; ++p) {
        const V2<S> k = kernel_pair<S>(vertex, V2<S>{state[p], state[p + n]}, sys.circulation[p], sys.delta,
                                       sys.kernel_form);
        fx += k.x;
        fy += k.y;
      }
      grid[j + i * lattice.ny] = std::sqrt(fx * fx + fy * fy) * scale;
    }
  }
  return grid;
}

// Plain ascending Euclidean norm, standing in for Eigen's VectorX::norm()
// (integrators.hpp:141, rom.hpp:313).
template <class S>
inline S norm2(const S* v, Index len) {
  S acc = S(0);
  for (Index k = 0; k < len; ++k) acc += v[k] * v[k];
  return std::sqrt(acc);
}

// integrators.hpp:47-53 — r = xi - x_prev - dt/2 (f_xi + f_prev), evaluated
// as the Eigen expression tree ((xi - x_prev) - (dt/2)*(f_xi + f_prev)).
template <class S>
inline void trapezoidal_residual(const S* xi, const S* f_xi, const S* x_prev, const S* f_prev, S dt,
                                 Index len, S* r) {
  const S h = dt / S(2);
  for (Index k = 0; k < len; ++k) r[k] = (xi[k] - x_prev[k]) - h * (f_xi[k] + f_prev[k]);
}

// integrators.hpp:55-66
struct NewtonConfig {
  double tol = 1e-10;
  int max_iters = 100;
  int jacobian_refresh_period = 1;
  void validate() const {
    if (!(tol > 0)) throw config_error("Newton tolerance must be positive");
    if (max_iters < 1) throw config_error("Newton max_iters must be >= 1");
    if (jacobian_refresh_period < 1) throw config_error("Jacobian refresh period must be >= 1");
  }
};

// integrators.hpp:69-79
template <class S>
struct PairwiseModel {
  ParticleSystem<S> sys;
  std::vector<S> velocity(const std::vector<S>& x) const { return pairwise_velocity<S>(x, sys); }
  BlockDiagonalJacobian<S> jacobian(const std::vector<S>& x) const {
    return inexact_kernel_jacobian<S>(x, sys);
  }
};

// integrators.hpp:104-111
template <class S>
struct StepResult {
  std::vector<S> x, f;
  int iterations = 0;
  bool converged = true;
  S relative_residual = S(0);
};

// integrators.hpp:117-201 — inexact Newton on the trapezoidal residual with
// per-particle 2x2 self-block inverses refreshed every p-th step.
template <class S, class Model>
class FomStepper {
 public:
  FomStepper(const Model& model, S dt, NewtonConfig cfg) : model_(model), dt_(dt), cfg_(cfg) {
    cfg_.validate();
    if (!(dt > S(0))) throw config_error("time step must be positive");
  }

  StepResult<S> step(const std::vector<S>& x_prev, const std::vector<S>& f_prev) {
    if (x_prev.size() % 2 != 0) throw config_error("state dimension must be even");
    const Index n = static_cast<Index>(x_prev.size() / 2);
    StepResult<S> out;
    std::vector<S> xi = x_prev;
    std::vector<S> f_xi = f_prev;
    std::vector<S> r(x_prev.size());
    S r0 = S(0);
    bool refreshed_this_step = false;
    const bool refresh_due =
        (step_index_ % cfg_.jacobian_refresh_period) == 0 || inv_blocks_.empty();
    int updates = 0;
    bool converged = false;
    S rel = S(0);
    while (true) {
      trapezoidal_residual<S>(xi.data(), f_xi.data(), x_prev.data(), f_prev.data(), dt_, 2 * n,
                              r.data());
      const S nr = norm2<S>(r.data(), 2 * n);
      if (updates == 0) {
        r0 = nr;
        if (r0 == S(0)) {
          converged = true;
          rel = S(0);
          break;
        }
      }
      rel = nr / r0;
      if (rel <= S(cfg_.tol)) {
        converged = true;
        break;
      }
      if (updates >= cfg_.max_iters) break;
      if (refresh_due && !refreshed_this_step) {
        refactor(xi, n);
        refreshed_this_step = true;
      }
      for (Index i = 0; i < n; ++i) {  // integrators.hpp:161-167
        const M2<S>& inv = inv_blocks_[static_cast<size_t>(i)];
        const S rhs0 = -r[i], rhs1 = -r[i + n];
        const S d0 = inv.a00 * rhs0 + inv.a01 * rhs1;
        const S d1 = inv.a10 * rhs0 + inv.a11 * rhs1;
        xi[i] += d0;
        xi[i + n] += d1;
      }
      ++updates;
      f_xi = model_.velocity(xi);
    }
    ++step_index_;
    out.x = std::move(xi);
    out.f = std::move(f_xi);
    out.iterations = updates;
    out.converged = converged;
    out.relative_residual = rel;
    return out;
  }

 private:
  // integrators.hpp:181-194
  void refactor(const std::vector<S>& xi, Index n) {
    const BlockDiagonalJacobian<S> jv = model_.jacobian(xi);
    inv_blocks_.resize(static_cast<size_t>(n));
    const S h = dt_ / S(2);
    for (Index i = 0; i < n; ++i) {
      const M2<S> j = jv.block(i);
      const M2<S> b{S(1) - h * j.a00, S(0) - h * j.a01, S(0) - h * j.a10, S(1) - h * j.a11};
      const S det = b.a00 * b.a11 - b.a01 * b.a10;
      if (det == S(0) || !std::isfinite(det))
        throw numerical_error("singular Newton block for particle " + std::to_string(i));
      inv_blocks_[static_cast<size_t>(i)] = {b.a11 / det, -b.a01 / det, -b.a10 / det, b.a00 / det};
    }
  }

  const Model& model_;
  S dt_;
  NewtonConfig cfg_;
  std::vector<M2<S>> inv_blocks_;
  Index step_index_ = 0;
};

// integrators.hpp:226-241
template <class S>
struct SimulateResult {
  std::vector<S> snapshots;  // column-major 2N x n_steps
  std::vector<int> iterations;
  std::vector<char> converged;
  std::vector<S> relative_residual;
};

// integrators.hpp:243-272 (timing instrumentation omitted)
template <class S, class Model>
inline SimulateResult<S> fom_simulate(const std::vector<S>& x0, const Model& model, S dt,
                                      Index n_steps, const NewtonConfig& cfg) {
  if (!(dt > S(0))) throw config_error("time step must be positive");
  if (n_steps < 0) throw config_error("negative step count");
  cfg.validate();
  SimulateResult<S> out;
  out.snapshots.resize(x0.size() * static_cast<size_t>(n_steps));
  FomStepper<S, Model> stepper(model, dt, cfg);
  std::vector<S> x = x0;
  std::vector<S> f = model.velocity(x0);
  for (Index s = 0; s < n_steps; ++s) {
    StepResult<S> res = stepper.step(x, f);
    x = std::move(res.x);
    f = std::move(res.f);
    std::copy(x.begin(), x.end(), out.snapshots.begin() + static_cast<size_t>(s) * x.size());
    out.iterations.push_back(res.iterations);
    out.converged.push_back(res.converged ? 1 : 0);
    out.relative_residual.push_back(res.relative_residual);
  }
  return out;
}

}  // namespace oracle
