// kat.cpp — pins the CPU ORACLE against the reference's own known-answer
// tests (test infrastructure only). Each case re-runs one reference test on
// the restatement, with the reference's seeds, generators (libstdc++
// std::mt19937_64 + <random> distributions, identical to the reference
// build's) and tolerances; the cited line is the reference test it ports.
// Exit code 0 iff every check passes. Prints one line per case.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "ptrom_oracle.hpp"
#include "ptrom_oracle_rom.hpp"
#include "ptrom_oracle_tree.hpp"

using namespace oracle;
using Vec = std::vector<double>;

static int g_fail = 0, g_checks = 0;
static std::string g_case;
#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) {                                                                  \
      ++g_fail;                                                                     \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool thrown = false;              \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      thrown = true;                  \
    } catch (...) {                   \
    }                                 \
    CHECK(thrown);                    \
  } while (0)

static bool approx(double a, double b, double eps) {
  // doctest::Approx(b).epsilon(eps): |a-b| < eps * (scale + max(|a|,|b|)), scale 1
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}
static double l2(const Vec& v) {
  double s = 0;
  for (double e : v) s += e * e;
  return std::sqrt(s);
}
static Vec vsub(const Vec& a, const Vec& b) {
  Vec r(a.size());
  for (size_t i = 0; i < a.size(); ++i) r[i] = a[i] - b[i];
  return r;
}
static double maxabs(const Vec& v) {
  double m = 0;
  for (double e : v) m = std::max(m, std::abs(e));
  return m;
}

static std::vector<std::pair<std::string, std::function<void()>>>& registry() {
  static std::vector<std::pair<std::string, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE_I(name, id) \
  static void CAT(tc_, id)(); \
  static Reg CAT(reg_, id)(name, CAT(tc_, id)); \
  static void CAT(tc_, id)()
#define TEST_CASE(name) TEST_CASE_I(name, __COUNTER__)

// ------------------------------------------------------------ kernel ------
// test_kernel.cpp:15-31
static Vec brute_velocity(const Vec& state, const Vec& gamma, double delta, const Vec* inflow) {
  const Index n = static_cast<Index>(gamma.size());
  Vec f(2 * n, 0.0);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      if (i == j) continue;
      const double rx = state[i] - state[j];
      const double ry = state[i + n] - state[j + n];
      const double den = rx * rx + ry * ry + delta;
      f[i] += gamma[j] / (2.0 * M_PI) * (-ry) / den;
      f[i + n] += gamma[j] / (2.0 * M_PI) * rx / den;
    }
  if (inflow)
    for (size_t k = 0; k < f.size(); ++k) f[k] += (*inflow)[k];
  return f;
}
// test_kernel.cpp:35-52 (k * g with the explicit 2N x 2N blocks)
static Vec block_matrix_velocity(const Vec& state, const Vec& gamma, double delta) {
  const Index n = static_cast<Index>(gamma.size());
  Vec f(2 * n, 0.0);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      if (i == j) continue;
      const double rx = state[i] - state[j];
      const double ry = state[i + n] - state[j + n];
      const double den = rx * rx + ry * ry + delta;
      f[i] += (-ry / den) * (gamma[j] / (2.0 * M_PI));
      f[i + n] += (rx / den) * (gamma[j] / (2.0 * M_PI));
    }
  return f;
}
// test_kernel.cpp:54-69
static ParticleSystem<double> random_system(std::mt19937_64& rng, Index n, double delta) {
  std::uniform_real_distribution<double> pos(-5.0, 5.0);
  std::uniform_real_distribution<double> circ(-2.0, 2.0);
  ParticleSystem<double> sys;
  sys.circulation.resize(n);
  for (Index i = 0; i < n; ++i) sys.circulation[i] = circ(rng);
  sys.delta = delta;
  return sys;
}
static Vec random_state(std::mt19937_64& rng, Index n) {
  std::uniform_real_distribution<double> pos(-5.0, 5.0);
  Vec x(2 * n);
  for (Index i = 0; i < 2 * n; ++i) x[i] = pos(rng);
  return x;
}

TEST_CASE("test_kernel.cpp:73 kernel_pair unit-distance values") {
  const double gamma = 2.0 * M_PI;
  auto k0 = kernel_pair<double>({0, 0}, {1, 0}, gamma, 0.0);
  CHECK(approx(k0.x, 0.0, 1e-15));
  CHECK(approx(k0.y, -1.0, 1e-15));
  auto k1 = kernel_pair<double>({0, 0}, {1, 0}, gamma, 1.0);
  CHECK(approx(k1.x, 0.0, 1e-15));
  CHECK(approx(k1.y, -0.5, 1e-15));
}

TEST_CASE("test_kernel.cpp:87 kernel_pair antisymmetry and orthogonality") {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-3.0, 3.0);
  for (int trial = 0; trial < 200; ++trial) {
    const double ax = u(rng), ay = u(rng), bx = u(rng), by = u(rng);
    if (std::hypot(ax - bx, ay - by) < 1e-8) continue;
    const double g = u(rng);
    auto kab = kernel_pair<double>({ax, ay}, {bx, by}, g, 0.0);
    auto kba = kernel_pair<double>({bx, by}, {ax, ay}, g, 0.0);
    const double nab = std::hypot(kab.x, kab.y);
    CHECK(std::hypot(kab.x + kba.x, kab.y + kba.y) <= 1e-14 * std::max(1.0, nab));
    CHECK(std::abs((ax - bx) * kab.x + (ay - by) * kab.y) <= 1e-13 * std::max(1.0, nab));
  }
}

TEST_CASE("test_kernel.cpp:103 kernel_pair denominator-scaled variant") {
  auto a = kernel_pair<double>({0, 0}, {1, 0}, 1.7, 0.0, KernelForm::standard);
  auto b = kernel_pair<double>({0, 0}, {1, 0}, 1.7, 0.0, KernelForm::denominator_scaled);
  CHECK(std::hypot(a.x - b.x, a.y - b.y) <= 1e-16);
  auto c = kernel_pair<double>({0, 0}, {1, 0}, 1.0, 3.0, KernelForm::denominator_scaled);
  CHECK(approx(c.y, -1.0 / (2.0 * M_PI + 3.0), 1e-15));
}

TEST_CASE("test_kernel.cpp:115 kernel_pair coincident points") {
  CHECK_THROWS_AS(kernel_pair<double>({1, 2}, {1, 2}, 1.0, 0.0), numerical_error);
  auto k = kernel_pair<double>({1, 2}, {1, 2}, 1.0, 0.5);
  CHECK(std::hypot(k.x, k.y) == 0.0);
}

TEST_CASE("test_kernel.cpp:123 pairwise_velocity two particles") {
  ParticleSystem<double> sys;
  sys.circulation = {1.5, -0.75};
  sys.delta = 0.1;
  Vec x = {0.0, 1.0, 0.0, 0.5};
  Vec f = pairwise_velocity<double>(x, sys);
  auto f1 = kernel_pair<double>({0, 0}, {1, 0.5}, sys.circulation[1], sys.delta);
  auto f2 = kernel_pair<double>({1, 0.5}, {0, 0}, sys.circulation[0], sys.delta);
  CHECK(approx(f[0], f1.x, 1e-15));
  CHECK(approx(f[2], f1.y, 1e-15));
  CHECK(approx(f[1], f2.x, 1e-15));
  CHECK(approx(f[3], f2.y, 1e-15));
}

TEST_CASE("test_kernel.cpp:141 pairwise_velocity zero circulation returns inflow") {
  ParticleSystem<double> sys;
  sys.circulation = Vec(3, 0.0);
  sys.delta = 0.0;
  sys.has_inflow = true;
  sys.inflow = {1, 2, 3, 4, 5, 6};
  Vec x = {0, 1, 2, 0, 1, 2};
  CHECK(l2(vsub(pairwise_velocity<double>(x, sys), sys.inflow)) == 0.0);
}

TEST_CASE("test_kernel.cpp:153 pairwise_velocity matches independent re-summation") {
  std::mt19937_64 rng(11);
  for (int trial = 0; trial < 25; ++trial) {
    const Index n = 3 + static_cast<Index>(rng() % 8);
    auto sys = random_system(rng, n, trial % 2 ? 0.3 : 0.0);
    const Vec x = random_state(rng, n);
    if (trial % 3 == 0) {
      sys.inflow = random_state(rng, n);
      sys.has_inflow = true;
    }
    const Vec f = pairwise_velocity<double>(x, sys);
    const Vec ref = brute_velocity(x, sys.circulation, sys.delta, sys.has_inflow ? &sys.inflow : nullptr);
    CHECK(l2(vsub(f, ref)) <= 1e-14 * std::max(1.0, l2(ref)));
  }
}

TEST_CASE("test_kernel.cpp:170 pairwise_velocity equals explicit block-matrix product") {
  std::mt19937_64 rng(13);
  for (int trial = 0; trial < 10; ++trial) {
    const Index n = 2 + static_cast<Index>(rng() % 10);
    const auto sys = random_system(rng, n, 0.25);
    const Vec x = random_state(rng, n);
    const Vec f = pairwise_velocity<double>(x, sys);
    const Vec ref = block_matrix_velocity(x, sys.circulation, sys.delta);
    CHECK(l2(vsub(f, ref)) <= 1e-13 * std::max(1.0, l2(ref)));
  }
}

TEST_CASE("test_kernel.cpp:182 pairwise_velocity input validation") {
  ParticleSystem<double> sys;
  sys.circulation = {1.0, 1.0};
  CHECK_THROWS_AS(pairwise_velocity<double>(Vec{1, 2, 3}, sys), config_error);
  CHECK_THROWS_AS(pairwise_velocity<double>(Vec{0, 1, 0, std::nan("")}, sys), config_error);
  sys.delta = 0.0;
  CHECK_THROWS_AS(pairwise_velocity<double>(Vec{1, 1, 2, 2}, sys), numerical_error);
}

TEST_CASE("test_kernel.cpp:197 inexact_kernel_jacobian two-particle block") {
  ParticleSystem<double> sys;
  sys.circulation = {0.0, 2.0 * M_PI};
  sys.delta = 0.0;
  const auto jac = inexact_kernel_jacobian<double>(Vec{0.0, 1.0, 0.0, 0.0}, sys);
  const auto b = jac.block(0);
  CHECK(approx(b.a00, 0.0, 1e-14));
  CHECK(approx(b.a01, -1.0, 1e-14));
  CHECK(approx(b.a10, -1.0, 1e-14));
  CHECK(approx(b.a11, 0.0, 1e-14));
}

TEST_CASE("test_kernel.cpp:212 inexact_kernel_jacobian matches central finite differences") {
  std::mt19937_64 rng(17);
  for (int trial = 0; trial < 10; ++trial) {
    const Index n = 5;
    const auto sys = random_system(rng, n, trial % 2 ? 0.2 : 0.0);
    const Vec x = random_state(rng, n);
    const auto jac = inexact_kernel_jacobian<double>(x, sys);
    const double h = 1e-6;
    for (Index i = 0; i < n; ++i) {
      double fd[2][2];
      for (int axis = 0; axis < 2; ++axis) {
        Vec xp = x, xm = x;
        const Index row = axis == 0 ? i : i + n;
        xp[row] += h;
        xm[row] -= h;
        const Vec fp = pairwise_velocity<double>(xp, sys);
        const Vec fm = pairwise_velocity<double>(xm, sys);
        fd[0][axis] = (fp[i] - fm[i]) / (2 * h);
        fd[1][axis] = (fp[i + n] - fm[i + n]) / (2 * h);
      }
      const auto b = jac.block(i);
      const double dn = std::sqrt(fd[0][0] * fd[0][0] + fd[0][1] * fd[0][1] + fd[1][0] * fd[1][0] + fd[1][1] * fd[1][1]);
      const double e = std::sqrt(std::pow(b.a00 - fd[0][0], 2) + std::pow(b.a01 - fd[0][1], 2) +
                                 std::pow(b.a10 - fd[1][0], 2) + std::pow(b.a11 - fd[1][1], 2));
      CHECK(e <= 1e-6 * std::max(1.0, dn));
    }
  }
}

TEST_CASE("test_kernel.cpp:238 inexact_kernel_jacobian zero circulation") {
  ParticleSystem<double> sys;
  sys.circulation = Vec(4, 0.0);
  sys.delta = 0.1;
  std::mt19937_64 rng(3);
  const Vec x = random_state(rng, 4);
  const auto jac = inexact_kernel_jacobian<double>(x, sys);
  for (Index i = 0; i < 4; ++i) {
    const auto b = jac.block(i);
    CHECK(b.a00 == 0.0 && b.a01 == 0.0 && b.a10 == 0.0 && b.a11 == 0.0);
  }
}

TEST_CASE("test_kernel.cpp:248 hamiltonian two-particle value") {
  ParticleSystem<double> sys;
  sys.circulation = {1.0, 1.0};
  const double e = std::exp(1.0);
  CHECK(approx(hamiltonian<double>(Vec{0.0, e, 0.0, 0.0}, sys), 1.0 / (2.0 * M_PI), 1e-14));
}

TEST_CASE("test_kernel.cpp:257 hamiltonian brute-force and translation invariance") {
  std::mt19937_64 rng(23);
  const Index n = 6;
  const auto sys = random_system(rng, n, 0.0);
  const Vec x = random_state(rng, n);
  double ref = 0.0;
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) {
      if (i == j) continue;
      ref += sys.circulation[j] * sys.circulation[i] * std::log(std::hypot(x[i] - x[j], x[i + n] - x[j + n]));
    }
  ref /= 4.0 * M_PI;
  const double h = hamiltonian<double>(x, sys);
  CHECK(approx(h, ref, 1e-13));
  Vec shifted = x;
  for (Index i = 0; i < n; ++i) {
    shifted[i] += 3.25;
    shifted[i + n] -= 1.5;
  }
  CHECK(approx(hamiltonian<double>(shifted, sys), h, 1e-12));
  Vec coincident = x;
  coincident[1] = coincident[0];
  coincident[1 + n] = coincident[n];
  CHECK_THROWS_AS((void)hamiltonian<double>(coincident, sys), numerical_error);
}

TEST_CASE("test_kernel.cpp:287 velocity_field_grid single vortex") {
  ParticleSystem<double> sys;
  sys.circulation = {2.0 * M_PI};
  sys.delta = 0.0;
  const Vec x{0.0, 0.0};
  const LatticeSpec<double> lattice{-1.0, 1.0, 2, 0.0, 1.0, 2};
  const double c_g = 1.25, l = 2.0, gamma_bar = 4.0;
  const Vec grid = velocity_field_grid<double>(x, sys, lattice, c_g, l, gamma_bar);
  CHECK(grid.size() == 4);
  CHECK(approx(grid[0 + 0 * 2], c_g * l / gamma_bar, 1e-13));
  CHECK(approx(grid[0 + 1 * 2], c_g * l / gamma_bar, 1e-13));
  CHECK(approx(grid[1 + 0 * 2], c_g * l / gamma_bar / std::sqrt(2.0), 1e-13));
  CHECK_THROWS_AS((void)velocity_field_grid<double>(x, sys, lattice, c_g, l, 0.0), config_error);
  const LatticeSpec<double> touching{-1.0, 1.0, 3, -1.0, 1.0, 3};
  CHECK_THROWS_AS((void)velocity_field_grid<double>(x, sys, touching, c_g, l, gamma_bar), numerical_error);
}

TEST_CASE("test_kernel.cpp:312 kernel evaluation counter") {
  kernel_eval_counter = 0;
  ParticleSystem<double> sys;
  sys.circulation = Vec(4, 1.0);
  sys.delta = 0.1;
  std::mt19937_64 rng(5);
  const Vec x = random_state(rng, 4);
  (void)pairwise_velocity<double>(x, sys);
  CHECK(kernel_eval_counter == 12);
}

// acceptance.cpp:123-141 — 100 random systems against the block-matrix route.
TEST_CASE("acceptance.cpp:123 criterion 1 pairwise vs block matrix (1e-13)") {
  std::mt19937_64 rng(1001);
  std::uniform_int_distribution<int> usize(2, 50);
  double worst = 0;
  for (int trial = 0; trial < 100; ++trial) {
    const Index n = usize(rng);
    std::uniform_real_distribution<double> upos(-5.0, 5.0);
    std::uniform_real_distribution<double> ug(0.5, 1.5);
    Vec x0(2 * n);
    ParticleSystem<double> sys;
    sys.circulation.resize(n);
    for (Index i = 0; i < n; ++i) {
      x0[i] = upos(rng);
      x0[i + n] = upos(rng);
      sys.circulation[i] = ug(rng);
    }
    sys.delta = 0.05;
    const Vec lib = pairwise_velocity<double>(x0, sys);
    const Vec blk = block_matrix_velocity(x0, sys.circulation, sys.delta);
    worst = std::max(worst, l2(vsub(lib, blk)) / l2(blk));
  }
  CHECK(worst <= 1e-13);
}

// -------------------------------------------------------- integrators ------
// test_integrators.cpp:16-31 — linear dynamics f = A x for one pseudo-particle.
struct LinearModel {
  double a00, a01, a10, a11;
  Vec velocity(const Vec& x) const { return {a00 * x[0] + a01 * x[1], a10 * x[0] + a11 * x[1]}; }
  BlockDiagonalJacobian<double> jacobian(const Vec&) const {
    auto j = BlockDiagonalJacobian<double>::Zero(1);
    j.add_block(0, {a00, a01, a10, a11});
    return j;
  }
};
// test_integrators.cpp:33-37 — x+ = (I - dt/2 A)^{-1} (I + dt/2 A) x
static void trapezoidal_exact(const LinearModel& m, const double* x, double dt, double* out) {
  const double h = dt / 2;
  const double l00 = 1 - h * m.a00, l01 = -h * m.a01, l10 = -h * m.a10, l11 = 1 - h * m.a11;
  const double r0 = (1 + h * m.a00) * x[0] + h * m.a01 * x[1];
  const double r1 = h * m.a10 * x[0] + (1 + h * m.a11) * x[1];
  const double det = l00 * l11 - l01 * l10;
  out[0] = (l11 * r0 - l01 * r1) / det;
  out[1] = (-l10 * r0 + l00 * r1) / det;
}
// test_integrators.cpp:41-60
struct CoRotation {
  double gamma, d, cx, cy;
  double omega() const { return gamma / (M_PI * d * d); }
  Vec state_at(double t) const {
    const double phi = omega() * t;
    const double ax = std::cos(phi) * d / 2, ay = std::sin(phi) * d / 2;
    return {cx + ax, cx - ax, cy + ay, cy - ay};
  }
  ParticleSystem<double> system() const {
    ParticleSystem<double> s;
    s.circulation = {gamma, gamma};
    s.delta = 0.0;
    return s;
  }
};
template <class Model>
static StepResult<double> fom_step(const Vec& x, const Model& model, double dt, NewtonConfig cfg) {
  FomStepper<double, Model> st(model, dt, cfg);
  return st.step(x, model.velocity(x));
}

TEST_CASE("test_integrators.cpp:74 trapezoidal residual algebra") {
  std::mt19937_64 rng(3);
  std::normal_distribution<double> dist;
  Vec xi(6), fxi(6), xp(6), fp(6), r(6);
  for (int i = 0; i < 6; ++i) {
    xi[i] = dist(rng);
    fxi[i] = dist(rng);
    xp[i] = dist(rng);
    fp[i] = dist(rng);
  }
  const double dt = 0.37;
  trapezoidal_residual<double>(xi.data(), fxi.data(), xp.data(), fp.data(), dt, 6, r.data());
  for (int i = 0; i < 6; ++i) CHECK(approx(r[i], xi[i] - xp[i] - dt / 2 * (fxi[i] + fp[i]), 1e-15));
}

TEST_CASE("test_integrators.cpp:91 implicit step matches the linear closed form") {
  LinearModel m{0.3, -1.1, 0.9, -0.2};
  NewtonConfig cfg;
  cfg.tol = 1e-13;
  Vec x = {1.0, -2.0};
  auto res = fom_step(x, m, 0.05, cfg);
  double e[2];
  trapezoidal_exact(m, x.data(), 0.05, e);
  CHECK(res.converged);
  CHECK(res.iterations == 1);
  CHECK(std::abs(res.x[0] - e[0]) <= 1e-13);
  CHECK(std::abs(res.x[1] - e[1]) <= 1e-13);
}

TEST_CASE("test_integrators.cpp:110 multi-step march matches iterated closed form") {
  LinearModel m{0.0, -1.0, 1.0, 0.0};
  NewtonConfig cfg;
  cfg.tol = 1e-13;
  const auto run = fom_simulate<double>(Vec{1.0, 0.0}, m, 0.02, 25, cfg);
  double e[2] = {1.0, 0.0};
  bool all = true;
  for (char c : run.converged) all = all && c;
  CHECK(all);
  for (int s = 0; s < 25; ++s) {
    double nx[2];
    trapezoidal_exact(m, e, 0.02, nx);
    e[0] = nx[0];
    e[1] = nx[1];
    CHECK(std::abs(run.snapshots[2 * s] - e[0]) <= 1e-12);
    CHECK(std::abs(run.snapshots[2 * s + 1] - e[1]) <= 1e-12);
  }
  CHECK(approx(std::hypot(run.snapshots[48], run.snapshots[49]), 1.0, 1e-12));
}

TEST_CASE("test_integrators.cpp:147 vortex pair co-rotates at the analytic rate") {
  const CoRotation pair{2.0 * M_PI, 2.0, 0.3, -0.8};
  PairwiseModel<double> model{pair.system()};
  NewtonConfig cfg;
  cfg.tol = 1e-12;
  const auto run = fom_simulate<double>(pair.state_at(0.0), model, 1e-3, 100, cfg);
  for (char c : run.converged) CHECK(c);
  const Vec last(run.snapshots.begin() + 99 * 4, run.snapshots.begin() + 100 * 4);
  const Vec expect = pair.state_at(1e-3 * 100.0);
  CHECK(maxabs(vsub(last, expect)) < 5e-6);
  const double r = std::hypot(last[0] - last[1], last[2] - last[3]);
  CHECK(std::abs(r - pair.d) / pair.d < 1e-7);
}

TEST_CASE("test_integrators.cpp:188 zero circulation leaves the state fixed") {
  ParticleSystem<double> sys;
  sys.circulation = Vec(3, 0.0);
  PairwiseModel<double> model{sys};
  Vec x = {0, 1, 2, 3, 4, 5};
  auto res = fom_step(x, model, 0.1, NewtonConfig{});
  CHECK(res.converged);
  CHECK(res.iterations == 0);
  CHECK(maxabs(vsub(res.x, x)) == 0.0);
  CHECK(maxabs(res.f) == 0.0);
}

TEST_CASE("test_integrators.cpp:202 stale Jacobian blocks still reach the same solution") {
  const CoRotation pair{4.0, 1.5, 0.0, 0.0};
  PairwiseModel<double> model{pair.system()};
  NewtonConfig fresh;
  fresh.tol = 1e-12;
  NewtonConfig stale = fresh;
  stale.jacobian_refresh_period = 5;
  const auto a = fom_simulate<double>(pair.state_at(0.0), model, 5e-3, 30, fresh);
  const auto b = fom_simulate<double>(pair.state_at(0.0), model, 5e-3, 30, stale);
  for (char c : a.converged) CHECK(c);
  for (char c : b.converged) CHECK(c);
  CHECK(maxabs(vsub(a.snapshots, b.snapshots)) < 1e-9);
}

TEST_CASE("test_integrators.cpp:218 iteration cap reports non-convergence honestly") {
  const CoRotation pair{2.0 * M_PI, 2.0, 0.0, 0.0};
  PairwiseModel<double> model{pair.system()};
  NewtonConfig cfg;
  cfg.tol = 1e-30;
  cfg.max_iters = 2;
  auto res = fom_step(pair.state_at(0.0), model, 1e-3, cfg);
  CHECK(!res.converged);
  CHECK(res.iterations == 2);
  CHECK(res.relative_residual > 0.0);
}

TEST_CASE("test_integrators.cpp:230 singular Newton block names the particle") {
  const double dt = 0.5;
  LinearModel m{2.0 / dt, 0.0, 0.0, 2.0 / dt};
  bool ok = false;
  try {
    (void)fom_step(Vec{1.0, 1.0}, m, dt, NewtonConfig{});
  } catch (const numerical_error& e) {
    ok = std::string(e.what()).find("particle 0") != std::string::npos;
  }
  CHECK(ok);
}

TEST_CASE("test_integrators.cpp:244 energy drift stays small on a small cloud") {
  std::mt19937_64 rng(17);
  std::uniform_real_distribution<double> pos(-1.0, 1.0);
  const Index n = 5;
  ParticleSystem<double> sys;
  sys.circulation = Vec(n, 1.5);
  Vec x0(2 * n);
  for (Index i = 0; i < 2 * n; ++i) x0[i] = pos(rng);
  PairwiseModel<double> model{sys};
  NewtonConfig cfg;
  cfg.tol = 1e-12;
  const double h0 = hamiltonian<double>(x0, sys);
  auto drift = [&](double dt, Index steps) {
    const auto run = fom_simulate<double>(x0, model, dt, steps, cfg);
    const Vec last(run.snapshots.end() - 2 * n, run.snapshots.end());
    return std::abs(hamiltonian<double>(last, sys) - h0) / std::abs(h0);
  };
  const double coarse = drift(1e-3, 50), fine = drift(5e-4, 100);
  CHECK(coarse < 1e-3);
  CHECK(fine < coarse / 2.5);
}

// ------------------------------------------------------------ quadtree ----
static void random_points(std::mt19937_64& rng, Index n, Vec& px, Vec& py, double scale = 10.0) {
  std::uniform_real_distribution<double> dist(-scale, scale);
  px.resize(n);
  py.resize(n);
  for (Index i = 0; i < n; ++i) {
    px[i] = dist(rng);
    py[i] = dist(rng);
  }
}
static Vec random_gamma(std::mt19937_64& rng, Index n) {
  std::uniform_real_distribution<double> dist(0.1, 2.0);
  Vec g(n);
  for (Index i = 0; i < n; ++i) g[i] = dist(rng);
  return g;
}
static Vec to_state(const Vec& px, const Vec& py) {
  Vec x(px);
  x.insert(x.end(), py.begin(), py.end());
  return x;
}

// test_quadtree.cpp:40-129
static void check_tree_invariants(const QuadTree<double>& tree, const Vec& px, const Vec& py, const Vec& gamma,
                                  Index cap) {
  const Index n = static_cast<Index>(px.size());
  CHECK(tree.size() == n);
  std::vector<char> seen(n, 0);
  for (Index k = 0; k < n; ++k) {
    const Index p = tree.perm[k];
    CHECK(p >= 0 && p < n && !seen[p]);
    seen[p] = 1;
    CHECK(tree.slot[p] == k);
  }
  const auto& root = tree.nodes[0];
  CHECK(root.begin == 0 && root.end == n && root.depth == 0);
  CHECK(approx(root.bounds[1] - root.bounds[0], root.width, 1e-15));
  CHECK(approx(root.bounds[3] - root.bounds[2], root.width, 1e-15));
  for (size_t id = 0; id < tree.nodes.size(); ++id) {
    const auto& nd = tree.nodes[id];
    CHECK(nd.begin < nd.end);
    double gs = 0, wx = 0, wy = 0, plx = 0, ply = 0;
    for (Index k = nd.begin; k < nd.end; ++k) {
      const Index p = tree.perm[k];
      CHECK(px[p] >= nd.bounds[0] - 1e-12 && px[p] <= nd.bounds[1] + 1e-12);
      CHECK(py[p] >= nd.bounds[2] - 1e-12 && py[p] <= nd.bounds[3] + 1e-12);
      gs += gamma[p];
      wx += gamma[p] * px[p];
      wy += gamma[p] * py[p];
      plx += px[p];
      ply += py[p];
    }
    CHECK(approx(nd.gamma_sum, gs, 1e-13));
    CHECK(nd.centroid_fallback == (gs == 0.0));
    const double ex = nd.centroid_fallback ? plx / double(nd.count()) : wx / gs;
    const double ey = nd.centroid_fallback ? ply / double(nd.count()) : wy / gs;
    CHECK(std::hypot(nd.centroid.x - ex, nd.centroid.y - ey) <= 1e-12 * (1.0 + std::hypot(ex, ey)));
    if (nd.leaf()) {
      CHECK(nd.count() <= cap || nd.depth >= kMaxTreeDepth);
    } else {
      Index cursor = nd.begin;
      const double cx = (nd.bounds[0] + nd.bounds[1]) / 2, cy = (nd.bounds[2] + nd.bounds[3]) / 2;
      for (int q = 0; q < 4; ++q) {
        if (nd.children[q] < 0) continue;
        const auto& ch = tree.nodes[nd.children[q]];
        CHECK(ch.begin == cursor);
        cursor = ch.end;
        CHECK(ch.depth == nd.depth + 1);
        CHECK(approx(ch.width, nd.width / 2, 1e-15));
        CHECK(ch.count() >= 1);
        for (Index k = ch.begin; k < ch.end; ++k) {
          const Index p = tree.perm[k];
          CHECK(((py[p] <= cy ? 0 : 1) * 2 + (px[p] <= cx ? 0 : 1)) == q);
        }
      }
      CHECK(cursor == nd.end);
    }
  }
  for (Index p = 0; p < n; ++p) {
    const auto leaf = tree.leaf_node[p];
    CHECK(leaf >= 0 && tree.nodes[leaf].leaf() && tree.contains(leaf, p));
  }
}

TEST_CASE("test_quadtree.cpp:133 four corner points split into one node per quadrant") {
  Vec px = {0, 1, 0, 1}, py = {0, 0, 1, 1}, g(4, 1.0);
  const auto tree = build_tree<double>(px, py, g, 1);
  CHECK(tree.nodes.size() == 5);
  CHECK(approx(tree.nodes[0].bounds[0], 0.0, 1e-12) && approx(tree.nodes[0].bounds[1], 1.0, 1e-12));
  CHECK(approx(tree.nodes[0].width, 1.0, 1e-12));
  for (int c = 0; c < 4; ++c) CHECK(tree.nodes[0].children[c] == c + 1);
  CHECK(tree.contains(1, 0) && tree.contains(2, 1) && tree.contains(3, 2) && tree.contains(4, 3));
  for (int c = 1; c <= 4; ++c) CHECK(tree.nodes[c].leaf());
  check_tree_invariants(tree, px, py, g, 1);
}

TEST_CASE("test_quadtree.cpp:157 points exactly on a split line go to the lower-left side") {
  Vec px = {0, 2, 1}, py = {0, 2, 1}, g(3, 1.0);
  const auto tree = build_tree<double>(px, py, g, 1);
  const auto& root = tree.nodes[0];
  CHECK(root.children[0] >= 0);
  CHECK(tree.nodes[root.children[0]].count() == 2);
  CHECK(tree.contains(root.children[0], 2));
  CHECK(root.children[1] == -1 && root.children[2] == -1);
  CHECK(root.children[3] >= 0 && tree.nodes[root.children[3]].count() == 1);
  check_tree_invariants(tree, px, py, g, 1);
}

TEST_CASE("test_quadtree.cpp:174 coincident points stop at the depth guard") {
  Vec px = {4.5, 4.5, 4.5}, py = {-2.0, -2.0, -2.0}, g(3, 1.0);
  const auto tree = build_tree<double>(px, py, g, 1);
  CHECK(approx(tree.nodes[0].width, 1.0, 1e-12));
  int deepest = 0;
  for (const auto& nd : tree.nodes) deepest = std::max(deepest, nd.depth);
  CHECK(deepest == kMaxTreeDepth);
  CHECK(tree.nodes[tree.leaf_node[0]].count() == 3);
  check_tree_invariants(tree, px, py, g, 1);
}

TEST_CASE("test_quadtree.cpp:188 random trees satisfy the structural invariants") {
  std::mt19937_64 rng(11);
  for (const Index n : {1, 2, 7, 40, 150})
    for (const Index cap : {Index{1}, Index{4}, Index{16}}) {
      Vec px, py;
      random_points(rng, n, px, py);
      if (n >= 7) {
        px[3] = px[1], py[3] = py[1];
        px[4] = px[1], py[4] = py[1];
      }
      const Vec g = random_gamma(rng, n);
      check_tree_invariants(build_tree<double>(px, py, g, cap), px, py, g, cap);
    }
}

TEST_CASE("test_quadtree.cpp:204 zero net circulation falls back to the arithmetic mean") {
  const auto tree = build_tree<double>(Vec{0, 1}, Vec{0, 1}, Vec{1.0, -1.0}, 2);
  CHECK(tree.nodes[0].centroid_fallback);
  CHECK(tree.nodes[0].gamma_sum == 0.0);
  CHECK(approx(tree.nodes[0].centroid.x, 0.5, 1e-12) && approx(tree.nodes[0].centroid.y, 0.5, 1e-12));
}

TEST_CASE("test_quadtree.cpp:217 build_tree input validation") {
  std::mt19937_64 rng(1);
  Vec px, py;
  random_points(rng, 4, px, py);
  CHECK_THROWS_AS(build_tree<double>(Vec{}, Vec{}, Vec{}, 1), config_error);
  CHECK_THROWS_AS(build_tree<double>(px, py, Vec(3, 1.0), 1), config_error);
  CHECK_THROWS_AS(build_tree<double>(px, py, Vec(4, 1.0), 0), config_error);
  Vec bad = px;
  bad[0] = std::nan("");
  CHECK_THROWS_AS(build_tree<double>(bad, py, Vec(4, 1.0), 1), config_error);
}

TEST_CASE("test_quadtree.cpp:228 opening-ratio acceptability boundary") {
  TreeNode<double> node{};
  node.width = 1.0;
  node.centroid = {2.0, 0.0};
  const V2<double> t{0.0, 0.0};
  CHECK(bh_prune_check<double>(node, t, 0.5));
  CHECK(!bh_prune_check<double>(node, t, 0.49));
  CHECK(!bh_prune_check<double>(node, t, 0.0));
  CHECK(bh_prune_check<double>(node, t, 10.0));
  node.centroid = t;
  CHECK(!bh_prune_check<double>(node, t, 10.0));
}

TEST_CASE("test_quadtree.cpp:241 neighborhood acceptability requires strict overlap") {
  const std::array<double, 4> leaf = {0, 1, 0, 1};
  CHECK(neighbor_prune_check<double>({2.5, 3.0, 0.0, 1.0}, leaf, 1.0, 1.0));
  CHECK(neighbor_prune_check<double>({2.0, 3.0, 0.0, 1.0}, leaf, 1.0, 1.0));
  CHECK(!neighbor_prune_check<double>({1.9, 3.0, 0.0, 1.0}, leaf, 1.0, 1.0));
  CHECK(neighbor_prune_check<double>({2.0, 3.0, 2.0, 3.0}, leaf, 1.0, 1.0));
  CHECK(!neighbor_prune_check<double>({2.5, 5.5, 0.0, 1.0}, leaf, 3.0, 1.0));
  CHECK(neighbor_prune_check<double>({2.5, 3.0, 0.0, 1.0}, leaf, 0.5, 1.0));
  CHECK(neighbor_prune_check<double>({1.0, 2.0, 0.0, 1.0}, leaf, 1.0, 0.0));
  CHECK(!neighbor_prune_check<double>({0.5, 2.0, 0.5, 2.0}, leaf, 1.0, 0.0));
}

TEST_CASE("test_quadtree.cpp:257 collected clusters and direct ids cover every other particle once") {
  std::mt19937_64 rng(29);
  const Index n = 120;
  Vec px, py;
  random_points(rng, n, px, py);
  const Vec g = random_gamma(rng, n);
  const auto tree = build_tree<double>(px, py, g, 4);
  for (const auto crit : {ClusterCriterion<double>::barnes_hut(0.7), ClusterCriterion<double>::neighbor(1.0),
                          ClusterCriterion<double>::barnes_hut(0.0), ClusterCriterion<double>::neighbor(0.0)})
    for (const Index target : {Index{0}, Index{17}, Index{119}}) {
      const auto cl = collect_clusters(tree, target, crit);
      CHECK(std::is_sorted(cl.direct_ids.begin(), cl.direct_ids.end()));
      CHECK(std::is_sorted(cl.cluster_nodes.begin(), cl.cluster_nodes.end()));
      std::set<Index> covered;
      for (const Index j : cl.direct_ids) {
        CHECK(j != target);
        CHECK(covered.insert(j).second);
      }
      for (const auto id : cl.cluster_nodes) {
        CHECK(!tree.contains(id, target));
        for (Index k = tree.nodes[id].begin; k < tree.nodes[id].end; ++k) CHECK(covered.insert(tree.perm[k]).second);
      }
      CHECK(covered.size() == static_cast<size_t>(n - 1));
    }
}

TEST_CASE("test_quadtree.cpp:289 tree velocity with theta 0 matches the pairwise sum") {
  std::mt19937_64 rng(47);
  const Index n = 200;
  Vec px, py;
  random_points(rng, n, px, py);
  const Vec state = to_state(px, py);
  ParticleSystem<double> sys;
  sys.circulation = random_gamma(rng, n);
  sys.delta = 0.05;
  const Vec naive = pairwise_velocity<double>(state, sys);
  const auto tree = build_tree<double>(px, py, sys.circulation, 4);
  CHECK(maxabs(vsub(bh_velocity<double>(tree, state, sys, ClusterCriterion<double>::barnes_hut(0.0)), naive)) <= 1e-12);
  CHECK(maxabs(vsub(bh_velocity<double>(tree, state, sys, ClusterCriterion<double>::neighbor(1e9)), naive)) <= 1e-12);
  const auto flat = build_tree<double>(px, py, sys.circulation, n);
  CHECK(maxabs(vsub(bh_velocity<double>(flat, state, sys, ClusterCriterion<double>::barnes_hut(0.0)), naive)) == 0.0);
}

TEST_CASE("test_quadtree.cpp:317 tree jacobian with theta 0 matches the pairwise self blocks") {
  std::mt19937_64 rng(53);
  const Index n = 60;
  Vec px, py;
  random_points(rng, n, px, py);
  const Vec state = to_state(px, py);
  ParticleSystem<double> sys;
  sys.circulation = random_gamma(rng, n);
  sys.delta = 0.1;
  const auto exact = inexact_kernel_jacobian<double>(state, sys);
  const auto tree = build_tree<double>(px, py, sys.circulation, 4);
  const auto treed = bh_jacobian<double>(tree, state, sys, ClusterCriterion<double>::barnes_hut(0.0));
  for (Index i = 0; i < n; ++i) {
    const auto a = treed.block(i), b = exact.block(i);
    CHECK(std::max({std::abs(a.a00 - b.a00), std::abs(a.a01 - b.a01), std::abs(a.a10 - b.a10),
                    std::abs(a.a11 - b.a11)}) <= 1e-12);
  }
}

TEST_CASE("test_quadtree.cpp:334 moderate opening ratio stays close to the exact field") {
  std::mt19937_64 rng(61);
  const Index n = 300;
  Vec px, py;
  random_points(rng, n, px, py, 50.0);
  const Vec state = to_state(px, py);
  ParticleSystem<double> sys;
  sys.circulation = random_gamma(rng, n);
  sys.delta = 0.5;
  const Vec naive = pairwise_velocity<double>(state, sys);
  const auto tree = build_tree<double>(px, py, sys.circulation, 8);
  const Vec approx_v = bh_velocity<double>(tree, state, sys, ClusterCriterion<double>::barnes_hut(0.5));
  CHECK(l2(vsub(approx_v, naive)) / l2(naive) < 1e-2);
  CHECK(l2(vsub(approx_v, naive)) > 0.0);
}

TEST_CASE("test_quadtree.cpp:351 inflow is added after the tree summation") {
  std::mt19937_64 rng(67);
  const Index n = 20;
  Vec px, py;
  random_points(rng, n, px, py);
  const Vec state = to_state(px, py);
  ParticleSystem<double> sys;
  sys.circulation = Vec(n, 0.0);
  sys.delta = 0.0;
  sys.has_inflow = true;
  sys.inflow.resize(2 * n);
  for (Index i = 0; i < 2 * n; ++i) sys.inflow[i] = 0.25 * double(i);
  const auto tree = build_tree<double>(px, py, sys.circulation, 4);
  CHECK(maxabs(vsub(bh_velocity<double>(tree, state, sys, ClusterCriterion<double>::neighbor(1.0)), sys.inflow)) == 0.0);
}

#include "kat_rom.inc"

int main() {
  for (auto& [name, fn] : registry()) {
    g_case = name;
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  FAIL [%s] unexpected exception: %s\n", name.c_str(), e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "[PASS]" : "[FAIL]", name.c_str());
  }
  std::printf("kat: %zu cases, %d checks, %d failures\n", registry().size(), g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
