// C++ consumer of the drop-in adapter (include/ptrom_b200.hpp): drives the
// oracle's FomStepper (a restatement of integrators.hpp:117-201, templated on
// the Model concept exactly like the reference's) with the B200-backed
// PairwiseModelVec, and compares against the all-CPU oracle run.
// Exit 0 on parity (1e-12 relative per snapshot).
#include <cmath>
#include <cstdio>
#include <vector>

#include "ptrom_b200.hpp"
#include "ptrom_oracle.hpp"

struct GpuModel {  // Model concept over the adapter, returning oracle types
  ptrom_b200::PairwiseModelVec m;
  std::vector<double> velocity(const std::vector<double>& x) const { return m.velocity(x); }
  oracle::BlockDiagonalJacobian<double> jacobian(const std::vector<double>& x) const {
    auto j = m.jacobian(x);
    return {j.dfx_dx, j.dfx_dy, j.dfy_dx, j.dfy_dy};
  }
};

int main() {
  const int n = 300;
  std::vector<double> x0(2 * n), g(n);
  for (int i = 0; i < n; ++i) {
    const double a = 0.37 * i, r = std::sqrt((i + 0.5) / n);
    x0[i] = r * std::cos(a);
    x0[i + n] = r * std::sin(a);
    g[i] = ((i * 7919) % 1000 - 500) * 1e-5;
  }
  const double delta = 1e-4;
  ptrom_b200::Context ctx(0);
  GpuModel gpu{ptrom_b200::PairwiseModelVec(ctx, g, delta)};
  oracle::ParticleSystem<double> sys;
  sys.circulation = g;
  sys.delta = delta;
  oracle::PairwiseModel<double> cpu{sys};
  oracle::NewtonConfig cfg;
  const auto a = oracle::fom_simulate<double>(x0, gpu, 1e-3, 10, cfg);
  const auto b = oracle::fom_simulate<double>(x0, cpu, 1e-3, 10, cfg);
  double worst = 0;
  for (int s = 0; s < 10; ++s) {
    double num = 0, den = 0;
    for (int k = 0; k < 2 * n; ++k) {
      const double d = a.snapshots[s * 2 * n + k] - b.snapshots[s * 2 * n + k];
      num += d * d;
      den += b.snapshots[s * 2 * n + k] * b.snapshots[s * 2 * n + k];
    }
    worst = std::fmax(worst, std::sqrt(num / den));
  }
  std::printf("adapter FomStepper parity: worst snapshot rel %.3e, pair evals %llu\n", worst,
              (unsigned long long)gpu.m.pair_evals());
  bool threw = false;
  try {
    ptrom_b200::PairwiseModelVec bad(ctx, {1.0, 1.0}, 0.0);
    bad.velocity({1.0, 1.0, 2.0, 2.0});
  } catch (const ptrom_b200::numerical_error&) {
    threw = true;
  }
  std::printf("coincident pair -> numerical_error: %s\n", threw ? "yes" : "no");
  return (worst <= 1e-12 && threw) ? 0 : 1;
}
