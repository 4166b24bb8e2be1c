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
#include "ptrom_oracle_tree.hpp"

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
  // BarnesHutModelVec (integrators.hpp:83-102) vs the oracle's BarnesHutModel
  const int nb = 5000;
  std::vector<double> xb(2 * nb), gb(nb);
  for (int i = 0; i < nb; ++i) {
    const double a = 2.399963 * i, r = std::sqrt((i + 0.5) / nb);
    xb[i] = r * std::cos(a);
    xb[i + nb] = r * std::sin(a);
    gb[i] = 1.0 / nb;
  }
  ptrom_b200::BarnesHutModelVec bh(ctx, gb, 1e-4, PTROM_CRIT_BARNES_HUT, 0.5, 16);
  oracle::ParticleSystem<double> sb;
  sb.circulation = gb;
  sb.delta = 1e-4;
  oracle::BarnesHutModel<double> obh{sb, oracle::ClusterCriterion<double>::barnes_hut(0.5), 16};
  const auto fv = bh.velocity(xb), ov = obh.velocity(xb);
  const auto jg = bh.jacobian(xb);
  const auto jo = obh.jacobian(xb);
  double num = 0, den = 0, jn = 0, jd = 0;
  for (int k = 0; k < 2 * nb; ++k) {
    num += (fv[k] - ov[k]) * (fv[k] - ov[k]);
    den += ov[k] * ov[k];
  }
  for (int k = 0; k < nb; ++k) {
    const double d[4] = {jg.dfx_dx[k] - jo.dfx_dx[k], jg.dfx_dy[k] - jo.dfx_dy[k], jg.dfy_dx[k] - jo.dfy_dx[k],
                         jg.dfy_dy[k] - jo.dfy_dy[k]};
    const double o[4] = {jo.dfx_dx[k], jo.dfx_dy[k], jo.dfy_dx[k], jo.dfy_dy[k]};
    for (int c = 0; c < 4; ++c) {
      jn += d[c] * d[c];
      jd += o[c] * o[c];
    }
  }
  const double bh_rel = std::sqrt(num / den), bhj_rel = std::sqrt(jn / jd);
  std::printf("BarnesHutModelVec parity: velocity rel %.3e, jacobian rel %.3e, pair evals %llu\n", bh_rel, bhj_rel,
              (unsigned long long)bh.pair_evals());
  return (worst <= 1e-12 && threw && bh_rel <= 1e-12 && bhj_rel <= 1e-12) ? 0 : 1;
}
