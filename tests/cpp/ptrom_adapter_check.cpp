// C++ consumer of the PTROM drop-in (include/ptrom_b200.hpp,
// ptrom_b200::ptrom_simulate / DevicePtrom): the offline products are built
// by the oracle's restatement of the reference's producers (build_pod,
// greedy_sample, build_gnat_operator, cluster_pod — the reference's own
// structs, nested index lists and all) and handed to the adapter with no
// hand-written marshalling. Checks rom.hpp:404-412 against the oracle: x_hat
// per step within 1e-12, equal iteration counts, and the in-place
// reassignment of the surrogate bit for bit. Exit 0 on parity.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ptrom_b200.hpp"
#include "ptrom_oracle_rom.hpp"

using namespace oracle;

static double lcg(unsigned long long& s) {  // uniform in (0, 1)
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((s >> 11) + 0.5) * 0x1p-53;
}

int main() {
  const Index n = 700, nsnap = 14, modes = 5, modes_r = 9, n_steps = 6;
  unsigned long long seed = 12345;
  Vec x0(2 * n), ga(n, 0.0), gb(n, 0.0);
  for (Index i = 0; i < n; ++i) {  // two patches, as BASELINE configs[3]
    const double r = 0.15 * std::sqrt(-2.0 * std::log(lcg(seed))), a = 2.0 * M_PI * lcg(seed);
    x0[i] = (i < n / 2 ? -0.5 : 0.5) + r * std::cos(a);
    x0[i + n] = r * std::sin(a);
    (i < n / 2 ? ga : gb)[i] = 2.0 / n;
  }
  Mat snaps(2 * n, nsnap), rsnaps(2 * n, nsnap);
  for (Index c = 0; c < nsnap; ++c)
    for (Index r = 0; r < 2 * n; ++r) {
      const double xr = x0[r % n], yr = x0[r % n + n];
      snaps(r, c) = x0[r] + 1e-2 * std::sin((c + 1) * xr + 0.3 * c * yr + 0.1 * r / n) * (lcg(seed) - 0.5);
      rsnaps(r, c) = lcg(seed) - 0.5;
    }
  const PODBasis basis = build_pod(snaps, modes, x0);
  const PODBasis residual = build_pod(rsnaps, modes_r, Vec(2 * n, 0.0));
  const std::vector<Index> ids = greedy_sample(residual.phi, 14);
  const GnatOperator op = build_gnat_operator(residual.phi, ids);
  Vec g1(n);
  for (Index i = 0; i < n; ++i) g1[i] = ga[i] + gb[i];
  const SurrogateSourceBasis built = cluster_pod(basis, g1, ids, ClusterCriterion<double>::neighbor(1.0), 1);

  ParticleSystem<double> sys;
  sys.circulation.resize(n);
  for (Index i = 0; i < n; ++i) sys.circulation[i] = ga[i] + 1.3 * gb[i];
  sys.delta = 2.5e-5;
  RomConfig cfg;
  cfg.tol = 1e-300;
  cfg.max_iters = 5;
  const double dt = 1e-3;

  SurrogateSourceBasis s_cpu = built, s_gpu = built;
  const RomTrajectory want = ptrom_simulate(basis, op, s_cpu, sys, dt, n_steps, cfg);
  ptrom_b200::Context ctx(0);
  RomTrajectory got;
  ptrom_b200::ptrom_simulate(ctx, basis, op, s_gpu, sys, dt, n_steps, cfg, got);

  int bad = 0;
  for (Index s = 0; s < n_steps; ++s) {
    double num = 0, den = 0;
    for (Index j = 0; j < modes; ++j) {
      const double d = got.x_hat(j, s) - want.x_hat(j, s);
      num += d * d;
      den += want.x_hat(j, s) * want.x_hat(j, s);
    }
    const double rel = std::sqrt(num / den);
    if (!(rel <= 1e-12)) {
      std::printf("step %ld: x_hat rel %.3e\n", (long)s, rel);
      ++bad;
    }
    if (got.iterations[s] != want.iterations[s]) {
      std::printf("step %ld: iterations %d vs %d\n", (long)s, got.iterations[s], want.iterations[s]);
      ++bad;
    }
  }
  // reassign_cluster_circulation mutated the surrogate (reduction.hpp:400-431, test_rom.cpp:454)
  if (s_gpu.phi_tilde.a != s_cpu.phi_tilde.a || s_gpu.gamma_tilde != s_cpu.gamma_tilde ||
      s_gpu.x0_tilde != s_cpu.x0_tilde || s_gpu.zero_gamma != s_cpu.zero_gamma ||
      s_gpu.direct_gamma != s_cpu.direct_gamma) {
    std::printf("reassigned surrogate tables differ from the oracle's\n");
    ++bad;
  }
  if (s_gpu.gamma_tilde == built.gamma_tilde) {
    std::printf("surrogate was not reassigned in place\n");
    ++bad;
  }
  std::printf("ptrom adapter: %ld clusters, %ld direct, %s\n", (long)s_gpu.gamma_tilde.size(),
              (long)s_gpu.direct_ids.size(), bad ? "FAIL" : "ok");
  return bad ? 1 : 0;
}
