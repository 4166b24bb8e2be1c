// rom_capi.cu — C ABI for the PTROM online path (include/ptrom_b200.h "ptrom").
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "comm.cuh"
#include "ops.cuh"
#include "rom.cuh"

namespace ptrom {
void rom_reassign_exact(ptrom_ctx* ctx, DSurrogate& s, const DBasis& b, const double* d_gamma);
void rom_basis_rowmajor(ptrom_ctx* ctx, DBasis& b);
void rom_reconstruct(ptrom_ctx* ctx, const DBasis& b, long long n_steps, const double* d_xhat, long long n_out,
                     const long long* d_dofs, double* d_out);
void rom_affine_tables(ptrom_ctx* ctx, const DSurrogate& s, const DBasis& b, const double* d_ga, const double* d_gb,
                       AffineTables& t);
unsigned long long rom_hyperpair(ptrom_ctx* ctx, const DSurrogate& s, const DGnat* g, const AffineTables* t,
                                 const EngineTables* et, int B, int xs, const double* d_xhat, const double* d_mu,
                                 const unsigned char* d_active, const double* d_xbar_in, double* d_xbar_out,
                                 double delta, int form, const double* d_inflow, long long n, RomScratch& w,
                                 double* d_f, double* d_jac, bool count_pairs);
unsigned long long rom_gnat_simulate(ptrom_ctx* ctx, const DSurrogate& s, const DGnat& g, const AffineTables* t,
                                     int B, const double* d_mu, double delta, int form, const double* d_inflow,
                                     long long n, double dt, long long n_steps, double tol, int max_iters,
                                     double alpha, double* d_xhat_out, int* d_iters, unsigned char* d_conv);
std::vector<long long> offline_greedy_sample(ptrom_ctx* ctx, long long n_dofs, int n_r, const double* phi_r,
                                             long long n_target, const std::vector<long long>& preseed);
std::vector<double> offline_gnat_operator(ptrom_ctx* ctx, long long n_dofs, int m_r, const double* phi_r,
                                          const std::vector<long long>& ids);
void offline_cluster_pod(ptrom_ctx* ctx, const DBasis& b, const double* d_gamma, long long leaf_cap, int crit_kind,
                         double crit_value, const std::vector<long long>& targets, DSurrogate& s,
                         std::vector<void*>& allocs, std::vector<int>& cluster_node_ids);
}  // namespace ptrom

using namespace ptrom;

namespace {

struct DevAllocs {
  std::vector<void*> p;
  ~DevAllocs() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  T* up(const T* h, size_t count) {
    T* d = nullptr;
    PTROM_CUDA(cudaMalloc(&d, std::max<size_t>(count, 1) * sizeof(T)));
    p.push_back(d);
    if (h && count) PTROM_CUDA(cudaMemcpy(d, h, count * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  template <class T>
  T* zeros(size_t count) {
    T* d = up<T>(nullptr, count);
    PTROM_CUDA(cudaMemset(d, 0, std::max<size_t>(count, 1) * sizeof(T)));
    return d;
  }
};

template <class F>
int guarded(ptrom_ctx* ctx, F&& fn) {
  if (!ctx) return PTROM_CONFIG_ERROR;
  try {
    cudaSetDevice(ctx->device);
    fn();
    ctx->err.clear();
    return PTROM_OK;
  } catch (const status_error& e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return PTROM_CUDA_ERROR;
  }
}

void check_finite(const double* v, size_t count, const char* what) {
  for (size_t i = 0; i < count; ++i)
    if (!std::isfinite(v[i])) config_fail(std::string(what) + ": non-finite input");
}

}  // namespace

struct ptrom_basis {
  int device = 0;
  DBasis b;
  DevAllocs mem;
};
struct ptrom_gnat_op {
  int device = 0;
  DGnat g;
  std::vector<long long> ids;
  DevAllocs mem;
};
struct ptrom_surrogate {
  int device = 0;
  DSurrogate s;
  std::vector<long long> target_ids;
  std::vector<int> cluster_node_ids;  // provenance (reduction.hpp:285), when built on the device
  long long n_membership = 0, n_cluster_list = 0, n_direct_list = 0;
  DevAllocs mem;
};

namespace {

// Shared argument checks of the batched entry points (rom.hpp:264-273,
// RomConfig::validate).
void validate_batch(const ptrom_basis* basis, const ptrom_gnat_op* op, const ptrom_surrogate* sur, int64_t n,
                    const double* gamma_a, const double* gamma_b, int64_t n_inst, const double* mu, double dt,
                    int64_t n_steps, double tol, int max_iters, double step_length) {
  if (!basis || !op || !sur) config_fail("null basis / operator / surrogate");
  if (!(dt > 0)) config_fail("time step must be positive");
  if (n_steps < 0) config_fail("negative step count");
  if (!(tol > 0)) config_fail("ROM tolerance must be positive");
  if (max_iters < 1) config_fail("ROM max_iters must be >= 1");
  if (!(step_length > 0)) config_fail("ROM step length must be positive");
  if (n != basis->b.n) config_fail("GnatSolver: basis dimension does not match particle count");
  if (sur->target_ids != op->ids) config_fail("GnatSolver: surrogate targets must equal the sampled particle ids");
  if (n_inst < 1) config_fail("batch needs at least one instance");
  check_finite(gamma_a, (size_t)n, "non-finite circulation");
  check_finite(gamma_b, (size_t)n, "non-finite circulation");
  check_finite(mu, (size_t)n_inst, "non-finite parameter");
}

// Batched affine march over host μ / Γa / Γb (SURVEY.md §8b
// ptrom_gnat_simulate_batch): affine member sums once, then batches of B
// instances; x_hat [n_inst][n_steps][M], iterations / converged
// [n_inst][n_steps] on the host. Returns the pair count.
unsigned long long batch_march(ptrom_ctx* ctx, const DBasis& b, const DGnat& g, const DSurrogate& s, long long n,
                               const double* gamma_a, const double* gamma_b, long long n_inst, const double* mu,
                               long long batch, double delta, int form, const double* inflow, double dt,
                               long long n_steps, double tol, int max_iters, double step_length, double* x_hat,
                               int* iterations, uint8_t* converged) {
  DevAllocs tmp;
  const double* dga = tmp.up(gamma_a, (size_t)n);
  const double* dgb = tmp.up(gamma_b, (size_t)n);
  const double* dinf = inflow ? tmp.up(inflow, (size_t)2 * n) : nullptr;
  AffineTables t;
  t.pa = tmp.zeros<double>((size_t)2 * s.n_c * s.m);
  t.pb = tmp.zeros<double>((size_t)2 * s.n_c * s.m);
  t.xa = tmp.zeros<double>((size_t)2 * s.n_c);
  t.xb = tmp.zeros<double>((size_t)2 * s.n_c);
  t.ga = tmp.zeros<double>((size_t)s.n_c);
  t.gb = tmp.zeros<double>((size_t)s.n_c);
  // direct circulations Γa[id], Γb[id]
  std::vector<long long> dids((size_t)s.u);
  PTROM_CUDA(cudaMemcpy(dids.data(), s.direct_ids, dids.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<double> dga_h(dids.size()), dgb_h(dids.size());
  for (size_t k = 0; k < dids.size(); ++k) {
    dga_h[k] = gamma_a[dids[k]];
    dgb_h[k] = gamma_b[dids[k]];
  }
  t.dga = tmp.up(dga_h.data(), dga_h.size());
  t.dgb = tmp.up(dgb_h.data(), dgb_h.size());
  rom_affine_tables(ctx, s, b, dga, dgb, t);
  const int m = b.m;
  const long long B = std::max<long long>(1, std::min<long long>(batch > 0 ? batch : 256, n_inst));
  const long long steps = std::max<long long>(n_steps, 1);
  double* dmu = tmp.up(mu, (size_t)n_inst);
  double* dxh = tmp.zeros<double>((size_t)B * m * steps);
  int* dit = tmp.zeros<int>((size_t)B * steps);
  unsigned char* dcv = tmp.zeros<unsigned char>((size_t)B * steps);
  unsigned long long pairs = 0;
  for (long long b0 = 0; b0 < n_inst; b0 += B) {
    const int nb = (int)std::min<long long>(B, n_inst - b0);
    pairs += rom_gnat_simulate(ctx, s, g, &t, nb, dmu + b0, delta, form, dinf, n, dt, n_steps, tol, max_iters,
                               step_length, dxh, dit, dcv);
    if (n_steps > 0) {
      PTROM_CUDA(cudaMemcpy(x_hat + (size_t)b0 * n_steps * m, dxh, (size_t)nb * n_steps * m * 8,
                            cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(iterations + (size_t)b0 * n_steps, dit, (size_t)nb * n_steps * 4,
                            cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(converged + (size_t)b0 * n_steps, dcv, (size_t)nb * n_steps, cudaMemcpyDeviceToHost));
    }
  }
  return pairs;
}

}  // namespace

extern "C" {

int ptrom_basis_create(ptrom_ctx* ctx, int64_t n_dofs, int64_t modes, const double* phi, const double* singular_values,
                       const double* x_ref, ptrom_basis** out) {
  return guarded(ctx, [&] {
    if (n_dofs <= 0 || n_dofs % 2 != 0) config_fail("state dimension must be even");
    if (modes < 1) config_fail("basis needs at least one mode");
    check_finite(phi, (size_t)(n_dofs * modes), "basis");
    check_finite(x_ref, (size_t)n_dofs, "basis reference state");
    auto* h = new ptrom_basis;
    h->device = ctx->device;
    try {
      h->b.n = n_dofs / 2;
      h->b.m = (int)modes;
      h->b.phi = h->mem.up(phi, (size_t)(n_dofs * modes));
      h->b.x_ref = h->mem.up(x_ref, (size_t)n_dofs);
      h->b.sv = h->mem.up(singular_values, singular_values ? (size_t)modes : 0);
      rom_basis_rowmajor(ctx, h->b);
      h->mem.p.push_back(h->b.rm);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void ptrom_basis_free(ptrom_basis* b) {
  if (b) {
    cudaSetDevice(b->device);
    delete b;
  }
}

// rom.hpp:45-64 reconstruct_output (dofs != NULL) / reconstruct_full (dofs == NULL).
int ptrom_reconstruct_output_f64(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_steps, const double* x_hat,
                                 int64_t n_dofs, const int64_t* dofs, double* out) {
  return guarded(ctx, [&] {
    if (!basis) config_fail("reconstruct_output: null basis");
    if (n_steps < 0) config_fail("reconstruct_output: negative step count");
    const long long nd = 2 * basis->b.n;
    const long long n_out = dofs ? n_dofs : nd;
    if (dofs)
      for (long long k = 0; k < n_dofs; ++k)
        if (dofs[k] < 0 || dofs[k] >= nd) config_fail("reconstruct_output: dof out of range");
    const int m = basis->b.m;
    double* dx = nullptr;
    double* dout = nullptr;
    long long* dd = nullptr;
    PTROM_CUDA(cudaMallocAsync(&dx, sizeof(double) * std::max<long long>(1, m * n_steps), ctx->stream));
    PTROM_CUDA(cudaMallocAsync(&dout, sizeof(double) * std::max<long long>(1, n_out * n_steps), ctx->stream));
    if (dofs) PTROM_CUDA(cudaMallocAsync(&dd, sizeof(long long) * std::max<long long>(1, n_dofs), ctx->stream));
    PTROM_CUDA(cudaMemcpyAsync(dx, x_hat, sizeof(double) * m * n_steps, cudaMemcpyHostToDevice, ctx->stream));
    if (dofs)
      PTROM_CUDA(cudaMemcpyAsync(dd, dofs, sizeof(long long) * n_dofs, cudaMemcpyHostToDevice, ctx->stream));
    rom_reconstruct(ctx, basis->b, n_steps, dx, n_out, dd, dout);
    PTROM_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n_out * n_steps, cudaMemcpyDeviceToHost, ctx->stream));
    PTROM_CUDA(cudaFreeAsync(dx, ctx->stream));
    PTROM_CUDA(cudaFreeAsync(dout, ctx->stream));
    if (dd) PTROM_CUDA(cudaFreeAsync(dd, ctx->stream));
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ptrom_dev_reconstruct_output_f64(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_steps, const double* d_xhat,
                                     int64_t n_dofs, const int64_t* d_dofs, double* d_out) {
  return guarded(ctx, [&] {
    if (!basis) config_fail("reconstruct_output: null basis");
    const long long n_out = d_dofs ? n_dofs : 2 * basis->b.n;
    rom_reconstruct(ctx, basis->b, n_steps, d_xhat, n_out, reinterpret_cast<const long long*>(d_dofs), d_out);
  });
}

int ptrom_gnat_op_create(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_samples, const int64_t* sample_ids,
                         int64_t m_r, const double* A, ptrom_gnat_op** out) {
  return guarded(ctx, [&] {
    if (!basis) config_fail("null basis");
    const DBasis& b = basis->b;
    if (n_samples < 1) config_fail("build_gnat_operator: no sample ids");
    std::vector<long long> ids(sample_ids, sample_ids + n_samples);
    if (!std::is_sorted(ids.begin(), ids.end()) || std::adjacent_find(ids.begin(), ids.end()) != ids.end())
      config_fail("GnatOperator: sample ids must be sorted and unique");
    if (ids.front() < 0 || ids.back() >= b.n) config_fail("build_gnat_operator: sample id out of range");
    if (m_r < 1 || m_r > 32) config_fail("ptrom online engine supports 1..32 residual modes");
    if (b.m > 32) config_fail("ptrom online engine supports at most 32 modes");
    check_finite(A, (size_t)(m_r * 2 * n_samples), "GNAT operator");
    auto* h = new ptrom_gnat_op;
    h->device = ctx->device;
    try {
      const long long ns = n_samples, rows = 2 * ns;
      const int mp = (b.m + 7) / 8 * 8;
      h->ids = ids;
      DGnat& g = h->g;
      g.n_s = ns;
      g.m_r = (int)m_r;
      g.m = b.m;
      g.mp = mp;
      g.ids = h->mem.up(ids.data(), ids.size());
      // A padded to 32 rows (zero rows do not change the least-squares problem)
      std::vector<double> Ap((size_t)32 * rows, 0.0);
      for (long long k = 0; k < rows; ++k)
        for (int i = 0; i < m_r; ++i) Ap[i + 32 * k] = A[i + m_r * k];
      g.A = h->mem.up(Ap.data(), Ap.size());
      // Φ̄ and x̄⁰ gathered on the host from the device basis (rom.hpp:279-289)
      std::vector<double> phi((size_t)2 * b.n * b.m), xr((size_t)2 * b.n);
      PTROM_CUDA(cudaMemcpy(phi.data(), b.phi, phi.size() * 8, cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(xr.data(), b.x_ref, xr.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<double> pb((size_t)rows * mp, 0.0), x0b((size_t)rows);
      for (long long k = 0; k < ns; ++k) {
        const long long p = ids[k];
        for (int j = 0; j < b.m; ++j) {
          pb[k + rows * j] = phi[p + 2 * b.n * j];
          pb[k + ns + rows * j] = phi[p + b.n + 2 * b.n * j];
        }
        x0b[k] = xr[p];
        x0b[k + ns] = xr[p + b.n];
      }
      g.phi_bar = h->mem.up(pb.data(), pb.size());
      g.x0_bar = h->mem.up(x0b.data(), x0b.size());
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void ptrom_gnat_op_free(ptrom_gnat_op* g) {
  if (g) {
    cudaSetDevice(g->device);
    delete g;
  }
}

int ptrom_surrogate_create(ptrom_ctx* ctx, int64_t modes, int64_t n_clusters, const double* phi_tilde,
                           const double* gamma_tilde, const double* x0_tilde, const uint8_t* zero_gamma,
                           const int64_t* membership_offsets, const int64_t* membership_ids, int64_t n_targets,
                           const int64_t* target_ids, const int64_t* cluster_offsets, const int64_t* cluster_list,
                           int64_t n_direct, const int64_t* direct_ids, const double* direct_phi,
                           const double* direct_x0, const double* direct_gamma, const int64_t* direct_offsets,
                           const int64_t* direct_list, ptrom_surrogate** out) {
  return guarded(ctx, [&] {
    if (n_targets < 1) config_fail("cluster_pod: no targets");
    if (modes < 1 || modes > 32) config_fail("surrogate supports 1..32 modes");
    auto* h = new ptrom_surrogate;
    h->device = ctx->device;
    try {
      DSurrogate& s = h->s;
      s.m = (int)modes;
      s.n_c = n_clusters;
      s.u = n_direct;
      s.n_t = n_targets;
      const size_t nc = (size_t)n_clusters, u = (size_t)n_direct, nt = (size_t)n_targets;
      h->n_membership = membership_offsets[nc];
      h->n_cluster_list = cluster_offsets[nt];
      h->n_direct_list = direct_offsets[nt];
      s.phi_tilde = h->mem.up(phi_tilde, 2 * nc * modes);
      s.x0_tilde = h->mem.up(x0_tilde, 2 * nc);
      s.gamma_tilde = h->mem.up(gamma_tilde, nc);
      s.zero_gamma = h->mem.up(zero_gamma, zero_gamma ? nc : 0);
      s.mem_off = h->mem.up(reinterpret_cast<const long long*>(membership_offsets), nc + 1);
      for (size_t c = 0; c < nc; ++c)
        s.max_members = std::max<long long>(s.max_members, membership_offsets[c + 1] - membership_offsets[c]);
      s.mem_ids = h->mem.up(reinterpret_cast<const long long*>(membership_ids), (size_t)membership_offsets[nc]);
      h->target_ids.assign(target_ids, target_ids + nt);
      s.target_ids = h->mem.up(reinterpret_cast<const long long*>(target_ids), nt);
      s.cl_off = h->mem.up(reinterpret_cast<const long long*>(cluster_offsets), nt + 1);
      std::vector<int> cl(cluster_list, cluster_list + cluster_offsets[nt]);
      for (int c : cl)
        if (c < 0 || c >= n_clusters) config_fail("surrogate: cluster index out of range");
      s.cl_list = h->mem.up(cl.data(), cl.size());
      s.d_off = h->mem.up(reinterpret_cast<const long long*>(direct_offsets), nt + 1);
      std::vector<int> dl(direct_list, direct_list + direct_offsets[nt]);
      for (int d : dl)
        if (d < 0 || d >= n_direct) config_fail("surrogate: direct index out of range");
      s.d_list = h->mem.up(dl.data(), dl.size());
      s.direct_ids = h->mem.up(reinterpret_cast<const long long*>(direct_ids), u);
      s.direct_phi = h->mem.up(direct_phi, 2 * u * modes);
      s.direct_x0 = h->mem.up(direct_x0, 2 * u);
      s.direct_gamma = h->mem.up(direct_gamma, u);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void ptrom_surrogate_free(ptrom_surrogate* s) {
  if (s) {
    cudaSetDevice(s->device);
    delete s;
  }
}

int ptrom_surrogate_export(ptrom_ctx* ctx, const ptrom_surrogate* sur, double* phi_tilde, double* gamma_tilde,
                           double* x0_tilde, uint8_t* zero_gamma, double* direct_gamma) {
  return guarded(ctx, [&] {
    const DSurrogate& s = sur->s;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) PTROM_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    d2h(phi_tilde, s.phi_tilde, (size_t)2 * s.n_c * s.m * 8);
    d2h(gamma_tilde, s.gamma_tilde, (size_t)s.n_c * 8);
    d2h(x0_tilde, s.x0_tilde, (size_t)2 * s.n_c * 8);
    d2h(zero_gamma, s.zero_gamma, (size_t)s.n_c);
    d2h(direct_gamma, s.direct_gamma, (size_t)s.u * 8);
  });
}

int ptrom_reassign_cluster_circulation_f64(ptrom_ctx* ctx, ptrom_surrogate* sur, int64_t n, const double* gamma,
                                           const ptrom_basis* basis) {
  return guarded(ctx, [&] {
    if (!sur || !basis) config_fail("null surrogate or basis");
    if (n != basis->b.n) config_fail("reassign_cluster_circulation: gamma size mismatch");
    check_finite(gamma, (size_t)n, "reassign_cluster_circulation");
    DevAllocs tmp;
    const double* dg = tmp.up(gamma, (size_t)n);
    rom_reassign_exact(ctx, sur->s, basis->b, dg);
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ptrom_hyperpair_f64(ptrom_ctx* ctx, const ptrom_surrogate* sur, const double* target_positions,
                        const double* x_hat, double delta, int form, int64_t n, const double* inflow, double* f,
                        double* jac, double* cluster_positions, double* direct_positions, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    if (!sur) config_fail("null surrogate");
    const DSurrogate& s = sur->s;
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    DevAllocs tmp;
    const long long nt = s.n_t;
    const double* dtp = tmp.up(target_positions, (size_t)2 * nt);
    const double* dxh = tmp.up(x_hat, (size_t)s.m);
    const double* dinf = inflow ? tmp.up(inflow, (size_t)2 * n) : nullptr;
    double* df = tmp.zeros<double>((size_t)2 * nt);
    double* dj = tmp.zeros<double>((size_t)4 * nt);
    RomScratch w;
    w.ensure(s, nt, 1);
    unsigned long long pairs = 0;
    try {
      pairs = rom_hyperpair(ctx, s, nullptr, nullptr, nullptr, 1, s.m, dxh, nullptr, nullptr, dtp, nullptr, delta,
                            form, dinf, n, w, df, dj, true);
      check_device_status(ctx);
      PTROM_CUDA(cudaMemcpy(f, df, 16 * nt, cudaMemcpyDeviceToHost));
      std::vector<double> jh((size_t)4 * nt);
      PTROM_CUDA(cudaMemcpy(jh.data(), dj, jh.size() * 8, cudaMemcpyDeviceToHost));
      for (long long t = 0; t < nt; ++t)
        for (int k = 0; k < 4; ++k) jac[k * nt + t] = jh[4 * t + k];
      if (cluster_positions) {
        // de-interleave (x, y) pairs into the reference's [x..., y...]
        PTROM_CUDA(cudaMemcpy2D(cluster_positions, 8, w.cxy, 16, 8, s.n_c, cudaMemcpyDeviceToHost));
        PTROM_CUDA(cudaMemcpy2D(cluster_positions + s.n_c, 8, reinterpret_cast<const double*>(w.cxy) + 1, 16, 8,
                                s.n_c, cudaMemcpyDeviceToHost));
      }
      if (direct_positions) {
        PTROM_CUDA(cudaMemcpy2D(direct_positions, 8, w.dxy, 16, 8, s.u, cudaMemcpyDeviceToHost));
        PTROM_CUDA(cudaMemcpy2D(direct_positions + s.u, 8, reinterpret_cast<const double*>(w.dxy) + 1, 16, 8, s.u,
                                cudaMemcpyDeviceToHost));
      }
    } catch (...) {
      w.release();
      throw;
    }
    w.release();
    if (n_pair_evals) *n_pair_evals = pairs;
  });
}

// rom.hpp:404-412: reassign (mutates the surrogate) + GnatSolver::simulate.
int ptrom_ptrom_simulate_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const ptrom_gnat_op* op, ptrom_surrogate* sur,
                             int64_t n, const double* gamma, double delta, int form, const double* inflow, double dt,
                             int64_t n_steps, double tol, int max_iters, double step_length, double* x_hat,
                             int* iterations, uint8_t* converged, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    if (!basis || !op || !sur) config_fail("null basis / operator / surrogate");
    if (!(dt > 0)) config_fail("time step must be positive");
    if (n_steps < 0) config_fail("negative step count");
    if (!(tol > 0)) config_fail("ROM tolerance must be positive");
    if (max_iters < 1) config_fail("ROM max_iters must be >= 1");
    if (!(step_length > 0)) config_fail("ROM step length must be positive");
    if (n != basis->b.n) config_fail("GnatSolver: basis dimension does not match particle count");
    if (sur->target_ids != op->ids) config_fail("GnatSolver: surrogate targets must equal the sampled particle ids");
    check_finite(gamma, (size_t)n, "non-finite circulation");
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    if (inflow) check_finite(inflow, (size_t)2 * n, "non-finite inflow");
    DevAllocs tmp;
    const double* dg = tmp.up(gamma, (size_t)n);
    const double* dinf = inflow ? tmp.up(inflow, (size_t)2 * n) : nullptr;
    rom_reassign_exact(ctx, sur->s, basis->b, dg);
    const int m = basis->b.m;
    double* dxh = tmp.zeros<double>((size_t)m * std::max<int64_t>(n_steps, 1));
    int* dit = tmp.zeros<int>((size_t)std::max<int64_t>(n_steps, 1));
    unsigned char* dcv = tmp.zeros<unsigned char>((size_t)std::max<int64_t>(n_steps, 1));
    const unsigned long long pairs = rom_gnat_simulate(ctx, sur->s, op->g, nullptr, 1, nullptr, delta, form, dinf, n,
                                                       dt, n_steps, tol, max_iters, step_length, dxh, dit, dcv);
    // x_hat: M x n_steps column-major (RomTrajectory::x_hat, rom.hpp:31)
    if (n_steps > 0) {
      PTROM_CUDA(cudaMemcpy(x_hat, dxh, (size_t)m * n_steps * 8, cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(iterations, dit, (size_t)n_steps * 4, cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(converged, dcv, (size_t)n_steps, cudaMemcpyDeviceToHost));
    }
    if (n_pair_evals) *n_pair_evals = pairs;
  });
}

// Batched online queries for an affine circulation Γ(μ) = Γa + μ Γb over
// n_inst parameters (SURVEY.md §8b ptrom_gnat_simulate_batch). The
// surrogate's topology is shared; its tables are not modified. Outputs:
// x_hat [n_inst][n_steps][M], iterations / converged [n_inst][n_steps].
int ptrom_ptrom_simulate_batch_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const ptrom_gnat_op* op,
                                   const ptrom_surrogate* sur, int64_t n, const double* gamma_a,
                                   const double* gamma_b, int64_t n_inst, const double* mu, int64_t batch,
                                   double delta, int form, const double* inflow, double dt, int64_t n_steps,
                                   double tol, int max_iters, double step_length, double* x_hat, int* iterations,
                                   uint8_t* converged, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_batch(basis, op, sur, n, gamma_a, gamma_b, n_inst, mu, dt, n_steps, tol, max_iters, step_length);
    const unsigned long long pairs =
        batch_march(ctx, basis->b, op->g, sur->s, n, gamma_a, gamma_b, n_inst, mu, batch, delta, form, inflow, dt,
                    n_steps, tol, max_iters, step_length, x_hat, iterations, converged);
    if (n_pair_evals) *n_pair_evals = pairs;
  });
}

// ------------------------------------------------------ offline producers --
int ptrom_greedy_sample_f64(ptrom_ctx* ctx, int64_t n_dofs, int64_t n_r, const double* phi_r, int64_t n_target,
                            int64_t n_preseed, const int64_t* preseed, int64_t* out_ids) {
  return guarded(ctx, [&] {
    std::vector<long long> pre(preseed, preseed + n_preseed);
    const std::vector<long long> ids = offline_greedy_sample(ctx, n_dofs, (int)n_r, phi_r, n_target, pre);
    std::copy(ids.begin(), ids.end(), out_ids);
  });
}

int ptrom_build_gnat_operator_f64(ptrom_ctx* ctx, int64_t n_dofs, int64_t m_r, const double* phi_r, int64_t n_s,
                                  const int64_t* ids, double* A) {
  return guarded(ctx, [&] {
    const std::vector<double> a = offline_gnat_operator(ctx, n_dofs, (int)m_r, phi_r, std::vector<long long>(ids, ids + n_s));
    std::copy(a.begin(), a.end(), A);
  });
}

int ptrom_cluster_pod_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const double* gamma, int64_t leaf_capacity,
                          int crit_kind, double crit_value, int64_t n_targets, const int64_t* targets,
                          ptrom_surrogate** out) {
  return guarded(ctx, [&] {
    if (!basis) config_fail("null basis");
    if (leaf_capacity < 1) config_fail("build_tree: leaf_capacity must be >= 1");
    if (crit_kind == PTROM_CRIT_BARNES_HUT ? !(crit_value >= 0) : !(crit_value >= 0))
      config_fail(crit_kind == PTROM_CRIT_BARNES_HUT ? "opening ratio must be >= 0"
                                                     : "neighborhood width factor must be >= 0");
    const long long n = basis->b.n;
    check_finite(gamma, (size_t)n, "cluster_pod");
    auto* h = new ptrom_surrogate;
    h->device = ctx->device;
    try {
      const double* dg = h->mem.up(gamma, (size_t)n);
      std::vector<long long> t(targets, targets + n_targets);
      offline_cluster_pod(ctx, basis->b, dg, leaf_capacity, crit_kind, crit_value, t, h->s, h->mem.p,
                          h->cluster_node_ids);
      h->target_ids = t;
      PTROM_CUDA(cudaMemcpy(&h->n_membership, h->s.mem_off + h->s.n_c, 8, cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(&h->n_cluster_list, h->s.cl_off + h->s.n_t, 8, cudaMemcpyDeviceToHost));
      PTROM_CUDA(cudaMemcpy(&h->n_direct_list, h->s.d_off + h->s.n_t, 8, cudaMemcpyDeviceToHost));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int ptrom_surrogate_sizes(const ptrom_surrogate* sur, int64_t* sizes) {
  if (!sur) return PTROM_CONFIG_ERROR;
  sizes[0] = sur->s.n_c;
  sizes[1] = sur->s.u;
  sizes[2] = sur->s.n_t;
  sizes[3] = sur->n_membership;
  sizes[4] = sur->n_cluster_list;
  sizes[5] = sur->n_direct_list;
  return PTROM_OK;
}

int ptrom_surrogate_export_lists(ptrom_ctx* ctx, const ptrom_surrogate* sur, int32_t* cluster_node_ids,
                                 int64_t* mem_off, int64_t* mem_ids, int64_t* cl_off, int64_t* cl_list,
                                 int64_t* direct_ids, int64_t* d_off, int64_t* d_list, double* direct_phi,
                                 double* direct_x0) {
  return guarded(ctx, [&] {
    const DSurrogate& s = sur->s;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) PTROM_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    if (cluster_node_ids) std::copy(sur->cluster_node_ids.begin(), sur->cluster_node_ids.end(), cluster_node_ids);
    d2h(mem_off, s.mem_off, (size_t)(s.n_c + 1) * 8);
    d2h(mem_ids, s.mem_ids, (size_t)sur->n_membership * 8);
    d2h(cl_off, s.cl_off, (size_t)(s.n_t + 1) * 8);
    d2h(d_off, s.d_off, (size_t)(s.n_t + 1) * 8);
    d2h(direct_ids, s.direct_ids, (size_t)s.u * 8);
    d2h(direct_phi, s.direct_phi, (size_t)2 * s.u * s.m * 8);
    d2h(direct_x0, s.direct_x0, (size_t)2 * s.u * 8);
    std::vector<int> tmp;
    auto widen = [&](int64_t* dst, const int* src, size_t count) {
      if (!dst || !count) return;
      tmp.resize(count);
      PTROM_CUDA(cudaMemcpy(tmp.data(), src, count * 4, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < count; ++i) dst[i] = tmp[i];
    };
    widen(cl_list, s.cl_list, (size_t)sur->n_cluster_list);
    widen(d_list, s.d_list, (size_t)sur->n_direct_list);
  });
}

}  // extern "C"

// ------------------------------------------------------- multi-GPU (§8e) --
namespace {

// Root's sizes and scalars, broadcast first so every rank can allocate its
// copies of the shared tables.
struct ShardHeader {
  long long n, n_inst, batch, n_steps;
  long long n_c, u, n_t, n_mem, n_cl, n_dl, n_s, max_members;
  double delta, dt, tol, step;
  int m, m_r, mp, form, max_iters, has_inflow, has_order, ok;
  char why[256];
};

// Device arrays of the online engine's shared tables (the row-major basis,
// the GNAT operator with its gathered rows, the surrogate): (member, bytes).
std::vector<std::pair<void**, size_t>> shared_fields(DBasis& b, DGnat& g, DSurrogate& s, const ShardHeader& h) {
  const size_t nc = (size_t)h.n_c, u = (size_t)h.u, nt = (size_t)h.n_t, m = (size_t)h.m;
  std::vector<std::pair<void**, size_t>> f = {
      {reinterpret_cast<void**>(&b.rm), (size_t)h.n * 2 * (m + 1) * 8},
      {reinterpret_cast<void**>(&g.ids), (size_t)h.n_s * 8},
      {reinterpret_cast<void**>(&g.A), (size_t)32 * 2 * h.n_s * 8},
      {reinterpret_cast<void**>(&g.phi_bar), (size_t)2 * h.n_s * h.mp * 8},
      {reinterpret_cast<void**>(&g.x0_bar), (size_t)2 * h.n_s * 8},
      {reinterpret_cast<void**>(&s.phi_tilde), 2 * nc * m * 8},
      {reinterpret_cast<void**>(&s.x0_tilde), 2 * nc * 8},
      {reinterpret_cast<void**>(&s.gamma_tilde), nc * 8},
      {reinterpret_cast<void**>(&s.zero_gamma), nc},
      {reinterpret_cast<void**>(&s.mem_off), (nc + 1) * 8},
      {reinterpret_cast<void**>(&s.mem_ids), (size_t)h.n_mem * 8},
      {reinterpret_cast<void**>(&s.target_ids), nt * 8},
      {reinterpret_cast<void**>(&s.cl_off), (nt + 1) * 8},
      {reinterpret_cast<void**>(&s.cl_list), (size_t)h.n_cl * 4},
      {reinterpret_cast<void**>(&s.d_off), (nt + 1) * 8},
      {reinterpret_cast<void**>(&s.d_list), (size_t)h.n_dl * 4},
      {reinterpret_cast<void**>(&s.direct_ids), u * 8},
      {reinterpret_cast<void**>(&s.direct_phi), 2 * u * m * 8},
      {reinterpret_cast<void**>(&s.direct_x0), 2 * u * 8},
      {reinterpret_cast<void**>(&s.direct_gamma), u * 8},
  };
  if (h.has_order) f.push_back({reinterpret_cast<void**>(&s.t_order), nt * 4});
  return f;
}

}  // namespace

extern "C" {

int ptrom_ptrom_simulate_batch_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int root, const ptrom_basis* basis,
                                           const ptrom_gnat_op* op, const ptrom_surrogate* sur, int64_t n,
                                           const double* gamma_a, const double* gamma_b, int64_t n_inst,
                                           const double* mu, int64_t batch, double delta, int form,
                                           const double* inflow, double dt, int64_t n_steps, double tol,
                                           int max_iters, double step_length, double* x_hat, int* iterations,
                                           uint8_t* converged, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    if (!comm) config_fail("null communicator");
    if (comm->device != ctx->device) config_fail("communicator and context are on different devices");
    if (root < 0 || root >= comm->world) config_fail("sharded batch: root outside [0, world)");
    const bool is_root = comm->rank == root;
    ShardHeader h{};
    if (is_root) {
      h.ok = 1;
      try {
        validate_batch(basis, op, sur, n, gamma_a, gamma_b, n_inst, mu, dt, n_steps, tol, max_iters, step_length);
        if (inflow) check_finite(inflow, (size_t)2 * n, "non-finite inflow");
      } catch (const status_error& e) {  // every rank must learn it before the collectives below
        h.ok = 0;
        std::strncpy(h.why, e.what(), sizeof(h.why) - 1);
      }
      if (h.ok) {
        const DSurrogate& s = sur->s;
        h.n = n;
        h.n_inst = n_inst;
        h.batch = batch;
        h.n_steps = n_steps;
        h.n_c = s.n_c;
        h.u = s.u;
        h.n_t = s.n_t;
        h.n_mem = sur->n_membership;
        h.n_cl = sur->n_cluster_list;
        h.n_dl = sur->n_direct_list;
        h.n_s = op->g.n_s;
        h.max_members = s.max_members;
        h.delta = delta;
        h.dt = dt;
        h.tol = tol;
        h.step = step_length;
        h.m = basis->b.m;
        h.m_r = op->g.m_r;
        h.mp = op->g.mp;
        h.form = form;
        h.max_iters = max_iters;
        h.has_inflow = inflow ? 1 : 0;
        h.has_order = s.t_order ? 1 : 0;
      }
    }
    comm_bcast_host(ctx, comm, &h, sizeof(h), root);
    if (!h.ok) config_fail(std::string("sharded batch: root rejected the arguments: ") + h.why);
    // host parameters (Γa, Γb, μ, inflow) in one broadcast
    const size_t np = (size_t)(2 * h.n + h.n_inst + (h.has_inflow ? 2 * h.n : 0));
    std::vector<double> par(np);
    if (is_root) {
      std::copy(gamma_a, gamma_a + h.n, par.begin());
      std::copy(gamma_b, gamma_b + h.n, par.begin() + h.n);
      std::copy(mu, mu + h.n_inst, par.begin() + 2 * h.n);
      if (h.has_inflow) std::copy(inflow, inflow + 2 * h.n, par.begin() + 2 * h.n + h.n_inst);
    }
    comm_bcast_host(ctx, comm, par.data(), np * 8, root);
    // shared device tables: root's own, a broadcast copy elsewhere
    DBasis b;
    DGnat g;
    DSurrogate s;
    DevAllocs copies;
    if (is_root) {
      b = basis->b;
      g = op->g;
      s = sur->s;
    } else {
      b.n = h.n;
      b.m = h.m;
      g.n_s = h.n_s;
      g.m_r = h.m_r;
      g.m = h.m;
      g.mp = h.mp;
      s.m = h.m;
      s.n_c = h.n_c;
      s.u = h.u;
      s.n_t = h.n_t;
      s.max_members = h.max_members;
      for (auto& [ptr, bytes] : shared_fields(b, g, s, h)) *ptr = copies.up<char>(nullptr, bytes);
    }
    std::vector<std::pair<void*, size_t>> bufs;
    for (auto& [ptr, bytes] : shared_fields(b, g, s, h)) bufs.push_back({*ptr, bytes});
    comm_bcast_many(ctx, comm, bufs, root);
    // this rank's instances, no communication during the march
    long long lo, hi;
    shard_bounds(h.n_inst, comm->rank, comm->world, lo, hi);
    const long long cnt = hi - lo, steps = h.n_steps, m = h.m;
    std::vector<double> xl((size_t)std::max<long long>(cnt * steps * m, 1));
    std::vector<int> il((size_t)std::max<long long>(cnt * steps, 1));
    std::vector<uint8_t> cl((size_t)std::max<long long>(cnt * steps, 1));
    unsigned long long pairs = 0;
    if (cnt > 0)
      pairs = batch_march(ctx, b, g, s, h.n, par.data(), par.data() + h.n, cnt, par.data() + 2 * h.n + lo, h.batch,
                          h.delta, h.form, h.has_inflow ? par.data() + 2 * h.n + h.n_inst : nullptr, h.dt, steps,
                          h.tol, h.max_iters, h.step, xl.data(), il.data(), cl.data());
    // gather in instance order: one record per instance (x̂, iterations, converged)
    long long max_cnt = 0;
    for (int r = 0; r < comm->world; ++r) {
      long long a, z;
      shard_bounds(h.n_inst, r, comm->world, a, z);
      max_cnt = std::max(max_cnt, z - a);
    }
    const size_t rec = (size_t)steps * (m * 8 + 4 + 1);
    std::vector<char> send((size_t)std::max<long long>(max_cnt, 1) * std::max<size_t>(rec, 1));
    for (long long i = 0; i < cnt; ++i) {
      char* p = send.data() + i * rec;
      std::memcpy(p, xl.data() + i * steps * m, steps * m * 8);
      std::memcpy(p + steps * m * 8, il.data() + i * steps, steps * 4);
      std::memcpy(p + steps * m * 8 + steps * 4, cl.data() + i * steps, steps);
    }
    std::vector<char> all(send.size() * comm->world);
    comm_allgather_host(ctx, comm, send.data(), all.data(), send.size());
    for (int r = 0; r < comm->world; ++r) {
      long long a, z;
      shard_bounds(h.n_inst, r, comm->world, a, z);
      for (long long i = a; i < z; ++i) {
        const char* p = all.data() + (size_t)r * send.size() + (i - a) * rec;
        if (x_hat) std::memcpy(x_hat + i * steps * m, p, steps * m * 8);
        if (iterations) std::memcpy(iterations + i * steps, p + steps * m * 8, steps * 4);
        if (converged) std::memcpy(converged + i * steps, p + steps * m * 8 + steps * 4, steps);
      }
    }
    if (n_pair_evals) *n_pair_evals = pairs;
  });
}

}  // extern "C"
