// offline.cu — PTROM offline producers needed to run the online path at
// scale without any CPU reference code:
//   greedy_sample        reduction.hpp:93-168   (device scoring + selection)
//   build_gnat_operator  reduction.hpp:182-220  (A = pinv(P Φ_r))
//   weighted_pod_space + build_weighted_pod_tree + cluster_pod
//                        reduction.hpp:74-77, 236-385 (device quadtree + traversal)
//
// Small dense factorizations (the gappy least-squares fits of greedy
// sampling, at most 2·n_samples x 31, and the n_d x m_r pseudo-inverse) run as
// a column-pivoted Householder QR on the host: they are O(rows · m_r²) index-
// sized problems next to the O(N · m_r) device scoring passes.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "ops.cuh"
#include "rom.cuh"
#include "tree.cuh"

namespace ptrom {

void tree_collect(ptrom_ctx* ctx, Tree& t, int crit_kind, double crit_value, const std::vector<long long>& targets,
                  std::vector<long long>& c_off, std::vector<int>& clusters, std::vector<long long>& d_off,
                  std::vector<long long>& direct);
void rom_reassign_exact(ptrom_ctx* ctx, DSurrogate& s, const DBasis& b, const double* d_gamma);

namespace {

// ---------------------------------------------------------- host dense LA --
// Column-pivoted Householder QR of a rows x cols column-major matrix.
struct PivotedQR {
  long long rows, cols;
  std::vector<double> a;     // R in the upper triangle, reflector tails below
  std::vector<double> taus;  // reflector scalars
  std::vector<int> piv;      // column j of R is input column piv[j]
  int rank = 0;

  PivotedQR(long long r, long long c, std::vector<double> m) : rows(r), cols(c), a(std::move(m)) {
    const long long k = std::min(rows, cols);
    piv.resize(cols);
    std::iota(piv.begin(), piv.end(), 0);
    taus.assign(k, 0.0);
    std::vector<double> cn(cols);
    for (long long j = 0; j < cols; ++j) {
      double s = 0;
      for (long long i = 0; i < rows; ++i) s += a[i + j * rows] * a[i + j * rows];
      cn[j] = s;
    }
    double first = 0;
    for (long long j = 0; j < k; ++j) {
      long long p = j;
      for (long long c2 = j + 1; c2 < cols; ++c2)
        if (cn[c2] > cn[p]) p = c2;
      if (p != j) {
        for (long long i = 0; i < rows; ++i) std::swap(a[i + j * rows], a[i + p * rows]);
        std::swap(cn[j], cn[p]);
        std::swap(piv[j], piv[p]);
      }
      double* col = &a[j * rows];
      double tail = 0;
      for (long long i = j + 1; i < rows; ++i) tail += col[i] * col[i];
      const double x0 = col[j];
      double beta = x0, tau = 0;
      if (tail > 0) {
        beta = -std::copysign(std::sqrt(x0 * x0 + tail), x0);
        tau = (beta - x0) / beta;
        const double scale = 1.0 / (x0 - beta);
        for (long long i = j + 1; i < rows; ++i) col[i] *= scale;
      }
      col[j] = beta;
      taus[j] = tau;
      for (long long c2 = j + 1; c2 < cols; ++c2) {
        double* cc = &a[c2 * rows];
        double w = cc[j];
        for (long long i = j + 1; i < rows; ++i) w += col[i] * cc[i];
        w *= tau;
        cc[j] -= w;
        for (long long i = j + 1; i < rows; ++i) cc[i] -= w * col[i];
        double s = 0;
        for (long long i = j + 1; i < rows; ++i) s += cc[i] * cc[i];
        cn[c2] = s;
      }
      if (j == 0) first = std::fabs(beta);
      if (std::fabs(beta) > 2.220446049250313e-16 * (double)k * first) rank = (int)j + 1;
    }
  }
  // y <- Q^T y
  void apply_qt(double* y) const {
    for (size_t j = 0; j < taus.size(); ++j) {
      if (taus[j] == 0) continue;
      const double* v = &a[j * rows];
      double w = y[j];
      for (long long i = (long long)j + 1; i < rows; ++i) w += v[i] * y[i];
      w *= taus[j];
      y[j] -= w;
      for (long long i = (long long)j + 1; i < rows; ++i) y[i] -= w * v[i];
    }
  }
  // basic least-squares solution (free variables zero)
  std::vector<double> solve(std::vector<double> b) const {
    apply_qt(b.data());
    std::vector<double> z(cols, 0.0), x(cols, 0.0);
    for (int i = rank - 1; i >= 0; --i) {
      double s = b[i];
      for (int j = i + 1; j < rank; ++j) s -= a[i + (long long)j * rows] * z[j];
      z[i] = s / a[i + (long long)i * rows];
    }
    for (long long j = 0; j < cols; ++j) x[piv[j]] = z[j];
    return x;
  }
};

// -------------------------------------------------------- greedy kernels ---
// work[:, q] = Φ_r[:, nb+q] − Φ_r[:, :nb]·coef[:, q]  (reduction.hpp:144)
__global__ void residual_columns_kernel(long long nd, int nb, int nci, const double* __restrict__ phi_r,
                                        const double* __restrict__ coef, double* __restrict__ work) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= nd * nci) return;
  const long long r = idx % nd;
  const int q = (int)(idx / nd);
  double s = 0.0;
  for (int c = 0; c < nb; ++c) s = __dadd_rn(s, __dmul_rn(phi_r[r + c * nd], coef[c + (long long)q * nb]));
  work[r + (long long)q * nd] = __dsub_rn(phi_r[r + (long long)(nb + q) * nd], s);
}

// reduction.hpp:150-158 scores (summed in the reference order); picked → -1.
__global__ void scores_kernel(long long n, int nci, const double* __restrict__ work,
                              const unsigned char* __restrict__ picked, double* __restrict__ score,
                              int* __restrict__ idx) {
  const long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= n) return;
  double s = 0.0;
  if (!picked[l]) {
    for (int q = 0; q < nci; ++q) {
      const double a = work[l + 2 * n * q], b = work[l + n + 2 * n * q];
      s = __dadd_rn(s, __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
    }
  } else {
    s = -1.0;
  }
  score[l] = s;
  idx[l] = (int)l;
}

__global__ void mark_kernel(int k, const int* __restrict__ ids, unsigned char* __restrict__ picked) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) picked[ids[i]] = 1;
}

// W = Φ σ in ascending-mode order (reduction.hpp:74-77)
__global__ void weighted_space_kernel(DBasis b, double* __restrict__ w) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= 2 * b.n) return;
  double s = 0.0;
  for (int j = 0; j < b.m; ++j) s = __dadd_rn(s, __dmul_rn(b.phi[r + j * 2 * b.n], b.sv[j]));
  w[r] = s;
}

__global__ void gather_members_kernel(long long nc, const long long* __restrict__ mem_off,
                                      const int* __restrict__ node_begin, const int* __restrict__ perm,
                                      long long* __restrict__ mem_ids) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const long long o = mem_off[c];
  const int b = node_begin[c];
  for (long long k = 0; k < mem_off[c + 1] - o; ++k) mem_ids[o + k] = perm[b + k];
}

__global__ void gather_direct_kernel(long long u, const long long* __restrict__ ids, DBasis b,
                                     const double* __restrict__ gamma, double* __restrict__ dphi,
                                     double* __restrict__ dx0, double* __restrict__ dg) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= u) return;
  const long long p = ids[k];
  for (int j = 0; j < b.m; ++j) {
    dphi[k + j * 2 * u] = b.phi[p + j * 2 * b.n];
    dphi[k + u + j * 2 * u] = b.phi[p + b.n + j * 2 * b.n];
  }
  dx0[k] = b.x_ref[p];
  dx0[k + u] = b.x_ref[p + b.n];
  dg[k] = gamma[p];
}

}  // namespace

// reduction.hpp:93-168 greedy_sample; phi_r host, column-major n_dofs x n_r.
std::vector<long long> offline_greedy_sample(ptrom_ctx* ctx, long long n_dofs, int n_r, const double* phi_r,
                                             long long n_target, const std::vector<long long>& preseed) {
  if (n_dofs % 2 != 0) config_fail("state dimension must be even");
  const long long n = n_dofs / 2;
  if (n_r < 1) config_fail("greedy_sample: empty residual basis");
  for (long long i = 0; i < n_dofs * n_r; ++i)
    if (!std::isfinite(phi_r[i])) config_fail("greedy_sample: non-finite residual basis");
  if (n_target < 1 || n_target > n)
    config_fail("greedy_sample: target count " + std::to_string(n_target) + " outside [1, " + std::to_string(n) + "]");
  cudaStream_t s = ctx->stream;
  std::vector<unsigned char> picked_h(n, 0);
  std::vector<long long> chosen;
  for (long long p : preseed) {
    if (p < 0 || p >= n) config_fail("greedy_sample: preseed id out of range");
    if (picked_h[p]) config_fail("greedy_sample: duplicate preseed id");
    picked_h[p] = 1;
    chosen.push_back(p);
  }
  if ((long long)chosen.size() > n_target) config_fail("greedy_sample: preseed larger than target count");
  const long long n_a = n_target - (long long)chosen.size();
  if (n_a > 0) {
    double *d_phi, *d_work, *d_coef, *d_score, *d_score_s;
    int *d_idx, *d_idx_s;
    unsigned char* d_picked;
    PTROM_CUDA(cudaMallocAsync(&d_phi, n_dofs * n_r * 8, s));
    PTROM_CUDA(cudaMemcpyAsync(d_phi, phi_r, n_dofs * n_r * 8, cudaMemcpyHostToDevice, s));
    const long long n_c = std::min<long long>(n_r, 2 * n_target);
    const long long n_it = std::min(n_c, n_a);
    const long long max_ci = n_c / n_it + 1;
    PTROM_CUDA(cudaMallocAsync(&d_work, n_dofs * max_ci * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_coef, (size_t)n_r * max_ci * 8 + 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_score, n * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_score_s, n * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_idx, n * 4, s));
    PTROM_CUDA(cudaMallocAsync(&d_idx_s, n * 4, s));
    PTROM_CUDA(cudaMallocAsync(&d_picked, n, s));
    PTROM_CUDA(cudaMemcpyAsync(d_picked, picked_h.data(), n, cudaMemcpyHostToDevice, s));
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, d_score, d_score_s, d_idx, d_idx_s, (int)n, 0, 64, s);
    void* d_tmp;
    PTROM_CUDA(cudaMallocAsync(&d_tmp, sort_bytes + 16, s));
    long long nb = 0;
    for (long long it = 1; it <= n_it; ++it) {
      const long long n_ci = n_c / n_it + (it <= n_c % n_it ? 1 : 0);
      const long long n_ai = n_a / n_it + (it <= n_a % n_it ? 1 : 0);
      if (it == 1) {
        PTROM_CUDA(cudaMemcpyAsync(d_work, d_phi, n_dofs * n_ci * 8, cudaMemcpyDeviceToDevice, s));
      } else {
        // gappy fit on the rows sampled so far (reduction.hpp:129-143)
        std::vector<long long> ids = chosen;
        std::sort(ids.begin(), ids.end());
        const long long rows = 2 * (long long)ids.size();
        std::vector<double> sb(rows * nb), rhs(rows * n_ci);
        for (long long k = 0; k < rows; ++k) {
          const long long r = k < (long long)ids.size() ? ids[k] : ids[k - ids.size()] + n;
          for (long long c = 0; c < nb; ++c) sb[k + c * rows] = phi_r[r + c * n_dofs];
          for (long long q = 0; q < n_ci; ++q) rhs[k + q * rows] = phi_r[r + (nb + q) * n_dofs];
        }
        PivotedQR qr(rows, nb, std::move(sb));
        std::vector<double> coef(nb * n_ci);
        for (long long q = 0; q < n_ci; ++q) {
          std::vector<double> col(rhs.begin() + q * rows, rhs.begin() + (q + 1) * rows);
          const std::vector<double> x = qr.solve(std::move(col));
          for (long long c = 0; c < nb; ++c) coef[c + q * nb] = x[c];
        }
        PTROM_CUDA(cudaMemcpyAsync(d_coef, coef.data(), coef.size() * 8, cudaMemcpyHostToDevice, s));
        residual_columns_kernel<<<(unsigned)((n_dofs * n_ci + 255) / 256), 256, 0, s>>>(n_dofs, (int)nb, (int)n_ci,
                                                                                       d_phi, d_coef, d_work);
      }
      scores_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, (int)n_ci, d_work, d_picked, d_score, d_idx);
      PTROM_LAUNCH_CHECK();
      // highest score first, lowest index among equal scores (stable sort)
      PTROM_CUDA(cub::DeviceRadixSort::SortPairsDescending(d_tmp, sort_bytes, d_score, d_score_s, d_idx, d_idx_s,
                                                           (int)n, 0, 64, s));
      std::vector<int> top(n_ai);
      PTROM_CUDA(cudaMemcpyAsync(top.data(), d_idx_s, n_ai * 4, cudaMemcpyDeviceToHost, s));
      mark_kernel<<<(unsigned)((n_ai + 255) / 256), 256, 0, s>>>((int)n_ai, d_idx_s, d_picked);
      PTROM_CUDA(cudaStreamSynchronize(s));
      for (int p : top) chosen.push_back(p);
      nb += n_ci;
    }
    void* fr[] = {d_phi, d_work, d_coef, d_score, d_score_s, d_idx, d_idx_s, d_picked, d_tmp};
    for (void* p : fr) cudaFreeAsync(p, s);
    PTROM_CUDA(cudaStreamSynchronize(s));
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// reduction.hpp:182-220: A = pinv(rows of Φ_r at the sampled dofs).
std::vector<double> offline_gnat_operator(long long n_dofs, int m_r, const double* phi_r,
                                          const std::vector<long long>& ids_in) {
  if (n_dofs % 2 != 0) config_fail("state dimension must be even");
  const long long n = n_dofs / 2;
  if (ids_in.empty()) config_fail("build_gnat_operator: no sample ids");
  std::vector<long long> ids = ids_in;
  std::sort(ids.begin(), ids.end());
  if (std::adjacent_find(ids.begin(), ids.end()) != ids.end()) config_fail("build_gnat_operator: duplicate sample ids");
  if (ids.front() < 0 || ids.back() >= n) config_fail("build_gnat_operator: sample id out of range");
  const long long nd = 2 * (long long)ids.size();
  if (nd < m_r)
    config_fail("build_gnat_operator: " + std::to_string(nd) + " sampled dofs cannot support " + std::to_string(m_r) +
                " residual modes (need 2 * samples >= modes)");
  std::vector<double> sm(nd * m_r);
  for (long long k = 0; k < nd; ++k) {
    const long long r = k < (long long)ids.size() ? ids[k] : ids[k - ids.size()] + n;
    for (int c = 0; c < m_r; ++c) sm[k + c * nd] = phi_r[r + c * n_dofs];
  }
  PivotedQR qr(nd, m_r, std::move(sm));
  if (qr.rank < m_r) {
    std::string cols;
    for (int k = qr.rank; k < m_r; ++k) cols += (cols.empty() ? "" : ", ") + std::to_string(qr.piv[k]);
    numerical_fail("build_gnat_operator: sampled residual basis has rank " + std::to_string(qr.rank) + " < " +
                   std::to_string(m_r) + "; dependent columns: " + cols);
  }
  // pinv = P R^{-1} Q1^T: form Q1 (nd x m_r) by applying the reflectors to the
  // first m_r identity columns, then back-substitute R on its rows.
  std::vector<double> q1((size_t)nd * m_r, 0.0);
  for (int j = 0; j < m_r; ++j) {
    double* col = &q1[(size_t)j * nd];
    col[j] = 1.0;
    for (int r = m_r - 1; r >= 0; --r) {  // Q e_j = H_0 ... H_{m_r-1} e_j
      if (qr.taus[r] == 0) continue;
      const double* v = &qr.a[(size_t)r * nd];
      double w = col[r];
      for (long long i = r + 1; i < nd; ++i) w += v[i] * col[i];
      w *= qr.taus[r];
      col[r] -= w;
      for (long long i = r + 1; i < nd; ++i) col[i] -= w * v[i];
    }
  }
  std::vector<double> A((size_t)m_r * nd);
  std::vector<double> z(m_r);
  for (long long k = 0; k < nd; ++k) {  // column k of pinv: R^{-1} (row k of Q1)^T, then P
    for (int i = m_r - 1; i >= 0; --i) {
      double s2 = q1[k + (size_t)i * nd];
      for (int j = i + 1; j < m_r; ++j) s2 -= qr.a[i + (size_t)j * nd] * z[j];
      z[i] = s2 / qr.a[i + (size_t)i * nd];
    }
    for (int j = 0; j < m_r; ++j) A[qr.piv[j] + (size_t)k * m_r] = z[j];
  }
  return A;
}

// build_weighted_pod_tree (leaf_capacity) + cluster_pod for `targets`, all
// tables on the device (reduction.hpp:236-385). Fills a DSurrogate whose
// arrays are owned by `allocs`.
void offline_cluster_pod(ptrom_ctx* ctx, const DBasis& b, const double* d_gamma, long long leaf_cap, int crit_kind,
                         double crit_value, const std::vector<long long>& targets, DSurrogate& s,
                         std::vector<void*>& allocs, std::vector<int>& cluster_node_ids) {
  cudaStream_t st = ctx->stream;
  auto dalloc = [&](size_t bytes) {
    void* p;
    PTROM_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    allocs.push_back(p);
    return p;
  };
  const long long n = b.n;
  for (long long t : targets)
    if (t < 0 || t >= n) config_fail("cluster_pod: target id out of range");
  if (targets.empty()) config_fail("cluster_pod: no targets");
  if (!b.sv) config_fail("cluster_pod: the basis needs singular values (weighted POD space)");
  // weighted POD space and its quadtree
  double* w;
  PTROM_CUDA(cudaMallocAsync(&w, 2 * n * 8, st));
  weighted_space_kernel<<<(unsigned)((2 * n + 255) / 256), 256, 0, st>>>(b, w);
  PTROM_LAUNCH_CHECK();
  Tree tree;
  tree_build(ctx, tree, n, w, w + n, d_gamma, leaf_cap, ctx->tree_seq_max);
  std::vector<long long> c_off, d_off, direct;
  std::vector<int> clusters;
  tree_collect(ctx, tree, crit_kind, crit_value, targets, c_off, clusters, d_off, direct);
  const long long nt = (long long)targets.size();
  // first-appearance dedupe by node id (reduction.hpp:325-331)
  std::vector<int> node_to_cluster(tree.nodes.count, -1);
  cluster_node_ids.clear();
  std::vector<int> cl_list(clusters.size());
  for (size_t k = 0; k < clusters.size(); ++k) {
    int& ix = node_to_cluster[clusters[k]];
    if (ix < 0) {
      ix = (int)cluster_node_ids.size();
      cluster_node_ids.push_back(clusters[k]);
    }
    cl_list[k] = ix;
  }
  // sorted near-field union and local indices (reduction.hpp:338-349)
  std::vector<long long> uni = direct;
  std::sort(uni.begin(), uni.end());
  uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
  std::vector<int> d_list(direct.size());
  for (size_t k = 0; k < direct.size(); ++k)
    d_list[k] = (int)(std::lower_bound(uni.begin(), uni.end(), direct[k]) - uni.begin());
  const long long nc = (long long)cluster_node_ids.size(), u = (long long)uni.size();
  // membership: perm slice of each cluster node, sorted ascending
  std::vector<int> nb(tree.nodes.count), ne(tree.nodes.count);
  PTROM_CUDA(cudaMemcpyAsync(nb.data(), tree.nodes.begin, nb.size() * 4, cudaMemcpyDeviceToHost, st));
  PTROM_CUDA(cudaMemcpyAsync(ne.data(), tree.nodes.end, ne.size() * 4, cudaMemcpyDeviceToHost, st));
  PTROM_CUDA(cudaStreamSynchronize(st));
  std::vector<long long> mem_off(nc + 1, 0);
  std::vector<int> cbeg(nc);
  for (long long c = 0; c < nc; ++c) {
    const int node = cluster_node_ids[c];
    cbeg[c] = nb[node];
    mem_off[c + 1] = mem_off[c] + (ne[node] - nb[node]);
  }
  s = DSurrogate{};
  s.m = b.m;
  s.n_c = nc;
  s.u = u;
  s.n_t = nt;
  for (long long c = 0; c < nc; ++c) s.max_members = std::max(s.max_members, mem_off[c + 1] - mem_off[c]);
  auto up = [&](const void* h, size_t bytes) {
    void* d = dalloc(bytes);
    if (bytes) PTROM_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    return d;
  };
  s.mem_off = (long long*)up(mem_off.data(), mem_off.size() * 8);
  long long* mem_tmp = (long long*)dalloc(mem_off[nc] * 8);
  s.mem_ids = (long long*)dalloc(mem_off[nc] * 8);
  int* d_cbeg = (int*)up(cbeg.data(), cbeg.size() * 4);
  if (nc > 0) {
    gather_members_kernel<<<(unsigned)((nc + 127) / 128), 128, 0, st>>>(nc, s.mem_off, d_cbeg, tree.perm, mem_tmp);
    size_t bytes = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, mem_tmp, s.mem_ids, mem_off[nc], nc, s.mem_off, s.mem_off + 1,
                                       st);
    void* tmp = dalloc(bytes + 16);
    PTROM_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, mem_tmp, s.mem_ids, mem_off[nc], nc, s.mem_off,
                                                  s.mem_off + 1, st));
  }
  s.target_ids = (long long*)up(targets.data(), nt * 8);
  {  // spatial processing order: targets sorted by their slot in the weighted tree
    std::vector<int> slot(n);
    PTROM_CUDA(cudaMemcpy(slot.data(), tree.slot, n * 4, cudaMemcpyDeviceToHost));
    std::vector<int> order(nt);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b2) { return slot[targets[a]] < slot[targets[b2]]; });
    s.t_order = (int*)up(order.data(), nt * 4);
  }
  s.cl_off = (long long*)up(c_off.data(), c_off.size() * 8);
  s.cl_list = (int*)up(cl_list.data(), cl_list.size() * 4);
  s.d_off = (long long*)up(d_off.data(), d_off.size() * 8);
  s.d_list = (int*)up(d_list.data(), d_list.size() * 4);
  s.direct_ids = (long long*)up(uni.data(), u * 8);
  s.phi_tilde = (double*)dalloc(2 * nc * b.m * 8);
  s.x0_tilde = (double*)dalloc(2 * nc * 8);
  s.gamma_tilde = (double*)dalloc(nc * 8);
  s.zero_gamma = (unsigned char*)dalloc(nc);
  s.direct_phi = (double*)dalloc(2 * u * b.m * 8);
  s.direct_x0 = (double*)dalloc(2 * u * 8);
  s.direct_gamma = (double*)dalloc(u * 8);
  // node tables (reduction.hpp:253-273 == reassign formula, ascending members)
  rom_reassign_exact(ctx, s, b, d_gamma);
  if (u > 0)
    gather_direct_kernel<<<(unsigned)((u + 127) / 128), 128, 0, st>>>(u, s.direct_ids, b, d_gamma, s.direct_phi,
                                                                      s.direct_x0, s.direct_gamma);
  PTROM_LAUNCH_CHECK();
  PTROM_CUDA(cudaStreamSynchronize(st));
  tree.free_all(st);
  cudaFreeAsync(w, st);
  PTROM_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ptrom
