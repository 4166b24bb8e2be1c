// offline.cu — PTROM offline producers needed to run the online path at
// scale without any CPU reference code:
//   greedy_sample        reduction.hpp:93-168   (device scoring + selection)
//   build_gnat_operator  reduction.hpp:182-220  (A = pinv(P Φ_r))
//   weighted_pod_space + build_weighted_pod_tree + cluster_pod
//                        reduction.hpp:74-77, 236-385 (device quadtree + traversal)
//
// The dense factorizations (the gappy least-squares fits of greedy sampling,
// up to 2·n_samples x 31 with their right-hand sides, and the n_d x m_r
// pseudo-inverse) run on the device as one cooperative column-pivoted
// Householder QR (dev_cpqr_kernel); only the k x k triangular solves of the
// fits (k ≤ 31) are finished on the host.
#include <cooperative_groups.h>
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

namespace cg = cooperative_groups;

// ------------------------------------------------------ device dense LA ---
// Column-pivoted Householder QR of a tall rows x ct column-major matrix in
// global memory, the first cp columns pivot-eligible and the rest right-hand
// sides that receive every reflector (so they end as Qᵀb). The algorithm is
// the host PivotedQR's below (the same pivot rule — largest remaining norm,
// lowest index on ties — the same reflector formulas and rank test), as one
// cooperative launch: CTA b owns rows [b·rows/G, (b+1)·rows/G), and each
// column step is three fixed-order grid reductions (the tail norm, the
// reflector's dot products, the updated norms), so it is deterministic.
constexpr int kQRT = 256;
constexpr int kQRMaxCols = 64;

struct DevQR {
  double* a;  // rows x ct, column-major (R and the reflector tails in place)
  long long rows;
  int ct, cp;
  double* taus;  // [cp]
  int* piv;      // [cp]: column j of R is input column piv[j]
  int* rank;     // [1]
  double* red;   // [3][G][kQRMaxCols] per-CTA partials
  double* rowj;  // [kQRMaxCols] row j of the columns right of j (published by its owner)
};

// fixed-order block sum (warp shuffles, then the warps in order), result in every thread
__device__ double qr_block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kQRT / 32; ++w) t += sh[w];
  return t;
}

__global__ void __launch_bounds__(kQRT) dev_cpqr_kernel(const __grid_constant__ DevQR q) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double cn[kQRMaxCols], wv[kQRMaxCols], sh[kQRT / 32];
  __shared__ int pv[kQRMaxCols];
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  const long long R = q.rows;
  const long long r0 = R * bid / G, r1 = R * (bid + 1) / G;
  const int ct = q.ct, cp = q.cp;
  double* a = q.a;
  auto col = [&](int c) { return a + (long long)c * R; };
  // three partial regions (tail norm, dot products, column norms): each is
  // read only between the two barriers that follow its writes
  auto publish = [&](int region, int c, double v) {  // thread 0 of each CTA: its partial for column c
    if (tid == 0) q.red[((long long)region * G + bid) * kQRMaxCols + c] = v;
  };
  auto gather = [&](int region, int c) {  // every CTA: the partials of column c in CTA order
    double t = 0.0;
    for (int b = 0; b < G; ++b) t += q.red[((long long)region * G + b) * kQRMaxCols + c];
    return t;
  };
  for (int c = tid; c < cp; c += kQRT) pv[c] = c;
  for (int c = 0; c < cp; ++c) {
    double s = 0.0;
    for (long long i = r0 + tid; i < r1; i += kQRT) s += col(c)[i] * col(c)[i];
    publish(2, c, qr_block_sum(s, sh));
  }
  grid.sync();
  for (int c = tid; c < cp; c += kQRT) cn[c] = gather(2, c);
  __syncthreads();
  const int k = (int)min((long long)cp, R);
  double first = 0.0;
  int rank = 0;
  for (int j = 0; j < k; ++j) {
    int p = j;
    for (int c2 = j + 1; c2 < cp; ++c2)
      if (cn[c2] > cn[p]) p = c2;
    if (p != j) {
      for (long long i = r0 + tid; i < r1; i += kQRT) {
        const double t = col(j)[i];
        col(j)[i] = col(p)[i];
        col(p)[i] = t;
      }
      __syncthreads();
      if (tid == 0) {
        const double t = cn[j];
        cn[j] = cn[p];
        cn[p] = t;
        const int ti = pv[j];
        pv[j] = pv[p];
        pv[p] = ti;
      }
      __syncthreads();
    }
    // tail norm Σ_{i>j} a_ij²; the owner of row j publishes row j of the columns right of j
    {
      double s = 0.0;
      for (long long i = max(r0, (long long)j + 1) + tid; i < r1; i += kQRT) s += col(j)[i] * col(j)[i];
      publish(0, j, qr_block_sum(s, sh));
      if (j >= r0 && j < r1)
        for (int c2 = j + tid; c2 < ct; c2 += kQRT) q.rowj[c2] = col(c2)[j];
    }
    grid.sync();
    const double tail = gather(0, j);
    const double x0 = q.rowj[j];
    double beta = x0, tau = 0.0, scale = 0.0;
    if (tail > 0) {
      beta = -copysign(sqrt(x0 * x0 + tail), x0);
      tau = (beta - x0) / beta;
      scale = 1.0 / (x0 - beta);
    }
    // reflector tail v = a_{i>j, j}·scale, then the dot products with the columns right of j
    for (long long i = max(r0, (long long)j + 1) + tid; i < r1; i += kQRT) col(j)[i] *= scale;
    __syncthreads();
    for (int c2 = j + 1; c2 < ct; ++c2) {
      double s = 0.0;
      for (long long i = max(r0, (long long)j + 1) + tid; i < r1; i += kQRT) s += col(j)[i] * col(c2)[i];
      publish(1, c2, qr_block_sum(s, sh));
    }
    grid.sync();
    for (int c2 = j + 1 + tid; c2 < ct; c2 += kQRT) wv[c2] = (q.rowj[c2] + gather(1, c2)) * tau;
    __syncthreads();
    if (j >= r0 && j < r1 && tid == 0) {
      col(j)[j] = beta;
      for (int c2 = j + 1; c2 < ct; ++c2) col(c2)[j] -= wv[c2];
    }
    for (int c2 = j + 1; c2 < ct; ++c2) {
      const double w = wv[c2];
      double s = 0.0;
      for (long long i = max(r0, (long long)j + 1) + tid; i < r1; i += kQRT) {
        const double v = col(c2)[i] - w * col(j)[i];
        col(c2)[i] = v;
        s += v * v;
      }
      if (c2 < cp) publish(2, c2, qr_block_sum(s, sh));
    }
    grid.sync();
    for (int c2 = j + 1 + tid; c2 < cp; c2 += kQRT) cn[c2] = gather(2, c2);
    __syncthreads();
    if (j == 0) first = fabs(beta);
    if (fabs(beta) > 2.220446049250313e-16 * (double)k * first) rank = j + 1;
    if (bid == 0 && tid == 0) q.taus[j] = tau;
  }
  if (bid == 0) {
    for (int c = tid; c < cp; c += kQRT) q.piv[c] = pv[c];
    if (tid == 0) *q.rank = rank;
  }
}

// Q1 = H_0 … H_{k−1} [e_0 … e_{m−1}] (rows x m, column-major) from the
// reflectors of dev_cpqr_kernel, applied in reverse order; one grid reduction
// per reflector (the owner of row r folds row r into its partial).
__global__ void __launch_bounds__(kQRT) dev_form_q1_kernel(const double* __restrict__ a, long long R, int m, int k,
                                                          const double* __restrict__ taus, double* __restrict__ q1,
                                                          double* __restrict__ red) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kQRT / 32], wv[kQRMaxCols];
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  const long long r0 = R * bid / G, r1 = R * (bid + 1) / G;
  for (int c = 0; c < m; ++c)
    for (long long i = r0 + tid; i < r1; i += kQRT) q1[i + (long long)c * R] = i == c ? 1.0 : 0.0;
  for (int r = k - 1; r >= 0; --r) {
    const double tau = taus[r];
    if (tau == 0.0) continue;  // CTA-uniform
    const double* v = a + (long long)r * R;
    for (int c = 0; c < m; ++c) {
      const double* qc = q1 + (long long)c * R;
      double s = (r >= r0 && r < r1) ? qc[r] : 0.0;
      s = (tid == 0) ? s : 0.0;
      for (long long i = max(r0, (long long)r + 1) + tid; i < r1; i += kQRT) s += v[i] * qc[i];
      const double t = qr_block_sum(s, sh);
      if (tid == 0) red[(long long)bid * kQRMaxCols + c] = t;
    }
    grid.sync();
    for (int c = tid; c < m; c += kQRT) {
      double t = 0.0;
      for (int b = 0; b < G; ++b) t += red[(long long)b * kQRMaxCols + c];
      wv[c] = t * tau;
    }
    __syncthreads();
    for (int c = 0; c < m; ++c) {
      double* qc = q1 + (long long)c * R;
      const double w = wv[c];
      if (r >= r0 && r < r1 && tid == 0) qc[r] -= w;
      for (long long i = max(r0, (long long)r + 1) + tid; i < r1; i += kQRT) qc[i] -= w * v[i];
    }
    grid.sync();  // red is rewritten by the next reflector
  }
}

// pinv column k = P R⁻¹ (row k of Q1)ᵀ (back substitution; R from the top
// m x m of the factorization), A is m x rows column-major.
__global__ void pinv_rows_kernel(const double* __restrict__ a, long long R, int m, const int* __restrict__ piv,
                                 const double* __restrict__ q1, double* __restrict__ A) {
  __shared__ double rs[kQRMaxCols * kQRMaxCols];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) rs[e] = a[(e % m) + (long long)(e / m) * R];
  __syncthreads();
  const long long kr = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (kr >= R) return;
  double z[kQRMaxCols];
  for (int i = m - 1; i >= 0; --i) {
    double s2 = q1[kr + (long long)i * R];
    for (int j = i + 1; j < m; ++j) s2 -= rs[i + j * m] * z[j];
    z[i] = s2 / rs[i + i * m];
  }
  for (int j = 0; j < m; ++j) A[piv[j] + kr * m] = z[j];
}

// sampled rows of Φ_r: row k ↦ ids[k] (k < nid), ids[k − nid] + n (x rows, then y rows),
// columns [c0, c0 + nc) into out (rows x nc, column-major)
__global__ void gather_rows_kernel(long long n_dofs, int nid, const long long* __restrict__ ids,
                                   const double* __restrict__ phi_r, int c0, int nc, double* __restrict__ out) {
  const long long rows = 2LL * nid;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= rows * nc) return;
  const long long k = e % rows;
  const int c = (int)(e / rows);
  const long long r = k < nid ? ids[k] : ids[k - nid] + n_dofs / 2;
  out[k + (long long)c * rows] = phi_r[r + (long long)(c0 + c) * n_dofs];
}

int coop_grid(ptrom_ctx* ctx, const void* kern, long long rows) {
  int occ = 0;
  PTROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kQRT, 0));
  const long long want = std::max<long long>(1, (rows + kQRT - 1) / kQRT);
  return (int)std::max<long long>(1, std::min<long long>(want, (long long)ctx->num_sms * std::max(1, occ)));
}

struct DevQRResult {
  int rank = 0;
  std::vector<int> piv;
  std::vector<double> top;  // the first min(rows, cp) rows of all ct columns (ld = that count)
};

// Factor d_a (rows x ct) in place on the device; returns rank, pivots and
// the top rows (R, and Qᵀb of the right-hand-side columns).
DevQRResult device_cpqr(ptrom_ctx* ctx, double* d_a, long long rows, int ct, int cp, double* d_taus, int* d_piv,
                        int* d_rank, double* d_red, double* d_rowj) {
  cudaStream_t s = ctx->stream;
  DevQR q{d_a, rows, ct, cp, d_taus, d_piv, d_rank, d_red, d_rowj};
  int G = coop_grid(ctx, (const void*)dev_cpqr_kernel, rows);
  void* args[] = {&q};
  PTROM_CUDA(cudaLaunchCooperativeKernel((const void*)dev_cpqr_kernel, dim3(G), dim3(kQRT), args, 0, s));
  PTROM_LAUNCH_CHECK();
  DevQRResult res;
  const int kt = (int)std::min<long long>(rows, cp);
  res.piv.resize(cp);
  res.top.resize((size_t)kt * ct);
  PTROM_CUDA(cudaMemcpyAsync(&res.rank, d_rank, 4, cudaMemcpyDeviceToHost, s));
  PTROM_CUDA(cudaMemcpyAsync(res.piv.data(), d_piv, cp * 4, cudaMemcpyDeviceToHost, s));
  if (kt > 0)
    PTROM_CUDA(cudaMemcpy2DAsync(res.top.data(), kt * 8, d_a, rows * 8, kt * 8, ct, cudaMemcpyDeviceToHost, s));
  PTROM_CUDA(cudaStreamSynchronize(s));
  return res;
}

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
    // device least-squares workspace (rows ≤ 2·n_target; basis + right-hand
    // sides nb + n_ci ≤ n_c columns)
    if (n_c > kQRMaxCols) config_fail("greedy_sample: at most 64 working vectors (residual modes)");
    double *d_fit, *d_taus, *d_red, *d_rowj;
    long long* d_ids;
    int *d_piv, *d_rank;
    PTROM_CUDA(cudaMallocAsync(&d_fit, (size_t)2 * n_target * n_c * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_ids, (size_t)n_target * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_taus, kQRMaxCols * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_piv, kQRMaxCols * 4, s));
    PTROM_CUDA(cudaMallocAsync(&d_rank, 4, s));
    PTROM_CUDA(cudaMallocAsync(&d_red, (size_t)3 * ctx->num_sms * 32 * kQRMaxCols * 8, s));
    PTROM_CUDA(cudaMallocAsync(&d_rowj, kQRMaxCols * 8, s));
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
        // gappy fit on the rows sampled so far (reduction.hpp:129-143): the
        // sampled basis with the n_ci right-hand sides appended, factored on
        // the device; the basic solution from the k x k top (free variables 0)
        std::vector<long long> ids = chosen;
        std::sort(ids.begin(), ids.end());
        const int nid = (int)ids.size();
        const long long rows = 2LL * nid;
        const int ct = (int)(nb + n_ci);
        PTROM_CUDA(cudaMemcpyAsync(d_ids, ids.data(), nid * 8, cudaMemcpyHostToDevice, s));
        gather_rows_kernel<<<(unsigned)((rows * ct + 255) / 256), 256, 0, s>>>(n_dofs, nid, d_ids, d_phi, 0, ct,
                                                                              d_fit);
        PTROM_LAUNCH_CHECK();
        const DevQRResult qr = device_cpqr(ctx, d_fit, rows, ct, (int)nb, d_taus, d_piv, d_rank, d_red, d_rowj);
        const int kt = (int)std::min<long long>(rows, nb);
        std::vector<double> coef(nb * n_ci, 0.0), z(nb);
        for (long long q = 0; q < n_ci; ++q) {
          const double* y = &qr.top[(size_t)(nb + q) * kt];  // Qᵀ b, first kt rows
          for (int i = qr.rank - 1; i >= 0; --i) {
            double s2 = y[i];
            for (int j = i + 1; j < qr.rank; ++j) s2 -= qr.top[i + (size_t)j * kt] * z[j];
            z[i] = s2 / qr.top[i + (size_t)i * kt];
          }
          for (int j = 0; j < qr.rank; ++j) coef[qr.piv[j] + q * nb] = z[j];
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
    void* fr[] = {d_phi, d_work, d_coef, d_score, d_score_s, d_idx, d_idx_s, d_picked, d_tmp,
                  d_fit, d_ids, d_taus, d_piv, d_rank, d_red, d_rowj};
    for (void* p : fr) cudaFreeAsync(p, s);
    PTROM_CUDA(cudaStreamSynchronize(s));
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// reduction.hpp:182-220: A = pinv(rows of Φ_r at the sampled dofs), on the
// device: the sampled rows (n_d x m_r) factored by dev_cpqr_kernel, the rank
// test of the COD, Q1 formed from the reflectors, and A = P R⁻¹ Q1ᵀ.
std::vector<double> offline_gnat_operator(ptrom_ctx* ctx, long long n_dofs, int m_r, const double* phi_r,
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
  if (m_r > kQRMaxCols) config_fail("build_gnat_operator: at most 64 residual modes");
  std::vector<double> sm(nd * m_r);
  for (long long k = 0; k < nd; ++k) {
    const long long r = k < (long long)ids.size() ? ids[k] : ids[k - ids.size()] + n;
    for (int c = 0; c < m_r; ++c) sm[k + c * nd] = phi_r[r + c * n_dofs];
  }
  cudaStream_t s = ctx->stream;
  double *d_a, *d_taus, *d_red, *d_rowj, *d_q1, *d_A;
  int *d_piv, *d_rank;
  const size_t red_n = (size_t)3 * ctx->num_sms * 32 * kQRMaxCols;
  PTROM_CUDA(cudaMallocAsync(&d_a, nd * m_r * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_taus, kQRMaxCols * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_red, red_n * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_rowj, kQRMaxCols * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_q1, nd * m_r * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_A, nd * m_r * 8, s));
  PTROM_CUDA(cudaMallocAsync(&d_piv, kQRMaxCols * 4, s));
  PTROM_CUDA(cudaMallocAsync(&d_rank, 4, s));
  struct Free {
    std::vector<void*> p;
    cudaStream_t s;
    ~Free() {
      for (void* q : p) cudaFreeAsync(q, s);
    }
  } guard{{d_a, d_taus, d_red, d_rowj, d_q1, d_A, d_piv, d_rank}, s};
  PTROM_CUDA(cudaMemcpyAsync(d_a, sm.data(), nd * m_r * 8, cudaMemcpyHostToDevice, s));
  const DevQRResult qr = device_cpqr(ctx, d_a, nd, m_r, m_r, d_taus, d_piv, d_rank, d_red, d_rowj);
  if (qr.rank < m_r) {
    std::string cols;
    for (int k = qr.rank; k < m_r; ++k) cols += (cols.empty() ? "" : ", ") + std::to_string(qr.piv[k]);
    numerical_fail("build_gnat_operator: sampled residual basis has rank " + std::to_string(qr.rank) + " < " +
                   std::to_string(m_r) + "; dependent columns: " + cols);
  }
  {
    long long R = nd;
    int m = m_r, k = m_r;
    int G = coop_grid(ctx, (const void*)dev_form_q1_kernel, nd);
    void* args[] = {&d_a, &R, &m, &k, &d_taus, &d_q1, &d_red};
    PTROM_CUDA(cudaLaunchCooperativeKernel((const void*)dev_form_q1_kernel, dim3(G), dim3(kQRT), args, 0, s));
    PTROM_LAUNCH_CHECK();
  }
  pinv_rows_kernel<<<(unsigned)((nd + 127) / 128), 128, 0, s>>>(d_a, nd, m_r, d_piv, d_q1, d_A);
  PTROM_LAUNCH_CHECK();
  std::vector<double> A((size_t)m_r * nd);
  PTROM_CUDA(cudaMemcpyAsync(A.data(), d_A, A.size() * 8, cudaMemcpyDeviceToHost, s));
  PTROM_CUDA(cudaStreamSynchronize(s));
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
