// rom.cu — PTROM online path on sm_100a, batched over parameter instances.
//
// Replaces, for B instances at once:
//   reassign_cluster_circulation  reduction.hpp:400-431
//   hyperpair                     rom.hpp:101-155
//   apply_residual_jacobian       rom.hpp:71-84
//   GnatSolver::simulate          rom.hpp:292-340 (Gauss–Newton on the sampled residual)
//   ptrom_simulate                rom.hpp:404-412
//
// Per Gauss–Newton evaluation of instance b:
//   1. source positions: clusters c (x̃⁰ + Φ̃x̂, or the affine (S_A + μS_B)/(G_A + μG_B) form),
//      direct sources (x⁰_d + Φ_d x̂), sampled targets x̄ = x̄⁰ + Φ̄x̂, as DMMA GEMMs
//      (positions_*_mma kernels; instance-minor layout [source][b] so a warp of 32 instances
//      reads one cluster's 32 positions coalesced).
//   2. hyperpair: a warp per (target, 32 instances), cluster list then direct list, fused
//      velocity + self-Jacobian (the reference's two calls kernel.hpp:29-73 per source).
//   3. gn_partial / gn_finish: split-K over the 2n_t sampled rows, 8 instances per CTA: residual
//      r̄, C = (I − h J)Φ̄ rows (row per lane, staged in shared memory), A·C on the FP64 tensor
//      cores (mma.sync m8n8k4 DMMA; tcgen05 has no fp64 kind), A·r̄ and Cᵀr̄; slice-ordered
//      reduction, then the reference's convergence logic on ‖Cᵀr̄‖.
//   4. qr_update: one warp per instance solves min‖AC·Δ + A r̄‖ by column-pivoted Householder QR
//      (lane i owns row i of the 32 x 16 system) and applies x̂ += αΔ.
//
// Cluster tables: the batch engine evaluates Φ̃(μ) = (S_A + μ S_B)/(G_A + μ G_B) with per-cluster
// member sums of an affine circulation Γ(μ) = Γ_a + μ Γ_b (mathematically the reference's
// Σ_p (Γ_p/ΣΓ) Φ_p) so no per-instance table is materialised. The
// single-instance drop-in (ptrom_ptrom_simulate_f64) instead reassigns exactly like the
// reference (sequential member order, w_p = Γ_p / Σ Γ) and runs the same engine with B = 1.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "ops.cuh"
#include "rom.cuh"

namespace ptrom {

namespace {


__device__ __forceinline__ double rcp64(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  double e = fma(-q, y, 1.0);
  e = fma(e, e, e);
  return fma(y, e, y);
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------- table preparation ---
// Row-major basis rows (DBasis::rm) for coalesced member gathers.
__global__ void basis_rowmajor_kernel(DBasis b) {
  const int W = 2 * (b.m + 1);
  const long long total = b.n * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / W;
    const int c = (int)(i % W);
    const int half = c / (b.m + 1), j = c % (b.m + 1);  // half 0 = x row, 1 = y row
    const long long row = p + half * b.n;
    b.rm[i] = j < b.m ? b.phi[row + (long long)j * 2 * b.n] : b.x_ref[row];
  }
}

// reduction.hpp:400-431 for one cluster per warp, members in the reference's
// sequential order: ΣΓ first (each chunk of 32 members gathered in parallel,
// then added in order via shuffles), then w_p = Γ_p / ΣΓ for 32 members at
// once (one division per lane), then lane j owns column j (mode j, or x_ref
// for j == m) of both rows and accumulates w_p·Φ(p, j) member by member.
// The arithmetic is the reference's, so Φ̃, x̃⁰ and Γ̃ are bit-identical.
// Clusters above `big` members (ctx->reassign_big, default 4096) take one CTA
// each (reassign_big_kernel); the rest a warp each.
__global__ void reassign_exact_kernel(DSurrogate s, DBasis b, const double* __restrict__ gamma, long long big) {
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= s.n_c) return;
  const long long b0 = s.mem_off[c], b1 = s.mem_off[c + 1];
  if (b1 - b0 > big) return;
  double gsum = 0.0;
  for (long long k0 = b0; k0 < b1; k0 += 32) {
    const int cnt = (int)min(32LL, b1 - k0);
    const double gv = lane < cnt ? gamma[s.mem_ids[k0 + lane]] : 0.0;
    for (int t = 0; t < cnt; ++t) gsum = __dadd_rn(gsum, __shfl_sync(0xffffffffu, gv, t));
  }
  const bool fb = gsum == 0.0;
  const double inv_count = __ddiv_rn(1.0, (double)(b1 - b0));
  const int W = 2 * (b.m + 1);
  for (int j0 = 0; j0 <= b.m; j0 += 32) {
    const int j = min(j0 + lane, b.m);  // lanes past m duplicate column m (not stored)
    double ax = 0.0, ay = 0.0;
    for (long long k0 = b0; k0 < b1; k0 += 32) {
      const int cnt = (int)min(32LL, b1 - k0);
      long long pl = 0;
      double wl = 0.0;
      if (lane < cnt) {
        pl = s.mem_ids[k0 + lane];
        wl = fb ? inv_count : __ddiv_rn(gamma[pl], gsum);
      }
#pragma unroll 8
      for (int t = 0; t < cnt; ++t) {
        const long long p = __shfl_sync(0xffffffffu, pl, t);
        const double w = __shfl_sync(0xffffffffu, wl, t);
        const double* row = b.rm + p * W;
        ax = __dadd_rn(ax, __dmul_rn(w, row[j]));
        ay = __dadd_rn(ay, __dmul_rn(w, row[b.m + 1 + j]));
      }
    }
    if (j0 + lane > b.m) continue;
    if (j < s.m) {
      s.phi_tilde[c + (long long)j * 2 * s.n_c] = ax;
      s.phi_tilde[c + s.n_c + (long long)j * 2 * s.n_c] = ay;
    } else {
      s.x0_tilde[c] = ax;
      s.x0_tilde[c + s.n_c] = ay;
      s.gamma_tilde[c] = gsum;
      s.zero_gamma[c] = fb ? 1 : 0;
    }
  }
}

__global__ void big_clusters_kernel(DSurrogate s, long long big, int* __restrict__ list, int* __restrict__ count) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c < s.n_c && s.mem_off[c + 1] - s.mem_off[c] > big) list[atomicAdd(count, 1)] = (int)c;
}

// reduction.hpp:400-431 for the large clusters, one CTA each. Warps 1..7
// stage the next chunk of members (ids and w_p = Γ_p/ΣΓ, then the row-major
// basis rows through cp.async — all loads of a chunk in flight at once) into
// the other shared-memory buffer while warp 0 runs the reference's sequential
// chains (lane j owns column j of both rows) over the current chunk. ΣΓ is
// the same producer/consumer pattern with lane 0 of warp 0 adding in order.
// Same arithmetic and order as reassign_exact_kernel: bit-identical tables.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void producers_sync(int nthr) { asm volatile("bar.sync 1, %0;" ::"r"(nthr)); }

constexpr int kBigGChunk = 2048;  // members per ΣΓ chunk
__global__ void __launch_bounds__(256) reassign_big_kernel(DSurrogate s, DBasis b, const double* __restrict__ gamma,
                                                           const int* __restrict__ list,
                                                           const int* __restrict__ count, int ch) {
  extern __shared__ double big_smem[];
  const int W = 2 * (b.m + 1);
  double* rows = big_smem;                 // [2][ch][W]
  double* wbuf = big_smem + 2 * ch * W;    // [2][max(ch, kBigGChunk)]
  const int wcap = max(ch, kBigGChunk);
  long long* sid = reinterpret_cast<long long*>(wbuf + 2 * wcap);  // [2][ch]
  __shared__ double s_gsum;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ptid = threadIdx.x - 32, pn = blockDim.x - 32;  // producer threads (warps 1..7)
  const int total = *count;
  for (int li = blockIdx.x; li < total; li += gridDim.x) {
    const long long c = list[li];
    const long long b0 = s.mem_off[c], b1 = s.mem_off[c + 1];
    // ---- ΣΓ in member order
    auto gstage = [&](long long k0, int buf, int tid0, int nthr) {
      const int cnt = (int)min((long long)kBigGChunk, b1 - k0);
      double* gb = wbuf + buf * wcap;
#pragma unroll 4
      for (int i = tid0; i < cnt; i += nthr) gb[i] = gamma[s.mem_ids[k0 + i]];
    };
    gstage(b0, 0, threadIdx.x, blockDim.x);
    __syncthreads();
    double gsum = 0.0;
    int buf = 0;
    for (long long k0 = b0; k0 < b1; k0 += kBigGChunk) {
      if (warp != 0) {
        if (k0 + kBigGChunk < b1) gstage(k0 + kBigGChunk, buf ^ 1, ptid, pn);
      } else if (lane == 0) {
        const int cnt = (int)min((long long)kBigGChunk, b1 - k0);
        const double* gb = wbuf + buf * wcap;
        int i = 0;
        for (; i + 8 <= cnt; i += 8) {  // loads issued ahead of the chain
          double v8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v8[u] = gb[i + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) gsum = __dadd_rn(gsum, v8[u]);
        }
        for (; i < cnt; ++i) gsum = __dadd_rn(gsum, gb[i]);
      }
      __syncthreads();
      buf ^= 1;
    }
    if (threadIdx.x == 0) s_gsum = gsum;
    __syncthreads();
    gsum = s_gsum;
    const bool fb = gsum == 0.0;
    const double inv_count = __ddiv_rn(1.0, (double)(b1 - b0));
    // ---- weighted rows
    auto stage = [&](long long k0, int bf, int tid0, int nthr, bool all) {
      const int cnt = (int)min((long long)ch, b1 - k0);
      double* rb = rows + (long long)bf * ch * W;
      for (int i = tid0; i < cnt; i += nthr) {
        const long long p = s.mem_ids[k0 + i];
        sid[bf * ch + i] = p;
        wbuf[bf * wcap + i] = fb ? inv_count : __ddiv_rn(gamma[p], gsum);
      }
      if (all) __syncthreads();
      else producers_sync(nthr);
      for (int e = tid0; e < cnt * W; e += nthr) {
        const int i = e / W, j = e - i * W;
        cp_async8(rb + e, b.rm + sid[bf * ch + i] * W + j);
      }
      cp_async_wait_all();
    };
    stage(b0, 0, threadIdx.x, blockDim.x, true);
    __syncthreads();
    // warp 0, lane l: columns l and l + 32 (mode j, or x_ref for j == m)
    double ax = 0.0, ay = 0.0, ax2 = 0.0, ay2 = 0.0;
    const int j = lane, j2 = lane + 32;
    buf = 0;
    for (long long k0 = b0; k0 < b1; k0 += ch) {
      if (warp != 0) {
        if (k0 + ch < b1) stage(k0 + ch, buf ^ 1, ptid, pn, false);
      } else if (j <= b.m) {
        const int cnt = (int)min((long long)ch, b1 - k0);
        const double* rb = rows + (long long)buf * ch * W;
        const double* wb = wbuf + buf * wcap;
        if (j2 <= b.m) {
          for (int i = 0; i < cnt; ++i) {
            const double w = wb[i];
            ax = __dadd_rn(ax, __dmul_rn(w, rb[i * W + j]));
            ay = __dadd_rn(ay, __dmul_rn(w, rb[i * W + b.m + 1 + j]));
            ax2 = __dadd_rn(ax2, __dmul_rn(w, rb[i * W + j2]));
            ay2 = __dadd_rn(ay2, __dmul_rn(w, rb[i * W + b.m + 1 + j2]));
          }
        } else {
          int i = 0;
          for (; i + 4 <= cnt; i += 4) {  // loads issued ahead of the chains
            double w4[4], vx4[4], vy4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              w4[u] = wb[i + u];
              vx4[u] = rb[(i + u) * W + j];
              vy4[u] = rb[(i + u) * W + b.m + 1 + j];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              ax = __dadd_rn(ax, __dmul_rn(w4[u], vx4[u]));
              ay = __dadd_rn(ay, __dmul_rn(w4[u], vy4[u]));
            }
          }
          for (; i < cnt; ++i) {
            const double w = wb[i];
            ax = __dadd_rn(ax, __dmul_rn(w, rb[i * W + j]));
            ay = __dadd_rn(ay, __dmul_rn(w, rb[i * W + b.m + 1 + j]));
          }
        }
      }
      __syncthreads();
      buf ^= 1;
    }
    auto put = [&](int jj, double vx, double vy) {
      if (jj < s.m) {
        s.phi_tilde[c + (long long)jj * 2 * s.n_c] = vx;
        s.phi_tilde[c + s.n_c + (long long)jj * 2 * s.n_c] = vy;
      } else {
        s.x0_tilde[c] = vx;
        s.x0_tilde[c + s.n_c] = vy;
        s.gamma_tilde[c] = gsum;
        s.zero_gamma[c] = fb ? 1 : 0;
      }
    };
    if (warp == 0 && j <= b.m) put(j, ax, ay);
    if (warp == 0 && j2 <= b.m) put(j2, ax2, ay2);
    __syncthreads();
  }
}

__global__ void direct_gamma_kernel(DSurrogate s, const double* __restrict__ gamma) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < s.u) s.direct_gamma[k] = gamma[s.direct_ids[k]];
}

// Affine member sums for Γ(μ) = Γa + μΓb: S_A, S_B (Φ rows), X_A, X_B
// (x_ref), G_A, G_B per cluster — an algebraic reformulation, so any order:
// one warp per (cluster, column), lanes striding over the members (large
// clusters are split across the lanes; rows come from the row-major basis).
__global__ void affine_tables_kernel(DSurrogate s, DBasis b, const double* __restrict__ ga,
                                     const double* __restrict__ gb, AffineTables t) {
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int cols = s.m + 1;
  if (wid >= s.n_c * cols) return;
  const long long c = wid / cols;
  const int j = (int)(wid % cols);
  const int W = 2 * (b.m + 1);
  double v[6] = {0, 0, 0, 0, 0, 0};  // sax say sbx sby ga gb
#pragma unroll 4
  for (long long k = s.mem_off[c] + lane; k < s.mem_off[c + 1]; k += 32) {
    const long long p = s.mem_ids[k];
    const double* row = b.rm + p * W;
    const double vx = row[j], vy = row[b.m + 1 + j];
    const double a = ga[p], bb = gb[p];
    v[0] = fma(a, vx, v[0]);
    v[1] = fma(a, vy, v[1]);
    v[2] = fma(bb, vx, v[2]);
    v[3] = fma(bb, vy, v[3]);
    v[4] += a;
    v[5] += bb;
  }
#pragma unroll
  for (int e = 0; e < 6; ++e)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[e] += __shfl_xor_sync(0xffffffffu, v[e], o);
  if (lane != 0) return;
  if (j < s.m) {
    t.pa[c + (long long)j * 2 * s.n_c] = v[0];
    t.pa[c + s.n_c + (long long)j * 2 * s.n_c] = v[1];
    t.pb[c + (long long)j * 2 * s.n_c] = v[2];
    t.pb[c + s.n_c + (long long)j * 2 * s.n_c] = v[3];
  } else {
    t.xa[c] = v[0];
    t.xa[c + s.n_c] = v[1];
    t.xb[c] = v[2];
    t.xb[c + s.n_c] = v[3];
    t.ga[c] = v[4];
    t.gb[c] = v[5];
  }
}

// Row-major engine tables from the column-major reference layouts.
__global__ void engine_tables_kernel(DSurrogate s, AffineTables t, DGnat g, int Q, int MP, EngineTables e) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nct = s.n_c * Q * MP, ndt = s.u * 2 * MP, npb = 2 * g.n_s * MP;
  if (idx < nct) {
    const long long c = idx / (Q * MP);
    const int q = (int)((idx / MP) % Q), k = (int)(idx % MP);
    double v = 0.0;
    if (k < s.m) {
      const long long row = c + ((q & 1) ? s.n_c : 0), col = (long long)k * 2 * s.n_c;
      v = Q == 2 ? s.phi_tilde[row + col] : (q < 2 ? t.pa[row + col] : t.pb[row + col]);
    }
    e.ct[idx] = v;
  } else if (idx < nct + ndt) {
    const long long i = idx - nct;
    const long long d = i / (2 * MP);
    const int q = (int)((i / MP) % 2), k = (int)(i % MP);
    e.dt[i] = k < s.m ? s.direct_phi[d + (q ? s.u : 0) + (long long)k * 2 * s.u] : 0.0;
  } else if (idx < nct + ndt + npb) {
    const long long i = idx - nct - ndt;
    const long long r = i / MP;
    const int k = (int)(i % MP);
    e.pbr[i] = g.phi_bar[r + (long long)k * 2 * g.n_s];
  }
}

// ------------------------------------------------------------ positions ---
// Clusters: exact mode cpos = x̃⁰ + Φ̃ x̂ (rom.hpp:113); affine mode
// cpos = (X_A + S_A x̂ + μ (X_B + S_B x̂)) / (G_A + μ G_B).
template <bool AFFINE>
__global__ void positions_clusters_kernel(DSurrogate s, AffineTables t, int B, int xs, const double* __restrict__ xhat,
                                          const double* __restrict__ mu, const unsigned char* __restrict__ active,
                                          double2* __restrict__ cxy, DeviceStatus* st) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= s.n_c * B) return;
  const long long c = idx / B;
  const int b = (int)(idx % B);
  if (active && !active[b]) return;
  const double* xh = xhat + (long long)b * xs;
  const long long ld = 2 * s.n_c;
  if (!AFFINE) {
    double ax = 0.0, ay = 0.0;
    for (int j = 0; j < s.m; ++j) {
      ax = fma(s.phi_tilde[c + j * ld], xh[j], ax);
      ay = fma(s.phi_tilde[c + s.n_c + j * ld], xh[j], ay);
    }
    cxy[idx] = make_double2(s.x0_tilde[c] + ax, s.x0_tilde[c + s.n_c] + ay);
  } else {
    double ax = t.xa[c], ay = t.xa[c + s.n_c], bx = t.xb[c], by = t.xb[c + s.n_c];
    for (int j = 0; j < s.m; ++j) {
      const double x = xh[j];
      ax = fma(t.pa[c + j * ld], x, ax);
      ay = fma(t.pa[c + s.n_c + j * ld], x, ay);
      bx = fma(t.pb[c + j * ld], x, bx);
      by = fma(t.pb[c + s.n_c + j * ld], x, by);
    }
    const double m = mu[b];
    const double g = t.ga[c] + m * t.gb[c];
    if (g == 0.0) latch_status(st, kStatusZeroClusterCirculation, c);
    const double ig = 1.0 / g;
    cxy[idx] = make_double2(fma(m, bx, ax) * ig, fma(m, by, ay) * ig);
  }
}


// Cluster positions as a DMMA GEMM. A warp tile is 8 instances x 4 clusters
// x (x, y) with K = MP modes: x̂ of 8 instances is the A operand, the table
// rows the B operand, so each lane's two accumulators are the (x, y) of one
// (instance, cluster) and the epilogue needs no exchange: one G(μ) and one
// reciprocal per lane, one 16-byte store. The bases (X_A, X_B or x̃⁰) seed
// the accumulators. Affine mode runs two chains (X_A + S_A x̂ and X_B + S_B x̂
// land in the same lane) and forms (a + μ b)/(G_A + μ G_B). Exact mode is one
// chain, x̃⁰ + Φ̃ x̂, and it also serves the direct sources (x⁰_d + Φ_d x̂,
// table [u][2][mp]). The CTA stages x̂ (and μ) of up to `ic` instances in
// shared memory once (row stride MP + 4 doubles: conflict-free fragments),
// and its 16 warps then sweep cluster tiles grid-stride.
template <int MP>
struct PosSmem {
  static constexpr int SX = MP + 4;
  static int ic(int B) {  // instances staged per pass: ≤ 96 KB of x̂
    const int cap = (12288 / SX) / 8 * 8;
    return std::min(cap, (B + 7) / 8 * 8);
  }
  static size_t bytes(int ic) { return (size_t)ic * (SX + 1) * 8; }
};

template <bool AFFINE, int MP>
__global__ void __launch_bounds__(512, 2) positions_clusters_mma_kernel(long long nc, const double* __restrict__ tab,
                                                                        const double* __restrict__ x0, AffineTables t,
                                                                        int B, int ic, const double* __restrict__ xhat,
                                                                        const double* __restrict__ mu,
                                                                        const unsigned char* __restrict__ active,
                                                                        double2* __restrict__ out,
                                                                        DeviceStatus* st) {
  constexpr int KS = MP / 4, SX = PosSmem<MP>::SX;
  extern __shared__ __align__(16) double pos_smem[];
  double* sxh = pos_smem;
  double* smu = pos_smem + (size_t)ic * SX;
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const long long ctiles = (nc + 3) / 4;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  const long long w0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int xy = lr & 1;
  for (int i0 = 0; i0 < B; i0 += ic) {
    const int icnt = min(ic, B - i0), ipad = (icnt + 7) & ~7;
    __syncthreads();
    for (int e = threadIdx.x; e < ipad * (MP / 2); e += blockDim.x) {
      const int r = e / (MP / 2), c2 = e % (MP / 2);
      const double2 v = r < icnt ? reinterpret_cast<const double2*>(xhat + (long long)(i0 + r) * MP)[c2]
                                 : make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(sxh + r * SX + 2 * c2) = v;
    }
    if (AFFINE)
      for (int e = threadIdx.x; e < icnt; e += blockDim.x) smu[e] = mu[i0 + e];
    __syncthreads();
    for (long long tile = w0; tile < ctiles; tile += wstride) {
      // B operand (k = lc, column n = lr): the table row of cluster
      // tile·4 + (lr >> 1), coordinate lr & 1, loaded once per tile
      const long long cb = tile * 4 + (lr >> 1);
      const double* trow = tab + (cb * (AFFINE ? 4 : 2) + xy) * (long long)MP;
      double a0[KS], a1[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        a0[k] = cb < nc ? trow[4 * k + lc] : 0.0;
        a1[k] = (AFFINE && cb < nc) ? trow[2 * MP + 4 * k + lc] : 0.0;
      }
      // accumulator owner: instance b0 + lr, cluster tile·4 + lc, (x, y) in
      // (d0, d1) — the x and y rows of one cluster are adjacent columns
      const long long ca = tile * 4 + lc;
      const bool c_ok = ca < nc;
      double bax = 0, bay = 0, bbx = 0, bby = 0;
      if (c_ok) {
        if (AFFINE) {
          bax = t.xa[ca];
          bay = t.xa[ca + nc];
          bbx = t.xb[ca];
          bby = t.xb[ca + nc];
        } else {
          bax = x0[ca];
          bay = x0[ca + nc];
        }
      }
      for (int b0 = 0; b0 < icnt; b0 += 8) {
        // D = X̂ · Tᵀ + base: the bases seed the accumulators
        double acc0[2] = {bax, bay}, acc1[2] = {bbx, bby};
        const double* xrow = sxh + (b0 + lr) * SX + lc;  // A operand: instance b0 + lr, k = lc
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          const double x = xrow[4 * k];
          dmma(acc0, x, a0[k]);
          if (AFFINE) dmma(acc1, x, a1[k]);
        }
        const int bl = b0 + lr, b = i0 + bl;
        if (!c_ok || bl >= icnt || (active && !active[b])) continue;
        double2 v;
        if (AFFINE) {
          // (a + μ b) / G(μ): one reciprocal (≤ 1 ulp, MUFU seed + cubic) for both coordinates
          const double m = smu[bl];
          const double G = fma(m, __ldg(t.gb + ca), __ldg(t.ga + ca));  // L1-resident across the tile
          if (G == 0.0) latch_status(st, kStatusZeroClusterCirculation, ca);
          const double ig = rcp64(G);
          v = make_double2(fma(m, acc1[0], acc0[0]) * ig, fma(m, acc1[1], acc0[1]) * ig);
        } else {
          v = make_double2(acc0[0], acc0[1]);
        }
        out[ca * B + b] = v;
      }
    }
  }
}

// Direct sources: x⁰_d + Φ_d x̂ (rom.hpp:114); Γ_d(μ) comes from the Γ tables.
__global__ void positions_direct_kernel(DSurrogate s, int B, int xs, const double* __restrict__ xhat,
                                        const unsigned char* __restrict__ active, double2* __restrict__ dxy) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= s.u * B) return;
  const long long k = idx / B;
  const int b = (int)(idx % B);
  if (active && !active[b]) return;
  const double* xh = xhat + (long long)b * xs;
  const long long ld = 2 * s.u;
  double ax = 0.0, ay = 0.0;
  for (int j = 0; j < s.m; ++j) {
    ax = fma(s.direct_phi[k + j * ld], xh[j], ax);
    ay = fma(s.direct_phi[k + s.u + j * ld], xh[j], ay);
  }
  dxy[idx] = make_double2(s.direct_x0[k] + ax, s.direct_x0[k + s.u] + ay);
}

// Sampled targets x̄ = x̄⁰ + Φ̄ x̂ (rom.hpp:306, 329); instance-major [b][row].
// A thread keeps one row of Φ̄ in registers and sweeps 32 instances (x̂
// staged in shared memory); stores are coalesced along the rows. Same
// sequential fma chain over the modes as the reference's dot product.
template <int MP>
__global__ void __launch_bounds__(256) positions_targets_kernel(DGnat g, int B, const double* __restrict__ xhat,
                                                               const unsigned char* __restrict__ active,
                                                               double* __restrict__ xbar) {
  constexpr int IB = 32;
  __shared__ double sx[IB * MP];
  __shared__ unsigned char sact[IB];
  const long long rows = 2 * g.n_s;
  const int b0 = blockIdx.y * IB, nb = min(IB, B - b0);
  for (int e = threadIdx.x; e < nb * MP; e += blockDim.x) sx[e] = xhat[(long long)b0 * MP + e];
  if (threadIdx.x < nb) sact[threadIdx.x] = active ? active[b0 + threadIdx.x] : 1;
  __syncthreads();
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double ph[MP];
#pragma unroll
  for (int j = 0; j < MP; ++j) ph[j] = j < g.m ? g.phi_bar[r + j * rows] : 0.0;
  const double x0 = g.x0_bar[r];
  for (int i = 0; i < nb; ++i) {
    if (!sact[i]) continue;
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < MP; ++j)
      if (j < g.m) a = fma(ph[j], sx[i * MP + j], a);
    xbar[(long long)(b0 + i) * rows + r] = x0 + a;
  }
}

// ------------------------------------------------------------- hyperpair ---
// rom.hpp:118-153 for (target t, instance b): clusters (skipping a centroid
// exactly on its target when delta == 0, rom.hpp:129), then direct sources
// (skipping the target's own id, rom.hpp:136), fused velocity + Jacobian,
// inflow at the target id. f: [b][2n_t], jac: [b][n_t][4].
// Γ/2π tables for hyperpair (built once per march): exact mode Γ̃_c/2π and
// Γ_d/2π (bit-identical to the reference's Γ·(1/2π) before the 1/q product),
// affine mode (G_A, G_B)/2π and (Γa_d, Γb_d)/2π as double2.
struct HpGamma {
  const double* gc = nullptr;    // [n_c] exact
  const double2* gab = nullptr;  // [n_c] affine
  const double* gd = nullptr;    // [u] exact
  const double2* gdab = nullptr; // [u] affine
  const int* self_loc = nullptr; // [n_t] the target's own slot in direct_ids, or -1
};

// Each target's own slot in the sorted near-field union (rom.hpp:140 skips it).
__global__ void hp_self_kernel(DSurrogate s, int* __restrict__ self_loc) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= s.n_t) return;
  const long long pid = s.target_ids[t];
  long long lo = 0, hi = s.u;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (s.direct_ids[mid] < pid) lo = mid + 1;
    else hi = mid;
  }
  self_loc[t] = (lo < s.u && s.direct_ids[lo] == pid) ? (int)lo : -1;
}

__global__ void hp_gamma_kernel(DSurrogate s, AffineTables t, bool affine, double* gc, double2* gab, double* gd,
                                double2* gdab) {
  const double inv2pi = 1.0 / (2.0 * M_PI);
  const long long total = s.n_c + s.u;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < s.n_c) {
      if (affine) gab[i] = make_double2(t.ga[i] * inv2pi, t.gb[i] * inv2pi);
      else gc[i] = s.gamma_tilde[i] * inv2pi;
    } else {
      const long long d = i - s.n_c;
      if (affine) gdab[d] = make_double2(t.dga[d] * inv2pi, t.dgb[d] * inv2pi);
      else gd[d] = s.direct_gamma[d] * inv2pi;
    }
  }
}

template <int IB, bool OFF32>
__global__ void __launch_bounds__(128, 7) hyperpair_kernel(DSurrogate s, AffineTables at, HpGamma hg,
                                                        const double* __restrict__ mu, int B,
                                                        const double* __restrict__ xbar,
                                                        const double2* __restrict__ cxy,
                                                        const double2* __restrict__ dxy, double dp, double delta, const double* __restrict__ inflow,
                                                        long long n, const unsigned char* __restrict__ active,
                                                        double* __restrict__ f, double* __restrict__ jac,
                                                        unsigned long long* __restrict__ pairs, DeviceStatus* st) {
  // Work mapping: with B >= IB a warp is (32/IB targets, IB-instance chunk)
  // and the chunk is the slow grid dimension, so concurrently resident warps
  // sweep spatially adjacent targets (t_order) for the same IB instances and
  // share the cluster positions in L2. With B < IB one thread per
  // (target, instance).
  const long long gidx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = s.n_t;
  unsigned long long cnt = 0;
  long long tt, bb_;
  if (B >= IB) {
    const long long wid = gidx >> 5;
    const int lane = (int)(gidx & 31);
    constexpr int TPW = 32 / IB;
    const long long tgroups = (nt + TPW - 1) / TPW;
    tt = (wid % tgroups) * TPW + lane / IB;
    bb_ = (wid / tgroups) * IB + lane % IB;
  } else {
    tt = gidx / B;
    bb_ = gidx % B;
  }
  if (tt < nt && bb_ < B) {
    const long long t = s.t_order ? s.t_order[tt] : tt;
    const int b = (int)bb_;
    if (!active || active[b]) {
      const double px = xbar[(long long)b * 2 * nt + t], py = xbar[(long long)b * 2 * nt + nt + t];
      const double inv2pi = 1.0 / (2.0 * M_PI);
      // Jacobian accumulators (kernel.hpp:53-61): A = Σ w·rx·ry, C = Σ w with
      // w = sv/q, and Σ w·(ry² − rx²) = S − δ'·C − 2·D from S = Σ sv and
      // D = Σ w·rx² (w·q = sv): one FP64 op fewer per interaction, with the
      // same O(ε·Σ|sv|) absolute rounding as the direct form.
      double fx = 0, fy = 0, ja = 0, jd = 0, jc = 0, js = 0;
      // gs = Γ/2π: sv = gs·(1/q) is the reference's Γ·(1/2π)·(1/q) (rom.hpp:131-132)
      auto add = [&](double sx, double sy, double gs) {
        const double rx = px - sx, ry = py - sy;
        const double q = fma(rx, rx, fma(ry, ry, dp));
        const double u = rcp64(q);
        const double sv = gs * u;
        fx = fma(-ry, sv, fx);
        fy = fma(rx, sv, fy);
        const double w = sv * u;
        const double wrx = w * rx;
        ja = fma(wrx, ry, ja);
        jd = fma(wrx, rx, jd);
        jc += w;
        js += sv;
      };
      const double mub = mu ? mu[b] : 0.0;
      auto cgam = [&](int ci) -> double {
        if (mu) {
          if (hg.gab) {
            const double2 v = hg.gab[ci];
            return fma(mub, v.y, v.x);
          }
          return fma(mub, at.gb[ci], at.ga[ci]) * inv2pi;
        }
        return hg.gc ? hg.gc[ci] : s.gamma_tilde[ci] * inv2pi;
      };
      const double2* cpb = cxy + b;
      // Cluster list, U entries per round: the U list reads, then the 2U
      // position loads are issued before any arithmetic (memory-level
      // parallelism for the L2/HBM-latency-bound gathers); order of the
      // accumulation is unchanged.
      constexpr int U = 4;
      const long long k0 = s.cl_off[t];
      const long long ke = s.cl_off[t + 1];
      unsigned skipped = 0;
      cnt = (unsigned long long)(ke - k0);
      // rom.hpp:129: a centroid coincident with the target is dropped when
      // delta == 0 (only then can it be singular); the check is hoisted out of
      // the δ > 0 loop.
      auto clusters = [&](auto check) {
        constexpr bool CHECK = decltype(check)::value;
        long long k = k0;
        // The next round's list entries are read one round ahead (clamped to
        // the list), so a round waits on the position gathers only.
        int cn[U] = {};
        if (k + U <= ke) {
#pragma unroll
          for (int u = 0; u < U; ++u) cn[u] = s.cl_list[k + u];
        }
        for (; k + U <= ke; k += U) {
          int ci[U];
          double sx[U], sy[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            ci[u] = cn[u];
            const long long kn = k + U + u;
            cn[u] = s.cl_list[kn < ke ? kn : k];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            // n_c·B < 2^32 (host-checked): 32-bit offsets, one IMAD.WIDE per gather
            const double2 p = OFF32 ? cpb[(unsigned)ci[u] * (unsigned)B] : cpb[(long long)ci[u] * B];
            sx[u] = p.x;
            sy[u] = p.y;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (CHECK && sx[u] == px && sy[u] == py) {
              ++skipped;
              continue;
            }
            add(sx[u], sy[u], cgam(ci[u]));
          }
        }
        for (; k < ke; ++k) {
          const int ci = s.cl_list[k];
          const double2 p = cpb[(long long)ci * B];
          const double sx = p.x, sy = p.y;
          if (CHECK && sx == px && sy == py) {
            ++skipped;
            continue;
          }
          add(sx, sy, cgam(ci));
        }
      };
      if (delta == 0.0)
        clusters(std::true_type{});
      else
        clusters(std::false_type{});
      cnt -= skipped;
      const long long pid = s.target_ids[t];
      const int self_loc = hg.self_loc ? hg.self_loc[t] : -1;
      auto dgam = [&](int loc) -> double {
        if (mu) {
          if (hg.gdab) {
            const double2 v = hg.gdab[loc];
            return fma(mub, v.y, v.x);
          }
          return fma(mub, at.dgb[loc], at.dga[loc]) * inv2pi;
        }
        return hg.gd ? hg.gd[loc] : s.direct_gamma[loc] * inv2pi;
      };
      const double2* dpb = dxy + b;
      long long kd = s.d_off[t];
      const long long kde = s.d_off[t + 1];
      for (; kd + 4 <= kde; kd += 4) {
        int loc[4];
        double sx[4], sy[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) loc[u] = s.d_list[kd + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 p = OFF32 ? dpb[(unsigned)loc[u] * (unsigned)B] : dpb[(long long)loc[u] * B];
          sx[u] = p.x;
          sy[u] = p.y;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (hg.self_loc ? loc[u] != self_loc : s.direct_ids[loc[u]] != pid) {
            add(sx[u], sy[u], dgam(loc[u]));
            ++cnt;
          }
      }
      for (; kd < kde; ++kd) {
        const int loc = s.d_list[kd];
        if (hg.self_loc ? loc == self_loc : s.direct_ids[loc] == pid) continue;
        const double2 p = dpb[(long long)loc * B];
        add(p.x, p.y, dgam(loc));
        ++cnt;
      }
      if (inflow) {
        fx = fx + inflow[pid];
        fy = fy + inflow[pid + n];
      }
      const double jb = fma(-2.0, jd, fma(-dp, jc, js));  // Σ w·(ry² − rx²)
      const double j00 = 2.0 * ja, j01 = jb - dp * jc, j10 = jb + dp * jc;
      if (!isfinite(fx) || !isfinite(fy) || !isfinite(j00) || !isfinite(j01) || !isfinite(j10))
        latch_status(st, kStatusNonFiniteVelocity, pid);
      f[(long long)b * 2 * nt + t] = fx;
      f[(long long)b * 2 * nt + nt + t] = fy;
      double* jj = jac + ((long long)b * nt + t) * 4;
      jj[0] = j00;
      jj[1] = j01;
      jj[2] = j10;
      jj[3] = -j00;
    }
  }
  using WR = cub::WarpReduce<unsigned long long>;
  __shared__ typename WR::TempStorage wt[4];
  const unsigned long long sum = WR(wt[threadIdx.x / 32]).Sum(cnt);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(pairs, sum);
}

// hyperpair for the batched march (engine Γ/2π tables present, n_c·B and
// u·B < 2^32): the same arithmetic and per-target summation order as
// hyperpair_kernel, with the table mode (affine (G_A, G_B)/2π or exact Γ̃/2π)
// and the δ = 0 coincidence check as template arguments, 32-bit list
// offsets, and the next round's list entries read without a clamp (the last
// round is peeled), so a round issues only its loads and the pair arithmetic.
// Warp = one target × 32 instances; the instance chunk is the slow index, and
// a CTA's WPC warps take WPC consecutive targets of t_order (they share most
// cluster positions in L1).
struct HpArgs {
  DSurrogate s;
  HpGamma hg;
  const double* mu;
  int B;
  const double* xbar;
  const double2* cxy;
  const double2* dxy;
  double dp;
  const double* inflow;
  long long n;
  const unsigned char* active;
  double* f;
  double* jac;
  unsigned long long* pairs;
  DeviceStatus* st;
  int* sm_ctr;  // per-SM work counters (hyperpair_engine_sm_kernel), zeroed before the launch
};

// Cache-hint probes for the engine kernel's loads (PTROM_HP_HINT, measured in
// profiles/r02_hp_hint_sweep.txt): 0 plain; 1 the list entries do not allocate in
// L1; 2 also the position gathers are kept (evict_last); 3 positions evict_last only.
#ifndef PTROM_HP_HINT
#define PTROM_HP_HINT 0
#endif
__device__ __forceinline__ unsigned hp_ld_list(const int* p) {
#if PTROM_HP_HINT == 1 || PTROM_HP_HINT == 2
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return (unsigned)v;
#else
  return (unsigned)*p;
#endif
}
__device__ __forceinline__ double2 hp_ld_pos(const double2* p) {
#if PTROM_HP_HINT == 2 || PTROM_HP_HINT == 3
  double2 v;
  asm volatile("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// One warp's item: target tt of t_order, instances [32·chunk, 32·chunk + 32).
// Returns the lane's interaction count.
template <bool AFFINE, bool CHECK, int U>
__device__ __forceinline__ unsigned long long hp_engine_item(const HpArgs& a, long long tt, long long chunk, int lane) {
  const DSurrogate& s = a.s;
  const HpGamma& hg = a.hg;
  const int B = a.B;
  const double dp = a.dp;
  const long long nt = s.n_t, n = a.n;
  const int b = (int)(chunk * 32 + lane);
  unsigned long long cnt = 0;
  const double* __restrict__ xbar = a.xbar;
  const double* __restrict__ mu = a.mu;
  const double* __restrict__ inflow = a.inflow;
  const double2* __restrict__ cxy = a.cxy;
  const double2* __restrict__ dxy = a.dxy;
  double* __restrict__ f = a.f;
  double* __restrict__ jac = a.jac;
  DeviceStatus* st = a.st;
  if (b < B && (!a.active || a.active[b])) {
    const long long t = s.t_order ? s.t_order[tt] : tt;
    const double px = xbar[(long long)b * 2 * nt + t], py = xbar[(long long)b * 2 * nt + nt + t];
    double fx = 0, fy = 0, ja = 0, jd = 0, jc = 0, js = 0;
    // the pair law of hyperpair_kernel (Jacobian B term as S − δ'C − 2D)
    auto add = [&](double sx, double sy, double gs) {
      const double rx = px - sx, ry = py - sy;
      const double q = fma(rx, rx, fma(ry, ry, dp));
      const double u = rcp64(q);
      const double sv = gs * u;
      fx = fma(-ry, sv, fx);
      fy = fma(rx, sv, fy);
      const double w = sv * u;
      const double wrx = w * rx;
      ja = fma(wrx, ry, ja);
      jd = fma(wrx, rx, jd);
      jc += w;
      js += sv;
    };
    const double mub = AFFINE ? mu[b] : 0.0;
    auto cgam = [&](unsigned ci) -> double {
      if (AFFINE) {
        const double2 v = __ldg(hg.gab + ci);
        return fma(mub, v.y, v.x);
      }
      return __ldg(hg.gc + ci);
    };
    const double2* cpb = cxy + b;
    const unsigned ub = (unsigned)B;
    const long long k0 = s.cl_off[t];
    const int* lp = s.cl_list + k0;
    const int nk = (int)(s.cl_off[t + 1] - k0);
    unsigned skipped = 0;
    cnt = (unsigned long long)nk;
    int i = 0;
    unsigned cn[U];
    if (nk >= U) {
#pragma unroll
      for (int u = 0; u < U; ++u) cn[u] = hp_ld_list(lp + u);
    }
    auto round = [&](const unsigned (&ci)[U]) {
      double2 p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) p[u] = hp_ld_pos(cpb + ci[u] * ub);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (CHECK && p[u].x == px && p[u].y == py) {  // rom.hpp:129 (δ = 0 only)
          ++skipped;
          continue;
        }
        add(p[u].x, p[u].y, cgam(ci[u]));
      }
    };
    const int* lq = lp + U;  // the next round's entries (immediate offsets)
    for (; i + 2 * U <= nk; i += U, lq += U) {
      unsigned ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ci[u] = cn[u];
        cn[u] = hp_ld_list(lq + u);
      }
      round(ci);
    }
    if (i + U <= nk) {
      round(cn);
      i += U;
    }
    for (; i < nk; ++i) {
      const unsigned ci = (unsigned)lp[i];
      const double2 p = cpb[ci * ub];
      if (CHECK && p.x == px && p.y == py) {
        ++skipped;
        continue;
      }
      add(p.x, p.y, cgam(ci));
    }
    cnt -= skipped;
    const int self_loc = hg.self_loc[t];
    const double2* dpb = dxy + b;
    const long long kd0 = s.d_off[t];
    const int* dl = s.d_list + kd0;
    const int nd = (int)(s.d_off[t + 1] - kd0);
    auto dgam = [&](unsigned loc) -> double {
      if (AFFINE) {
        const double2 v = hg.gdab[loc];
        return fma(mub, v.y, v.x);
      }
      return hg.gd[loc];
    };
    int j = 0;
    for (; j + 4 <= nd; j += 4) {
      unsigned loc[4];
      double2 p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) loc[u] = (unsigned)dl[j + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] = dpb[loc[u] * ub];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if ((int)loc[u] != self_loc) {  // rom.hpp:140
          add(p[u].x, p[u].y, dgam(loc[u]));
          ++cnt;
        }
    }
    for (; j < nd; ++j) {
      const unsigned loc = (unsigned)dl[j];
      if ((int)loc == self_loc) continue;
      const double2 p = dpb[loc * ub];
      add(p.x, p.y, dgam(loc));
      ++cnt;
    }
    const long long pid = s.target_ids[t];
    if (inflow) {
      fx = fx + inflow[pid];
      fy = fy + inflow[pid + n];
    }
    const double jb = fma(-2.0, jd, fma(-dp, jc, js));  // Σ w·(ry² − rx²)
    const double j00 = 2.0 * ja, j01 = jb - dp * jc, j10 = jb + dp * jc;
    if (!isfinite(fx) || !isfinite(fy) || !isfinite(j00) || !isfinite(j01) || !isfinite(j10))
      latch_status(st, kStatusNonFiniteVelocity, pid);
    f[(long long)b * 2 * nt + t] = fx;
    f[(long long)b * 2 * nt + nt + t] = fy;
    double* jj = jac + ((long long)b * nt + t) * 4;
    jj[0] = j00;
    jj[1] = j01;
    jj[2] = j10;
    jj[3] = -j00;
  }
  return cnt;
}

__device__ __forceinline__ void hp_count(unsigned long long cnt, int lane, unsigned long long* pairs) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(pairs, cnt);
}

// Static mapping: warp w → (target w mod n_t, chunk w / n_t); a CTA's WPC
// warps take WPC consecutive targets of t_order.
template <bool AFFINE, bool CHECK, int WPC, int MINB, int U>
__global__ void __launch_bounds__(WPC * 32, MINB) hyperpair_engine_kernel(const __grid_constant__ HpArgs a) {
  const int lane = threadIdx.x & 31;
  const long long wid = blockIdx.x * (long long)WPC + (threadIdx.x >> 5);
  const long long nt = a.s.n_t;
  const long long tt = wid % nt, chunk = wid / nt;
  if (chunk * 32 >= a.B) return;
  hp_count(hp_engine_item<AFFINE, CHECK, U>(a, tt, chunk, lane), lane, a.pairs);
}

// Per-SM mapping (persistent CTAs): SM i owns the targets
// [i·n_t/S, (i+1)·n_t/S) of t_order for every chunk (S = %nsmid), and its
// warps pull items chunk-major from the SM's counter, so all warps resident
// on one SM sweep neighbouring targets of one chunk together (their cluster
// positions meet in the SM's L1). A warp whose SM range is exhausted moves on
// to the next SM's counter (load balance at the tail).
template <bool AFFINE, bool CHECK, int WPC, int MINB, int U>
__global__ void __launch_bounds__(WPC * 32, MINB) hyperpair_engine_sm_kernel(const __grid_constant__ HpArgs a) {
  const int lane = threadIdx.x & 31;
  unsigned smid, nsm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsm));
  nsm = min(nsm, (unsigned)RomScratch::kSmCtr);  // counters allocated (smid >= kSmCtr folds below)
  smid %= nsm;
  const long long nt = a.s.n_t;
  const long long chunks = (a.B + 31) / 32;
  unsigned long long cnt = 0;
  for (unsigned v = 0; v < nsm; ++v) {
    const unsigned sm = (smid + v) % nsm;
    const long long lo = nt * sm / nsm, hi = nt * (sm + 1) / nsm, len = hi - lo;
    if (len == 0) continue;
    const long long items = len * chunks;
    while (true) {
      int item = 0;
      if (lane == 0) item = atomicAdd(a.sm_ctr + sm, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= items) break;
      cnt += hp_engine_item<AFFINE, CHECK, U>(a, lo + item % len, item / len, lane);
    }
  }
  hp_count(cnt, lane, a.pairs);
}

// ------------------------------------------------------ Gauss–Newton ---
// Split-K Gauss–Newton projections: CTA = 8 instances (one warp each) x one
// slice of the sampled rows, 32 rows per chunk. Each chunk's operands are
// staged by cp.async into a two-stage shared-memory ring while the previous
// chunk computes: the A columns and the Φ̄ rows (x and y rows of each
// sampled particle) once per CTA, and per instance warp the x̄, x̄_prev, f̄,
// f̄_prev slices plus the row's half of the 2x2 Jacobian block. Lane l forms
// the residual r̄ and C-row coefficients for row l (rom.hpp:71-84):
// C = Φ̄_own − h·(J_a Φ̄_x + J_b Φ̄_y) = α Φ̄_x + β Φ̄_y; A·C goes to DMMA
// (mma.sync m8n8k4 f64), 4 rows per k-step. Partials [slice][b][32·M + 32 +
// M] are reduced in slice order by gn_finish_kernel (deterministic).

template <int M>
struct GnSmem {
  static constexpr int AS = 36;         // A chunk row stride (doubles), kk-major
  static constexpr int PS = 2 * M + 8;  // Φ̄ chunk row stride: [Φ̄_x (M) | Φ̄_y (M)], ≡ 8 mod 16
  static constexpr int WS = 2 * 32 + 4 * 32;  // per warp: J halves (32 x 2), x̄ x̄p f̄ f̄p (4 x 32)
  static constexpr int STAGE = 32 * AS + 32 * PS + 8 * WS;
  static constexpr int BYTES = (2 * STAGE + 8 * 3 * 32) * 8;
};

template <int M>
__global__ void __launch_bounds__(256, M <= 16 ? 3 : 2) gn_partial_kernel(DGnat g, EngineTables et, int B, double h,
                                                         const double* __restrict__ xbar,
                                                         const double* __restrict__ xprev,
                                                         const double* __restrict__ fbar,
                                                         const double* __restrict__ fprev,
                                                         const double* __restrict__ jac, GnState st_,
                                                         long long slice_len, double* __restrict__ part) {
  using L = GnSmem<M>;
  constexpr int MR = 32, TI = MR / 8, TN = M / 8, PART = MR * M + MR + M, AS = L::AS, PS = L::PS;
  extern __shared__ __align__(16) double gn_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  const bool ok = b < B && st_.active[b];
  const long long nt = g.n_s, rows = 2 * nt;
  const long long bb = ok ? b : 0;
  // lanes 0-15 stage x̄ (f̄), lanes 16-31 x̄_prev (f̄_prev)
  const double* wsrc0 = (lane < 16 ? xbar : xprev) + bb * rows;
  const double* wsrc1 = (lane < 16 ? fbar : fprev) + bb * rows;
  const double* jb = jac + bb * nt * 4;
  const int lr = lane >> 2, lc = lane & 3;
  const bool need_ac = ok && !(st_.evals[b] >= st_.max_iters);
  double* coef = gn_smem + 2 * L::STAGE + warp * 3 * 32;  // r̄, α, β per row of the chunk
  const long long k_begin = blockIdx.y * slice_len, k_end = min(rows, k_begin + slice_len);
  const int n_chunks = (int)((k_end - k_begin + 31) / 32);

  auto issue = [&](int c) {
    double* st = gn_smem + (c & 1) * L::STAGE;
    const long long k0 = k_begin + 32LL * c;
    // A: 32 columns x 32 rows = 512 16-byte units
    for (int u = threadIdx.x; u < 512; u += 256) {
      const int kk = u >> 4, i2 = u & 15;
      const bool v = k0 + kk < k_end;
      cp_async16z(st + kk * AS + 2 * i2, g.A + (v ? (k0 + kk) * MR + 2 * i2 : 0), v);
    }
    // Φ̄ rows of the chunk's particles: 32 x 2M doubles = 32·M units
    double* sp = st + 32 * AS;
    for (int u = threadIdx.x; u < 32 * M; u += 256) {
      const int kk = u / M, q = u % M, half = q / (M / 2), c2 = q % (M / 2);
      const long long r = k0 + kk;
      const bool v = r < k_end;
      const long long t = r < nt ? r : r - nt;
      cp_async16z(sp + kk * PS + half * M + 2 * c2, et.pbr + (v ? (t + half * nt) * M + 2 * c2 : 0), v);
    }
    if (ok) {
      double* sw = st + 32 * AS + 32 * PS + warp * L::WS;
      const long long r = k0 + lane;
      const bool v = r < k_end;
      const long long t = r < nt ? r : r - nt;
      cp_async16z(sw + 2 * lane, jb + (v ? 4 * t + (r < nt ? 0 : 2) : 0), v);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int uu = lane + 32 * e, arr = uu >> 4, q = uu & 15;
        const bool vv = k0 + 2 * q < k_end;
        cp_async16z(sw + 64 + arr * 32 + 2 * q, (e ? wsrc1 : wsrc0) + (vv ? k0 + 2 * q : 0), vv);
      }
    }
  };

  double acc[TI][TN][2];
  double ar[TI];
  double gr[TN];
#pragma unroll
  for (int i = 0; i < TI; ++i) {
    ar[i] = 0.0;
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) gr[j] = 0.0;

  if (n_chunks > 0) issue(0);
  cp_async_commit();
  for (int c = 0; c < n_chunks; ++c) {
    if (c + 1 < n_chunks) issue(c + 1);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const double* st = gn_smem + (c & 1) * L::STAGE;
    const double* sA = st;
    const double* sp = st + 32 * AS;
    if (ok) {
      const double* sw = st + 32 * AS + 32 * PS + warp * L::WS;
      const long long r = k_begin + 32LL * c + lane;
      const double ja = sw[2 * lane], jbv = sw[2 * lane + 1];
      const double x = sw[64 + lane], xp = sw[96 + lane], f = sw[128 + lane], fp = sw[160 + lane];
      const bool xrow = r < nt;
      const double hja = __dmul_rn(h, ja), hjb = __dmul_rn(h, jbv);
      coef[lane] = __dsub_rn(__dsub_rn(x, xp), __dmul_rn(h, __dadd_rn(f, fp)));
      coef[32 + lane] = xrow ? 1.0 - hja : -hja;
      coef[64 + lane] = xrow ? -hjb : 1.0 - hjb;
      __syncwarp();
#pragma unroll
      for (int s4 = 0; s4 < 8; ++s4) {
        const int kk = 4 * s4 + lc;
        const double rvv = coef[kk], al = coef[32 + kk], be = coef[64 + kk];
        double av[TI];
#pragma unroll
        for (int i = 0; i < TI; ++i) {
          av[i] = sA[kk * AS + i * 8 + lr];
          ar[i] = fma(av[i], rvv, ar[i]);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const double cvv = fma(al, sp[kk * PS + j * 8 + lr], be * sp[kk * PS + M + j * 8 + lr]);
          gr[j] = fma(cvv, rvv, gr[j]);
          if (need_ac) {
#pragma unroll
            for (int i = 0; i < TI; ++i) dmma(acc[i][j], av[i], cvv);
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  if (!ok) return;
  double* out = part + ((long long)blockIdx.y * B + b) * PART;
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int row = i * 8 + lr, col = j * 8 + lc * 2;
      out[row + col * MR] = acc[i][j][0];
      out[row + (col + 1) * MR] = acc[i][j][1];
    }
#pragma unroll
  for (int i = 0; i < TI; ++i) {
    double v = ar[i];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (lc == 0) out[MR * M + i * 8 + lr] = v;
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    double v = gr[j];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (lc == 0) out[MR * M + MR + j * 8 + lr] = v;
  }
}

// Slice-ordered reduction + the convergence logic of rom.hpp:309-324.
template <int M>
__global__ void gn_finish_kernel(int B, int S, const double* __restrict__ part, GnState st_) {
  constexpr int MR = 32, PART = MR * M + MR + M;
  const int b = blockIdx.x;
  if (!st_.active[b]) return;
  __shared__ double grad[M];
  for (int e = threadIdx.x; e < PART; e += blockDim.x) {
    double v = 0.0;
    for (int sl = 0; sl < S; ++sl) v += part[((long long)sl * B + b) * PART + e];
    if (e < MR * M) st_.ac[(long long)b * MR * M + e] = v;
    else if (e < MR * M + MR) st_.ar[(long long)b * MR + (e - MR * M)] = v;
    else grad[e - MR * M - MR] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int m = 0; m < M; ++m) ss += grad[m] * grad[m];
    const double gn = sqrt(ss);
    const int evals = ++st_.evals[b];
    bool done = false, conv = false;
    if (evals == 1) {
      st_.g0[b] = gn;
      if (gn == 0.0) done = conv = true;
    } else if (gn / st_.g0[b] <= st_.tol) {
      done = conv = true;
    }
    if (!done && evals - 1 >= st_.max_iters) done = true;
    st_.converged[b] = conv ? 1 : 0;
    if (done) st_.active[b] = 0;
    else atomicAdd(st_.n_active, 1);
  }
}

// --------------------------------------------------------------- update ---
// rom.hpp:325-329: Δ = argmin ‖(A C) Δ + A r̄‖ (ColPivHouseholderQR), x̂ += αΔ.
// One warp per instance; lane i owns row i of the MR x M system.
template <int MR, int M>
__global__ void qr_update_kernel(int B, GnState st_, double alpha, double* __restrict__ xhat) {
  const int b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B || !st_.active[b]) return;
  static_assert(MR == 32, "one lane per residual mode (padded)");
  double a[M];
  const double* ac = st_.ac + (long long)b * MR * M;
#pragma unroll
  for (int j = 0; j < M; ++j) a[j] = ac[lane + j * MR];
  double rhs = -st_.ar[(long long)b * MR + lane];
  int perm[M];
#pragma unroll
  for (int j = 0; j < M; ++j) perm[j] = j;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  double rdiag[M];
  int rank = 0;
  double maxpiv = 0.0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    // pivot: largest remaining column norm (rows >= j)
    int best = j;
    double bestn = -1.0;
#pragma unroll
    for (int c = j; c < M; ++c) {
      const double nc = wsum(lane >= j ? a[c] * a[c] : 0.0);
      if (nc > bestn) {
        bestn = nc;
        best = c;
      }
    }
#pragma unroll
    for (int c = j + 1; c < M; ++c)
      if (c == best) {
        const double t = a[j];
        a[j] = a[c];
        a[c] = t;
        const int tp = perm[j];
        perm[j] = perm[c];
        perm[c] = tp;
      }
    // Householder on column j, rows >= j (Eigen's makeHouseholder convention)
    const double x0 = __shfl_sync(0xffffffffu, a[j], j);
    const double tail = wsum(lane > j ? a[j] * a[j] : 0.0);
    double beta = x0, tau = 0.0, denom = 1.0;
    if (tail > 2.2250738585072014e-308) {
      beta = sqrt(x0 * x0 + tail);
      if (x0 >= 0) beta = -beta;
      tau = (beta - x0) / beta;
      denom = x0 - beta;
    }
    const double v = lane == j ? 1.0 : (lane > j ? a[j] / denom : 0.0);
    // apply H = I - tau v v^T to the remaining columns and the rhs
#pragma unroll
    for (int c = j + 1; c < M; ++c) {
      const double w = tau * wsum(v * a[c]);
      a[c] -= w * v;
    }
    rhs -= tau * wsum(v * rhs) * v;
    rdiag[j] = beta;
    if (j == 0) maxpiv = fabs(beta);
    if (fabs(beta) > 2.220446049250313e-16 * M * maxpiv) rank = j + 1;
    if (lane == j) a[j] = beta;
    else if (lane > j) a[j] = 0.0;
  }
  // back substitution on the leading rank rows (lane i holds row i of R)
  double z[M];
#pragma unroll
  for (int j = 0; j < M; ++j) z[j] = 0.0;
  for (int i = rank - 1; i >= 0; --i) {
    double s = __shfl_sync(0xffffffffu, rhs, i);
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (j > i && j < rank) s -= __shfl_sync(0xffffffffu, a[j], i) * z[j];
    z[i] = s / rdiag[i];
  }
  if (lane == 0) {
    double* xh = xhat + (long long)b * M;
#pragma unroll
    for (int j = 0; j < M; ++j) xh[perm[j]] += alpha * z[j];
  }
}

__global__ void record_step_kernel(int B, int M, int MP, long long step, long long n_steps,
                                   const double* __restrict__ xhat, GnState st_, double* __restrict__ xhat_out,
                                   int* __restrict__ iters, unsigned char* __restrict__ conv) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  for (int j = 0; j < M; ++j) xhat_out[((long long)b * n_steps + step) * M + j] = xhat[(long long)b * MP + j];
  iters[(long long)b * n_steps + step] = st_.evals[b];
  conv[(long long)b * n_steps + step] = st_.converged[b];
}

__global__ void reset_step_kernel(int B, GnState st_) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  st_.evals[b] = 0;
  st_.active[b] = 1;
  st_.converged[b] = 0;
}

int blocks_for(long long count, int tpb) { return (int)std::max(1LL, (count + tpb - 1) / tpb); }

}  // namespace

// reconstruct_output / reconstruct_full (rom.hpp:45-64): out(k, s) = x_ref[d_k] + Φ(d_k,:)·x̂(:, s).
// One thread per output row d_k keeps Φ's row in registers (M ≤ 32; one
// coalesced read of Φ per column) and walks the steps with x̂ staged in
// shared memory (≤ 32 steps per stage); writes are coalesced along k.
template <int MAXM>
__global__ void __launch_bounds__(128) reconstruct_kernel(DBasis b, long long n_steps, const double* __restrict__ xh,
                                                          long long n_out, const long long* __restrict__ dofs,
                                                          double* __restrict__ out) {
  constexpr int SS = 32;
  __shared__ double xs[SS * MAXM];
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nd = 2 * b.n;
  const int m = b.m;
  long long d = k < n_out ? (dofs ? dofs[k] : k) : 0;
  double row[MAXM];
#pragma unroll
  for (int j = 0; j < MAXM; ++j) row[j] = (j < m && k < n_out) ? b.phi[d + j * nd] : 0.0;
  const double xr = k < n_out ? b.x_ref[d] : 0.0;
  for (long long s0 = 0; s0 < n_steps; s0 += SS) {
    const int cnt = (int)min((long long)SS, n_steps - s0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * m; e += blockDim.x) xs[e] = xh[s0 * m + e];
    __syncthreads();
    if (k < n_out) {
      for (int s = 0; s < cnt; ++s) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < MAXM; ++j)
          if (j < m) acc = fma(row[j], xs[s * m + j], acc);
        out[k + (s0 + s) * n_out] = acc + xr;
      }
    }
  }
}

// ------------------------------------------------------------- drivers ---
void rom_reconstruct(ptrom_ctx* ctx, const DBasis& b, long long n_steps, const double* d_xhat, long long n_out,
                     const long long* d_dofs, double* d_out) {
  if (n_out <= 0 || n_steps <= 0) return;
  if (b.m > 32) throw status_error(PTROM_CONFIG_ERROR, "reconstruct: at most 32 modes");
  reconstruct_kernel<32><<<blocks_for(n_out, 128), 128, 0, ctx->stream>>>(b, n_steps, d_xhat, n_out, d_dofs, d_out);
  PTROM_LAUNCH_CHECK();
}

void rom_basis_rowmajor(ptrom_ctx* ctx, DBasis& b) {
  PTROM_CUDA(cudaMalloc(&b.rm, sizeof(double) * std::max<long long>(1, b.n * 2 * (b.m + 1))));
  basis_rowmajor_kernel<<<std::max(1, ctx->num_sms * 8), 256, 0, ctx->stream>>>(b);
  PTROM_LAUNCH_CHECK();
}

void rom_reassign_exact(ptrom_ctx* ctx, DSurrogate& s, const DBasis& b, const double* d_gamma) {
  if (s.n_c > 0) {
    if (b.m > 63) throw status_error(PTROM_CONFIG_ERROR, "reassign: at most 63 modes");
    const long long big_thr = std::max<long long>(32, ctx->reassign_big);
    // Clusters above big_thr members: one CTA each. Their count is known on
    // the host from the membership offsets' maximum, which the surrogate
    // records when it is built (max_members); the CTA path is launched only
    // when some cluster needs it.
    if (s.max_members > big_thr) {
      int* big;  // [0] count, then the list of clusters above big_thr members
      PTROM_CUDA(cudaMallocAsync(&big, sizeof(int) * (s.n_c + 1), ctx->stream));
      PTROM_CUDA(cudaMemsetAsync(big, 0, sizeof(int), ctx->stream));
      big_clusters_kernel<<<blocks_for(s.n_c, 256), 256, 0, ctx->stream>>>(s, big_thr, big + 1, big);
      // members per weighted-pass chunk: the largest multiple of 32 (<= 256)
      // whose double-buffered rows fit the opt-in shared memory of one CTA
      const size_t row = sizeof(double) * 2 * (b.m + 1);
      const size_t fixed_b = sizeof(double) * 2 * kBigGChunk;
      int ch = 256;
      auto bytes = [&](int c) {
        return 2 * (size_t)c * row + sizeof(double) * 2 * (size_t)std::max(c, kBigGChunk) +
               sizeof(long long) * 2 * (size_t)c;
      };
      while (ch > 32 && bytes(ch) > (size_t)ctx->smem_optin) ch -= 32;
      (void)fixed_b;
      const size_t smem = bytes(ch);
      PTROM_CUDA(cudaFuncSetAttribute(reassign_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      reassign_big_kernel<<<ctx->num_sms, 256, smem, ctx->stream>>>(s, b, d_gamma, big + 1, big, ch);
      PTROM_CUDA(cudaFreeAsync(big, ctx->stream));
    }
    reassign_exact_kernel<<<blocks_for(s.n_c * 32, 256), 256, 0, ctx->stream>>>(s, b, d_gamma, big_thr);
  }
  if (s.u > 0) direct_gamma_kernel<<<blocks_for(s.u, 256), 256, 0, ctx->stream>>>(s, d_gamma);
  PTROM_LAUNCH_CHECK();
}

void rom_affine_tables(ptrom_ctx* ctx, const DSurrogate& s, const DBasis& b, const double* d_ga, const double* d_gb,
                       AffineTables& t) {
  const long long work = s.n_c * (s.m + 1);
  if (work > 0) affine_tables_kernel<<<blocks_for(work * 32, 256), 256, 0, ctx->stream>>>(s, b, d_ga, d_gb, t);
  PTROM_LAUNCH_CHECK();
}

template <int MP>
void launch_positions_mma(ptrom_ctx* ctx, const DSurrogate& s, const AffineTables* t, const EngineTables& et, int B,
                          const double* d_xhat, const double* d_mu, const unsigned char* d_active, RomScratch& w) {
  cudaStream_t st = ctx->stream;
  AffineTables empty{};
  const AffineTables& tt = t ? *t : empty;
  if (s.n_c > 0) {
    const int ic = PosSmem<MP>::ic(B);
    const size_t smem = PosSmem<MP>::bytes(ic);
    const long long ctiles = (s.n_c + 3) / 4;
    const int grid = (int)std::max<long long>(1, std::min<long long>(2LL * ctx->num_sms, (ctiles + 15) / 16));
    if (t) {
      PTROM_CUDA(cudaFuncSetAttribute(positions_clusters_mma_kernel<true, MP>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      positions_clusters_mma_kernel<true, MP><<<grid, 512, smem, st>>>(s.n_c, et.ct, nullptr, tt, B, ic, d_xhat, d_mu,
                                                                      nullptr, w.cxy, ctx->d_status);
    } else {
      PTROM_CUDA(cudaFuncSetAttribute(positions_clusters_mma_kernel<false, MP>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      positions_clusters_mma_kernel<false, MP><<<grid, 512, smem, st>>>(s.n_c, et.ct, s.x0_tilde, tt, B, ic, d_xhat,
                                                                       d_mu, nullptr, w.cxy, ctx->d_status);
    }
  }
  if (s.u > 0) {
    // source positions are written for every instance: hyperpair skips the
    // inactive ones (their x̂ is frozen), so the stores stay vectorised
    const int ic = PosSmem<MP>::ic(B);
    const size_t smem = PosSmem<MP>::bytes(ic);
    const long long dtiles = (s.u + 3) / 4;
    const int grid = (int)std::max<long long>(1, std::min<long long>(2LL * ctx->num_sms, (dtiles + 15) / 16));
    PTROM_CUDA(cudaFuncSetAttribute(positions_clusters_mma_kernel<false, MP>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    positions_clusters_mma_kernel<false, MP><<<grid, 512, smem, st>>>(s.u, et.dt, s.direct_x0, tt, B, ic, d_xhat,
                                                                     nullptr, nullptr, w.dxy, ctx->d_status);
  }
  PTROM_LAUNCH_CHECK();
}

// Positions + hyperpair for B instances (active mask may be null). With
// engine tables (the batched march) source positions use the DMMA kernels;
// without (single hyperpair calls) the scalar ones.
unsigned long long rom_hyperpair(ptrom_ctx* ctx, const DSurrogate& s, const DGnat* g, const AffineTables* t,
                                 const EngineTables* et, int B, int xs, const double* d_xhat, const double* d_mu,
                                 const unsigned char* d_active, const double* d_xbar_in, double* d_xbar_out,
                                 double delta, int form, const double* d_inflow, long long n, RomScratch& w,
                                 double* d_f, double* d_jac, bool count_pairs) {
  cudaStream_t st = ctx->stream;
  AffineTables empty{};
  const AffineTables& tt = t ? *t : empty;
  if (et) {
    switch (xs) {
      case 8: launch_positions_mma<8>(ctx, s, t, *et, B, d_xhat, d_mu, d_active, w); break;
      case 16: launch_positions_mma<16>(ctx, s, t, *et, B, d_xhat, d_mu, d_active, w); break;
      case 24: launch_positions_mma<24>(ctx, s, t, *et, B, d_xhat, d_mu, d_active, w); break;
      default: launch_positions_mma<32>(ctx, s, t, *et, B, d_xhat, d_mu, d_active, w); break;
    }
  } else {
    if (s.n_c > 0) {
      if (t)
        positions_clusters_kernel<true><<<blocks_for(s.n_c * B, 256), 256, 0, st>>>(s, tt, B, xs, d_xhat, d_mu, d_active,
                                                                                   w.cxy, ctx->d_status);
      else
        positions_clusters_kernel<false><<<blocks_for(s.n_c * B, 256), 256, 0, st>>>(s, tt, B, xs, d_xhat, d_mu,
                                                                                    d_active, w.cxy, ctx->d_status);
    }
    if (s.u > 0)
      positions_direct_kernel<<<blocks_for(s.u * B, 256), 256, 0, st>>>(s, B, xs, d_xhat, d_active, w.dxy);
  }
  const double* xbar = d_xbar_in;
  if (g) {
    const dim3 grid((unsigned)((2 * g->n_s + 255) / 256), (unsigned)((B + 31) / 32));
    switch (g->mp) {
      case 8: positions_targets_kernel<8><<<grid, 256, 0, st>>>(*g, B, d_xhat, d_active, d_xbar_out); break;
      case 16: positions_targets_kernel<16><<<grid, 256, 0, st>>>(*g, B, d_xhat, d_active, d_xbar_out); break;
      case 24: positions_targets_kernel<24><<<grid, 256, 0, st>>>(*g, B, d_xhat, d_active, d_xbar_out); break;
      default: positions_targets_kernel<32><<<grid, 256, 0, st>>>(*g, B, d_xhat, d_active, d_xbar_out); break;
    }
    xbar = d_xbar_out;
  }
  PTROM_LAUNCH_CHECK();
  if (count_pairs) PTROM_CUDA(cudaMemsetAsync(w.pairs, 0, 8, st));
  {
    ProfScope prof(ctx);
    // IB = 32: one 256-byte segment per position row and instance chunk (8-instance
    // chunks doubled the DRAM traffic: half-used L2 lines).
    constexpr int IB = 32;
    const long long threads = B >= IB ? ((s.n_t + 32 / IB - 1) / (32 / IB)) * 32 * ((B + IB - 1) / IB) : s.n_t * B;
    HpGamma hg;
    if (et) {
      hg.self_loc = et->hself;
      hg.gc = et->hgc;
      hg.gab = et->hgab;
      hg.gd = et->hgd;
      hg.gdab = et->hgdab;
    }
    const bool off32 = (double)std::max(s.n_c, s.u) * (double)B < 4294967296.0;
    const int var = ctx->hp_variant;
    // the engine maps 32 instances to a warp: below 32 instances (the
    // single-instance drop-in, small batches) the generic kernel's one thread
    // per (target, instance) keeps the lanes full
    if (et && off32 && s.n_t > 0 && var != 1 && B >= 32) {
      // batched march: hyperpair_engine_kernel (template table mode, no clamps)
      HpArgs ha{s, hg, t ? d_mu : nullptr, B, xbar, w.cxy, w.dxy, effective_delta(delta, form), d_inflow, n,
                d_active, d_f, d_jac, w.pairs, ctx->d_status, w.sm_ctr};
      const long long warps = s.n_t * ((B + 31) / 32);
      const bool chk = delta == 0.0;
      auto launch = [&](auto wpc_tag, auto minb_tag, auto u_tag, auto per_sm_tag) {
        constexpr int WPC = decltype(wpc_tag)::value, MINB = decltype(minb_tag)::value, UU = decltype(u_tag)::value;
        if constexpr (decltype(per_sm_tag)::value) {
          PTROM_CUDA(cudaMemsetAsync(w.sm_ctr, 0, sizeof(int) * RomScratch::kSmCtr, st));
          const unsigned blocks = (unsigned)(ctx->num_sms * MINB);
          auto k = t ? (chk ? hyperpair_engine_sm_kernel<true, true, WPC, MINB, UU>
                            : hyperpair_engine_sm_kernel<true, false, WPC, MINB, UU>)
                     : (chk ? hyperpair_engine_sm_kernel<false, true, WPC, MINB, UU>
                            : hyperpair_engine_sm_kernel<false, false, WPC, MINB, UU>);
          k<<<blocks, WPC * 32, 0, st>>>(ha);
        } else {
          const unsigned blocks = (unsigned)((warps + WPC - 1) / WPC);
          auto k = t ? (chk ? hyperpair_engine_kernel<true, true, WPC, MINB, UU>
                            : hyperpair_engine_kernel<true, false, WPC, MINB, UU>)
                     : (chk ? hyperpair_engine_kernel<false, true, WPC, MINB, UU>
                            : hyperpair_engine_kernel<false, false, WPC, MINB, UU>);
          k<<<blocks, WPC * 32, 0, st>>>(ha);
        }
      };
      // Measured on config 4 (B = 512, tools/sweep_hp.py, profiles/r02_sweep_hyperpair.jsonl):
      // generic kernel 4.92 ms; engine U = 4 at 28 / 32 / 36 warps per SM 5.01 / 4.55 / 4.42 ms;
      // U = 3 at 36 warps (56 registers) 4.40 ms (default); fewer registers spill (U = 2/3 at
      // 40-44 warps: 4.7-9.0 ms); per-SM target ranges 4.84 ms.
      using C4 = std::integral_constant<int, 4>;
      using C3 = std::integral_constant<int, 3>;
      using C9 = std::integral_constant<int, 9>;
      switch (var) {
        case 2: launch(C4{}, std::integral_constant<int, 8>{}, C4{}, std::false_type{}); break;  // U = 4, 32 warps/SM
        case 3: launch(C4{}, std::integral_constant<int, 8>{}, C4{}, std::true_type{}); break;   // per-SM target ranges
        default: launch(C4{}, C9{}, C3{}, std::false_type{}); break;                 // U = 3, 36 warps/SM
      }
    } else {
      auto hk = off32 ? hyperpair_kernel<IB, true> : hyperpair_kernel<IB, false>;
      hk<<<blocks_for(threads, 128), 128, 0, st>>>(s, tt, hg, t ? d_mu : nullptr, B, xbar, w.cxy, w.dxy,
                                                   effective_delta(delta, form), delta, d_inflow, n, d_active, d_f,
                                                   d_jac, w.pairs, ctx->d_status);
    }
  }
  PTROM_LAUNCH_CHECK();
  unsigned long long h = 0;
  if (count_pairs) {
    PTROM_CUDA(cudaMemcpyAsync(&h, w.pairs, 8, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaStreamSynchronize(st));
  }
  return h;
}

void RomScratch::ensure(const DSurrogate& s, long long nt, int B) {
  const size_t need_c = (size_t)std::max<long long>(1, s.n_c) * B, need_d = (size_t)std::max<long long>(1, s.u) * B;
  if (need_c > cap_c) {
    cudaFree(cxy);
    PTROM_CUDA(cudaMalloc(&cxy, need_c * 16));
    cap_c = need_c;
  }
  if (need_d > cap_d) {
    cudaFree(dxy);
    PTROM_CUDA(cudaMalloc(&dxy, need_d * 16));
    cap_d = need_d;
  }
  if (!pairs) PTROM_CUDA(cudaMalloc(&pairs, 16));
  if (!sm_ctr) PTROM_CUDA(cudaMalloc(&sm_ctr, sizeof(int) * kSmCtr));
  (void)nt;
}
void RomScratch::release() {
  void* ps[] = {cxy, dxy, pairs, sm_ctr};
  for (void* p : ps)
    if (p) cudaFree(p);
  *this = RomScratch{};
}

// GnatSolver::simulate (rom.hpp:292-340) for B instances in lock step.
// Outputs: xhat_out [B][n_steps][M], iters/conv [B][n_steps].
template <int MP>
unsigned long long gnat_simulate_t(ptrom_ctx* ctx, const DSurrogate& s, const DGnat& g, const AffineTables* t, int B,
                                   const double* d_mu, double delta, int form, const double* d_inflow, long long n,
                                   double dt, long long n_steps, double tol, int max_iters, double alpha,
                                   double* d_xhat_out, int* d_iters, unsigned char* d_conv) {
  cudaStream_t st = ctx->stream;
  const long long nt = g.n_s, rows = 2 * nt;
  RomScratch w;
  w.ensure(s, nt, B);
  struct Bufs {
    std::vector<void*> p;
    cudaStream_t s;
    RomScratch* w;
    ~Bufs() {
      for (void* q : p) cudaFreeAsync(q, s);
      cudaStreamSynchronize(s);
      w->release();
    }
  } bufs{{}, st, &w};
  auto alloc = [&](size_t bytes) {
    void* q;
    PTROM_CUDA(cudaMallocAsync(&q, std::max<size_t>(bytes, 8), st));
    bufs.p.push_back(q);
    return q;
  };
  double* xhat = (double*)alloc((size_t)B * MP * 8);
  double* xbar = (double*)alloc((size_t)B * rows * 8);
  double* xprev = (double*)alloc((size_t)B * rows * 8);
  double* fbar = (double*)alloc((size_t)B * rows * 8);
  double* fprev = (double*)alloc((size_t)B * rows * 8);
  double* jac = (double*)alloc((size_t)B * nt * 4 * 8);
  GnState gs;
  gs.ac = (double*)alloc((size_t)B * 32 * MP * 8);
  gs.ar = (double*)alloc((size_t)B * 32 * 8);
  gs.g0 = (double*)alloc((size_t)B * 8);
  gs.evals = (int*)alloc((size_t)B * 4);
  gs.active = (unsigned char*)alloc(B);
  gs.converged = (unsigned char*)alloc(B);
  gs.n_active = (int*)alloc(4);
  gs.tol = tol;
  gs.max_iters = max_iters;
  EngineTables et;
  et.q = t ? 4 : 2;
  et.ct = (double*)alloc((size_t)s.n_c * et.q * MP * 8);
  et.dt = (double*)alloc((size_t)s.u * 2 * MP * 8);
  et.pbr = (double*)alloc((size_t)rows * MP * 8);
  {
    AffineTables empty{};
    const long long total = s.n_c * et.q * MP + s.u * 2 * MP + rows * MP;
    engine_tables_kernel<<<blocks_for(total, 256), 256, 0, st>>>(s, t ? *t : empty, g, et.q, MP, et);
    PTROM_LAUNCH_CHECK();
  }
  if (t) {
    et.hgab = (double2*)alloc((size_t)std::max<long long>(1, s.n_c) * 16);
    et.hgdab = (double2*)alloc((size_t)std::max<long long>(1, s.u) * 16);
  } else {
    et.hgc = (double*)alloc((size_t)std::max<long long>(1, s.n_c) * 8);
    et.hgd = (double*)alloc((size_t)std::max<long long>(1, s.u) * 8);
  }
  et.hself = (int*)alloc((size_t)std::max<long long>(1, s.n_t) * 4);
  if (s.n_t > 0) hp_self_kernel<<<blocks_for(s.n_t, 256), 256, 0, st>>>(s, et.hself);
  {
    AffineTables empty2{};
    hp_gamma_kernel<<<std::max(1, ctx->num_sms * 4), 256, 0, st>>>(s, t ? *t : empty2, t != nullptr, et.hgc, et.hgab,
                                                                   et.hgd, et.hgdab);
    PTROM_LAUNCH_CHECK();
  }
  // split-K shape: ~4 CTAs per SM over ceil(B/8) instance groups
  const long long groups = (B + 7) / 8;
  const int S = (int)std::max<long long>(1, std::min<long long>(64, (8LL * ctx->num_sms + groups - 1) / groups));
  const long long slice_len = ((rows + S - 1) / S + 31) / 32 * 32;
  const size_t gn_smem = GnSmem<MP>::BYTES;
  PTROM_CUDA(cudaFuncSetAttribute(gn_partial_kernel<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gn_smem));
  double* part = (double*)alloc((size_t)S * B * (32 * MP + 32 + MP) * 8);
  int* h_active = nullptr;
  PTROM_CUDA(cudaMallocHost(&h_active, 4));
  PTROM_CUDA(cudaMemsetAsync(xhat, 0, (size_t)B * MP * 8, st));
  PTROM_CUDA(cudaMemsetAsync(w.pairs, 0, 8, st));
  const double h = dt / 2.0;
  // rom.hpp:298-300: x̄_prev = x̄⁰, f̄_prev = hyperpair(x̄⁰, 0). The step-start
  // evaluation of rom.hpp:306-307 (x̄ = x̄⁰ + Φ̄x̂, (f̄, J) = hyperpair(x̄, x̂))
  // is at the x̂ of the previous evaluation of every instance, so it is the
  // same deterministic computation on the same inputs: its result is already
  // in (x̄, f̄, J) — at step 0 from this call (x̂ = 0 gives x̄ = x̄⁰ exactly, and
  // the fused kernel returns the velocity-only call's f̄ bit for bit), later
  // from the last evaluation of the previous step (inactive instances keep
  // theirs). It is reused instead of recomputed; x̄_prev/f̄_prev get copies.
  rom_hyperpair(ctx, s, &g, t, &et, B, MP, xhat, d_mu, nullptr, nullptr, xbar, delta, form, d_inflow, n, w, fbar,
                jac, false);
  const size_t row_bytes = (size_t)B * rows * 8;
  PTROM_CUDA(cudaMemcpyAsync(xprev, xbar, row_bytes, cudaMemcpyDeviceToDevice, st));
  PTROM_CUDA(cudaMemcpyAsync(fprev, fbar, row_bytes, cudaMemcpyDeviceToDevice, st));
  for (long long step = 0; step < n_steps; ++step) {
    reset_step_kernel<<<blocks_for(B, 256), 256, 0, st>>>(B, gs);
    while (true) {
      PTROM_CUDA(cudaMemsetAsync(gs.n_active, 0, 4, st));
      gn_partial_kernel<MP><<<dim3((unsigned)((B + 7) / 8), (unsigned)S), 256, gn_smem, st>>>(
          g, et, B, h, xbar, xprev, fbar, fprev, jac, gs, slice_len, part);
      gn_finish_kernel<MP><<<B, 128, 0, st>>>(B, S, part, gs);
      PTROM_LAUNCH_CHECK();
      PTROM_CUDA(cudaMemcpyAsync(h_active, gs.n_active, 4, cudaMemcpyDeviceToHost, st));
      PTROM_CUDA(cudaStreamSynchronize(st));
      if (*h_active == 0) break;
      qr_update_kernel<32, MP><<<blocks_for(B, 4), 128, 0, st>>>(B, gs, alpha, xhat);
      PTROM_LAUNCH_CHECK();
      rom_hyperpair(ctx, s, &g, t, &et, B, MP, xhat, d_mu, gs.active, nullptr, xbar, delta, form, d_inflow, n, w,
                    fbar, jac, false);
    }
    record_step_kernel<<<blocks_for(B, 128), 128, 0, st>>>(B, g.m, MP, step, n_steps, xhat, gs, d_xhat_out, d_iters,
                                                            d_conv);
    PTROM_LAUNCH_CHECK();
    // rom.hpp:336-337: history <- accepted state; (x̄, f̄, J) stay as the next
    // step's start evaluation
    PTROM_CUDA(cudaMemcpyAsync(xprev, xbar, row_bytes, cudaMemcpyDeviceToDevice, st));
    PTROM_CUDA(cudaMemcpyAsync(fprev, fbar, row_bytes, cudaMemcpyDeviceToDevice, st));
  }
  unsigned long long pairs = 0;
  PTROM_CUDA(cudaMemcpyAsync(&pairs, w.pairs, 8, cudaMemcpyDeviceToHost, st));
  PTROM_CUDA(cudaStreamSynchronize(st));
  cudaFreeHost(h_active);
  check_device_status(ctx);
  return pairs;
}

unsigned long long rom_gnat_simulate(ptrom_ctx* ctx, const DSurrogate& s, const DGnat& g, const AffineTables* t,
                                     int B, const double* d_mu, double delta, int form, const double* d_inflow,
                                     long long n, double dt, long long n_steps, double tol, int max_iters,
                                     double alpha, double* d_xhat_out, int* d_iters, unsigned char* d_conv) {
  if (g.m_r > 32 || g.m > 32) config_fail("ptrom online engine supports at most 32 modes and 32 residual modes");
  switch (g.mp) {
    case 8:
      return gnat_simulate_t<8>(ctx, s, g, t, B, d_mu, delta, form, d_inflow, n, dt, n_steps, tol, max_iters, alpha,
                                d_xhat_out, d_iters, d_conv);
    case 16:
      return gnat_simulate_t<16>(ctx, s, g, t, B, d_mu, delta, form, d_inflow, n, dt, n_steps, tol, max_iters, alpha,
                                 d_xhat_out, d_iters, d_conv);
    case 24:
      return gnat_simulate_t<24>(ctx, s, g, t, B, d_mu, delta, form, d_inflow, n, dt, n_steps, tol, max_iters, alpha,
                                 d_xhat_out, d_iters, d_conv);
    default:
      return gnat_simulate_t<32>(ctx, s, g, t, B, d_mu, delta, form, d_inflow, n, dt, n_steps, tol, max_iters, alpha,
                                 d_xhat_out, d_iters, d_conv);
  }
}

}  // namespace ptrom
