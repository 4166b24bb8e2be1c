// allpairs.cu — O(N^2) regularized Biot–Savart evaluation on sm_100a.
//
// Replaces the scalar double loops of the reference:
//   pairwise_velocity       kernel.hpp:107-129  (kernel_pair kernel.hpp:29-42)
//   inexact_kernel_jacobian kernel.hpp:154-170  (kernel_pair_jacobian kernel.hpp:45-73)
//
// Both kernel forms reduce to one law with Γ' = Γ/(2π):
//   standard:           pre = Γ/(2π(d²+δ))       = Γ'/(d²+δ)
//   denominator_scaled: pre = Γ/(2πd²+δ)         = Γ'/(d²+δ/(2π))
// so the device works with q = d² + δ' (δ' = δ or δ/2π) and s = Γ'/q:
//   v  += s·(−ry, rx)
//   J  += s/q·[[2rx·ry, ry²−rx²−δ'], [ry²−rx²+δ', −2rx·ry]]
// and the Jacobian is accumulated as A=Σw·rx·ry, B=Σw·(ry²−rx²), C=Σw
// (w = s/q): J = [[2A, B−δ'C], [B+δ'C, −2A]].
//
// Work decomposition (FP64-pipe bound):
//   grid.x = target tiles of TPB·T targets (T targets per thread kept in
//   registers), grid.y = source chunks chosen so grid.x·grid.y fills whole
//   waves of resident blocks on 148 SMs. Each block streams its source chunk
//   through shared memory in tiles of TPB sources (double2 position + Γ'
//   broadcast loads) and writes one partial per (target, chunk); a reduce
//   kernel sums the chunks in ascending order (fixed-order, deterministic),
//   adds the inflow and latches a numerical error on a non-finite result
//   (a coincident pair with δ = 0, the reference's throw at kernel.hpp:38-39).
//
// Reciprocal (the FP64 pipe is the bound):
//  * fast path (δ' ∈ [2^-62, 2^60] and every coordinate of the tile and of the
//    block's targets below 2^29, so q ∈ [2^-62, 2^62)): two targets share one
//    reciprocal of P = q1·q2 (Montgomery); the double P is re-biased into an
//    fp32 bit pattern with integer ops (ALU pipe), seeded with MUFU.RCP (fp32,
//    ≤ 2^-22 rel incl. truncation) and refined by one fp64 Newton step:
//    |rel err| ≤ 1e-13 per term. 9 FP64 + 2 ALU/MUFU ops per velocity pair.
//  * safe path (δ' tiny or huge coordinates, masked self tiles): MUFU.RCP64H
//    seed + cubic correction y0(1+e+e²) (~1 ulp, 10 FP64 ops); q = 0
//    propagates inf/NaN so a coincident pair with δ = 0 is detected.
#include <algorithm>
#include <cmath>

#include "ops.cuh"
#include "pair_tile.cuh"

namespace ptrom {

constexpr int kMaxPeers = 8;  // ranks whose source blocks one kernel reads in place

// Source position loaders. SrcFlat: the SoA state of one device.
// SrcPeers: the sources are split over G ranks (offsets off[0..G]); rank r's
// SoA block (x then y, off[r+1]-off[r] each) lives in its own HBM and is read
// in place over NVLink (CUDA IPC mappings) — the per-evaluation exchange of
// the sharded FOM fused into the tile loads instead of an all-gather.
struct SrcFlat {
  const double* xs;
  const double* ys;
  __device__ __forceinline__ void load(long long j, double& x, double& y) const {
    x = xs[j];
    y = ys[j];
  }
};
struct SrcPeers {
  const double* base[kMaxPeers];
  long long off[kMaxPeers + 1];
  int G;
  __device__ __forceinline__ void load(long long j, double& x, double& y) const {
    int r = 0;
#pragma unroll
    for (int q = 1; q < kMaxPeers; ++q) r += (q < G && j >= off[q]) ? 1 : 0;
    const long long jl = j - off[r], m = off[r + 1] - off[r];
    x = base[r][jl];
    y = base[r][m + jl];
  }
};

// Velocity epilogue fused into the tile kernel: the last CTA to finish a
// target tile (arrival counter per tile) adds that tile's chunk partials in
// chunk order — the same fixed order as reduce_velocity_f64_kernel, so the
// result is bit-identical — adds the inflow, latches non-finite results and
// writes f; f == nullptr keeps the separate reduction.
struct FusedOut {
  double* f = nullptr;
  long long ld = 0, n_total = 0;
  const double* inflow = nullptr;
  unsigned* tile_ctr = nullptr;
  DeviceStatus* st = nullptr;
};

template <int TPB, int T, int UNR, int MINB, bool VEL, bool JAC, int F4 = 4, class Src = SrcFlat>
__global__ void __launch_bounds__(TPB, MINB) allpairs_f64_kernel(long long n, Src src,
                                                           const double* __restrict__ gam, double inv2pi,
                                                           double dp, long long t_begin, long long t_count,
                                                           long long chunk_len, double* __restrict__ part,
                                                           const double* __restrict__ txs,
                                                           const double* __restrict__ tys, long long t_base,
                                                           int self_excl, FusedOut fo) {
  // Targets i in [t_begin, t_begin + t_count) are rows i - t_base of
  // (txs, tys); self_excl = targets are sources with the same global index,
  // so pair (i, i) is skipped. External targets (lattice vertices,
  // kernel.hpp:213-238) pass self_excl = 0.
  constexpr int NCOMP = (VEL ? 2 : 0) + (JAC ? 3 : 0);
  __shared__ double2 sp[TPB];
  __shared__ double sg[TPB];

  const int tid = threadIdx.x;
  const long long tile0 = t_begin + (long long)blockIdx.x * (TPB * T);
  double tx[T], ty[T], fx[T], fy[T], ja[T], jb[T], jc[T];
  long long ti[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const long long i = tile0 + k * TPB + tid;
    const bool ok = i < t_begin + t_count;
    ti[k] = ok ? i : -1;
    tx[k] = ok ? txs[i - t_base] : 0.0;
    ty[k] = ok ? tys[i - t_base] : 0.0;
    fx[k] = fy[k] = ja[k] = jb[k] = jc[k] = 0.0;
  }
  const long long tile_end = min(tile0 + (long long)TPB * T, t_begin + t_count);

  const long long cbeg = (long long)blockIdx.y * chunk_len;
  const long long cend = min(n, cbeg + chunk_len);

  bool my_ok = true, my_ok4 = true;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    my_ok = my_ok && coord_ok(tx[k]) && coord_ok(ty[k]);
    my_ok4 = my_ok4 && coord_ok4(tx[k]) && coord_ok4(ty[k]);
  }
  // δ' bounded on both sides so the Montgomery product stays inside the fp32
  // seed's range (rcp_seed_via_f32 needs P ∈ [2^-126, 2^126)):
  //   2-way: q ∈ [2^-62, 2^61 + 2^60]  → P = q1 q2 < 2^124
  //   4-way: q ∈ [2^-31, 2^31 + 2^29]  → P = q1 q2 q3 q4 < 2^125.3
  // (also false for δ' = inf / NaN); otherwise the tile takes the safe path.
  const bool targets_ok = __syncthreads_and(my_ok) && dp >= 0x1p-62 && dp <= 0x1p60;
  const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-31 && dp <= 0x1p29;

  // Register prefetch of the first source tile.
  double px = 0.0, py = 0.0, pg = 0.0;
  if (cbeg + tid < cend) {
    src.load(cbeg + tid, px, py);
    pg = gam[cbeg + tid] * inv2pi;
  }
  for (long long j0 = cbeg; j0 < cend; j0 += TPB) {
    const int cnt = (int)min((long long)TPB, cend - j0);
    sp[tid] = make_double2(px, py);
    sg[tid] = pg;
    const bool fast4 = __syncthreads_and(coord_ok4(px) && coord_ok4(py)) && targets_ok4;
    const bool fast = fast4 || (__syncthreads_and(coord_ok(px) && coord_ok(py)) && targets_ok);
    const long long jn = j0 + TPB + tid;  // prefetch the next tile while computing
    if (jn < cend) {
      src.load(jn, px, py);
      pg = gam[jn] * inv2pi;
    }
    // The self pair (kernel.hpp:118 skips j == i) needs masking only for the
    // Jacobian or on the safe path: on the fast paths δ' > 0, so for the
    // velocity it has r = 0, q = δ', s finite and adds exactly ±0 to f.
    const bool masked = self_excl && (j0 < tile_end) && (tile0 < j0 + cnt) && (JAC || !fast);
    if (masked)
      tile_f64<T, UNR, VEL, JAC, true, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
    else if (fast4)
      tile_f64<T, UNR, VEL, JAC, false, F4>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
    else if (fast)
      tile_f64<T, UNR, VEL, JAC, false, 2>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
    else
      tile_f64<T, UNR, VEL, JAC, false, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
    __syncthreads();
  }

  double* out = part + (long long)blockIdx.y * NCOMP * t_count;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    if (ti[k] < 0) continue;
    const long long li = ti[k] - t_begin;
    int c = 0;
    if (VEL) {
      out[(c++) * t_count + li] = fx[k];
      out[(c++) * t_count + li] = fy[k];
    }
    if (JAC) {
      out[(c++) * t_count + li] = ja[k];
      out[(c++) * t_count + li] = jb[k];
      out[(c++) * t_count + li] = jc[k];
    }
  }
  if (VEL && !JAC && fo.f) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(fo.tile_ctr + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // chunk partials summed in ascending chunk order (bit-identical to the
    // separate reduction); U chunks of every target are loaded before they
    // are added, so the tail is ~nch/U L2 round trips, not nch
    constexpr int U = T <= 2 ? 8 : (T <= 4 ? 4 : 2);
    const int nch = (int)gridDim.y;
    double sxs[T], sys[T];
    long long lis[T];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      sxs[k] = sys[k] = 0.0;
      lis[k] = ti[k] >= 0 ? ti[k] - t_begin : 0;
    }
    int c = 0;
    for (; c + U <= nch; c += U) {
      double vx[T][U], vy[T][U];
#pragma unroll
      for (int k = 0; k < T; ++k)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          vx[k][u] = __ldcg(part + ((long long)(c + u) * 2 + 0) * t_count + lis[k]);
          vy[k][u] = __ldcg(part + ((long long)(c + u) * 2 + 1) * t_count + lis[k]);
        }
#pragma unroll
      for (int k = 0; k < T; ++k)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          sxs[k] += vx[k][u];
          sys[k] += vy[k][u];
        }
    }
    for (; c < nch; ++c)
#pragma unroll
      for (int k = 0; k < T; ++k) {
        sxs[k] += __ldcg(part + ((long long)c * 2 + 0) * t_count + lis[k]);
        sys[k] += __ldcg(part + ((long long)c * 2 + 1) * t_count + lis[k]);
      }
#pragma unroll
    for (int k = 0; k < T; ++k) {
      if (ti[k] < 0) continue;
      const long long li = lis[k];
      double sx = sxs[k], sy = sys[k];
      const long long i = ti[k];
      if (fo.inflow) {
        sx = sx + fo.inflow[i];
        sy = sy + fo.inflow[i + fo.n_total];
      }
      if (!isfinite(sx) || !isfinite(sy)) latch_status(fo.st, kStatusNonFiniteVelocity, i);
      fo.f[li] = sx;
      fo.f[li + fo.ld] = sy;
    }
    if (tid == 0) fo.tile_ctr[blockIdx.x] = 0;  // ready for the next launch
  }
}

// Fixed-order chunk reduction + inflow + finiteness latch.
__global__ void reduce_velocity_f64_kernel(long long n, long long t_begin, long long t_count, int n_chunks,
                                           const double* __restrict__ part, int ncomp,
                                           const double* __restrict__ inflow, double* __restrict__ f, long long ld,
                                           DeviceStatus* st) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < t_count;
       li += (long long)gridDim.x * blockDim.x) {
    // ascending chunk order; 8 chunks loaded ahead of their adds
    double fx = 0.0, fy = 0.0;
    int c = 0;
    for (; c + 8 <= n_chunks; c += 8) {
      double vx[8], vy[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        vx[u] = part[((long long)(c + u) * ncomp + 0) * t_count + li];
        vy[u] = part[((long long)(c + u) * ncomp + 1) * t_count + li];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        fx += vx[u];
        fy += vy[u];
      }
    }
    for (; c < n_chunks; ++c) {
      fx += part[((long long)c * ncomp + 0) * t_count + li];
      fy += part[((long long)c * ncomp + 1) * t_count + li];
    }
    const long long i = t_begin + li;
    if (inflow) {
      fx = fx + inflow[i];
      fy = fy + inflow[i + n];
    }
    if (!isfinite(fx) || !isfinite(fy)) latch_status(st, kStatusNonFiniteVelocity, i);
    f[li] = fx;
    f[li + ld] = fy;
  }
}

// Jacobian assembly from (A, B, C) partials; optionally the Newton-block
// inverse of (I − h·J) (integrators.hpp:181-194, reference rounding order).
template <bool INVERT>
__global__ void reduce_jacobian_f64_kernel(long long t_begin, long long t_count, int n_chunks,
                                           const double* __restrict__ part, int ncomp, int off, double dp,
                                           double h, double* __restrict__ jxx, double* __restrict__ jxy,
                                           double* __restrict__ jyx, double* __restrict__ jyy,
                                           double* __restrict__ inv, DeviceStatus* st) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < t_count;
       li += (long long)gridDim.x * blockDim.x) {
    // ascending chunk order; 8 chunks loaded ahead of their adds
    double a = 0.0, b = 0.0, c = 0.0;
    int ch = 0;
    for (; ch + 8 <= n_chunks; ch += 8) {
      double va[8], vb[8], vc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* pc = part + (long long)(ch + u) * ncomp * t_count + li;
        va[u] = pc[(off + 0) * t_count];
        vb[u] = pc[(off + 1) * t_count];
        vc[u] = pc[(off + 2) * t_count];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a += va[u];
        b += vb[u];
        c += vc[u];
      }
    }
    for (; ch < n_chunks; ++ch) {
      const double* pc = part + (long long)ch * ncomp * t_count + li;
      a += pc[(off + 0) * t_count];
      b += pc[(off + 1) * t_count];
      c += pc[(off + 2) * t_count];
    }
    const double j00 = 2.0 * a, j11 = -2.0 * a;
    const double j01 = b - dp * c, j10 = b + dp * c;
    const long long i = t_begin + li;
    if (!INVERT) {
      if (!isfinite(j00) || !isfinite(j01) || !isfinite(j10)) latch_status(st, kStatusNonFiniteJacobian, i);
      jxx[li] = j00;
      jxy[li] = j01;
      jyx[li] = j10;
      jyy[li] = j11;
    } else {
      const double b00 = __dsub_rn(1.0, __dmul_rn(h, j00));
      const double b01 = __dsub_rn(0.0, __dmul_rn(h, j01));
      const double b10 = __dsub_rn(0.0, __dmul_rn(h, j10));
      const double b11 = __dsub_rn(1.0, __dmul_rn(h, j11));
      const double det = __dsub_rn(__dmul_rn(b00, b11), __dmul_rn(b01, b10));
      if (det == 0.0 || !isfinite(det)) latch_status(st, kStatusSingularBlock, i);
      double* o = inv + 4 * li;
      o[0] = __ddiv_rn(b11, det);
      o[1] = __ddiv_rn(-b01, det);
      o[2] = __ddiv_rn(-b10, det);
      o[3] = __ddiv_rn(b00, det);
    }
  }
}

// ----------------------------------------------------------------- fp32 ---
// fp32 pairs (tile_f32, pair_tile.cuh); each shared-memory tile is summed in
// fp32 and promoted into fp64 accumulators (blocked summation keeps the fp32
// result within 1e-5 of the fp64 oracle at N = 65,536).
template <int TPB, int T>
__global__ void __launch_bounds__(TPB) allpairs_f32_kernel(long long n, const float* __restrict__ xs,
                                                           const float* __restrict__ ys,
                                                           const float* __restrict__ gam, float inv2pi, float dp,
                                                           long long t_begin, long long t_count,
                                                           long long chunk_len, double* __restrict__ part) {
  __shared__ float2 sp[TPB];
  __shared__ float sg[TPB];
  const int tid = threadIdx.x;
  const long long tile0 = t_begin + (long long)blockIdx.x * (TPB * T);
  float tx[T], ty[T];
  double fx[T], fy[T];
  long long ti[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const long long i = tile0 + k * TPB + tid;
    const bool ok = i < t_begin + t_count;
    ti[k] = ok ? i : -1;
    tx[k] = ok ? xs[i] : 0.f;
    ty[k] = ok ? ys[i] : 0.f;
    fx[k] = fy[k] = 0.0;
  }
  bool my_ok = true;
#pragma unroll
  for (int k = 0; k < T; ++k) my_ok = my_ok && coord_ok_f32(tx[k]) && coord_ok_f32(ty[k]);
  const bool targets_ok = __syncthreads_and(my_ok) && dp >= 0x1p-30f && dp <= 0x1p28f;
  const long long tile_end = min(tile0 + (long long)TPB * T, t_begin + t_count);
  const long long cbeg = (long long)blockIdx.y * chunk_len;
  const long long cend = min(n, cbeg + chunk_len);
  float px = 0.f, py = 0.f, pg = 0.f;
  if (cbeg + tid < cend) {
    px = xs[cbeg + tid];
    py = ys[cbeg + tid];
    pg = gam[cbeg + tid] * inv2pi;
  }
  for (long long j0 = cbeg; j0 < cend; j0 += TPB) {
    const int cnt = (int)min((long long)TPB, cend - j0);
    sp[tid] = make_float2(px, py);
    sg[tid] = pg;
    const bool fast = __syncthreads_and(coord_ok_f32(px) && coord_ok_f32(py)) && targets_ok;
    const long long jn = j0 + TPB + tid;
    if (jn < cend) {
      px = xs[jn];
      py = ys[jn];
      pg = gam[jn] * inv2pi;
    }
    // the self pair adds exactly ±0 on the fast path (δ' > 0), so only the
    // safe path masks the diagonal
    const bool masked = (j0 < tile_end) && (tile0 < j0 + cnt) && !fast;
    float ax[T], ay[T];
#pragma unroll
    for (int k = 0; k < T; ++k) ax[k] = ay[k] = 0.f;
    if (masked)
      tile_f32<T, true, false>(cnt, sp, sg, j0, tx, ty, ti, dp, ax, ay);
    else if (fast)
      tile_f32<T, false, true>(cnt, sp, sg, j0, tx, ty, ti, dp, ax, ay);
    else
      tile_f32<T, false, false>(cnt, sp, sg, j0, tx, ty, ti, dp, ax, ay);
#pragma unroll
    for (int k = 0; k < T; ++k) {
      fx[k] += (double)ax[k];
      fy[k] += (double)ay[k];
    }
    __syncthreads();
  }
  double* out = part + (long long)blockIdx.y * 2 * t_count;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    if (ti[k] < 0) continue;
    const long long li = ti[k] - t_begin;
    out[li] = fx[k];
    out[t_count + li] = fy[k];
  }
}

__global__ void reduce_velocity_f32_kernel(long long n, long long t_begin, long long t_count, int n_chunks,
                                           const double* __restrict__ part, const float* __restrict__ inflow,
                                           float* __restrict__ f, long long ld, DeviceStatus* st) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < t_count;
       li += (long long)gridDim.x * blockDim.x) {
    double fx = 0.0, fy = 0.0;
    for (int c = 0; c < n_chunks; ++c) {
      fx += part[((long long)c * 2 + 0) * t_count + li];
      fy += part[((long long)c * 2 + 1) * t_count + li];
    }
    const long long i = t_begin + li;
    float ox = (float)fx, oy = (float)fy;
    if (inflow) {
      ox = ox + inflow[i];
      oy = oy + inflow[i + n];
    }
    if (!isfinite(ox) || !isfinite(oy)) latch_status(st, kStatusNonFiniteVelocity, i);
    f[li] = ox;
    f[li + ld] = oy;
  }
}

// ------------------------------------------------------------ launchers ---
int choose_source_chunks(ptrom_ctx* ctx, long long n_tiles, long long n_sources, int resident_per_sm,
                         long long min_chunk) {
  const long long slots = (long long)ctx->num_sms * std::max(1, resident_per_sm);
  const long long max_chunks = std::max(1LL, std::min(512LL, n_sources / std::max(1LL, min_chunk)));
  int best = 1;
  double best_eff = -1.0;
  for (long long c = 1; c <= max_chunks; ++c) {
    const long long blocks = n_tiles * c;
    const double waves = (double)blocks / (double)slots;
    const double eff = waves / std::ceil(waves);  // fraction of the last-wave slots in use
    // Prefer fewer chunks unless more chunks give a clearly better wave fill.
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = (int)c;
    }
    if (blocks >= 8 * slots) break;
  }
  return best;
}

namespace {

constexpr int kTPB = 128;
constexpr int kReduceThreads = 256;
// Set by dev_velocity_* for the duration of one launch: fuse the chunk
// reduction into the tile kernel (FusedOut).
thread_local const FusedOut* g_fuse = nullptr;
// dev_jacobian_reserve_f64: size the scratch arena of a launch without
// launching it (graph capture cannot allocate)
thread_local bool g_size_only = false;

template <class K>
int resident_blocks(K kernel, int tpb) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, tpb, 0);
  return std::max(occ, 1);
}

int reduce_grid(ptrom_ctx* ctx, long long count) {
  long long g = (count + kReduceThreads - 1) / kReduceThreads;
  return (int)std::max(1LL, std::min(g, (long long)ctx->num_sms * 8));
}

template <int TPB, int T, int UNR, int MINB, bool VEL, bool JAC, int F4, class Src>
void launch_allpairs_src(ptrom_ctx* ctx, long long n, Src src, const double* gamma, double dp, long long t_begin,
                         long long t_count, double** part_out, int* chunks_out, const double* tx, const double* ty,
                         long long t_base, int self_excl) {
  auto kern = allpairs_f64_kernel<TPB, T, UNR, MINB, VEL, JAC, F4, Src>;
  static int occ = resident_blocks(kern, TPB);
  constexpr int NCOMP = (VEL ? 2 : 0) + (JAC ? 3 : 0);
  const long long tiles = (t_count + TPB * T - 1) / (TPB * T);
  // short source ranges (small N) may split into chunks of 32 sources
  int chunks = choose_source_chunks(ctx, tiles, n, occ, T <= 2 ? 32 : 2 * TPB);
  // Sources beyond a third of L2 (x, y, Γ: 24 B each): split them into chunks
  // of ≤ 40 MB. CTAs are scheduled tile-fastest, so the resident waves stream
  // one chunk at a time and keep it L2-resident instead of re-reading the
  // whole source set from HBM per wave (config 5: 100 MB of sources).
  constexpr long long kL2ChunkBytes = 40ll << 20;
  chunks = (int)std::min<long long>(512, std::max<long long>(chunks, (n * 24 + kL2ChunkBytes - 1) / kL2ChunkBytes));
  const long long chunk_len = (n + chunks - 1) / chunks;
  ctx->scratch.reset();
  ctx->scratch.reserve((size_t)chunks * NCOMP * t_count * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)chunks * NCOMP * t_count);
  if (g_size_only) {
    *part_out = part;
    *chunks_out = chunks;
    return;
  }
  dim3 grid((unsigned)tiles, (unsigned)chunks);
  const double inv2pi = 1.0 / (2.0 * M_PI);
  {
    ProfScope prof(ctx);
    FusedOut fo{};
    if (VEL && !JAC && g_fuse) {
      fo = *g_fuse;
      if (ctx->tile_ctr_cap < (size_t)tiles) {  // zero-initialised once; the kernel leaves it zeroed
        if (ctx->tile_ctr) PTROM_CUDA(cudaFree(ctx->tile_ctr));
        const size_t cap = std::max<size_t>((size_t)tiles, 4096);
        PTROM_CUDA(cudaMalloc(&ctx->tile_ctr, cap * sizeof(unsigned)));
        PTROM_CUDA(cudaMemset(ctx->tile_ctr, 0, cap * sizeof(unsigned)));
        ctx->tile_ctr_cap = cap;
      }
      fo.tile_ctr = ctx->tile_ctr;
    }
    kern<<<grid, TPB, 0, ctx->stream>>>(n, src, gamma, inv2pi, dp, t_begin, t_count, chunk_len, part, tx, ty, t_base,
                                        self_excl, fo);
  }
  PTROM_LAUNCH_CHECK();
  *part_out = part;
  *chunks_out = chunks;
}

template <int TPB, int T, int UNR, int MINB, bool VEL, bool JAC, int F4 = 4>
void launch_allpairs_f64_t(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double dp,
                           long long t_begin, long long t_count, double** part_out, int* chunks_out,
                           const double* tx, const double* ty, const SrcPeers* peers, long long t_base) {
  if (peers) {
    launch_allpairs_src<TPB, T, UNR, MINB, VEL, JAC, F4>(ctx, n, *peers, gamma, dp, t_begin, t_count, part_out,
                                                         chunks_out, tx, ty, t_base, 1);
    return;
  }
  const bool external = tx != nullptr;
  launch_allpairs_src<TPB, T, UNR, MINB, VEL, JAC, F4>(ctx, n, SrcFlat{x, x + n}, gamma, dp, t_begin, t_count,
                                                       part_out, chunks_out, external ? tx : x,
                                                       external ? ty : x + n, external ? t_base : 0,
                                                       external ? 0 : 1);
}

using LaunchFn = void (*)(ptrom_ctx*, long long, const double*, const double*, double, long long, long long,
                          double**, int*, const double*, const double*, const SrcPeers*, long long);

// Velocity-kernel shapes (TPB, targets/thread, source unroll, min blocks/SM);
// entry 0 is the default, the rest are kept for tools/tune_allpairs.py
// (PTROM_ALLPAIRS_VARIANT selects one at context creation). Sweep on B200 at
// N = 65,536 with the unmasked fast diagonal (profiles/r01_tune_allpairs_sweeps.jsonl):
// (128,8,2,1) 21.6 TFLOP/s, (64,8,2,1) 21.4, (128,8,4,1) 21.4, (64,8,4,1) 21.2,
// (128,4,8,4) 21.1, (32,8,2,1) 21.1, (128,8,3,1) 21.0, (64,8,3,1) 20.8.
#define PTROM_VEL_VARIANTS(X) \
  X(128, 8, 2, 1, 4)          \
  X(64, 8, 2, 1, 4)           \
  X(128, 4, 8, 4, 4)          \
  X(128, 8, 3, 1, 4)          \
  X(64, 8, 2, 6, 4)           \
  X(64, 8, 4, 1, 4)           \
  X(64, 8, 3, 1, 4)           \
  X(128, 8, 4, 1, 4)          \
  X(64, 12, 2, 1, 4)          \
  X(96, 8, 2, 1, 4)           \
  X(32, 8, 2, 1, 4)           \
  X(64, 16, 1, 1, 4)          \
  X(128, 8, 2, 1, 5)          \
  X(64, 8, 2, 1, 5)           \
  X(128, 8, 4, 1, 5)

#define PTROM_VEL_ENTRY(TPB, T, UNR, MINB, F4) launch_allpairs_f64_t<TPB, T, UNR, MINB, true, false, F4>,
const LaunchFn kVelVariants[] = {PTROM_VEL_VARIANTS(PTROM_VEL_ENTRY)};
constexpr int kNumVelVariants = sizeof(kVelVariants) / sizeof(kVelVariants[0]);

// Small target sets get one target per thread (more blocks); large sets
// keep several targets per thread in registers to amortize the shared loads.
template <bool VEL, bool JAC>
void launch_allpairs_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double dp,
                         long long t_begin, long long t_count, double** part, int* chunks,
                         const double* tx = nullptr, const double* ty = nullptr, const SrcPeers* peers = nullptr,
                         long long t_base = 0) {
  // Few target tiles x few source chunks would not fill the 148 SMs with
  // 8 targets per thread (e.g. N = 4,096): use 2 per thread (4x the tiles).
  const long long wide_blocks = ((t_count + 1023) / 1024) * std::max(1LL, n / 256);
  if (t_count < 4096 || wide_blocks < 8LL * ctx->num_sms) {
    launch_allpairs_f64_t<kTPB, 2, 4, 1, VEL, JAC>(ctx, n, x, gamma, dp, t_begin, t_count, part, chunks, tx, ty,
                                                   peers, t_base);
  } else if (VEL && !JAC) {
    const int v = (ctx->allpairs_variant >= 0 && ctx->allpairs_variant < kNumVelVariants) ? ctx->allpairs_variant : 0;
    kVelVariants[v](ctx, n, x, gamma, dp, t_begin, t_count, part, chunks, tx, ty, peers, t_base);
  } else {
    launch_allpairs_f64_t<kTPB, 4, 4, 1, VEL, JAC>(ctx, n, x, gamma, dp, t_begin, t_count, part, chunks, tx, ty,
                                                   peers, t_base);
  }
}

// Lattice speeds (kernel.hpp:213-238): |Σ_p kernel_pair(vertex, p)|·scale per
// vertex; grid column-major ny x nx (vertex t = i·ny + j).
__global__ void lattice_vertices_kernel(double x_min, double x_max, long long nx, double y_min, double y_max,
                                        long long ny, double* __restrict__ vx, double* __restrict__ vy) {
  const long long count = nx * ny;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / ny, j = t - i * ny;
    // LatticeSpec::x_at / y_at (kernel.hpp:205-206), reference rounding order
    vx[t] = __dadd_rn(x_min, __ddiv_rn(__dmul_rn(__dsub_rn(x_max, x_min), (double)i), (double)(nx - 1)));
    vy[t] = __dadd_rn(y_min, __ddiv_rn(__dmul_rn(__dsub_rn(y_max, y_min), (double)j), (double)(ny - 1)));
  }
}

__global__ void lattice_speed_kernel(long long count, int n_chunks, const double* __restrict__ part, double scale,
                                     double* __restrict__ grid, DeviceStatus* st) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    double fx = 0.0, fy = 0.0;
    for (int c = 0; c < n_chunks; ++c) {
      fx += part[((long long)c * 2 + 0) * count + t];
      fy += part[((long long)c * 2 + 1) * count + t];
    }
    const double speed = __dmul_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(fx, fx), __dmul_rn(fy, fy))), scale);
    if (!isfinite(speed)) latch_status(st, kStatusNonFiniteVelocity, t);
    grid[t] = speed;
  }
}

}  // namespace

double effective_delta(double delta, int form) { return form == PTROM_FORM_STANDARD ? delta : delta / (2.0 * M_PI); }

void dev_velocity_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                      const double* inflow, long long t_begin, long long t_end, double* f, long long ld) {
  const long long t_count = t_end - t_begin;
  if (t_count <= 0) return;
  if (t_begin == 0 && t_count == n && ld == n && sym_velocity_applies(ctx, n)) {  // every target: unordered pairs
    dev_velocity_sym_f64(ctx, n, x, gamma, delta, form, inflow, f);
    return;
  }
  double* part;
  int chunks;
  if ((double)n * (double)t_count > 268435456.0) {  // large: the separate reduction is cheaper than a serial tail
    launch_allpairs_f64<true, false>(ctx, n, x, gamma, effective_delta(delta, form), t_begin, t_count, &part,
                                     &chunks);
    reduce_velocity_f64_kernel<<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
        n, t_begin, t_count, chunks, part, 2, inflow, f, ld, ctx->d_status);
    PTROM_LAUNCH_CHECK();
    return;
  }
  // small (launch-bound, e.g. the N = 4,096 FOM): one launch, reduction fused
  FusedOut fo;
  fo.f = f;
  fo.ld = ld;
  fo.n_total = n;
  fo.inflow = inflow;
  fo.st = ctx->d_status;
  g_fuse = &fo;
  try {
    launch_allpairs_f64<true, false>(ctx, n, x, gamma, effective_delta(delta, form), t_begin, t_count, &part,
                                     &chunks);
  } catch (...) {
    g_fuse = nullptr;
    throw;
  }
  g_fuse = nullptr;
}

// Kirchhoff–Routh energy (kernel.hpp:174-191): H = Σ_{i<j} Γi Γj log|r_ij| / 2π.
// Blocks own TPB·T targets i and a source chunk; only pairs j > i are
// evaluated (blocks and tiles entirely at or below the diagonal skip). Each
// target accumulates Σ_j Γj·log(d²) in its registers (log|r| = ½ log d²,
// within one ulp of the reference's log(sqrt(d²))); the fixed-order reduce
// below multiplies by Γi and sums targets in a fixed tree, so the result is
// bit-reproducible. d² == 0 latches the lexicographically first pair
// (encoded i·n + j), the reference's throw at kernel.hpp:185-187.
template <int TPB, int T>
__global__ void __launch_bounds__(TPB) hamiltonian_f64_kernel(long long n, const double* __restrict__ xs,
                                                              const double* __restrict__ ys,
                                                              const double* __restrict__ gam, long long chunk_len,
                                                              double* __restrict__ part, DeviceStatus* st) {
  __shared__ double2 sp[TPB];
  __shared__ double sg[TPB];
  const int tid = threadIdx.x;
  const long long tile0 = (long long)blockIdx.x * (TPB * T);
  const long long tile_end = min(tile0 + (long long)TPB * T, n);
  double tx[T], ty[T], acc[T];
  long long ti[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const long long i = tile0 + k * TPB + tid;
    ti[k] = i < n ? i : LLONG_MAX;  // out-of-range rows never see j > i
    tx[k] = i < n ? xs[i] : 0.0;
    ty[k] = i < n ? ys[i] : 0.0;
    acc[k] = 0.0;
  }
  const long long cbeg = max((long long)blockIdx.y * chunk_len, tile0 + 1);
  const long long cend = min(n, (long long)(blockIdx.y + 1) * chunk_len);
  for (long long j0 = cbeg; j0 < cend; j0 += TPB) {
    const int cnt = (int)min((long long)TPB, cend - j0);
    if (tid < cnt) {
      sp[tid] = make_double2(xs[j0 + tid], ys[j0 + tid]);
      sg[tid] = gam[j0 + tid];
    }
    __syncthreads();
    const bool full = j0 >= tile_end;  // every source above every target of the block
    for (int jj = 0; jj < cnt; ++jj) {
      const double2 p = sp[jj];
      const double g = sg[jj];
      const long long j = j0 + jj;
#pragma unroll
      for (int k = 0; k < T; ++k) {
        const double rx = __dsub_rn(tx[k], p.x), ry = __dsub_rn(ty[k], p.y);
        double d2 = __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry));
        const bool use = full || j > ti[k];
        if (use && d2 == 0.0) latch_status(st, kStatusCoincidentPair, ti[k] * n + j);
        d2 = use ? d2 : 1.0;
        acc[k] = fma(use ? g : 0.0, log(d2), acc[k]);
      }
    }
    __syncthreads();
  }
  double* out = part + (long long)blockIdx.y * n;
#pragma unroll
  for (int k = 0; k < T; ++k)
    if (ti[k] < n) out[ti[k]] = acc[k];
}

constexpr int kHamBlocks = 296;

__global__ void hamiltonian_reduce_kernel(long long n, int n_chunks, const double* __restrict__ part,
                                          const double* __restrict__ gam, double* __restrict__ block_sums) {
  __shared__ double red[kReduceThreads];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int c = 0; c < n_chunks; ++c) a += part[(long long)c * n + i];
    s = fma(gam[i], a, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kReduceThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) block_sums[blockIdx.x] = red[0];
}

__global__ void hamiltonian_finish_kernel(int nb, const double* __restrict__ block_sums, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += block_sums[b];
  out[0] = 0.5 * s / (2.0 * M_PI);
}

void dev_hamiltonian_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double* out) {
  constexpr int TPB = 128, T = 2;
  auto kern = hamiltonian_f64_kernel<TPB, T>;
  static int occ = resident_blocks(kern, TPB);
  const long long tiles = (n + TPB * T - 1) / (TPB * T);
  // About half of the (tile, chunk) blocks sit below the diagonal and exit at once.
  const int chunks = choose_source_chunks(ctx, (tiles + 1) / 2, n, occ, 2 * TPB);
  const long long chunk_len = (n + chunks - 1) / chunks;
  ctx->scratch.reset();
  ctx->scratch.reserve(((size_t)chunks * n + kHamBlocks) * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)chunks * n);
  double* bs = ctx->scratch.take<double>(kHamBlocks);
  PTROM_CUDA(cudaMemsetAsync(part, 0, (size_t)chunks * n * sizeof(double), ctx->stream));
  ctx->status_pair_n = n;
  {
    ProfScope prof(ctx);
    kern<<<dim3((unsigned)tiles, (unsigned)chunks), TPB, 0, ctx->stream>>>(n, x, x + n, gamma, chunk_len, part,
                                                                           ctx->d_status);
  }
  PTROM_LAUNCH_CHECK();
  hamiltonian_reduce_kernel<<<kHamBlocks, kReduceThreads, 0, ctx->stream>>>(n, chunks, part, gamma, bs);
  hamiltonian_finish_kernel<<<1, 32, 0, ctx->stream>>>(kHamBlocks, bs, out);
  PTROM_LAUNCH_CHECK();
}

// Target-sharded velocity reading the other ranks' source blocks in place
// (SrcPeers): rows [t_begin, t_end) are this rank's particles, stored at
// tx/ty (row i at tx[i - t_begin]); Γ and the inflow are full replicated
// arrays. Result as dev_velocity_f64.
void dev_velocity_peers_f64(ptrom_ctx* ctx, long long n, int n_peers, const double* const* peer_base,
                            const long long* peer_off, const double* gamma, double delta, int form,
                            const double* inflow, long long t_begin, long long t_end, const double* tx,
                            const double* ty, double* f, long long ld) {
  const long long t_count = t_end - t_begin;
  if (t_count <= 0) return;
  if (n_peers < 1 || n_peers > kMaxPeers) throw status_error(PTROM_CONFIG_ERROR, "peer count outside [1, 8]");
  SrcPeers sp{};
  sp.G = n_peers;
  for (int r = 0; r < n_peers; ++r) sp.base[r] = peer_base[r];
  for (int r = 0; r <= n_peers; ++r) sp.off[r] = peer_off[r];
  for (int r = n_peers + 1; r <= kMaxPeers; ++r) sp.off[r] = n;
  for (int r = n_peers; r < kMaxPeers; ++r) sp.base[r] = nullptr;
  double* part;
  int chunks;
  launch_allpairs_f64<true, false>(ctx, n, nullptr, gamma, effective_delta(delta, form), t_begin, t_count, &part,
                                   &chunks, tx, ty, &sp, t_begin);
  reduce_velocity_f64_kernel<<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
      n, t_begin, t_count, chunks, part, 2, inflow, f, ld, ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

void dev_velocity_field_grid_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta,
                                 int form, double x_min, double x_max, long long nx, double y_min, double y_max,
                                 long long ny, double scale, double* grid) {
  const long long count = nx * ny;
  double* vx;
  PTROM_CUDA(cudaMallocAsync(&vx, 2 * count * sizeof(double), ctx->stream));
  double* vy = vx + count;
  lattice_vertices_kernel<<<reduce_grid(ctx, count), kReduceThreads, 0, ctx->stream>>>(x_min, x_max, nx, y_min,
                                                                                         y_max, ny, vx, vy);
  PTROM_LAUNCH_CHECK();
  double* part;
  int chunks;
  launch_allpairs_f64<true, false>(ctx, n, x, gamma, effective_delta(delta, form), 0, count, &part, &chunks, vx, vy);
  lattice_speed_kernel<<<reduce_grid(ctx, count), kReduceThreads, 0, ctx->stream>>>(count, chunks, part, scale, grid,
                                                                                     ctx->d_status);
  PTROM_LAUNCH_CHECK();
  PTROM_CUDA(cudaFreeAsync(vx, ctx->stream));
}

void dev_jacobian_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                      long long t_begin, long long t_end, double* jxx, double* jxy, double* jyx, double* jyy,
                      double dt_for_inverse, double* inv) {
  const long long t_count = t_end - t_begin;
  if (t_count <= 0) return;
  double* part;
  int chunks;
  const double dp = effective_delta(delta, form);
  if (t_begin == 0 && t_count == n && sym_velocity_applies(ctx, n))  // every target: unordered pairs
    dev_jacobian_sym_part(ctx, n, x, gamma, dp, &part, &chunks, false);
  else
    launch_allpairs_f64<false, true>(ctx, n, x, gamma, dp, t_begin, t_count, &part, &chunks);
  if (inv) {
    reduce_jacobian_f64_kernel<true><<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
        t_begin, t_count, chunks, part, 3, 0, dp, dt_for_inverse / 2.0, nullptr, nullptr, nullptr, nullptr, inv,
        ctx->d_status);
  } else {
    reduce_jacobian_f64_kernel<false><<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
        t_begin, t_count, chunks, part, 3, 0, dp, 0.0, jxx, jxy, jyx, jyy, nullptr, ctx->d_status);
  }
  PTROM_LAUNCH_CHECK();
}

void dev_jacobian_reduce_f64(ptrom_ctx* ctx, const double* part, int chunks, long long t_begin, long long t_count,
                             double dp, double dt_for_inverse, double* jxx, double* jxy, double* jyx, double* jyy,
                             double* inv) {
  if (t_count <= 0) return;
  if (inv)
    reduce_jacobian_f64_kernel<true><<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
        t_begin, t_count, chunks, part, 3, 0, dp, dt_for_inverse / 2.0, nullptr, nullptr, nullptr, nullptr, inv,
        ctx->d_status);
  else
    reduce_jacobian_f64_kernel<false><<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
        t_begin, t_count, chunks, part, 3, 0, dp, 0.0, jxx, jxy, jyx, jyy, nullptr, ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

void dev_jacobian_reserve_f64(ptrom_ctx* ctx, long long n, long long t_count) {
  if (t_count <= 0) return;
  double* part;
  int chunks;
  if (t_count == n && sym_velocity_applies(ctx, n)) {
    dev_jacobian_sym_part(ctx, n, nullptr, nullptr, 1.0, &part, &chunks, true);
    return;
  }
  g_size_only = true;
  try {
    launch_allpairs_f64<false, true>(ctx, n, nullptr, nullptr, 1.0, 0, t_count, &part, &chunks);
  } catch (...) {
    g_size_only = false;
    throw;
  }
  g_size_only = false;
}

void dev_velocity_f32(ptrom_ctx* ctx, long long n, const float* x, const float* gamma, float delta, int form,
                      const float* inflow, long long t_begin, long long t_end, float* f, long long ld) {
  const long long t_count = t_end - t_begin;
  if (t_count <= 0) return;
  if (t_begin == 0 && t_count == n && ld == n && sym_velocity_applies(ctx, n)) {  // every target: unordered pairs
    dev_velocity_sym_f32(ctx, n, x, gamma, delta, form, inflow, f);
    return;
  }
  constexpr int T = 8;
  auto kern = allpairs_f32_kernel<kTPB, T>;
  static int occ = resident_blocks(kern, kTPB);
  const long long tiles = (t_count + kTPB * T - 1) / (kTPB * T);
  const int chunks = choose_source_chunks(ctx, tiles, n, occ, 2 * kTPB);
  const long long chunk_len = (n + chunks - 1) / chunks;
  ctx->scratch.reset();
  ctx->scratch.reserve((size_t)chunks * 2 * t_count * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)chunks * 2 * t_count);
  const float dp = (float)effective_delta((double)delta, form);
  const float inv2pi = (float)(1.0 / (2.0 * M_PI));
  {
    ProfScope prof(ctx);
    kern<<<dim3((unsigned)tiles, (unsigned)chunks), kTPB, 0, ctx->stream>>>(n, x, x + n, gamma, inv2pi, dp,
                                                                             t_begin, t_count, chunk_len, part);
  }
  PTROM_LAUNCH_CHECK();
  reduce_velocity_f32_kernel<<<reduce_grid(ctx, t_count), kReduceThreads, 0, ctx->stream>>>(
      n, t_begin, t_count, chunks, part, inflow, f, ld, ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

}  // namespace ptrom
