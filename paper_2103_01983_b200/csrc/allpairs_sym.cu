// allpairs_sym.cu — the full self-evaluation f = pairwise_velocity(x)
// (kernel.hpp:107-129, every target against every source) computed once per
// UNORDERED pair. Pair (i, j) and pair (j, i) share d² (r_ji = −r_ij
// exactly, so q = d² + δ' has the same bits) and one reciprocal u = 1/q;
// they differ only in the weight (Γ'_j for target i, Γ'_i for target j) and
// the sign of r. Per unordered pair the FP64 pipe executes ~12.75 ops
// against 2 × 9 for the two ordered pairs of allpairs_f64_kernel.
//
// Decomposition (fixed-order, deterministic): the particles are cut into nb
// blocks of B (a multiple of 1,024). A CTA takes one block pair (I, J),
// I ≤ J, and walks block I in passes of 1,024 targets (128 threads x 8 in
// registers, with Γ'_i) against block J's sources staged through shared
// memory in tiles of 128:
//  * I side: each thread accumulates its 8 targets in registers over the
//    whole block J and writes part[J][·][i] once;
//  * J side: within a warp the sources of a 32-source batch rotate over the
//    lanes (lane l takes source (l + s) mod 32 at sub-step s) and the
//    per-source accumulator travels with them — after the FMA it moves one
//    lane down (one shuffle), so after 32 sub-steps lane l holds the warp's
//    sum for source l with no reduction tree. The 4 warps' sums are added in
//    warp order and accumulated over the passes into part[I][·][j], which
//    only this CTA touches.
//  * diagonal blocks (I = J) are evaluated one-sided (tile_f64, self pair
//    excluded) — 1/nb of the work.
// part[K][c][i] is thus written by exactly one CTA for every (K, i), and
// f_i = Σ_K part[K][·][i] (ascending K) + inflow in a fixed order.
// Reciprocals: 4-way Montgomery (one MUFU.RCP64H seed + cubic correction per
// four pairs) on range-guarded tiles, MUFU.RCP64H + cubic correction per pair
// otherwise (which also propagates q = 0 as inf/NaN for a coincident pair
// with δ = 0, the reference's throw at kernel.hpp:38-39).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "comm.cuh"
#include "ops.cuh"
#include "pair_tile.cuh"

namespace ptrom {
namespace {

constexpr int kSTPB = 128;                 // threads per CTA
constexpr int kST = 8;                     // targets per thread
constexpr int kSPass = kSTPB * kST;        // targets per pass (1,024)
constexpr long long kSymMinN = 16384;
#ifndef PTROM_SYM_UNR
#define PTROM_SYM_UNR 16
#endif
constexpr int kSymUnr = PTROM_SYM_UNR;     // sub-steps unrolled in the fp64 velocity batch loop      // below: the one-sided kernels (launch-bound sizes)

__device__ __forceinline__ double rcp_cubic(double q) {
  const double y0 = rcp_seed(q);
  double e = fma(-q, y0, 1.0);
  e = fma(e, e, e);
  return fma(y0, e, y0);
}

__device__ __forceinline__ void decode_pair(long long k, int& I, int& J) {
  int j = (int)((sqrt(8.0 * (double)k + 1.0) - 1.0) * 0.5);
  while ((long long)(j + 1) * (j + 2) / 2 <= k) ++j;
  while ((long long)j * (j + 1) / 2 > k) --j;
  J = j;
  I = (int)(k - (long long)j * (j + 1) / 2);
}

// One rotated source against the thread's 8 targets: I-side into (fx, fy),
// J-side into (wx, wy). Off-diagonal items always have a full target block
// (only the last block can be ragged and I < J); TAIL: a source beyond n
// adds exactly 0 to the targets (selected, so its dummy position can never
// inject inf/NaN), and its own accumulator is never stored.
template <bool FAST4, bool TAIL>
__device__ __forceinline__ void sym_pairs(double px, double py, double g, bool vj, const double (&tx)[kST],
                                          const double (&ty)[kST], const double (&gi)[kST], double dp,
                                          double (&fx)[kST], double (&fy)[kST], double& wx, double& wy) {
#pragma unroll
  for (int k = 0; k < kST; k += 4) {
    double rx[4], ry[4], q[4], u[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      rx[m] = tx[k + m] - px;
      ry[m] = ty[k + m] - py;
      q[m] = fma(rx[m], rx[m], fma(ry[m], ry[m], dp));
    }
    if (FAST4) {  // u_m = 1/q_m from one reciprocal of (q0 q1)(q2 q3)
      const double p01 = q[0] * q[1], p23 = q[2] * q[3];
      const double P = p01 * p23;
      // MUFU.RCP64H seed + cubic step (~1 ulp): one FP64 op more than the
      // fp32-seeded Newton step but no integer re-biasing (measured 1.3% faster)
      const double uP = rcp_cubic(P);
      const double u01 = uP * p23, u23 = uP * p01;
      u[0] = u01 * q[1];
      u[1] = u01 * q[0];
      u[2] = u23 * q[3];
      u[3] = u23 * q[2];
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) u[m] = rcp_cubic(q[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double a = g * u[m];                // Γ'_j / q: target i's weight (kernel.hpp:37-41)
      const double b = gi[k + m] * u[m];  // Γ'_i / q: source j's weight, r_ji = −r_ij
      if (TAIL) a = vj ? a : 0.0;         // a source beyond n (its own sum is discarded)
      fx[k + m] = fma(-ry[m], a, fx[k + m]);
      fy[k + m] = fma(rx[m], a, fy[k + m]);
      wx = fma(ry[m], b, wx);
      wy = fma(-rx[m], b, wy);
    }
  }
}

template <bool TAIL>
__device__ void sym_item(long long n, const double* __restrict__ xs, const double* __restrict__ ys,
                         const double* __restrict__ gam, double inv2pi, double dp, long long B, int I, int J,
                         double* __restrict__ part, long long ps, double2* sp, double* sg, double2 (*sj)[kSTPB]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i_blk = (long long)I * B, j_blk = (long long)J * B;
  const long long j_end = min(j_blk + B, n);
  const int passes = (int)((min(i_blk + B, n) - i_blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long i0 = i_blk + (long long)pass * kSPass;
    double tx[kST], ty[kST], gi[kST], fx[kST], fy[kST];
    bool my_ok4 = true;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      const bool ok = i < n;
      tx[k] = ok ? xs[i] : 0.0;
      ty[k] = ok ? ys[i] : 0.0;
      gi[k] = ok ? gam[i] * inv2pi : 0.0;
      fx[k] = fy[k] = 0.0;
      my_ok4 = my_ok4 && coord_ok4(tx[k]) && coord_ok4(ty[k]);
    }
    const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-31 && dp <= 0x1p29;
    for (long long t0 = j_blk; t0 < j_end; t0 += kSTPB) {
      const long long j = t0 + tid;
      const bool vj = j < n;
      const double px = vj ? xs[j] : 0.0, py = vj ? ys[j] : 0.0;
      const double pg = vj ? gam[j] * inv2pi : 0.0;
      // each 32-source batch is staged twice in a row, so lane l reads its
      // rotated sources (l + s) mod 32 at the linear offsets l + s
      sp[2 * tid - lane] = make_double2(px, py);  // [batch][0..63]: row 64·warp
      sp[2 * tid - lane + 32] = make_double2(px, py);
      sg[2 * tid - lane] = pg;
      sg[2 * tid - lane + 32] = pg;
      const bool fast4 = __syncthreads_and(coord_ok4(px) && coord_ok4(py)) && targets_ok4;
      const int cnt = (int)min((long long)kSTPB, j_end - t0);
      for (int b0 = 0; b0 < kSTPB; b0 += 32) {
        double wx = 0.0, wy = 0.0;
        if (b0 < cnt) {  // CTA-uniform
          const double2* bp = sp + 2 * b0 + lane;
          const double* bg = sg + 2 * b0 + lane;
          const int nxt = (lane + 1) & 31;
          // the tier is uniform over the tile: one loop per tier, no branch per sub-step
          auto batch = [&](auto fast_tag) {
            constexpr bool F = decltype(fast_tag)::value;
#pragma unroll kSymUnr
            for (int s = 0; s < 32; ++s) {
              const double2 p = bp[s];
              const double g = bg[s];
              const bool v = !TAIL || b0 + ((lane + s) & 31) < cnt;
              sym_pairs<F, TAIL>(p.x, p.y, g, v, tx, ty, gi, dp, fx, fy, wx, wy);
              // the accumulator follows its source one lane down
              wx = __shfl_sync(0xffffffffu, wx, nxt);
              wy = __shfl_sync(0xffffffffu, wy, nxt);
            }
          };
          if (fast4)
            batch(std::true_type{});
          else
            batch(std::false_type{});
        }
        sj[warp][b0 + lane] = make_double2(wx, wy);  // lane holds source b0 + lane
      }
      __syncthreads();
      if (vj) {  // the 4 warps in order, accumulated over the passes
        double2 acc = sj[0][tid];
#pragma unroll
        for (int w = 1; w < kSTPB / 32; ++w) {
          acc.x += sj[w][tid].x;
          acc.y += sj[w][tid].y;
        }
        double* px_ = part + (long long)I * 2 * ps + j;
        if (pass == 0) {
          px_[0] = acc.x;
          px_[ps] = acc.y;
        } else {
          px_[0] = px_[0] + acc.x;
          px_[ps] = px_[ps] + acc.y;
        }
      }
      __syncthreads();
    }
    double* out = part + (long long)J * 2 * ps;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      if (i < n) {
        out[i] = fx[k];
        out[ps + i] = fy[k];
      }
    }
  }
}

// Diagonal block: one-sided, self pair excluded (allpairs_f64_kernel's tile loop).
__device__ void diag_item(long long n, const double* __restrict__ xs, const double* __restrict__ ys,
                          const double* __restrict__ gam, double inv2pi, double dp, long long B, int I,
                          double* __restrict__ part, long long ps, double2* sp, double* sg) {
  constexpr int T = kST, TPB = kSTPB;
  const int tid = threadIdx.x;
  const long long blk = (long long)I * B, blk_end = min(blk + B, n);
  const int passes = (int)((blk_end - blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long tile0 = blk + (long long)pass * kSPass;
    double tx[T], ty[T], fx[T], fy[T], ja[T], jb[T], jc[T];
    long long ti[T];
    bool my_ok = true, my_ok4 = true;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const long long i = tile0 + k * TPB + tid;
      const bool ok = i < blk_end;
      ti[k] = ok ? i : -1;
      tx[k] = ok ? xs[i] : 0.0;
      ty[k] = ok ? ys[i] : 0.0;
      fx[k] = fy[k] = ja[k] = jb[k] = jc[k] = 0.0;
      my_ok = my_ok && coord_ok(tx[k]) && coord_ok(ty[k]);
      my_ok4 = my_ok4 && coord_ok4(tx[k]) && coord_ok4(ty[k]);
    }
    const long long tile_end = min(tile0 + (long long)kSPass, blk_end);
    const bool targets_ok = __syncthreads_and(my_ok) && dp >= 0x1p-62 && dp <= 0x1p60;
    const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-31 && dp <= 0x1p29;
    for (long long j0 = blk; j0 < blk_end; j0 += TPB) {
      const int cnt = (int)min((long long)TPB, blk_end - j0);
      const long long j = j0 + tid;
      const double px = j < blk_end ? xs[j] : 0.0, py = j < blk_end ? ys[j] : 0.0;
      sp[tid] = make_double2(px, py);
      sg[tid] = j < blk_end ? gam[j] * inv2pi : 0.0;
      const bool fast4 = __syncthreads_and(coord_ok4(px) && coord_ok4(py)) && targets_ok4;
      const bool fast = fast4 || (__syncthreads_and(coord_ok(px) && coord_ok(py)) && targets_ok);
      const bool masked = (j0 < tile_end) && (tile0 < j0 + cnt) && !fast;
      if (masked)
        tile_f64<T, 2, true, false, true, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else if (fast4)
        tile_f64<T, 2, true, false, false, 4>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else if (fast)
        tile_f64<T, 2, true, false, false, 2>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else
        tile_f64<T, 2, true, false, false, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      __syncthreads();
    }
    double* out = part + (long long)I * 2 * ps;
#pragma unroll
    for (int k = 0; k < T; ++k)
      if (ti[k] >= 0) {
        out[ti[k]] = fx[k];
        out[ps + ti[k]] = fy[k];
      }
  }
}

// part rows have stride ps (≥ n); the grid covers items [k0, k0 + gridDim.x)
// of the nb(nb+1)/2 block pairs (a rank's share in the sharded evaluation).
__global__ void __launch_bounds__(kSTPB, 4) allpairs_sym_kernel(long long n, const double* __restrict__ xs,
                                                                const double* __restrict__ ys,
                                                                const double* __restrict__ gam, double inv2pi,
                                                                double dp, long long B, double* __restrict__ part,
                                                                long long ps, long long k0) {
  __shared__ double2 sp[2 * kSTPB];  // sym items: each batch twice; diagonal items: the first kSTPB
  __shared__ double sg[2 * kSTPB];
  __shared__ double2 sj[kSTPB / 32][kSTPB];
  int I, J;
  decode_pair(k0 + blockIdx.x, I, J);
  if (I == J) {
    diag_item(n, xs, ys, gam, inv2pi, dp, B, I, part, ps, sp, sg);
    return;
  }
  const bool tail = (long long)(J + 1) * B > n;  // only the last block can be ragged (I < J)
  if (tail)
    sym_item<true>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
  else
    sym_item<false>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
}

// f_i = Σ_K part[K][·][i] in ascending K (fixed order) + inflow, for the
// rows [r0, r0 + m) of part (row stride ps) → f (ld m); target ids t0 + row.
__global__ void reduce_sym_kernel(long long n, int nb, const double* __restrict__ part, long long ps, long long r0,
                                  long long m, long long t0, const double* __restrict__ inflow,
                                  double* __restrict__ f, DeviceStatus* st) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < m;
       li += (long long)gridDim.x * blockDim.x) {
    const long long r = r0 + li;
    double sx = 0.0, sy = 0.0;
    int k = 0;
    for (; k + 8 <= nb; k += 8) {
      double vx[8], vy[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        vx[u] = part[(long long)(k + u) * 2 * ps + r];
        vy[u] = part[((long long)(k + u) * 2 + 1) * ps + r];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sx += vx[u];
        sy += vy[u];
      }
    }
    for (; k < nb; ++k) {
      sx += part[(long long)k * 2 * ps + r];
      sy += part[((long long)k * 2 + 1) * ps + r];
    }
    const long long i = t0 + li;
    if (inflow) {
      sx = sx + inflow[i];
      sy = sy + inflow[i + n];
    }
    if (!isfinite(sx) || !isfinite(sy)) latch_status(st, kStatusNonFiniteVelocity, i);
    f[li] = sx;
    f[li + m] = sy;
  }
}

// ------------------------------------------------------------- Jacobian ---
// The self-block Jacobian (inexact_kernel_jacobian, kernel.hpp:154-170) over
// unordered pairs: its terms w·(rx ry, ry² − rx², 1) with w = Γ'/q² are even
// in r, so pair (i, j) and pair (j, i) share q, u = 1/q, u² and the two
// products and differ only in Γ'. Per unordered pair ~19 FP64 ops against
// 2 × 14 one-sided. Same block decomposition as the velocity; part holds
// (A, B, C) = Σ w·(rx ry, ry² − rx², 1) per target as [K][3][n], the layout
// of the one-sided kernel's chunk partials (reduce_jacobian_f64_kernel).
template <bool FAST4, bool TAIL>
__device__ __forceinline__ void sym_pairs_jac(double px, double py, double g, bool vj, const double (&tx)[kST],
                                              const double (&ty)[kST], const double (&gi)[kST], double dp,
                                              double (&ja)[kST], double (&jb)[kST], double (&jc)[kST],
                                              double& wa, double& wb, double& wc) {
#pragma unroll
  for (int k = 0; k < kST; k += 4) {
    double rx[4], ry[4], q[4], u[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      rx[m] = tx[k + m] - px;
      ry[m] = ty[k + m] - py;
      q[m] = fma(rx[m], rx[m], fma(ry[m], ry[m], dp));
    }
    if (FAST4) {
      const double p01 = q[0] * q[1], p23 = q[2] * q[3];
      const double uP = rcp_cubic(p01 * p23);
      const double u01 = uP * p23, u23 = uP * p01;
      u[0] = u01 * q[1];
      u[1] = u01 * q[0];
      u[2] = u23 * q[3];
      u[3] = u23 * q[2];
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) u[m] = rcp_cubic(q[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double uu = u[m] * u[m];
      const double t1 = rx[m] * ry[m];
      const double t2 = fma(ry[m], ry[m], -(rx[m] * rx[m]));
      double a = g * uu;                // Γ'_j / q²: target i's weight (kernel.hpp:53-61)
      const double b = gi[k + m] * uu;  // Γ'_i / q²: source j's weight
      if (TAIL) a = vj ? a : 0.0;
      ja[k + m] = fma(a, t1, ja[k + m]);
      jb[k + m] = fma(a, t2, jb[k + m]);
      jc[k + m] += a;
      wa = fma(b, t1, wa);
      wb = fma(b, t2, wb);
      wc += b;
    }
  }
}

template <bool TAIL>
__device__ void sym_item_jac(long long n, const double* __restrict__ xs, const double* __restrict__ ys,
                             const double* __restrict__ gam, double inv2pi, double dp, long long B, int I, int J,
                             double* __restrict__ part, long long ps, double2* sp, double* sg, double (*sj)[kSTPB][3]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i_blk = (long long)I * B, j_blk = (long long)J * B;
  const long long j_end = min(j_blk + B, n);
  const int passes = (int)((min(i_blk + B, n) - i_blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long i0 = i_blk + (long long)pass * kSPass;
    double tx[kST], ty[kST], gi[kST], ja[kST], jb[kST], jc[kST];
    bool my_ok4 = true;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      const bool ok = i < n;
      tx[k] = ok ? xs[i] : 0.0;
      ty[k] = ok ? ys[i] : 0.0;
      gi[k] = ok ? gam[i] * inv2pi : 0.0;
      ja[k] = jb[k] = jc[k] = 0.0;
      my_ok4 = my_ok4 && coord_ok4(tx[k]) && coord_ok4(ty[k]);
    }
    // u² = 1/q² must stay normal too: the 4-way tier's q ∈ [2^-31, 2^31] keeps it in range
    const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-31 && dp <= 0x1p29;
    for (long long t0 = j_blk; t0 < j_end; t0 += kSTPB) {
      const long long j = t0 + tid;
      const bool vj = j < n;
      const double px = vj ? xs[j] : 0.0, py = vj ? ys[j] : 0.0;
      const double pg = vj ? gam[j] * inv2pi : 0.0;
      sp[2 * tid - lane] = make_double2(px, py);
      sp[2 * tid - lane + 32] = make_double2(px, py);
      sg[2 * tid - lane] = pg;
      sg[2 * tid - lane + 32] = pg;
      const bool fast4 = __syncthreads_and(coord_ok4(px) && coord_ok4(py)) && targets_ok4;
      const int cnt = (int)min((long long)kSTPB, j_end - t0);
      for (int b0 = 0; b0 < kSTPB; b0 += 32) {
        double wa = 0.0, wb = 0.0, wc = 0.0;
        if (b0 < cnt) {
          const double2* bp = sp + 2 * b0 + lane;
          const double* bg = sg + 2 * b0 + lane;
          const int nxt = (lane + 1) & 31;
          auto batch = [&](auto fast_tag) {
            constexpr bool F = decltype(fast_tag)::value;
#pragma unroll 8
            for (int s = 0; s < 32; ++s) {
              const double2 p = bp[s];
              const double g = bg[s];
              const bool v = !TAIL || b0 + ((lane + s) & 31) < cnt;
              sym_pairs_jac<F, TAIL>(p.x, p.y, g, v, tx, ty, gi, dp, ja, jb, jc, wa, wb, wc);
              wa = __shfl_sync(0xffffffffu, wa, nxt);
              wb = __shfl_sync(0xffffffffu, wb, nxt);
              wc = __shfl_sync(0xffffffffu, wc, nxt);
            }
          };
          if (fast4)
            batch(std::true_type{});
          else
            batch(std::false_type{});
        }
        sj[warp][b0 + lane][0] = wa;
        sj[warp][b0 + lane][1] = wb;
        sj[warp][b0 + lane][2] = wc;
      }
      __syncthreads();
      if (vj) {
        double acc[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          acc[c] = sj[0][tid][c];
#pragma unroll
          for (int w = 1; w < kSTPB / 32; ++w) acc[c] += sj[w][tid][c];
        }
        double* pj = part + (long long)I * 3 * ps + j;
#pragma unroll
        for (int c = 0; c < 3; ++c) pj[c * ps] = pass == 0 ? acc[c] : pj[c * ps] + acc[c];
      }
      __syncthreads();
    }
    double* out = part + (long long)J * 3 * ps;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      if (i < n) {
        out[i] = ja[k];
        out[ps + i] = jb[k];
        out[2 * ps + i] = jc[k];
      }
    }
  }
}

// Diagonal block: one-sided (tile_f64's Jacobian path, self pair masked).
__device__ void diag_item_jac(long long n, const double* __restrict__ xs, const double* __restrict__ ys,
                              const double* __restrict__ gam, double inv2pi, double dp, long long B, int I,
                              double* __restrict__ part, long long ps, double2* sp, double* sg) {
  constexpr int T = kST, TPB = kSTPB;
  const int tid = threadIdx.x;
  const long long blk = (long long)I * B, blk_end = min(blk + B, n);
  const int passes = (int)((blk_end - blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long tile0 = blk + (long long)pass * kSPass;
    double tx[T], ty[T], fx[T], fy[T], ja[T], jb[T], jc[T];
    long long ti[T];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const long long i = tile0 + k * TPB + tid;
      const bool ok = i < blk_end;
      ti[k] = ok ? i : -1;
      tx[k] = ok ? xs[i] : 0.0;
      ty[k] = ok ? ys[i] : 0.0;
      fx[k] = fy[k] = ja[k] = jb[k] = jc[k] = 0.0;
    }
    const long long tile_end = min(tile0 + (long long)kSPass, blk_end);
    for (long long j0 = blk; j0 < blk_end; j0 += TPB) {
      const int cnt = (int)min((long long)TPB, blk_end - j0);
      const long long j = j0 + tid;
      sp[tid] = make_double2(j < blk_end ? xs[j] : 0.0, j < blk_end ? ys[j] : 0.0);
      sg[tid] = j < blk_end ? gam[j] * inv2pi : 0.0;
      __syncthreads();
      // the Jacobian always masks the self pair where the tile meets the diagonal
      if ((j0 < tile_end) && (tile0 < j0 + cnt))
        tile_f64<T, 2, false, true, true, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else
        tile_f64<T, 2, false, true, false, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      __syncthreads();
    }
    double* out = part + (long long)I * 3 * ps;
#pragma unroll
    for (int k = 0; k < T; ++k)
      if (ti[k] >= 0) {
        out[ti[k]] = ja[k];
        out[ps + ti[k]] = jb[k];
        out[2 * ps + ti[k]] = jc[k];
      }
  }
}

__global__ void __launch_bounds__(kSTPB, 3) allpairs_sym_jac_kernel(long long n, const double* __restrict__ xs,
                                                                    const double* __restrict__ ys,
                                                                    const double* __restrict__ gam, double inv2pi,
                                                                    double dp, long long B, double* __restrict__ part,
                                                                    long long ps, long long k0) {
  __shared__ double2 sp[2 * kSTPB];
  __shared__ double sg[2 * kSTPB];
  __shared__ double sj[kSTPB / 32][kSTPB][3];
  int I, J;
  decode_pair(k0 + blockIdx.x, I, J);
  if (I == J) {
    diag_item_jac(n, xs, ys, gam, inv2pi, dp, B, I, part, ps, sp, sg);
    return;
  }
  if ((long long)(J + 1) * B > n)
    sym_item_jac<true>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
  else
    sym_item_jac<false>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
}

// ----------------------------------------------------------------- fp32 ---
// The same unordered-pair decomposition at S = float (kernel.hpp:107-129
// instantiated for float): fp32 pair arithmetic, four targets sharing one
// MUFU.RCP of (q0 q1)(q2 q3) on range-guarded tiles (tile_f32's guard), one
// MUFU.RCP per pair otherwise. Blocked summation as in allpairs_f32_kernel:
// the I side is summed in fp32 per 128-source tile and promoted into fp64
// accumulators; the J side per 32-source batch (32 lanes x 8 targets) in
// fp32, the warps' batch sums and the passes in fp64; part rows are fp64.
template <bool FAST4, bool TAIL>
__device__ __forceinline__ void sym_pairs_f32(float px, float py, float g, bool vj, const float (&tx)[kST],
                                              const float (&ty)[kST], const float (&gi)[kST], float dp,
                                              float (&fx)[kST], float (&fy)[kST], float& wx, float& wy) {
#pragma unroll
  for (int k = 0; k < kST; k += 4) {
    float rx[4], ry[4], q[4], u[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      rx[m] = tx[k + m] - px;
      ry[m] = ty[k + m] - py;
      q[m] = fmaf(rx[m], rx[m], fmaf(ry[m], ry[m], dp));
    }
    if (FAST4) {  // u_m = 1/q_m from one reciprocal of (q0 q1)(q2 q3)
      const float p01 = q[0] * q[1], p23 = q[2] * q[3];
      const float uP = rcp_approx(p01 * p23);
      const float u01 = uP * p23, u23 = uP * p01;
      u[0] = u01 * q[1];
      u[1] = u01 * q[0];
      u[2] = u23 * q[3];
      u[3] = u23 * q[2];
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) u[m] = rcp_approx(q[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      float a = g * u[m];                // Γ'_j / q: target i's weight
      const float b = gi[k + m] * u[m];  // Γ'_i / q: source j's weight, r_ji = −r_ij
      if (TAIL) a = vj ? a : 0.f;        // a source beyond n (its own sum is discarded)
      fx[k + m] = fmaf(-ry[m], a, fx[k + m]);
      fy[k + m] = fmaf(rx[m], a, fy[k + m]);
      wx = fmaf(ry[m], b, wx);
      wy = fmaf(-rx[m], b, wy);
    }
  }
}

template <bool TAIL>
__device__ void sym_item_f32(long long n, const float* __restrict__ xs, const float* __restrict__ ys,
                             const float* __restrict__ gam, float inv2pi, float dp, long long B, int I, int J,
                             double* __restrict__ part, long long ps, float2* sp, float* sg, double2 (*sj)[kSTPB]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i_blk = (long long)I * B, j_blk = (long long)J * B;
  const long long j_end = min(j_blk + B, n);
  const int passes = (int)((min(i_blk + B, n) - i_blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long i0 = i_blk + (long long)pass * kSPass;
    float tx[kST], ty[kST], gi[kST];
    double dfx[kST], dfy[kST];
    bool my_ok4 = true;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      const bool ok = i < n;
      tx[k] = ok ? xs[i] : 0.f;
      ty[k] = ok ? ys[i] : 0.f;
      gi[k] = ok ? gam[i] * inv2pi : 0.f;
      dfx[k] = dfy[k] = 0.0;
      my_ok4 = my_ok4 && coord_ok_f32(tx[k]) && coord_ok_f32(ty[k]);
    }
    const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-30f && dp <= 0x1p28f;
    for (long long t0 = j_blk; t0 < j_end; t0 += kSTPB) {
      const long long j = t0 + tid;
      const bool vj = j < n;
      const float px = vj ? xs[j] : 0.f, py = vj ? ys[j] : 0.f;
      const float pg = vj ? gam[j] * inv2pi : 0.f;
      sp[2 * tid - lane] = make_float2(px, py);  // each 32-source batch twice (rotated linear reads)
      sp[2 * tid - lane + 32] = make_float2(px, py);
      sg[2 * tid - lane] = pg;
      sg[2 * tid - lane + 32] = pg;
      const bool fast4 = __syncthreads_and(coord_ok_f32(px) && coord_ok_f32(py)) && targets_ok4;
      const int cnt = (int)min((long long)kSTPB, j_end - t0);
      float fx[kST], fy[kST];
#pragma unroll
      for (int k = 0; k < kST; ++k) fx[k] = fy[k] = 0.f;
      for (int b0 = 0; b0 < kSTPB; b0 += 32) {
        float wx = 0.f, wy = 0.f;
        if (b0 < cnt) {  // CTA-uniform
          const float2* bp = sp + 2 * b0 + lane;
          const float* bg = sg + 2 * b0 + lane;
          const int nxt = (lane + 1) & 31;
          auto batch = [&](auto fast_tag) {
            constexpr bool F = decltype(fast_tag)::value;
#pragma unroll 16
            for (int s = 0; s < 32; ++s) {
              const float2 p = bp[s];
              const float g = bg[s];
              const bool v = !TAIL || b0 + ((lane + s) & 31) < cnt;
              sym_pairs_f32<F, TAIL>(p.x, p.y, g, v, tx, ty, gi, dp, fx, fy, wx, wy);
              wx = __shfl_sync(0xffffffffu, wx, nxt);  // the accumulator follows its source one lane down
              wy = __shfl_sync(0xffffffffu, wy, nxt);
            }
          };
          if (fast4)
            batch(std::true_type{});
          else
            batch(std::false_type{});
        }
        sj[warp][b0 + lane] = make_double2((double)wx, (double)wy);
      }
#pragma unroll
      for (int k = 0; k < kST; ++k) {
        dfx[k] += (double)fx[k];
        dfy[k] += (double)fy[k];
      }
      __syncthreads();
      if (vj) {
        double2 acc = sj[0][tid];
#pragma unroll
        for (int w = 1; w < kSTPB / 32; ++w) {
          acc.x += sj[w][tid].x;
          acc.y += sj[w][tid].y;
        }
        double* px_ = part + (long long)I * 2 * ps + j;
        if (pass == 0) {
          px_[0] = acc.x;
          px_[ps] = acc.y;
        } else {
          px_[0] = px_[0] + acc.x;
          px_[ps] = px_[ps] + acc.y;
        }
      }
      __syncthreads();
    }
    double* out = part + (long long)J * 2 * ps;
#pragma unroll
    for (int k = 0; k < kST; ++k) {
      const long long i = i0 + k * kSTPB + tid;
      if (i < n) {
        out[i] = dfx[k];
        out[ps + i] = dfy[k];
      }
    }
  }
}

// Diagonal block, fp32: one-sided (allpairs_f32_kernel's tile loop). On the
// fast path the self pair adds exactly ±0 (δ' > 0); the safe path masks it.
__device__ void diag_item_f32(long long n, const float* __restrict__ xs, const float* __restrict__ ys,
                              const float* __restrict__ gam, float inv2pi, float dp, long long B, int I,
                              double* __restrict__ part, long long ps, float2* sp, float* sg) {
  constexpr int T = kST, TPB = kSTPB;
  const int tid = threadIdx.x;
  const long long blk = (long long)I * B, blk_end = min(blk + B, n);
  const int passes = (int)((blk_end - blk + kSPass - 1) / kSPass);
  for (int pass = 0; pass < passes; ++pass) {
    const long long tile0 = blk + (long long)pass * kSPass;
    float tx[T], ty[T];
    double dfx[T], dfy[T];
    long long ti[T];
    bool my_ok = true;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const long long i = tile0 + k * TPB + tid;
      const bool ok = i < blk_end;
      ti[k] = ok ? i : -1;
      tx[k] = ok ? xs[i] : 0.f;
      ty[k] = ok ? ys[i] : 0.f;
      dfx[k] = dfy[k] = 0.0;
      my_ok = my_ok && coord_ok_f32(tx[k]) && coord_ok_f32(ty[k]);
    }
    const long long tile_end = min(tile0 + (long long)kSPass, blk_end);
    const bool targets_ok = __syncthreads_and(my_ok) && dp >= 0x1p-30f && dp <= 0x1p28f;
    for (long long j0 = blk; j0 < blk_end; j0 += TPB) {
      const int cnt = (int)min((long long)TPB, blk_end - j0);
      const long long j = j0 + tid;
      const float px = j < blk_end ? xs[j] : 0.f, py = j < blk_end ? ys[j] : 0.f;
      sp[tid] = make_float2(px, py);
      sg[tid] = j < blk_end ? gam[j] * inv2pi : 0.f;
      const bool fast = __syncthreads_and(coord_ok_f32(px) && coord_ok_f32(py)) && targets_ok;
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
        dfx[k] += (double)ax[k];
        dfy[k] += (double)ay[k];
      }
      __syncthreads();
    }
    double* out = part + (long long)I * 2 * ps;
#pragma unroll
    for (int k = 0; k < T; ++k)
      if (ti[k] >= 0) {
        out[ti[k]] = dfx[k];
        out[ps + ti[k]] = dfy[k];
      }
  }
}

__global__ void __launch_bounds__(kSTPB, 4) allpairs_sym_f32_kernel(long long n, const float* __restrict__ xs,
                                                                    const float* __restrict__ ys,
                                                                    const float* __restrict__ gam, float inv2pi,
                                                                    float dp, long long B,
                                                                    double* __restrict__ part, long long ps,
                                                                    long long k0) {
  __shared__ float2 sp[2 * kSTPB];
  __shared__ float sg[2 * kSTPB];
  __shared__ double2 sj[kSTPB / 32][kSTPB];
  int I, J;
  decode_pair(k0 + blockIdx.x, I, J);
  if (I == J) {
    diag_item_f32(n, xs, ys, gam, inv2pi, dp, B, I, part, ps, sp, sg);
    return;
  }
  if ((long long)(J + 1) * B > n)
    sym_item_f32<true>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
  else
    sym_item_f32<false>(n, xs, ys, gam, inv2pi, dp, B, I, J, part, ps, sp, sg, sj);
}

// f_i = (float)(Σ_K part[K][·][i], ascending K) + inflow (the rounding of
// reduce_velocity_f32_kernel).
__global__ void reduce_sym_f32_kernel(long long n, int nb, const double* __restrict__ part,
                                      const float* __restrict__ inflow, float* __restrict__ f, DeviceStatus* st) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k < nb; ++k) {
      sx += part[(long long)k * 2 * n + i];
      sy += part[((long long)k * 2 + 1) * n + i];
    }
    float ox = (float)sx, oy = (float)sy;
    if (inflow) {
      ox = ox + inflow[i];
      oy = oy + inflow[i + n];
    }
    if (!isfinite(ox) || !isfinite(oy)) latch_status(st, kStatusNonFiniteVelocity, i);
    f[i] = ox;
    f[i + n] = oy;
  }
}

}  // namespace

bool sym_velocity_applies(ptrom_ctx* ctx, long long n) {
  if (n < kSymMinN) return false;
  const char* v = std::getenv("PTROM_ALLPAIRS_SYM");
  if (v && v[0] == '0') return false;
  (void)ctx;
  return true;
}

// Block size: a multiple of 1,024 whose block pairs (split over `world`
// ranks) fill the resident CTAs in whole waves best, with the partial buffer
// (nb x 2 x n doubles) ≤ 12 GB (24 GB when sharded).
static long long choose_sym_block(long long n, int resident, int world) {
  long long best = 0;
  double best_eff = -1.0;
  const double cap = world > 1 ? 24e9 : 12e9;
  for (long long B = kSPass; B <= std::max<long long>(kSPass, n); B *= 2) {
    const long long nb = (n + B - 1) / B;
    if ((double)nb * 2.0 * (double)n * 8.0 > cap) continue;
    const double items = (double)(nb * (nb + 1) / 2) / world;
    const double waves = items / resident;
    double eff = waves / std::ceil(waves);
    if (items < 2.0 * resident) eff *= items / (2.0 * resident);  // too few items to balance
    if (eff > best_eff + 0.01) {
      best_eff = eff;
      best = B;
    }
  }
  return best ? best : kSPass;
}

static int sym_occupancy() {
  static int occ = [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, allpairs_sym_kernel, kSTPB, 0);
    return std::max(o, 1);
  }();
  return occ;
}

static void launch_sym_items(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double dp,
                             long long B, double* part, long long ps, long long k0, long long count) {
  if (count <= 0) return;
  ProfScope prof(ctx);
  allpairs_sym_kernel<<<(unsigned)count, kSTPB, 0, ctx->stream>>>(n, x, x + n, gamma, 1.0 / (2.0 * M_PI), dp, B, part,
                                                                   ps, k0);
}

void dev_velocity_sym_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                          const double* inflow, double* f) {
  const long long B = choose_sym_block(n, ctx->num_sms * sym_occupancy(), 1);
  const long long nb = (n + B - 1) / B;
  const long long items = nb * (nb + 1) / 2;
  ctx->scratch.reset();
  ctx->scratch.reserve((size_t)nb * 2 * n * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)nb * 2 * n);
  launch_sym_items(ctx, n, x, gamma, effective_delta(delta, form), B, part, n, 0, items);
  PTROM_LAUNCH_CHECK();
  const long long rg = std::min<long long>((n + 255) / 256, (long long)ctx->num_sms * 8);
  reduce_sym_kernel<<<(unsigned)std::max<long long>(rg, 1), 256, 0, ctx->stream>>>(n, (int)nb, part, n, 0, n, 0,
                                                                                  inflow, f, ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

static int sym_f32_occupancy() {
  static int occ = [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, allpairs_sym_f32_kernel, kSTPB, 0);
    return std::max(o, 1);
  }();
  return occ;
}

void dev_velocity_sym_f32(ptrom_ctx* ctx, long long n, const float* x, const float* gamma, float delta, int form,
                          const float* inflow, float* f) {
  const long long B = choose_sym_block(n, ctx->num_sms * sym_f32_occupancy(), 1);
  const long long nb = (n + B - 1) / B;
  const long long items = nb * (nb + 1) / 2;
  ctx->scratch.reset();
  ctx->scratch.reserve((size_t)nb * 2 * n * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)nb * 2 * n);
  const float dp = (float)effective_delta((double)delta, form);
  {
    ProfScope prof(ctx);
    allpairs_sym_f32_kernel<<<(unsigned)items, kSTPB, 0, ctx->stream>>>(n, x, x + n, gamma,
                                                                        (float)(1.0 / (2.0 * M_PI)), dp, B, part, n, 0);
  }
  PTROM_LAUNCH_CHECK();
  const long long rg = std::min<long long>((n + 255) / 256, (long long)ctx->num_sms * 8);
  reduce_sym_f32_kernel<<<(unsigned)std::max<long long>(rg, 1), 256, 0, ctx->stream>>>(n, (int)nb, part, inflow, f,
                                                                                      ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

static int sym_jac_occupancy() {
  static int occ = [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, allpairs_sym_jac_kernel, kSTPB, 0);
    return std::max(o, 1);
  }();
  return occ;
}

// The Jacobian's (A, B, C) partials over unordered pairs into the context
// scratch ([nb][3][n]); size_only sizes the scratch without launching (before
// a graph capture).
void dev_jacobian_sym_part(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double dp,
                           double** part_out, int* nb_out, bool size_only) {
  const long long B = choose_sym_block(n, ctx->num_sms * sym_jac_occupancy(), 1);
  const long long nb = (n + B - 1) / B;
  const long long items = nb * (nb + 1) / 2;
  ctx->scratch.reset();
  ctx->scratch.reserve((size_t)nb * 3 * n * sizeof(double) + 4096);
  double* part = ctx->scratch.take<double>((size_t)nb * 3 * n);
  *part_out = part;
  *nb_out = (int)nb;
  if (size_only) return;
  ProfScope prof(ctx);
  allpairs_sym_jac_kernel<<<(unsigned)items, kSTPB, 0, ctx->stream>>>(n, x, x + n, gamma, 1.0 / (2.0 * M_PI), dp, B,
                                                                      part, n, 0);
  PTROM_LAUNCH_CHECK();
}

// Sharded: rank r computes its contiguous share of the block pairs into a
// zeroed [nb][3][n] buffer, one reduce-scatter hands it the partial rows of
// its own targets (one non-zero contributor per element: exact), and the
// one-sided reduction forms the Newton blocks of rows [r·n/G, (r+1)·n/G):
// bit-identical to the single-GPU evaluation's rows.
void dev_jacobian_sym_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, long long n, const double* x_full,
                                  const double* gamma, double delta, int form, double dt_for_inverse,
                                  double* inv_local) {
  const int G = comm->world;
  const long long B = choose_sym_block(n, ctx->num_sms * sym_jac_occupancy(), G);
  const long long nb = (n + B - 1) / B;
  const long long items = nb * (nb + 1) / 2;
  const long long m = n / G;
  const double dp = effective_delta(delta, form);
  ctx->scratch.reset();
  ctx->scratch.reserve(((size_t)nb * 3 * n + (size_t)nb * 3 * m) * sizeof(double) + 8192);
  double* part = ctx->scratch.take<double>((size_t)nb * 3 * n);
  double* mine = ctx->scratch.take<double>((size_t)nb * 3 * m);
  PTROM_CUDA(cudaMemsetAsync(part, 0, (size_t)nb * 3 * n * sizeof(double), ctx->stream));
  const long long k_lo = items * comm->rank / G, k_hi = items * (comm->rank + 1) / G;
  if (k_hi > k_lo) {
    ProfScope prof(ctx);
    allpairs_sym_jac_kernel<<<(unsigned)(k_hi - k_lo), kSTPB, 0, ctx->stream>>>(
        n, x_full, x_full + n, gamma, 1.0 / (2.0 * M_PI), dp, B, part, n, k_lo);
  }
  PTROM_LAUNCH_CHECK();
  comm_reduce_scatter_rows(ctx, comm, part, 3 * nb, n, mine);
  dev_jacobian_reduce_f64(ctx, mine, (int)nb, (long long)comm->rank * m, m, dp, dt_for_inverse, nullptr, nullptr,
                          nullptr, nullptr, inv_local);
}

bool sym_sharded_applies(ptrom_ctx* ctx, long long n, int world) {
  return world > 1 && n % world == 0 && sym_velocity_applies(ctx, n);
}

// Target-sharded full evaluation over unordered pairs: every rank holds all
// positions (x_full), computes its contiguous share of the block pairs into a
// zeroed partial buffer, and one reduce-scatter (row by row) hands each rank
// the partial rows of its own targets — every element has exactly one
// non-zero contributor, so the sum is exact and the result is bit-identical
// to the single-GPU evaluation; then the same fixed-order reduction.
void dev_velocity_sym_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, long long n, const double* x_full,
                                  const double* gamma, double delta, int form, const double* inflow, double* f_local) {
  const int G = comm->world;
  const long long B = choose_sym_block(n, ctx->num_sms * sym_occupancy(), G);
  const long long nb = (n + B - 1) / B;
  const long long items = nb * (nb + 1) / 2;
  const long long m = n / G;
  ctx->scratch.reset();
  ctx->scratch.reserve(((size_t)nb * 2 * n + (size_t)nb * 2 * m) * sizeof(double) + 8192);
  double* part = ctx->scratch.take<double>((size_t)nb * 2 * n);
  double* mine = ctx->scratch.take<double>((size_t)nb * 2 * m);
  PTROM_CUDA(cudaMemsetAsync(part, 0, (size_t)nb * 2 * n * sizeof(double), ctx->stream));
  const long long k_lo = items * comm->rank / G, k_hi = items * (comm->rank + 1) / G;
  launch_sym_items(ctx, n, x_full, gamma, effective_delta(delta, form), B, part, n, k_lo, k_hi - k_lo);
  PTROM_LAUNCH_CHECK();
  comm_reduce_scatter_rows(ctx, comm, part, 2 * nb, n, mine);
  const long long rg = std::min<long long>((m + 255) / 256, (long long)ctx->num_sms * 8);
  reduce_sym_kernel<<<(unsigned)std::max<long long>(rg, 1), 256, 0, ctx->stream>>>(
      n, (int)nb, mine, m, 0, m, (long long)comm->rank * m, inflow, f_local, ctx->d_status);
  PTROM_LAUNCH_CHECK();
}

}  // namespace ptrom
