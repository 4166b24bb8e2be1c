// pair_tile.cuh — the fp64 pair arithmetic of one source tile against a
// thread's register-resident targets, shared by the all-pairs kernels
// (allpairs.cu) and the persistent small-system FOM kernel
// (fom_persistent.cu). See allpairs.cu for the reciprocal tiers.
#pragma once

#include "common.cuh"

namespace ptrom {

__device__ __forceinline__ double rcp_seed(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  return y;
}
// fp32 reciprocal seed of a double q ∈ [2^-126, 2^126) through integer
// exponent re-biasing (no FP64-pipe conversion instructions); outside that
// range the re-biased exponent wraps or the fp32 reciprocal flushes, so every
// caller guards the range (allpairs_f64_kernel targets_ok / targets_ok4).
__device__ __forceinline__ double rcp_seed_via_f32(double q) {
  const int hi = __double2hiint(q), lo = __double2loint(q);
  const unsigned fb = __funnelshift_l((unsigned)lo, (unsigned)hi, 3) - (896u << 23);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint_as_float(fb)));
  const unsigned rb = __float_as_uint(r);
  return __hiloint2double((int)((rb >> 3) + (896u << 20)), (int)(rb << 29));
}
__device__ __forceinline__ bool coord_ok(double v) {  // |v| < 2^29 (also false for inf/NaN)
  return (__double2hiint(v) & 0x7fffffff) < 0x41C00000;
}
__device__ __forceinline__ bool coord_ok4(double v) {  // |v| < 2^14: q ∈ [δ', 2^31]
  return (__double2hiint(v) & 0x7fffffff) < 0x40D00000;
}
__device__ __forceinline__ float rcp_approx(float q) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(q));
  return y;
}

// ----------------------------------------------------------------- fp64 ---
// Per-pair accumulation given s = Γ'/q and u = 1/q (u only used for JAC).
template <bool VEL, bool JAC>
__device__ __forceinline__ void accumulate(double rx, double ry, double s, double u, double& fx, double& fy,
                                           double& ja, double& jb, double& jc) {
  if (JAC) {
    const double w = s * u;  // Γ'/q²
    const double t = w * rx;
    ja = fma(t, ry, ja);
    const double rx2 = rx * rx;
    jb = fma(w, fma(ry, ry, -rx2), jb);
    jc += w;
  }
  if (VEL) {
    fx = fma(-ry, s, fx);
    fy = fma(rx, s, fy);
  }
}

// One source tile against T register-resident targets of this thread.
//  FAST: targets are taken two at a time and share one reciprocal
//        (Montgomery): u = 1/(q1·q2) from the fp32 seed + one Newton step,
//        then 1/q1 = q2·u, 1/q2 = q1·u. Per pair 9 FP64 ops and 2 ALU/MUFU
//        ops instead of 9 + 4 (the SMSP dispatch, not the FP64 pipe, is the
//        limit: tools/fp64mix.cu). Needs q ∈ [2^-62, 2^61] (tile guard).
//  safe: MUFU.RCP64H + cubic correction per pair (propagates q = 0 as inf/NaN).
template <int T, int UNR, bool VEL, bool JAC, bool MASK, int FAST>
__device__ __forceinline__ void tile_f64(int cnt, const double2* __restrict__ sp, const double* __restrict__ sg,
                                         long long j0, const double (&tx)[T], const double (&ty)[T],
                                         const long long (&ti)[T], double dp, double (&fx)[T], double (&fy)[T],
                                         double (&ja)[T], double (&jb)[T], double (&jc)[T]) {
#pragma unroll UNR
  for (int jj = 0; jj < cnt; ++jj) {
    const double2 p = sp[jj];
    const double g = sg[jj];
    if ((FAST == 4 || FAST == 5) && !MASK && (T % 4 == 0)) {
      // four targets share one reciprocal: P = (q1 q2)(q3 q4), q ∈ [2^-31, 2^31]
#pragma unroll
      for (int k = 0; k < T; k += 4) {
        double rx[4], ry[4], q[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          rx[m] = tx[k + m] - p.x;
          ry[m] = ty[k + m] - p.y;
          q[m] = fma(rx[m], rx[m], fma(ry[m], ry[m], dp));
        }
        const double p01 = q[0] * q[1], p23 = q[2] * q[3];
        const double P = p01 * p23;
        double uP;  // 1/P
        if (FAST == 5) {  // MUFU.RCP64H seed (~2^-20) + cubic correction
          const double y0 = rcp_seed(P);
          double e = fma(-P, y0, 1.0);
          e = fma(e, e, e);
          uP = fma(y0, e, y0);
        } else {  // fp32 seed via exponent rebias (≤ 2^-22) + one Newton step
          const double y0 = rcp_seed_via_f32(P);
          const double e = fma(-P, y0, 1.0);
          uP = fma(y0, e, y0);
        }
        if (JAC) {
          const double u01 = uP * p23, u23 = uP * p01;  // 1/(q0 q1), 1/(q2 q3)
          const double u[4] = {u01 * q[1], u01 * q[0], u23 * q[3], u23 * q[2]};
#pragma unroll
          for (int m = 0; m < 4; ++m)
            accumulate<VEL, JAC>(rx[m], ry[m], g * u[m], u[m], fx[k + m], fy[k + m], ja[k + m], jb[k + m],
                                 jc[k + m]);
        } else {
          const double gu = g * uP;
          const double g01 = gu * p23, g23 = gu * p01;  // Γ'/(q0 q1), Γ'/(q2 q3)
          const double sv[4] = {g01 * q[1], g01 * q[0], g23 * q[3], g23 * q[2]};
#pragma unroll
          for (int m = 0; m < 4; ++m)
            accumulate<VEL, JAC>(rx[m], ry[m], sv[m], 0.0, fx[k + m], fy[k + m], ja[k + m], jb[k + m], jc[k + m]);
        }
      }
    } else if (FAST >= 2 && !MASK && (T % 2 == 0)) {
#pragma unroll
      for (int k = 0; k < T; k += 2) {
        const double rx1 = tx[k] - p.x, ry1 = ty[k] - p.y;
        const double rx2 = tx[k + 1] - p.x, ry2 = ty[k + 1] - p.y;
        const double q1 = fma(rx1, rx1, fma(ry1, ry1, dp));
        const double q2 = fma(rx2, rx2, fma(ry2, ry2, dp));
        const double P = q1 * q2;
        const double y0 = rcp_seed_via_f32(P);
        const double e = fma(-P, y0, 1.0);
        if (JAC) {
          const double uP = fma(y0, e, y0);  // 1/(q1 q2)
          const double u1 = q2 * uP, u2 = q1 * uP;
          accumulate<VEL, JAC>(rx1, ry1, g * u1, u1, fx[k], fy[k], ja[k], jb[k], jc[k]);
          accumulate<VEL, JAC>(rx2, ry2, g * u2, u2, fx[k + 1], fy[k + 1], ja[k + 1], jb[k + 1], jc[k + 1]);
        } else {
          const double gu = g * fma(y0, e, y0);  // Γ'/(q1 q2)
          accumulate<VEL, JAC>(rx1, ry1, gu * q2, 0.0, fx[k], fy[k], ja[k], jb[k], jc[k]);
          accumulate<VEL, JAC>(rx2, ry2, gu * q1, 0.0, fx[k + 1], fy[k + 1], ja[k + 1], jb[k + 1], jc[k + 1]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < T; ++k) {
        const double rx = tx[k] - p.x;
        const double ry = ty[k] - p.y;
        double q = fma(rx, rx, fma(ry, ry, dp));
        double gs = g;
        if (MASK) {
          const bool self = (j0 + jj) == ti[k];  // kernel.hpp:118 `if (j == i) continue;`
          q = self ? 1.0 : q;
          gs = self ? 0.0 : gs;
        }
        const double y0 = rcp_seed(q);
        double e = fma(-q, y0, 1.0);
        e = fma(e, e, e);
        if (JAC) {
          const double u = fma(y0, e, y0);  // 1/q
          accumulate<VEL, JAC>(rx, ry, gs * u, u, fx[k], fy[k], ja[k], jb[k], jc[k]);
        } else {
          const double g0 = gs * y0;
          accumulate<VEL, JAC>(rx, ry, fma(g0, e, g0), 0.0, fx[k], fy[k], ja[k], jb[k], jc[k]);
        }
      }
    }
  }
}

// ----------------------------------------------------------------- fp32 ---
// One source tile against T register-resident fp32 targets (the fp32 pair
// law of kernel.hpp:107-129 at S = float; allpairs.cu / allpairs_sym.cu).
// MUFU.RCP (16/clk/SM) would bound a reciprocal per pair at 1/8 of the FMA
// rate, so on the fast path four targets share one reciprocal of
// P = (q0 q1)(q2 q3) (tile guard: |coords| < 2^13 and δ' in [2^-30, 2^28]
// keep P inside the normal fp32 range); the safe path (and the masked
// diagonal tiles) keep one MUFU.RCP per pair.
__device__ __forceinline__ bool coord_ok_f32(float v) { return fabsf(v) < 8192.f; }

template <int T, bool MASK, bool FAST>
__device__ __forceinline__ void tile_f32(int cnt, const float2* __restrict__ sp, const float* __restrict__ sg,
                                         long long j0, const float (&tx)[T], const float (&ty)[T],
                                         const long long (&ti)[T], float dp, float (&ax)[T], float (&ay)[T]) {
#pragma unroll 4
  for (int jj = 0; jj < cnt; ++jj) {
    const float2 p = sp[jj];
    const float g = sg[jj];
    if (FAST && !MASK && (T % 4 == 0)) {
#pragma unroll
      for (int k = 0; k < T; k += 4) {
        float rx[4], ry[4], q[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          rx[m] = tx[k + m] - p.x;
          ry[m] = ty[k + m] - p.y;
          q[m] = fmaf(rx[m], rx[m], fmaf(ry[m], ry[m], dp));
        }
        const float p01 = q[0] * q[1], p23 = q[2] * q[3];
        const float gu = g * rcp_approx(p01 * p23);  // Γ'/(q0 q1 q2 q3)
        const float g01 = gu * p23, g23 = gu * p01;  // Γ'/(q0 q1), Γ'/(q2 q3)
        const float sv[4] = {g01 * q[1], g01 * q[0], g23 * q[3], g23 * q[2]};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          ax[k + m] = fmaf(-ry[m], sv[m], ax[k + m]);
          ay[k + m] = fmaf(rx[m], sv[m], ay[k + m]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < T; ++k) {
        const float rx = tx[k] - p.x;
        const float ry = ty[k] - p.y;
        float q = fmaf(rx, rx, fmaf(ry, ry, dp));
        float gs = g;
        if (MASK) {
          const bool self = (j0 + jj) == ti[k];
          q = self ? 1.f : q;
          gs = self ? 0.f : gs;
        }
        const float s = gs * rcp_approx(q);
        ax[k] = fmaf(-ry, s, ax[k]);
        ay[k] = fmaf(rx, s, ay[k]);
      }
    }
  }
}


}  // namespace ptrom
