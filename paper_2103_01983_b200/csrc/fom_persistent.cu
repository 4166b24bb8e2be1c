// fom_persistent.cu — the implicit-trapezoidal FOM (FomStepper::step +
// fom_simulate, integrators.hpp:117-201, 243-272) for small systems as ONE
// cooperative persistent kernel: the whole trajectory, every Newton
// iteration and every decision, without a host round trip or a kernel
// launch (config 1, N = 4,096: ~400 velocity/Jacobian evaluations of 16.7M
// pairs each, which as separate launches are bound by launch latency and
// graph-node overhead, not by the FP64 pipe).
//
// Work of one evaluation: items = target tiles (TPB threads x T targets in
// registers; 256 x 2 by default) x source chunks, taken grid-stride by the
// resident CTAs, each writing its partials part[chunk][comp][target] (the
// same tile arithmetic as allpairs.cu, pair_tile.cuh). Between phases a grid
// barrier; per-target phases (chunk reduction, residual, Newton blocks,
// update, record) use one fixed thread→target mapping, so they need no
// barrier among themselves.
// ‖r‖: per-CTA fixed-order partials, then every CTA sums them in the same
// fixed order, so all CTAs take the reference's decision (integrators.hpp:
// 140-155) identically; the partials are double-buffered by call parity.
// Residual, Newton blocks and update use the reference's rounding order
// (_rn intrinsics), as fom.cu.
//
// A Newton iteration costs two grid barriers (tiles → residual + norm):
//  * the update ξ + blocks·(−r) is formed in the residual phase into the
//    second ξ buffer (before the norm's barrier); when the step continues the
//    two buffers are swapped — no update phase, no third barrier;
//  * a step's Jacobian point is the previous step's accepted ξ, whose
//    velocity was that step's last evaluation: the evaluation expected to be
//    the last (the previous step's update count) forms the (A, B, C)
//    partials in the same tile pass (shared r, q and reciprocal), and the
//    next step forms its Newton blocks from them before its first residual,
//    into the second block buffer, adopted only when the refresh happens
//    (the reference refreshes inside the loop, after the r0 == 0 exit). A
//    wrong guess costs one separate Jacobian pass, never a different result
//    path: decisions, counters and error latches are the reference's.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "ops.cuh"
#include "pair_tile.cuh"

namespace cg = cooperative_groups;

// Tile phases inlined (as separate __noinline__ functions they measured
// 14.4 -> 17.6 us per evaluation); sources unrolled PTROM_FOM_UNR at a time.
#ifndef PTROM_FOM_NOINLINE
#define PTROM_FOM_NOINLINE
#endif
#ifndef PTROM_FOM_UNR
#define PTROM_FOM_UNR 8
#endif

namespace ptrom {
namespace {

// Threads per CTA is a template argument (128, 256 or 512; tuning knob
// PTROM_FOM_TPB): the tile phases want ≥ 4 warps per SM sub-partition to hide
// the FP64 latency, the grid barriers want few CTAs.
// Targets per thread in a tile item (2 or 4; PTROM_FOM_TPT) likewise.
constexpr long long kPersistentMaxN = 16384;

struct PFom {
  long long n;
  const double* g;       // Γ (n)
  const double* inflow;  // 2n or null
  double dp;             // effective delta
  double h;              // dt / 2
  double* xp;            // x_prev (2n); holds x0 on entry
  double* fp;            // f_prev (2n)
  double* xi;            // ξ
  double* xi2;           // the other ξ buffer (speculative Newton update, swapped in)
  double* fxi;           // f_ξ
  double* r;             // residual
  double* inv;           // 4n Newton blocks
  double* inv2;          // blocks formed ahead of the refresh that adopts them (swapped in)
  double* part;          // [nch][2][n] velocity partials
  double* part_j;        // [nch][3][n] Jacobian (A, B, C) partials
  double* block_part;    // [2][gridDim] per-CTA partial ‖r‖² (double-buffered by parity)
  double* snaps;         // 2n x n_steps
  int* iters;
  unsigned char* conv;
  double* rel_out;
  long long n_steps;
  double tol;
  int max_iters, refresh;
  int nch, n_tiles;
  long long chunk_len;
  long long* counters;  // [0] velocity evaluations, [1] Jacobian evaluations
  DeviceStatus* st;
  unsigned long long* prof;  // PTROM_FOM_PROFILE phase times, or null
};

// Fixed-order block sum of one double per thread (warp shuffles, then the
// warps in order); the result in every thread.
template <int TPB>
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < TPB / 32; ++w) s = __dadd_rn(s, red[w]);
  return s;
}

// One tile item's partials (allpairs_f64_kernel's tile loop on SrcFlat).
template <int TPB, int T, bool VEL, bool JAC>
__device__ PTROM_FOM_NOINLINE void pair_items(const PFom& P, const double* __restrict__ x, double2* sp, double* sg) {
  constexpr int kPTile = TPB * T;
  const double inv2pi = 1.0 / (2.0 * M_PI);
  const long long n = P.n;
  const int tid = threadIdx.x;
  const int n_items = P.n_tiles * P.nch;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int tile = item % P.n_tiles, chunk = item / P.n_tiles;
    const long long tile0 = (long long)tile * kPTile;
    double tx[T], ty[T], fx[T], fy[T], ja[T], jb[T], jc[T];
    long long ti[T];
    bool my_ok = true, my_ok4 = true;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const long long i = tile0 + k * TPB + tid;
      const bool ok = i < n;
      ti[k] = ok ? i : -1;
      tx[k] = ok ? x[i] : 0.0;
      ty[k] = ok ? x[n + i] : 0.0;
      fx[k] = fy[k] = ja[k] = jb[k] = jc[k] = 0.0;
      my_ok = my_ok && coord_ok(tx[k]) && coord_ok(ty[k]);
      my_ok4 = my_ok4 && coord_ok4(tx[k]) && coord_ok4(ty[k]);
    }
    const long long tile_end = min(tile0 + (long long)kPTile, n);
    const long long cbeg = (long long)chunk * P.chunk_len, cend = min(n, cbeg + P.chunk_len);
    const double dp = P.dp;
    // the first source tile's loads are issued with the target loads (one
    // L2 round trip after the grid barrier, not two)
    double px = 0.0, py = 0.0, pg = 0.0;
    if (cbeg + tid < cend) {
      px = x[cbeg + tid];
      py = x[n + cbeg + tid];
      pg = P.g[cbeg + tid] * inv2pi;
    }
    const bool targets_ok = __syncthreads_and(my_ok) && dp >= 0x1p-62 && dp <= 0x1p60;
    const bool targets_ok4 = __syncthreads_and(my_ok4) && dp >= 0x1p-31 && dp <= 0x1p29;
    for (long long j0 = cbeg; j0 < cend; j0 += TPB) {
      const int cnt = (int)min((long long)TPB, cend - j0);
      sp[tid] = make_double2(px, py);
      sg[tid] = pg;
      const bool fast4 = __syncthreads_and(coord_ok4(px) && coord_ok4(py)) && targets_ok4;
      const bool fast = fast4 || (__syncthreads_and(coord_ok(px) && coord_ok(py)) && targets_ok);
      const long long jn = j0 + TPB + tid;
      if (jn < cend) {
        px = x[jn];
        py = x[n + jn];
        pg = P.g[jn] * inv2pi;
      }
      const bool masked = (j0 < tile_end) && (tile0 < j0 + cnt) && (JAC || !fast);
      if (masked)
        tile_f64<T, PTROM_FOM_UNR, VEL, JAC, true, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else if (fast)
        tile_f64<T, PTROM_FOM_UNR, VEL, JAC, false, 2>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      else
        tile_f64<T, PTROM_FOM_UNR, VEL, JAC, false, 0>(cnt, sp, sg, j0, tx, ty, ti, dp, fx, fy, ja, jb, jc);
      __syncthreads();
    }
    double* out = P.part + (long long)chunk * 2 * n;
    double* outj = P.part_j + (long long)chunk * 3 * n;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      if (ti[k] < 0) continue;
      if (VEL) {
        out[ti[k]] = fx[k];
        out[n + ti[k]] = fy[k];
      }
      if (JAC) {
        outj[ti[k]] = ja[k];
        outj[n + ti[k]] = jb[k];
        outj[2 * n + ti[k]] = jc[k];
      }
    }
  }
}

// [velocity chunk reduction →] residual r = ξ − x_prev − h(f_ξ + f_prev)
// (integrators.hpp:47-53) → ‖r‖ (every CTA, same fixed order). One fixed
// thread→target mapping for every per-target phase.
// With spec_out, the Newton update ξ + blocks·(−r) this residual would lead to
// (newton_update's arithmetic, the current blocks) is also written to spec_out:
// if the step continues, the kernel swaps the two ξ buffers instead of running
// an update phase and its grid barrier.
template <int TPB>
__device__ double residual_norm(const PFom& P, const double* xi, double* spec_out, const double* blocks,
                                bool with_velocity, int parity, double* red, cg::grid_group& grid) {
  const long long n = P.n;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, gs = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = g0; i < n; i += gs) {
    // the thread's own state is loaded together with the chunk partials (one
    // L2 round trip; f_ξ stays in registers instead of being stored and re-read)
    const double xi0 = xi[i], xi1 = xi[n + i], xp0 = P.xp[i], xp1 = P.xp[n + i];
    const double fp0 = P.fp[i], fp1 = P.fp[n + i];
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    if (spec_out) {
      const double* b = blocks + 4 * i;
      b0 = b[0];
      b1 = b[1];
      b2 = b[2];
      b3 = b[3];
    }
    double sx, sy;
    if (with_velocity) {  // chunk partials in ascending chunk order (fixed), + inflow
      sx = sy = 0.0;
      int c = 0;
      for (; c + 16 <= P.nch; c += 16) {  // 16 chunks loaded ahead of their adds
        double vx[16], vy[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          vx[u] = __ldcg(P.part + (long long)(c + u) * 2 * n + i);
          vy[u] = __ldcg(P.part + ((long long)(c + u) * 2 + 1) * n + i);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          sx += vx[u];
          sy += vy[u];
        }
      }
      for (; c < P.nch; ++c) {
        sx += __ldcg(P.part + (long long)c * 2 * n + i);
        sy += __ldcg(P.part + ((long long)c * 2 + 1) * n + i);
      }
      if (P.inflow) {
        sx = sx + P.inflow[i];
        sy = sy + P.inflow[n + i];
      }
      if (!isfinite(sx) || !isfinite(sy)) latch_status(P.st, kStatusNonFiniteVelocity, i);
      P.fxi[i] = sx;
      P.fxi[n + i] = sy;
    } else {
      sx = P.fxi[i];
      sy = P.fxi[n + i];
    }
    const double v0 = __dsub_rn(__dsub_rn(xi0, xp0), __dmul_rn(P.h, __dadd_rn(sx, fp0)));
    const double v1 = __dsub_rn(__dsub_rn(xi1, xp1), __dmul_rn(P.h, __dadd_rn(sy, fp1)));
    P.r[i] = v0;
    P.r[n + i] = v1;
    acc = __dadd_rn(acc, __dmul_rn(v0, v0));
    acc = __dadd_rn(acc, __dmul_rn(v1, v1));
    if (spec_out) {  // newton_update's arithmetic
      const double rhs0 = -v0, rhs1 = -v1;
      const double d0 = __dadd_rn(__dmul_rn(b0, rhs0), __dmul_rn(b1, rhs1));
      const double d1 = __dadd_rn(__dmul_rn(b2, rhs0), __dmul_rn(b3, rhs1));
      spec_out[i] = __dadd_rn(xi0, d0);
      spec_out[n + i] = __dadd_rn(xi1, d1);
    }
  }
  double* bp = P.block_part + (long long)parity * gridDim.x;
  const double s = block_sum<TPB>(acc, red);
  if (threadIdx.x == 0) bp[blockIdx.x] = s;
  grid.sync();
  // every CTA: the same partials in the same order; only the CTAs that own
  // targets under the grid-stride mapping contributed, and their partials
  // are loaded together (one L2 round trip, not one per partial)
  const int nb = (int)min((long long)gridDim.x, (n + blockDim.x - 1) / blockDim.x);
  const int lane = threadIdx.x & 31;
  double v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = lane + 32 * u < nb ? __ldcg(bp + lane + 32 * u) : 0.0;
  double tot = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) tot = __dadd_rn(tot, v[u]);
  for (int b = lane + 256; b < nb; b += 32) tot = __dadd_rn(tot, __ldcg(bp + b));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot = __dadd_rn(tot, __shfl_down_sync(0xffffffffu, tot, o));
  tot = __shfl_sync(0xffffffffu, tot, 0);
  return sqrt(tot);
}

// Newton blocks (I − h·J)^-1 at ξ from the Jacobian partials
// (integrators.hpp:181-194, reduce_jacobian_f64_kernel<true>'s rounding).
// Returns the thread's first singular block (or -1); latched at once unless
// the blocks are formed ahead of a refresh that may not happen (the caller
// latches when it adopts them).
__device__ long long newton_blocks(const PFom& P, double* inv, bool latch) {
  long long first_singular = -1;
  const long long n = P.n;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, gs = (long long)gridDim.x * blockDim.x;
  for (long long i = g0; i < n; i += gs) {
    double a = 0.0, b = 0.0, c = 0.0;
    int ch = 0;
    for (; ch + 8 <= P.nch; ch += 8) {  // ascending chunks, 8 loaded ahead of their adds
      double va[8], vb[8], vc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* pc = P.part_j + (long long)(ch + u) * 3 * n + i;
        va[u] = __ldcg(pc);
        vb[u] = __ldcg(pc + n);
        vc[u] = __ldcg(pc + 2 * n);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a += va[u];
        b += vb[u];
        c += vc[u];
      }
    }
    for (; ch < P.nch; ++ch) {
      const double* pc = P.part_j + (long long)ch * 3 * n + i;
      a += __ldcg(pc);
      b += __ldcg(pc + n);
      c += __ldcg(pc + 2 * n);
    }
    const double j00 = 2.0 * a, j11 = -2.0 * a;
    const double j01 = b - P.dp * c, j10 = b + P.dp * c;
    const double b00 = __dsub_rn(1.0, __dmul_rn(P.h, j00));
    const double b01 = __dsub_rn(0.0, __dmul_rn(P.h, j01));
    const double b10 = __dsub_rn(0.0, __dmul_rn(P.h, j10));
    const double b11 = __dsub_rn(1.0, __dmul_rn(P.h, j11));
    const double det = __dsub_rn(__dmul_rn(b00, b11), __dmul_rn(b01, b10));
    if (det == 0.0 || !isfinite(det)) {
      if (latch) latch_status(P.st, kStatusSingularBlock, i);
      if (first_singular < 0) first_singular = i;
    }
    double* o = inv + 4 * i;
    o[0] = __ddiv_rn(b11, det);
    o[1] = __ddiv_rn(-b01, det);
    o[2] = __ddiv_rn(-b10, det);
    o[3] = __ddiv_rn(b00, det);
  }
  return first_singular;
}

// ξ += blocks · (−r) (integrators.hpp:161-167, newton_update_kernel's rounding).
__device__ void newton_update(const PFom& P, const double* inv, double* xi) {
  const long long n = P.n;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, gs = (long long)gridDim.x * blockDim.x;
  for (long long i = g0; i < n; i += gs) {
    const double* b = inv + 4 * i;
    const double rhs0 = -P.r[i], rhs1 = -P.r[n + i];
    const double d0 = __dadd_rn(__dmul_rn(b[0], rhs0), __dmul_rn(b[1], rhs1));
    const double d1 = __dadd_rn(__dmul_rn(b[2], rhs0), __dmul_rn(b[3], rhs1));
    xi[i] = __dadd_rn(xi[i], d0);
    xi[n + i] = __dadd_rn(xi[n + i], d1);
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// PTROM_FOM_PROFILE: CTA 0 accumulates the wall time (ns) of each phase
// kind into P.prof[0..7]: 0 velocity tiles, 1 barrier after them, 2 reduction
// + residual + norm, 3 Jacobian tiles, 4 barrier after them, 5 blocks +
// update, 6 barrier after the update, 7 record.
#define PF_MARK(k)                                          \
  if (P.prof && threadIdx.x == 0 && blockIdx.x == 0) {      \
    const unsigned long long t_ = gtimer();                 \
    P.prof[k] += t_ - t_last;                               \
    t_last = t_;                                            \
  }

template <int TPB, int T>
__global__ void __launch_bounds__(TPB) fom_persistent_kernel(PFom P) {
  unsigned long long t_last = P.prof ? gtimer() : 0;
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 sp[TPB];
  __shared__ double sg[TPB];
  __shared__ double red[TPB / 32];
  const long long n = P.n;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, gs = (long long)gridDim.x * blockDim.x;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  double* xi = P.xi;    // the current iterate
  double* xi2 = P.xi2;  // the speculative next iterate (swapped in when the step continues)
  double* inv = P.inv;  // the Newton blocks in use / the buffer early refreshes are formed into
  double* inv2 = P.inv2;
  // f = velocity(x0) (integrators.hpp:257-259); ξ = x_prev, f_ξ = f_prev. The
  // first step's Jacobian point is x0 too: both in one tile pass.
  pair_items<TPB, T, true, true>(P, P.xp, sp, sg);
  bool jac_ready = true;  // part_j holds the Jacobian partials at the current ξ
  grid.sync();
  for (long long i = g0; i < n; i += gs) {
    double sx = 0.0, sy = 0.0;
    for (int c = 0; c < P.nch; ++c) {
      sx += __ldcg(P.part + (long long)c * 2 * n + i);
      sy += __ldcg(P.part + ((long long)c * 2 + 1) * n + i);
    }
    if (P.inflow) {
      sx = sx + P.inflow[i];
      sy = sy + P.inflow[n + i];
    }
    if (!isfinite(sx) || !isfinite(sy)) latch_status(P.st, kStatusNonFiniteVelocity, i);
    P.fp[i] = P.fxi[i] = sx;
    P.fp[n + i] = P.fxi[n + i] = sy;
    xi[i] = P.xp[i];
    xi[n + i] = P.xp[n + i];
  }
  long long evals = 1, jevals = 0;
  int parity = 0;
  bool have_blocks = false;
  int predicted = -1;  // the previous step's update count: its last evaluation is the next Jacobian point
  for (long long s = 0; s < P.n_steps; ++s) {
    const bool refresh_due = (s % P.refresh) == 0 || !have_blocks;
    const bool next_refresh = s + 1 < P.n_steps && ((s + 1) % P.refresh) == 0;
    bool refreshed = false, converged = false;
    int updates = 0;
    double r0 = 0.0, rel = 0.0;
    // f_ξ = f_prev: no evaluation. The update is formed speculatively with the
    // blocks the step's first update will use: the current ones, or — when a
    // refresh is due and the Jacobian partials at this ξ are ready — the new
    // blocks, formed into the second buffer and adopted only if the refresh
    // happens (a step that converges at once leaves the old blocks in place).
    const bool early_blocks = refresh_due && jac_ready;
    const long long early_singular = early_blocks ? newton_blocks(P, inv2, false) : -1;
    bool spec = early_blocks || (have_blocks && !refresh_due);
    double nr = residual_norm<TPB>(P, xi, spec ? xi2 : nullptr, early_blocks ? inv2 : inv, false, parity, red, grid);
    parity ^= 1;
    while (true) {  // integrators.hpp:140-178
      if (updates == 0) {
        r0 = nr;
        if (r0 == 0.0) {
          converged = true;
          rel = 0.0;
          break;
        }
      }
      rel = nr / r0;
      if (rel <= P.tol) {
        converged = true;
        break;
      }
      if (updates >= P.max_iters) break;
      PF_MARK(7);
      if (refresh_due && !refreshed) {
        if (early_blocks) {  // formed before the residual: adopt them
          double* t = inv;
          inv = inv2;
          inv2 = t;
          if (early_singular >= 0) latch_status(P.st, kStatusSingularBlock, early_singular);
        } else {  // Jacobian not evaluated together with the velocity at this ξ
          pair_items<TPB, T, false, true>(P, xi, sp, sg);
          PF_MARK(3);
          grid.sync();
          PF_MARK(4);
          newton_blocks(P, inv, true);  // same thread→target mapping as the update below
          spec = false;           // no speculative update with these blocks
        }
        refreshed = have_blocks = true;
        ++jevals;
      }
      if (spec) {  // ξ ← the update formed with the residual (stored before the norm's grid barrier)
        double* t = xi;
        xi = xi2;
        xi2 = t;
        PF_MARK(5);
      } else {
        newton_update(P, inv, xi);
        PF_MARK(5);
        grid.sync();  // every ξ updated before any tile reads the sources
        PF_MARK(6);
      }
      ++updates;
      jac_ready = false;  // ξ moved
      // the evaluation expected to be the step's last (the previous step's
      // update count) also forms the next step's Jacobian partials at the same ξ
      const bool fuse = next_refresh && updates == predicted;
      const unsigned long long tc0 = (P.prof && threadIdx.x == 0) ? gtimer() : 0;
      if (fuse)
        pair_items<TPB, T, true, true>(P, xi, sp, sg);
      else
        pair_items<TPB, T, true, false>(P, xi, sp, sg);
      jac_ready = fuse;
      ++evals;
      PF_MARK(0);
      const unsigned long long tc1 = (P.prof && threadIdx.x == 0) ? gtimer() : 0;
      grid.sync();
      PF_MARK(1);
      if (P.prof && threadIdx.x == 0) {  // per-CTA view: own tile time, own wait in the barrier
        P.prof[8 + blockIdx.x] += tc1 - tc0;
        P.prof[8 + gridDim.x + blockIdx.x] += gtimer() - tc1;
      }
      spec = true;  // blocks are current for the rest of the step
      nr = residual_norm<TPB>(P, xi, xi2, inv, true, parity, red, grid);
      parity ^= 1;
      PF_MARK(2);
    }
    predicted = updates;
    // the accepted state is the next step's history and initial guess
    // (integrators.hpp:262-264, 130-131), recorded as a snapshot column
    double* col = P.snaps + s * 2 * n;
    for (long long i = g0; i < n; i += gs) {
      const double x0 = xi[i], x1 = xi[n + i];
      col[i] = x0;
      col[n + i] = x1;
      P.xp[i] = x0;
      P.xp[n + i] = x1;
      P.fp[i] = P.fxi[i];
      P.fp[n + i] = P.fxi[n + i];
    }
    if (lead) {
      P.iters[s] = updates;
      P.conv[s] = converged ? 1 : 0;
      P.rel_out[s] = rel;
    }
  }
  if (lead) {
    P.counters[0] = evals;
    P.counters[1] = jevals;
  }
}

}  // namespace

bool fom_persistent_applies(ptrom_ctx* ctx, long long n) {
  if (n > kPersistentMaxN || n < 2) return false;
  const char* v = std::getenv("PTROM_FOM_PERSISTENT");
  if (v && v[0] == '0') return false;
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
  return coop != 0;
}

FomResult fom_simulate_persistent(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma,
                                  double delta, int form, const double* d_inflow, double dt, long long n_steps,
                                  double tol, int max_iters, int refresh, double* snapshots_out, int* iters,
                                  unsigned char* conv, double* rel_out) {
  cudaStream_t st = ctx->stream;
  // CTA shape (tuning knobs PTROM_FOM_TPB x PTROM_FOM_PCTAS x PTROM_FOM_TPT:
  // threads per CTA, CTAs per SM, targets per thread). Every phase ends in a
  // grid barrier whose cost grows with the CTA count (1.5 us at 148 CTAs, the
  // slowest CTA waits on), and the tile phase wants warps: 256 x 1 x 2
  // measured 9.29 ms per config-1 trajectory, 128 x 2 x 2 10.06, 512 x 1 x 2
  // 9.76 (37 source chunks to reduce instead of 18), 128 x 4 x 2 10.31
  // (profiles/r02_fom_shape_sweep.txt).
  int tpb = 256, per_sm = 1, tpt = 2;
  if (const char* v = std::getenv("PTROM_FOM_TPB")) tpb = std::atoi(v);
  if (tpb != 128 && tpb != 256 && tpb != 512) tpb = 256;
  if (const char* v = std::getenv("PTROM_FOM_TPT")) tpt = std::atoi(v);
  if (tpt != 1 && tpt != 2 && tpt != 4) tpt = 2;
  if (const char* v = std::getenv("PTROM_FOM_PCTAS")) per_sm = std::max(1, std::atoi(v));
  auto pick = [&](auto t) -> const void* {
    constexpr int T = decltype(t)::value;
    return tpb == 512   ? (const void*)fom_persistent_kernel<512, T>
           : tpb == 256 ? (const void*)fom_persistent_kernel<256, T>
                        : (const void*)fom_persistent_kernel<128, T>;
  };
  const void* kernel = tpt == 4   ? pick(std::integral_constant<int, 4>{})
                       : tpt == 1 ? pick(std::integral_constant<int, 1>{})
                                  : pick(std::integral_constant<int, 2>{});
  int occ = 0;
  PTROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, tpb, 0));
  const int grid = ctx->num_sms * std::max(1, std::min(occ, per_sm));
  const int kPTile = tpb * tpt;
  PFom P{};
  P.n = n;
  P.g = d_gamma;
  P.inflow = d_inflow;
  P.dp = effective_delta(delta, form);
  P.h = dt / 2.0;
  P.n_steps = n_steps;
  P.tol = tol;
  P.max_iters = max_iters;
  P.refresh = refresh;
  P.n_tiles = (int)((n + kPTile - 1) / kPTile);
  P.nch = (int)std::max(1LL, std::min<long long>(grid / P.n_tiles, n / 32));
  P.chunk_len = (n + P.nch - 1) / P.nch;
  P.st = ctx->d_status;
  std::vector<void*> bufs;
  struct Free {
    std::vector<void*>* b;
    cudaStream_t s;
    ~Free() {
      for (void* p : *b) cudaFreeAsync(p, s);
    }
  } guard{&bufs, st};
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    PTROM_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 8), st));
    bufs.push_back(p);
    return p;
  };
  const size_t dim = 2 * (size_t)n;
  P.xp = (double*)alloc(dim * 8);
  P.fp = (double*)alloc(dim * 8);
  P.xi = (double*)alloc(dim * 8);
  P.xi2 = (double*)alloc(dim * 8);
  P.fxi = (double*)alloc(dim * 8);
  P.r = (double*)alloc(dim * 8);
  P.inv = (double*)alloc(4 * (size_t)n * 8);
  P.inv2 = (double*)alloc(4 * (size_t)n * 8);
  P.part = (double*)alloc((size_t)P.nch * 2 * n * 8);
  P.part_j = (double*)alloc((size_t)P.nch * 3 * n * 8);
  P.block_part = (double*)alloc(2 * (size_t)grid * 8);
  const bool own_snaps = snapshots_out == nullptr;
  P.snaps = (double*)alloc(dim * std::max<long long>(n_steps, 1) * 8);
  P.iters = (int*)alloc(std::max<long long>(n_steps, 1) * 4);
  P.conv = (unsigned char*)alloc(std::max<long long>(n_steps, 1));
  P.rel_out = (double*)alloc(std::max<long long>(n_steps, 1) * 8);
  P.counters = (long long*)alloc(16);
  const bool prof = std::getenv("PTROM_FOM_PROFILE") != nullptr;
  if (prof) {
    P.prof = (unsigned long long*)alloc(64 + 16 * (size_t)grid);
    PTROM_CUDA(cudaMemsetAsync(P.prof, 0, 64 + 16 * (size_t)grid, st));
  }
  PTROM_CUDA(cudaMemcpyAsync(P.xp, d_x0, dim * 8, cudaMemcpyDeviceToDevice, st));
  void* args[] = {&P};
  PTROM_CUDA(cudaLaunchCooperativeKernel(kernel, dim3(grid), dim3(tpb), args, 0, st));
  PTROM_LAUNCH_CHECK();
  long long cnt[2] = {0, 0};
  if (n_steps > 0) {
    PTROM_CUDA(cudaMemcpyAsync(iters, P.iters, n_steps * 4, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaMemcpyAsync(conv, P.conv, n_steps, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaMemcpyAsync(rel_out, P.rel_out, n_steps * 8, cudaMemcpyDeviceToHost, st));
    if (!own_snaps)
      PTROM_CUDA(cudaMemcpyAsync(snapshots_out, P.snaps, dim * n_steps * 8, cudaMemcpyDefault, st));
  }
  PTROM_CUDA(cudaMemcpyAsync(cnt, P.counters, 16, cudaMemcpyDeviceToHost, st));
  unsigned long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::vector<unsigned long long> pc(prof ? 2 * (size_t)grid : 0);
  if (prof) {
    PTROM_CUDA(cudaMemcpyAsync(pr, P.prof, 64, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaMemcpyAsync(pc.data(), P.prof + 8, 16 * (size_t)grid, cudaMemcpyDeviceToHost, st));
  }
  PTROM_CUDA(cudaStreamSynchronize(st));
  if (prof)
    fprintf(stderr, "fom_persistent grid %d x %d x %d nch %d: vel %.3f ms, sync %.3f, reduce+norm %.3f, jac %.3f, sync %.3f, "
                    "blocks+update %.3f, sync %.3f, other %.3f\n",
            grid, tpb, tpt, P.nch, pr[0] * 1e-6, pr[1] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6, pr[4] * 1e-6, pr[5] * 1e-6,
            pr[6] * 1e-6, pr[7] * 1e-6);
  if (prof) {  // velocity phase per CTA: tile time (min / median / max) and the smallest barrier wait
    std::vector<unsigned long long> a(pc.begin(), pc.begin() + grid), w(pc.begin() + grid, pc.end());
    std::sort(a.begin(), a.end());
    std::sort(w.begin(), w.end());
    const double per = 1e-3 / std::max<long long>(cnt[0] - 1, 1);
    fprintf(stderr, "  velocity phase per evaluation, per CTA: tiles min %.2f / median %.2f / max %.2f us; barrier wait min "
                    "%.2f / median %.2f / max %.2f us\n",
            a.front() * per, a[grid / 2] * per, a.back() * per, w.front() * per, w[grid / 2] * per, w.back() * per);
  }
  check_device_status(ctx);
  FomResult out;
  out.velocity_evals = cnt[0];
  out.jacobian_evals = cnt[1];
  return out;
}

}  // namespace ptrom
