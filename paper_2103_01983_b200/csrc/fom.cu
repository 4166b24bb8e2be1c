// fom.cu — device-resident implicit-trapezoidal FOM (inexact Newton).
//
// Replaces FomStepper::step / refactor (integrators.hpp:117-201) and
// fom_simulate (integrators.hpp:243-272) for the PairwiseModel
// (integrators.hpp:69-79). State, velocity, residual and the per-particle
// 2x2 inverse blocks stay in HBM for the whole trajectory; the host only
// sees one 8-byte residual norm per Newton iteration (the convergence test
// integrators.hpp:140-155 needs it) and the snapshot columns.
//
// Elementwise arithmetic follows the reference rounding order with explicit
// _rn intrinsics (no FMA contraction), so given identical velocities the
// residual and update are bit-identical to the oracle. ‖r‖ is a fixed-order
// two-level reduction (per-thread strided sums, warp/block trees in a fixed
// shape, then the block partials in index order): deterministic run to run.
#include <cmath>
#include <vector>

#include "ops.cuh"

namespace ptrom {

namespace {

constexpr int kNormThreads = 256;
constexpr int kNormBlocks = 296;  // 2 x 148 SMs; fixed so the reduction shape is fixed

// r = (xi - x_prev) - h*(f_xi + f_prev) on rows k and k+ld, k < m
// (integrators.hpp:47-53), with fixed-order partial sums of r².
__global__ void __launch_bounds__(kNormThreads) residual_kernel(long long m, long long ld,
                                                                const double* __restrict__ xi,
                                                                const double* __restrict__ fxi,
                                                                const double* __restrict__ xp,
                                                                const double* __restrict__ fp, double h,
                                                                double* __restrict__ r,
                                                                double* __restrict__ block_part) {
  double acc = 0.0;
  const long long rows = 2 * m;
  for (long long e = blockIdx.x * (long long)kNormThreads + threadIdx.x; e < rows;
       e += (long long)gridDim.x * kNormThreads) {
    const long long k = e < m ? e : (e - m) + ld;
    const double v = __dsub_rn(__dsub_rn(xi[k], xp[k]), __dmul_rn(h, __dadd_rn(fxi[k], fp[k])));
    r[k] = v;
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  __shared__ double warp_sum[kNormThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) s = __dadd_rn(s, warp_sum[w]);
    block_part[blockIdx.x] = s;
  }
}

__global__ void sum_blocks_kernel(int nb, const double* __restrict__ block_part, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s = __dadd_rn(s, block_part[b]);
    *out = s;
  }
}

// integrators.hpp:161-167: d = inv * (-r); x += d (reference rounding order).
__global__ void newton_update_kernel(long long m, long long ld, const double* __restrict__ inv,
                                     const double* __restrict__ r, double* __restrict__ x) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x) {
    const double* b = inv + 4 * k;
    const double rhs0 = -r[k], rhs1 = -r[k + ld];
    const double d0 = __dadd_rn(__dmul_rn(b[0], rhs0), __dmul_rn(b[1], rhs1));
    const double d1 = __dadd_rn(__dmul_rn(b[2], rhs0), __dmul_rn(b[3], rhs1));
    x[k] = __dadd_rn(x[k], d0);
    x[k + ld] = __dadd_rn(x[k + ld], d1);
  }
}

int grid_for(ptrom_ctx* ctx, long long count, int tpb) {
  long long g = (count + tpb - 1) / tpb;
  return (int)std::max(1LL, std::min(g, (long long)ctx->num_sms * 8));
}

}  // namespace

void dev_residual_f64(ptrom_ctx* ctx, long long m, long long ld, const double* xi, const double* fxi,
                      const double* xp, const double* fp, double dt, double* r, double* norm2, double* block_part) {
  residual_kernel<<<kNormBlocks, kNormThreads, 0, ctx->stream>>>(m, ld, xi, fxi, xp, fp, dt / 2.0, r, block_part);
  PTROM_LAUNCH_CHECK();
  sum_blocks_kernel<<<1, 32, 0, ctx->stream>>>(kNormBlocks, block_part, norm2);
  PTROM_LAUNCH_CHECK();
}

void dev_newton_update_f64(ptrom_ctx* ctx, long long m, long long ld, const double* inv, const double* r,
                           double* x) {
  newton_update_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(m, ld, inv, r, x);
  PTROM_LAUNCH_CHECK();
}

size_t residual_block_part_count() { return kNormBlocks; }

// ----------------------------------------------------------- fom_simulate --
// integrators.hpp:243-272 + FomStepper::step integrators.hpp:126-178.
// All buffers are device-resident; host copies only x0 in and snapshots out.
FomResult fom_simulate_device(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma, double delta,
                              int form, const double* d_inflow, double dt, long long n_steps, double tol,
                              int max_iters, int refresh, double* h_snapshots, int* iters, unsigned char* conv,
                              double* rel_out) {
  FomResult out;
  const size_t dim = (size_t)2 * n;
  double *x_prev, *f_prev, *xi, *fxi, *r, *inv, *norm2, *block_part;
  PTROM_CUDA(cudaMallocAsync(&x_prev, dim * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&f_prev, dim * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&xi, dim * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&fxi, dim * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&r, dim * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&inv, (size_t)4 * n * sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&norm2, sizeof(double), ctx->stream));
  PTROM_CUDA(cudaMallocAsync(&block_part, kNormBlocks * sizeof(double), ctx->stream));
  double* h_norm2 = nullptr;
  PTROM_CUDA(cudaMallocHost(&h_norm2, sizeof(double)));
  struct Free {
    ptrom_ctx* c;
    std::vector<void*> d;
    double* h;
    ~Free() {
      for (void* p : d) cudaFreeAsync(p, c->stream);
      cudaFreeHost(h);
    }
  } guard{ctx, {x_prev, f_prev, xi, fxi, r, inv, norm2, block_part}, h_norm2};

  auto read_norm = [&]() -> double {
    PTROM_CUDA(cudaMemcpyAsync(h_norm2, norm2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
    check_device_status(ctx);  // a singular block or non-finite velocity raised on device
    return std::sqrt(*h_norm2);
  };

  // x = x0; f = model.velocity(x0)   (integrators.hpp:257-259)
  PTROM_CUDA(cudaMemcpyAsync(x_prev, d_x0, dim * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  dev_velocity_f64(ctx, n, x_prev, d_gamma, delta, form, d_inflow, 0, n, f_prev, n);
  ++out.velocity_evals;
  bool have_blocks = false;
  for (long long s = 0; s < n_steps; ++s) {
    // xi = x_prev; f_xi = f_prev   (integrators.hpp:130-131)
    PTROM_CUDA(cudaMemcpyAsync(xi, x_prev, dim * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    PTROM_CUDA(cudaMemcpyAsync(fxi, f_prev, dim * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    const bool refresh_due = (s % refresh) == 0 || !have_blocks;
    bool refreshed = false;
    int updates = 0;
    bool converged = false;
    double r0 = 0.0, rel = 0.0;
    while (true) {
      dev_residual_f64(ctx, n, n, xi, fxi, x_prev, f_prev, dt, r, norm2, block_part);
      const double nr = read_norm();
      if (updates == 0) {
        r0 = nr;
        if (r0 == 0.0) {
          converged = true;
          rel = 0.0;
          break;
        }
      }
      rel = nr / r0;
      if (rel <= tol) {
        converged = true;
        break;
      }
      if (updates >= max_iters) break;
      if (refresh_due && !refreshed) {
        dev_jacobian_f64(ctx, n, xi, d_gamma, delta, form, 0, n, nullptr, nullptr, nullptr, nullptr, dt, inv);
        refreshed = true;
        have_blocks = true;
      }
      dev_newton_update_f64(ctx, n, n, inv, r, xi);
      ++updates;
      dev_velocity_f64(ctx, n, xi, d_gamma, delta, form, d_inflow, 0, n, fxi, n);
      ++out.velocity_evals;
    }
    // accepted state becomes the next step's history (integrators.hpp:262-264)
    std::swap(x_prev, xi);
    std::swap(f_prev, fxi);
    if (h_snapshots)
      PTROM_CUDA(cudaMemcpyAsync(h_snapshots + (size_t)s * dim, x_prev, dim * sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx->stream));
    iters[s] = updates;
    conv[s] = converged ? 1 : 0;
    rel_out[s] = rel;
  }
  guard.d = {x_prev, f_prev, xi, fxi, r, inv, norm2, block_part};
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  check_device_status(ctx);
  return out;
}

}  // namespace ptrom
