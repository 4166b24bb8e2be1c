// fp64mix.cu — what limits the all-pairs inner loop? Same shared-memory tile
// structure as csrc/allpairs.cu with the per-pair body swapped by MODE:
//  0 fast path as shipped (DADD x2, DFMA x2, int rebias + MUFU.RCP, DFMA, DMUL, DFMA, DFMA x2)
//  1 no MUFU (rebias only, y0 = rebias(q))
//  2 no MUFU, no rebias (y0 = q)
//  3 MUFU.RCP64H + cubic (10 FP64 ops)
//  4 9 DFMA with the same dependency shape but no conversions
//  5 fast path with 8 targets/thread
// Prints pairs/clk/SM and FP64-op utilization per mode.
#include <cuda_runtime.h>

#include <cstdio>

template <int MODE>
__device__ __forceinline__ void pair(double tx, double ty, double2 p, double g, double dp, double& fx, double& fy) {
  const double rx = tx - p.x, ry = ty - p.y;
  const double q = fma(rx, rx, fma(ry, ry, dp));
  double y0, e;
  if (MODE == 0 || MODE == 1) {
    const int hi = __double2hiint(q), lo = __double2loint(q);
    unsigned fb = __funnelshift_l((unsigned)lo, (unsigned)hi, 3) - (896u << 23);
    float r;
    if (MODE == 0)
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint_as_float(fb)));
    else
      r = __uint_as_float(fb ^ 0x7f000000u);
    const unsigned rb = __float_as_uint(r);
    y0 = __hiloint2double((int)((rb >> 3) + (896u << 20)), (int)(rb << 29));
    e = fma(-q, y0, 1.0);
  } else if (MODE == 2 || MODE == 4) {
    y0 = q;
    e = fma(-q, y0, 1.0);
  } else {
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(q));
    e = fma(-q, y0, 1.0);
    e = fma(e, e, e);
  }
  const double g0 = g * y0;
  const double s = fma(g0, e, g0);
  fx = fma(-ry, s, fx);
  fy = fma(rx, s, fy);
}

__device__ __forceinline__ double seed32(double q) {
  const int hi = __double2hiint(q), lo = __double2loint(q);
  const unsigned fb = __funnelshift_l((unsigned)lo, (unsigned)hi, 3) - (896u << 23);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint_as_float(fb)));
  const unsigned rb = __float_as_uint(r);
  return __hiloint2double((int)((rb >> 3) + (896u << 20)), (int)(rb << 29));
}
// Two targets against one source sharing one reciprocal of q1*q2.
__device__ __forceinline__ void pair2(double tx1, double ty1, double tx2, double ty2, double2 p, double g, double dp,
                                      double& fx1, double& fy1, double& fx2, double& fy2) {
  const double rx1 = tx1 - p.x, ry1 = ty1 - p.y, rx2 = tx2 - p.x, ry2 = ty2 - p.y;
  const double q1 = fma(rx1, rx1, fma(ry1, ry1, dp));
  const double q2 = fma(rx2, rx2, fma(ry2, ry2, dp));
  const double P = q1 * q2;
  const double y0 = seed32(P);
  const double e = fma(-P, y0, 1.0);
  const double gu = g * fma(y0, e, y0);  // g / (q1 q2)
  const double s1 = gu * q2, s2 = gu * q1;
  fx1 = fma(-ry1, s1, fx1);
  fy1 = fma(rx1, s1, fy1);
  fx2 = fma(-ry2, s2, fx2);
  fy2 = fma(rx2, s2, fy2);
}

template <int MODE, int T>
__global__ void __launch_bounds__(128) mix_kernel(const double* xs, const double* ys, const double* gs, int n,
                                                  int reps, double dp, double* out) {
  __shared__ double2 sp[128];
  __shared__ double sg[128];
  double tx[T], ty[T], fx[T], fy[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int i = (blockIdx.x * 128 * T + k * 128 + threadIdx.x) % n;
    tx[k] = xs[i];
    ty[k] = ys[i];
    fx[k] = fy[k] = 0.0;
  }
  for (int r = 0; r < reps; ++r) {
    const int j = (r * 128 + threadIdx.x) % n;
    sp[threadIdx.x] = make_double2(xs[j], ys[j]);
    sg[threadIdx.x] = gs[j];
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < 128; ++jj) {
      const double2 p = sp[jj];
      const double g = sg[jj];
      if (MODE == 9) {
#pragma unroll
        for (int k = 0; k < T; k += 2)
          pair2(tx[k], ty[k], tx[k + 1], ty[k + 1], p, g, dp, fx[k], fy[k], fx[k + 1], fy[k + 1]);
      } else {
#pragma unroll
        for (int k = 0; k < T; ++k) pair<MODE>(tx[k], ty[k], p, g, dp, fx[k], fy[k]);
      }
    }
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < T; ++k) s += fx[k] + fy[k];
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MODE, int T>
void run(const char* name, int fp64_ops, const double* x, const double* y, const double* g, int n, double* out,
         int sms, int clk_khz) {
  const int reps = 64;
  const int blocks = sms * 6 * 4;
  auto k = mix_kernel<MODE, T>;
  k<<<blocks, 128>>>(x, y, g, n, reps, 2.5e-5, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<blocks, 128>>>(x, y, g, n, reps, 2.5e-5, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double pairs = double(blocks) * 128 * T * reps * 128;
  const double per_clk_sm = pairs / (ms * 1e-3) / (sms * clk_khz * 1e3);
  std::printf("{\"mode\": \"%s\", \"T\": %d, \"ms\": %.3f, \"pairs_per_clk_sm\": %.3f, \"fp64_util_at_max_clk\": %.3f}\n",
              name, T, ms, per_clk_sm, per_clk_sm * fp64_ops / 64.0);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 1 << 16;
  double *x, *y, *g, *out;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMalloc(&g, n * 8);
  cudaMalloc(&out, 1 << 26);
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = 0.25 * ((i * 7919) % 1000 - 500) / 500.0;
  cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  for (int i = 0; i < n; ++i) h[i] = 0.25 * ((i * 104729) % 1000 - 500) / 500.0;
  cudaMemcpy(y, h, n * 8, cudaMemcpyHostToDevice);
  for (int i = 0; i < n; ++i) h[i] = 1.0 / n;
  cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
  run<0, 4>("fast", 9, x, y, g, n, out, sms, clk);
  run<1, 4>("no_mufu", 9, x, y, g, n, out, sms, clk);
  run<2, 4>("no_mufu_no_rebias", 9, x, y, g, n, out, sms, clk);
  run<3, 4>("rcp64h_cubic", 10, x, y, g, n, out, sms, clk);
  run<0, 8>("fast_T8", 9, x, y, g, n, out, sms, clk);
  run<2, 8>("no_mufu_no_rebias_T8", 9, x, y, g, n, out, sms, clk);
  run<0, 2>("fast_T2", 9, x, y, g, n, out, sms, clk);
  run<9, 4>("montgomery_T4", 9, x, y, g, n, out, sms, clk);
  run<9, 8>("montgomery_T8", 9, x, y, g, n, out, sms, clk);
  run<9, 2>("montgomery_T2", 9, x, y, g, n, out, sms, clk);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
