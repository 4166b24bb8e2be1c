// peaks.cu — microbenchmarks for the roofline denominators MEASURED_PEAKS.json
// lacks (SURVEY.md §8d "Peaks"): FP64 DFMA, FP32 FFMA, MUFU.RCP64H and FP64
// DMMA (mma.sync m8n8k4) throughput, plus the accuracy of the MUFU.RCP64H seed
// and of the cubic correction used by the all-pairs kernel.
// Built as tools/libptrom_peaks.so (called in-process by bench.py) and as a
// standalone binary printing one JSON line.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

namespace {

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;
}

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5f) out[0] = s;
}

__global__ void rcp64_kernel(double* out) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double y;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[k]));
      x[k] = y;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double* out) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void rcp_accuracy_kernel(const double* q, int n, double* err_seed, double* err_cubic,
                                    double* err_newton1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = q[i];
  double y0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(v));
  const double exact = __drcp_rn(v);
  double e = fma(-v, y0, 1.0);
  const double y1 = fma(y0, e, y0);
  const double e2 = fma(e, e, e);
  const double y3 = fma(y0, e2, y0);
  err_seed[i] = fabs(y0 - exact) / exact;
  err_newton1[i] = fabs(y1 - exact) / exact;
  err_cubic[i] = fabs(y3 - exact) / exact;
}

template <class F>
double time_ms(F&& launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms;
}

}  // namespace

extern "C" int ptrom_peaks(int device, double* out /* 9 values */) {
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d;
  cudaMalloc(&d, 1 << 20);
  const int blocks = sms * 8, tpb = 256;
  const double threads = double(blocks) * tpb;
  const double ms_d = time_ms([&] { dfma_kernel<<<blocks, tpb>>>(d, 0.999, 1e-3); });
  const double ms_f = time_ms([&] { ffma_kernel<<<blocks, tpb>>>((float*)d, 0.999f, 1e-3f); });
  const double ms_r = time_ms([&] { rcp64_kernel<<<blocks, tpb>>>(d); });
  const double ms_m = time_ms([&] { dmma_kernel<<<blocks, tpb>>>(d); });
  out[0] = threads * kIters * 8 * 2 / (ms_d * 1e-3) / 1e12;        // FP64 TFLOP/s (DFMA)
  out[1] = threads * kIters * 8 * 2 / (ms_f * 1e-3) / 1e12;        // FP32 TFLOP/s (FFMA)
  out[2] = threads * (kIters / 4) * 8 / (ms_r * 1e-3) / 1e12;      // MUFU.RCP64H T/s
  out[3] = (threads / 32) * (kIters / 4) * 4 * 512 / (ms_m * 1e-3) / 1e12;  // DMMA TFLOP/s
  // accuracy over q in [1e-8, 1e4] (log-uniform)
  const int n = 1 << 20;
  std::vector<double> hq(n);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    hq[i] = std::pow(10.0, -8.0 + 12.0 * double(s >> 11) * 0x1.0p-53);
  }
  double *dq, *e0, *e3, *e1;
  cudaMalloc(&dq, n * sizeof(double));
  cudaMalloc(&e0, n * sizeof(double));
  cudaMalloc(&e3, n * sizeof(double));
  cudaMalloc(&e1, n * sizeof(double));
  cudaMemcpy(dq, hq.data(), n * sizeof(double), cudaMemcpyHostToDevice);
  rcp_accuracy_kernel<<<(n + 255) / 256, 256>>>(dq, n, e0, e3, e1);
  std::vector<double> h0(n), h3(n), h1(n);
  cudaMemcpy(h0.data(), e0, n * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(h3.data(), e3, n * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(h1.data(), e1, n * sizeof(double), cudaMemcpyDeviceToHost);
  double m0 = 0, m3 = 0, m1 = 0;
  for (int i = 0; i < n; ++i) {
    m0 = std::fmax(m0, h0[i]);
    m3 = std::fmax(m3, h3[i]);
    m1 = std::fmax(m1, h1[i]);
  }
  out[4] = m0;  // max rel error of the MUFU.RCP64H seed
  out[5] = m1;  // after one Newton step
  out[6] = m3;  // after the cubic correction (used by allpairs.cu)
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
  out[7] = clk / 1000.0;  // max SM clock MHz
  out[8] = sms;
  cudaFree(d);
  cudaFree(dq);
  cudaFree(e0);
  cudaFree(e3);
  cudaFree(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

#ifdef PEAKS_MAIN
int main() {
  double o[9];
  int rc = ptrom_peaks(0, o);
  std::printf(
      "{\"fp64_dfma_tflops\": %.3f, \"fp32_ffma_tflops\": %.3f, \"mufu_rcp64h_tops\": %.4f, "
      "\"dmma_fp64_tflops\": %.3f, \"rcp_seed_max_rel_err\": %.3e, \"rcp_newton1_max_rel_err\": %.3e, "
      "\"rcp_cubic_max_rel_err\": %.3e, \"sm_max_mhz\": %.0f, \"sms\": %.0f, \"rc\": %d}\n",
      o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8], rc);
  return rc;
}
#endif
