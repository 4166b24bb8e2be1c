// Do FP64 DMMA (mma.sync m8n8k4) and DFMA share execution hardware on B200?
// Runs DFMA-only, DMMA-only and mixed (independent chains in the same warp)
// and reports achieved FP64 TFLOP/s for each.
#include <cuda_runtime.h>
#include <cstdio>
template <int NF, int NM>
__global__ void k(double* out, int iters) {
  double x[NF > 0 ? NF : 1];
  double c[NM > 0 ? NM : 1][2];
  for (int i = 0; i < NF; ++i) x[i] = threadIdx.x + i;
  for (int i = 0; i < NM; ++i) c[i][0] = c[i][1] = 0;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NF; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < NF; ++i) s += x[i];
  for (int i = 0; i < NM; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int NF, int NM>
void run(double* d, int sms) {
  const int blocks = sms * 4, tpb = 256, iters = 2048;
  k<NF, NM><<<blocks, tpb>>>(d, iters);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<NF, NM><<<blocks, tpb>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double thr = double(blocks) * tpb;
  const double f_dfma = thr * iters * NF * 2;
  const double f_dmma = thr / 32 * iters * NM * 512;
  printf("{\"dfma_per_iter\": %d, \"dmma_per_iter\": %d, \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
         NF, NM, ms, f_dfma / ms / 1e9, f_dmma / ms / 1e9, (f_dfma + f_dmma) / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 64);
  run<8, 0>(d, sms); run<0, 4>(d, sms); run<8, 1>(d, sms); run<8, 2>(d, sms); run<16, 1>(d, sms); run<4, 4>(d, sms);
  return 0;
}
