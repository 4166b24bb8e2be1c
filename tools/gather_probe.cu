// tools/gather_probe.cu — measurement only (not part of the product): nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_probe.cu
// L1 gather microbenchmark: a warp reads 512 B per "cluster" (32 lanes x 16 B)
// from clusters picked by a per-warp index list: (a) one LDG.128 per lane
// ([c][32] double2), (b) four LDG.32 per lane (planes [c][4][32] u32).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k128(const double2* __restrict__ pos, const int* __restrict__ list, int nl, double* out) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double ax = 0, ay = 0;
  const int* l = list + (w & 1023) * nl;
  for (int i = 0; i < nl; i += 4) {
    double2 p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = __ldg(pos + (unsigned)l[i + u] * 32u + lane);
#pragma unroll
    for (int u = 0; u < 4; ++u) { ax += p[u].x; ay += p[u].y; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ax + ay;
}
__global__ void k32(const unsigned* __restrict__ pl, const int* __restrict__ list, int nl, double* out) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double ax = 0, ay = 0;
  const int* l = list + (w & 1023) * nl;
  for (int i = 0; i < nl; i += 4) {
    double2 p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned* b = pl + (unsigned)l[i + u] * 128u + lane;
      const unsigned a0 = __ldg(b), a1 = __ldg(b + 32), a2 = __ldg(b + 64), a3 = __ldg(b + 96);
      p[u] = make_double2(__hiloint2double((int)a1, (int)a0), __hiloint2double((int)a3, (int)a2));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { ax += p[u].x; ay += p[u].y; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ax + ay;
}
int main() {
  for (int nc : {256, 4096, 65536, 1 << 20}) {
    const int nl = 256;
    double2* pos; unsigned* pl; int* list; double* out;
    cudaMalloc(&pos, (size_t)nc * 32 * 16); cudaMalloc(&pl, (size_t)nc * 128 * 4);
    cudaMemset(pos, 0, (size_t)nc * 512); cudaMemset(pl, 0, (size_t)nc * 512);
    int* h = new int[1024 * nl];
    unsigned s = 1;
    for (int i = 0; i < 1024 * nl; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % nc; }
    cudaMalloc(&list, 1024 * nl * 4); cudaMemcpy(list, h, 1024 * nl * 4, cudaMemcpyHostToDevice);
    const int blocks = 148 * 36 / 4, threads = 128;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float t128 = 0, t32 = 0, ms;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a); k128<<<blocks, threads>>>(pos, list, nl, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); t128 = ms;
      cudaEventRecord(a); k32<<<blocks, threads>>>(pl, list, nl, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); t32 = ms;
    }
    const double gathers = (double)blocks * threads / 32 * nl;
    printf("clusters %7d (%6.1f MB): LDG.128 %.3f ms (%.1f GB/s), 4xLDG.32 %.3f ms (%.1f GB/s)\n", nc, nc * 512.0 / 1e6,
           t128, gathers * 512 / t128 / 1e6, t32, gathers * 512 / t32 / 1e6);
    cudaFree(pos); cudaFree(pl); cudaFree(list); cudaFree(out); delete[] h;
  }
}
