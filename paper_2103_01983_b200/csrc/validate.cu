// validate.cu — the reference's input checks (ParticleSystem::validate and
// check_state, kernel.hpp:84-103) run on the device copies of the host API's
// inputs. The finiteness scans read the uploaded arrays at HBM speed instead
// of walking them on one host core (≈ 2 ms per 3M doubles). The errors are
// raised before any compute and in the reference's order.
#include <cmath>

#include "ops.cuh"

namespace ptrom {

namespace {

template <class S>
__global__ void nonfinite_kernel(const S* __restrict__ g, long long ng, const S* __restrict__ inf, long long ninf,
                                 const S* __restrict__ x, long long nx, unsigned* __restrict__ flag) {
  const long long len = ng > nx ? (ng > ninf ? ng : ninf) : (nx > ninf ? nx : ninf);
  unsigned m = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    if (i < ng && !isfinite(g[i])) m |= 1u;
    if (i < ninf && !isfinite(inf[i])) m |= 2u;
    if (i < nx && !isfinite(x[i])) m |= 4u;
  }
  m = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(flag, m);
}

}  // namespace

template <class S>
void validate_uploaded(ptrom_ctx* ctx, long long n, const S* dx, const S* dg, S delta, const S* di,
                       const char* who) {
  cudaStream_t st = ctx->stream;
  unsigned* flag;
  PTROM_CUDA(cudaMallocAsync(&flag, sizeof(unsigned), st));
  PTROM_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), st));
  const long long len = 2 * n;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(4LL * ctx->num_sms, (len + 255) / 256));
  nonfinite_kernel<S><<<blocks, 256, 0, st>>>(dg, dg ? n : 0, di, di ? 2 * n : 0, dx, dx ? 2 * n : 0, flag);
  PTROM_LAUNCH_CHECK();
  PTROM_CUDA(cudaMemcpyAsync(ctx->h_counts, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  PTROM_CUDA(cudaFreeAsync(flag, st));
  PTROM_CUDA(cudaStreamSynchronize(st));
  const unsigned m = (unsigned)ctx->h_counts[0];
  // kernel.hpp:84-93 order: circulation, δ, inflow; then check_state
  if (m & 1u) config_fail("non-finite circulation");
  if (!(delta >= S(0))) config_fail("negative desingularization constant");
  if (m & 2u) config_fail("non-finite inflow");
  if (m & 4u) config_fail(std::string(who) + ": non-finite state");
}

template void validate_uploaded<double>(ptrom_ctx*, long long, const double*, const double*, double, const double*,
                                        const char*);
template void validate_uploaded<float>(ptrom_ctx*, long long, const float*, const float*, float, const float*,
                                       const char*);

}  // namespace ptrom
