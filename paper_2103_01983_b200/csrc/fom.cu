// fom.cu — device-resident implicit-trapezoidal FOM (inexact Newton).
//
// Replaces FomStepper::step / refactor (integrators.hpp:117-201) and
// fom_simulate (integrators.hpp:243-272) for the PairwiseModel
// (integrators.hpp:69-79). State, velocity, residual and the per-particle
// 2x2 inverse blocks stay in HBM for the whole trajectory.
//
// Control flow on the device: one FOM step is a CUDA graph whose Newton loop
// is a conditional WHILE node; the residual kernel's last block evaluates the
// reference's convergence test (integrators.hpp:140-155: ‖r‖/‖r0‖ ≤ tol,
// update cap, r0 == 0) and sets the loop condition, and a nested IF node runs
// the Jacobian/Newton-block refresh on the steps it is due. The host enqueues
// the step graph n_steps times with no synchronization in between; iteration
// counts, flags, ‖r‖/‖r0‖ and snapshots are recorded on the device and copied
// out once. (PTROM_FOM_GRAPH=0 selects the host-driven loop, one 8-byte
// norm read per iteration.)
//
// Elementwise arithmetic follows the reference rounding order with explicit
// _rn intrinsics (no FMA contraction), so given identical velocities the
// residual and update are bit-identical to the oracle. ‖r‖ is a fixed-order
// two-level reduction (per-thread strided sums, warp/block trees in a fixed
// shape, then the block partials in index order): deterministic run to run.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ops.cuh"

namespace ptrom {

namespace {

constexpr int kNormThreads = 256;
constexpr int kNormBlocks = 296;  // 2 x 148 SMs: the most blocks a residual reduction uses
// Residual blocks for m rows of each half: one block per 1,024 of the 2m rows,
// capped at kNormBlocks. A function of m alone, so every entry point (graph,
// host loop, sharded ranks of the same m) reduces in the same fixed shape.
inline int norm_blocks(long long m) {
  return (int)std::max(1LL, std::min<long long>(kNormBlocks, (2 * m + 1023) / 1024));
}

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

// Fixed-order sum of the block partials by one warp: lane l adds blocks
// l, l+32, ... in order, then a fixed shuffle tree (deterministic).
__device__ __forceinline__ double warp_sum_blocks(int nb, const double* __restrict__ block_part) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s = __dadd_rn(s, block_part[b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  return __shfl_sync(0xffffffffu, s, 0);
}

__global__ void sum_blocks_kernel(int nb, const double* __restrict__ block_part, double* __restrict__ out) {
  const double s = warp_sum_blocks(nb, block_part);
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = s;
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

// Per-trajectory control block of the device-driven Newton loop.
struct FomCtl {
  long long step;
  long long evals;  // velocity evaluations (the reference's counter / N(N-1))
  long long jac_evals;  // Newton-block refreshes (inexact_kernel_jacobian evaluations)
  double r0, rel;
  int updates, converged, have_blocks, refreshed, do_refresh;
  unsigned ticket;  // residual blocks done (the last one decides)
};

// integrators.hpp:140-155 on the device: ‖r‖ from the fixed-order block
// partials, the reference's decisions, and the loop / refresh conditions.
__device__ void fom_decide(FomCtl* c, double s, double tol, int max_iters, int refresh,
                           cudaGraphConditionalHandle h_loop) {
  const double nr = sqrt(s);
  const int upd = c->updates;
  bool cont = false, do_ref = false;
  if (upd == 0) {
    c->r0 = nr;
    if (nr == 0.0) {
      c->converged = 1;
      c->rel = 0.0;
      c->do_refresh = 0;
      cudaGraphSetConditional(h_loop, 0);
      return;
    }
  }
  const double rel = nr / c->r0;
  c->rel = rel;
  if (rel <= tol) {
    c->converged = 1;
  } else if (upd < max_iters) {
    cont = true;
    const bool due = (c->step % refresh) == 0 || !c->have_blocks;
    do_ref = due && !c->refreshed;
    if (do_ref) c->refreshed = c->have_blocks = 1;
    c->updates = upd + 1;
    c->evals += 1;
  }
  c->do_refresh = do_ref ? 1 : 0;
  cudaGraphSetConditional(h_loop, cont ? 1u : 0u);
}

// residual_kernel + fom_decide in one launch: the last block to finish sums
// the block partials (same fixed order) and decides.
__global__ void __launch_bounds__(kNormThreads) residual_decide_kernel(
    long long m, long long ld, const double* __restrict__ xi, const double* __restrict__ fxi,
    const double* __restrict__ xp, const double* __restrict__ fp, double h, double* __restrict__ r,
    double* __restrict__ block_part, FomCtl* c, double tol, int max_iters, int refresh,
    cudaGraphConditionalHandle h_loop) {
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
  __shared__ bool s_last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sb = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) sb = __dadd_rn(sb, warp_sum[w]);
    block_part[blockIdx.x] = sb;
    __threadfence();
    s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  double sum = 0.0;
  for (int b = lane; b < (int)gridDim.x; b += 32) sum = __dadd_rn(sum, __ldcg(block_part + b));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum = __dadd_rn(sum, __shfl_down_sync(0xffffffffu, sum, o));
  if (lane == 0) {
    c->ticket = 0;
    fom_decide(c, sum, tol, max_iters, refresh, h_loop);
  }
}

// First node of the loop body: arms the IF node of the Newton-block refresh.
__global__ void fom_refresh_gate_kernel(FomCtl* c, cudaGraphConditionalHandle h_refresh) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cudaGraphSetConditional(h_refresh, c->do_refresh ? 1u : 0u);
    if (c->do_refresh) c->jac_evals += 1;
  }
}

// StepResult + snapshot column of the accepted state (integrators.hpp:262-268).
// The accepted state also becomes the history (integrators.hpp:262-264):
// x_prev ← ξ, f_prev ← f_ξ; ξ and f_ξ already hold the next step's initial
// guess (integrators.hpp:130-131), so no copies run at the start of a step.
__global__ void fom_record_kernel(const FomCtl* c, long long dim, const double* __restrict__ x,
                                  const double* __restrict__ fx, double* __restrict__ x_prev,
                                  double* __restrict__ f_prev, double* __restrict__ snaps, int* __restrict__ iters,
                                  unsigned char* __restrict__ conv, double* __restrict__ rel) {
  const long long s = c->step;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < dim; k += (long long)gridDim.x * blockDim.x) {
    const double v = x[k];
    snaps[s * dim + k] = v;
    x_prev[k] = v;
    f_prev[k] = fx[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    iters[s] = c->updates;
    conv[s] = (unsigned char)c->converged;
    rel[s] = c->rel;
  }
}

__global__ void fom_advance_kernel(FomCtl* c) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  c->step += 1;
  c->updates = 0;
  c->converged = 0;
  c->refreshed = 0;
  c->rel = 0.0;
}

// Small systems (2m ≤ kOneBlockRows rows, e.g. config 1's 8,192): the
// residual, its fixed-order norm and (DECIDE) the Newton decision in one
// block of 1,024 threads — no block partials, fence or arrival ticket on the
// per-iteration critical path. Every entry point uses this shape for such m.
constexpr int kOneBlockThreads = 1024;
constexpr int kOneBlockPer = 8;  // rows per thread, all loads issued before the sums
constexpr long long kOneBlockRows = (long long)kOneBlockThreads * kOneBlockPer;
template <bool DECIDE>
__global__ void __launch_bounds__(kOneBlockThreads) residual_one_block_kernel(
    long long m, long long ld, const double* __restrict__ xi, const double* __restrict__ fxi,
    const double* __restrict__ xp, const double* __restrict__ fp, double h, double* __restrict__ r,
    double* __restrict__ norm2, FomCtl* c, double tol, int max_iters, int refresh, cudaGraphConditionalHandle h_loop) {
  const long long rows = 2 * m;
  double v[kOneBlockPer];
#pragma unroll
  for (int i = 0; i < kOneBlockPer; ++i) {
    const long long e = threadIdx.x + (long long)i * kOneBlockThreads;
    v[i] = 0.0;
    if (e < rows) {
      const long long k = e < m ? e : (e - m) + ld;
      v[i] = __dsub_rn(__dsub_rn(xi[k], xp[k]), __dmul_rn(h, __dadd_rn(fxi[k], fp[k])));
      r[k] = v[i];
    }
  }
  double acc = 0.0;  // the same per-thread order as the strided loop
#pragma unroll
  for (int i = 0; i < kOneBlockPer; ++i) acc = __dadd_rn(acc, __dmul_rn(v[i], v[i]));
  __shared__ double warp_sum[kOneBlockThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < kOneBlockThreads / 32; ++w) sum = __dadd_rn(sum, warp_sum[w]);
    if (DECIDE) fom_decide(c, sum, tol, max_iters, refresh, h_loop);
    else *norm2 = sum;
  }
}

int grid_for(ptrom_ctx* ctx, long long count, int tpb) {
  long long g = (count + tpb - 1) / tpb;
  return (int)std::max(1LL, std::min(g, (long long)ctx->num_sms * 8));
}

}  // namespace

void dev_residual_f64(ptrom_ctx* ctx, long long m, long long ld, const double* xi, const double* fxi,
                      const double* xp, const double* fp, double dt, double* r, double* norm2, double* block_part) {
  if (2 * m <= kOneBlockRows) {
    residual_one_block_kernel<false><<<1, kOneBlockThreads, 0, ctx->stream>>>(m, ld, xi, fxi, xp, fp, dt / 2.0, r,
                                                                             norm2, nullptr, 0.0, 0, 1, 0);
    PTROM_LAUNCH_CHECK();
    return;
  }
  const int nb = norm_blocks(m);
  residual_kernel<<<nb, kNormThreads, 0, ctx->stream>>>(m, ld, xi, fxi, xp, fp, dt / 2.0, r, block_part);
  PTROM_LAUNCH_CHECK();
  sum_blocks_kernel<<<1, 32, 0, ctx->stream>>>(nb, block_part, norm2);
  PTROM_LAUNCH_CHECK();
}

void dev_newton_update_f64(ptrom_ctx* ctx, long long m, long long ld, const double* inv, const double* r,
                           double* x) {
  newton_update_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(m, ld, inv, r, x);
  PTROM_LAUNCH_CHECK();
}

size_t residual_block_part_count() { return kNormBlocks; }

// Device-driven trajectory: the step graph (see the file comment) launched
// n_steps times back to back; one synchronization at the end.
static FomResult fom_simulate_graph(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma,
                                    double delta, int form, const double* d_inflow, double dt, long long n_steps,
                                    double tol, int max_iters, int refresh, double* h_snapshots, int* iters,
                                    unsigned char* conv, double* rel_out) {
  FomResult out;
  // Capture needs a real stream (the caller's may be the legacy default one):
  // run the whole trajectory on a private stream ordered after ctx->stream.
  cudaStream_t caller = ctx->stream, st = nullptr;
  PTROM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    cudaEvent_t ev;
    PTROM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PTROM_CUDA(cudaEventRecord(ev, caller));
    PTROM_CUDA(cudaStreamWaitEvent(st, ev, 0));
    cudaEventDestroy(ev);
  }
  struct StreamGuard {
    ptrom_ctx* c;
    cudaStream_t caller, own;
    ~StreamGuard() {
      c->stream = caller;
      cudaStreamSynchronize(own);
      cudaStreamDestroy(own);
    }
  } sguard{ctx, caller, st};
  ctx->stream = st;
  const long long dim = 2 * n;
  std::vector<void*> bufs;
  auto alloc = [&](size_t bytes) {
    void* p;
    PTROM_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    bufs.push_back(p);
    return p;
  };
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t s_body = nullptr, s_ref = nullptr;
  struct Cleanup {
    std::vector<void*>* b;
    cudaGraphExec_t* e;
    cudaGraph_t* g;
    cudaStream_t *s1, *s2;
    ~Cleanup() {
      if (*e) cudaGraphExecDestroy(*e);
      if (*g) cudaGraphDestroy(*g);
      if (*s1) cudaStreamDestroy(*s1);
      if (*s2) cudaStreamDestroy(*s2);
      for (void* p : *b) cudaFree(p);
    }
  } cleanup{&bufs, &exec, &graph, &s_body, &s_ref};
  double* x_prev = (double*)alloc(dim * 8);
  double* f_prev = (double*)alloc(dim * 8);
  double* xi = (double*)alloc(dim * 8);
  double* fxi = (double*)alloc(dim * 8);
  double* r = (double*)alloc(dim * 8);
  double* inv = (double*)alloc(4 * n * 8);
  double* block_part = (double*)alloc(kNormBlocks * 8);
  double* snaps = (double*)alloc((size_t)dim * std::max<long long>(n_steps, 1) * 8);
  int* d_iters = (int*)alloc(std::max<long long>(n_steps, 1) * 4);
  unsigned char* d_conv = (unsigned char*)alloc(std::max<long long>(n_steps, 1));
  double* d_rel = (double*)alloc(std::max<long long>(n_steps, 1) * 8);
  FomCtl* ctl = (FomCtl*)alloc(sizeof(FomCtl));
  PTROM_CUDA(cudaMemsetAsync(ctl, 0, sizeof(FomCtl), st));

  // x = x0; f = model.velocity(x0)   (integrators.hpp:257-259); the Jacobian
  // path's scratch is sized without evaluating it (capture cannot allocate)
  PTROM_CUDA(cudaMemcpyAsync(x_prev, d_x0, dim * 8, cudaMemcpyDeviceToDevice, st));
  dev_jacobian_reserve_f64(ctx, n, n);
  dev_velocity_f64(ctx, n, x_prev, d_gamma, delta, form, d_inflow, 0, n, f_prev, n);
  ++out.velocity_evals;
  PTROM_CUDA(cudaStreamSynchronize(st));

  const double h = dt / 2.0;
  PTROM_CUDA(cudaStreamCreateWithFlags(&s_body, cudaStreamNonBlocking));
  PTROM_CUDA(cudaStreamCreateWithFlags(&s_ref, cudaStreamNonBlocking));
  const bool prof = ctx->prof_on;
  ctx->prof_on = false;  // no event nodes inside conditional bodies
  cudaGraphConditionalHandle h_loop, h_ref;
  // ξ = x_prev, f_ξ = f_prev (integrators.hpp:130-131) for the first step;
  // later steps inherit them from fom_record_kernel
  PTROM_CUDA(cudaMemcpyAsync(xi, x_prev, dim * 8, cudaMemcpyDeviceToDevice, st));
  PTROM_CUDA(cudaMemcpyAsync(fxi, f_prev, dim * 8, cudaMemcpyDeviceToDevice, st));
  PTROM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  // pre: r; decide
  // the loop node's handle must exist before the kernel that sets it
  cudaStreamCaptureStatus cs;
  cudaGraph_t g_cap;
  PTROM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g_cap, nullptr, nullptr));
  PTROM_CUDA(cudaGraphConditionalHandleCreate(&h_loop, g_cap, 0, 0));
  auto residual_decide = [&](cudaStream_t on) {
    if (2 * n <= kOneBlockRows)
      residual_one_block_kernel<true><<<1, kOneBlockThreads, 0, on>>>(n, n, xi, fxi, x_prev, f_prev, h, r, nullptr,
                                                                       ctl, tol, max_iters, refresh, h_loop);
    else
      residual_decide_kernel<<<norm_blocks(n), kNormThreads, 0, on>>>(n, n, xi, fxi, x_prev, f_prev, h, r, block_part,
                                                                      ctl, tol, max_iters, refresh, h_loop);
  };
  residual_decide(st);
  {
    // WHILE (continue): [IF refresh: Newton blocks]; update; velocity; r; decide
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    PTROM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g_cap, &deps, &ndeps));
    cudaGraphNodeParams prm = {};
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = h_loop;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    cudaGraphNode_t loop_node;
    PTROM_CUDA(cudaGraphAddNode(&loop_node, g_cap, deps, ndeps, &prm));
    PTROM_CUDA(cudaStreamUpdateCaptureDependencies(st, &loop_node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = prm.conditional.phGraph_out[0];

    PTROM_CUDA(cudaStreamBeginCaptureToGraph(s_body, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    PTROM_CUDA(cudaGraphConditionalHandleCreate(&h_ref, body, 0, 0));
    fom_refresh_gate_kernel<<<1, 32, 0, s_body>>>(ctl, h_ref);
    cudaStream_t saved = ctx->stream;
    {
      const cudaGraphNode_t* bdeps = nullptr;
      size_t nbdeps = 0;
      cudaGraph_t g_body;
      PTROM_CUDA(cudaStreamGetCaptureInfo(s_body, &cs, nullptr, &g_body, &bdeps, &nbdeps));
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = h_ref;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      cudaGraphNode_t if_node;
      PTROM_CUDA(cudaGraphAddNode(&if_node, g_body, bdeps, nbdeps, &ip));
      PTROM_CUDA(cudaStreamUpdateCaptureDependencies(s_body, &if_node, 1, cudaStreamSetCaptureDependencies));
      cudaGraph_t ref_body = ip.conditional.phGraph_out[0];
      PTROM_CUDA(cudaStreamBeginCaptureToGraph(s_ref, ref_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      ctx->stream = s_ref;  // integrators.hpp:181-194 refactor at ξ
      dev_jacobian_f64(ctx, n, xi, d_gamma, delta, form, 0, n, nullptr, nullptr, nullptr, nullptr, dt, inv);
      cudaGraph_t tmp;
      PTROM_CUDA(cudaStreamEndCapture(s_ref, &tmp));
    }
    ctx->stream = s_body;
    newton_update_kernel<<<grid_for(ctx, n, 256), 256, 0, s_body>>>(n, n, inv, r, xi);
    dev_velocity_f64(ctx, n, xi, d_gamma, delta, form, d_inflow, 0, n, fxi, n);
    residual_decide(s_body);
    ctx->stream = saved;
    cudaGraph_t tmp;
    PTROM_CUDA(cudaStreamEndCapture(s_body, &tmp));
  }
  // post: record the accepted state, it becomes the history (integrators.hpp:262-264)
  fom_record_kernel<<<grid_for(ctx, dim, 256), 256, 0, st>>>(ctl, dim, xi, fxi, x_prev, f_prev, snaps, d_iters, d_conv,
                                                             d_rel);
  fom_advance_kernel<<<1, 32, 0, st>>>(ctl);
  PTROM_CUDA(cudaStreamEndCapture(st, &graph));
  ctx->prof_on = prof;
  PTROM_CUDA(cudaGraphInstantiate(&exec, graph, 0));

  for (long long s = 0; s < n_steps; ++s) PTROM_CUDA(cudaGraphLaunch(exec, st));
  FomCtl hc;
  PTROM_CUDA(cudaMemcpyAsync(&hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
  if (n_steps > 0) {
    PTROM_CUDA(cudaMemcpyAsync(iters, d_iters, n_steps * 4, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaMemcpyAsync(conv, d_conv, n_steps, cudaMemcpyDeviceToHost, st));
    PTROM_CUDA(cudaMemcpyAsync(rel_out, d_rel, n_steps * 8, cudaMemcpyDeviceToHost, st));
    if (h_snapshots)
      PTROM_CUDA(cudaMemcpyAsync(h_snapshots, snaps, (size_t)dim * n_steps * 8, cudaMemcpyDefault, st));
  }
  PTROM_CUDA(cudaStreamSynchronize(st));
  check_device_status(ctx);
  out.velocity_evals += hc.evals;
  out.jacobian_evals += hc.jac_evals;
  return out;
}

// ----------------------------------------------------------- fom_simulate --
// integrators.hpp:243-272 + FomStepper::step integrators.hpp:126-178.
// All buffers are device-resident; host copies only x0 in and snapshots out.
FomResult fom_simulate_device(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma, double delta,
                              int form, const double* d_inflow, double dt, long long n_steps, double tol,
                              int max_iters, int refresh, double* h_snapshots, int* iters, unsigned char* conv,
                              double* rel_out) {
  const char* mode = std::getenv("PTROM_FOM_GRAPH");
  if (!(mode && mode[0] == '0') && fom_persistent_applies(ctx, n))  // small systems: one persistent kernel
    return fom_simulate_persistent(ctx, n, d_x0, d_gamma, delta, form, d_inflow, dt, n_steps, tol, max_iters, refresh,
                                   h_snapshots, iters, conv, rel_out);
  if (!(mode && mode[0] == '0'))
    return fom_simulate_graph(ctx, n, d_x0, d_gamma, delta, form, d_inflow, dt, n_steps, tol, max_iters, refresh,
                              h_snapshots, iters, conv, rel_out);
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
        ++out.jacobian_evals;
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
                                 cudaMemcpyDefault, ctx->stream));
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
