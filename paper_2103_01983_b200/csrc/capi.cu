// capi.cu — the C ABI (include/ptrom_b200.h): context lifecycle, status
// mapping and the host-buffer drop-in entry points. Validation mirrors the
// reference's ParticleSystem::validate / check_state (kernel.hpp:84-103) so
// status codes and messages match the reference's exceptions.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ops.cuh"

namespace ptrom {

void check_device_status(ptrom_ctx* ctx) {
  PTROM_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(DeviceStatus), cudaMemcpyDeviceToHost,
                             ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  const DeviceStatus st = *ctx->h_status;
  if (st.kind == kStatusOk) return;
  DeviceStatus clear{0, 0, LLONG_MAX};
  PTROM_CUDA(cudaMemcpy(ctx->d_status, &clear, sizeof(clear), cudaMemcpyHostToDevice));
  switch (st.kind) {
    case kStatusSingularBlock:  // integrators.hpp:187-189
      numerical_fail("singular Newton block for particle " + std::to_string(st.index));
    case kStatusZeroClusterCirculation:
      numerical_fail("affine circulation batch: cluster " + std::to_string(st.index) +
                     " has zero net circulation for some mu (use the per-instance ptrom_simulate)");
    case kStatusCoincidentPair: {  // kernel.hpp:185-187
      const long long pn = std::max(1LL, ctx->status_pair_n);
      numerical_fail("hamiltonian: coincident particles " + std::to_string(st.index / pn) + " and " +
                     std::to_string(st.index % pn));
    }
    case kStatusNonFiniteJacobian:  // kernel.hpp:55-56 / 64-65
      numerical_fail("kernel_pair_jacobian: coincident target/source with zero desingularization (target " +
                     std::to_string(st.index) + ")");
    default:  // kernel.hpp:38-39
      numerical_fail("kernel_pair: coincident target/source with zero desingularization (target " +
                     std::to_string(st.index) + ")");
  }
}

namespace {

template <class F>
int guarded(ptrom_ctx* ctx, F&& fn) {
  if (!ctx) return PTROM_CONFIG_ERROR;
  try {
    cudaSetDevice(ctx->device);
    fn();
    ctx->err.clear();
    return PTROM_OK;
  } catch (const status_error& e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return PTROM_CUDA_ERROR;
  }
}

// kernel.hpp:84-93 ParticleSystem::validate: the host-side part (size and
// form). The finiteness and δ checks run on the uploaded copies
// (validate_uploaded, validate.cu) in the reference's order.
void validate_shape(long long n, int form) {
  if (n <= 0) config_fail("particle system is empty");
  if (form != PTROM_FORM_STANDARD && form != PTROM_FORM_DENOMINATOR_SCALED) config_fail("unknown kernel form");
}

void check_rows(long long n, long long b, long long e) {
  if (n <= 0) config_fail("particle system is empty");
  if (b < 0 || e > n || b > e) config_fail("target range outside [0, n]");
}

template <class S>
S* stage_in(ptrom_ctx* ctx, const S* h, size_t count) {
  if (!h) return nullptr;
  S* d = ctx->io.take<S>(count);
  PTROM_CUDA(cudaMemcpyAsync(d, h, count * sizeof(S), cudaMemcpyHostToDevice, ctx->stream));
  return d;
}

}  // namespace
}  // namespace ptrom

using namespace ptrom;

extern "C" {

const char* ptrom_build_info(void) {
  return "libptrom_b200 sm_100a: allpairs f64/f32 (MUFU.RCP64H+cubic), fom, tree, ptrom-online";
}

int ptrom_create(int device, void* stream, ptrom_ctx** out) {
  if (!out) return PTROM_CONFIG_ERROR;
  *out = nullptr;
  auto* ctx = new ptrom_ctx;
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(stream);
  const int rc = guarded(ctx, [&] {
    PTROM_CUDA(cudaSetDevice(device));
    int sms = 0;
    PTROM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0;
    PTROM_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) throw status_error(PTROM_CUDA_ERROR, "libptrom_b200 requires an sm_100a (B200) device");
    ctx->num_sms = sms;
    // Keep freed stream-ordered allocations (tree / ROM scratch) in the pool
    // instead of returning them to the OS at every synchronization.
    cudaMemPool_t pool;
    PTROM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    PTROM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    if (const char* v = std::getenv("PTROM_ALLPAIRS_VARIANT")) ctx->allpairs_variant = std::atoi(v);
    if (const char* v = std::getenv("PTROM_TREE_SEQ_MAX")) ctx->tree_seq_max = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("PTROM_TREE_BUILD")) ctx->tree_build_mode = std::string(v) == "levels" ? 1 : 0;
    if (const char* v = std::getenv("PTROM_REASSIGN_BIG")) ctx->reassign_big = std::max(32LL, std::atoll(v));
    PTROM_CUDA(cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    PTROM_CUDA(cudaMalloc(&ctx->d_status, sizeof(DeviceStatus)));
    PTROM_CUDA(cudaMallocHost(&ctx->h_status, sizeof(DeviceStatus)));
    PTROM_CUDA(cudaMallocHost(&ctx->h_counts, 128 * sizeof(int)));  // also holds the Morton build state
    DeviceStatus clear{0, 0, LLONG_MAX};
    PTROM_CUDA(cudaMemcpy(ctx->d_status, &clear, sizeof(clear), cudaMemcpyHostToDevice));
  });
  if (rc != PTROM_OK) {
    ptrom_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return PTROM_OK;
}

void ptrom_destroy(ptrom_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_counts) cudaFreeHost(ctx->h_counts);
  if (ctx->tile_ctr) cudaFree(ctx->tile_ctr);
  if (ctx->scratch.base) cudaFree(ctx->scratch.base);
  if (ctx->io.base) cudaFree(ctx->io.base);
  for (auto& pr : ctx->prof_events) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  delete ctx;
}

const char* ptrom_last_error(const ptrom_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ptrom_set_stream(ptrom_ctx* ctx, void* stream) {
  return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

int ptrom_set_tuning(ptrom_ctx* ctx, const char* key, int64_t value) {
  return guarded(ctx, [&] {
    const std::string k = key ? key : "";
    if (k == "reassign_big_members") ctx->reassign_big = std::max<long long>(32, value);
    else if (k == "tree_seq_max") ctx->tree_seq_max = (int)std::max<int64_t>(1, value);
    else if (k == "tree_build_mode") ctx->tree_build_mode = value ? 1 : 0;
    else if (k == "allpairs_variant") ctx->allpairs_variant = (int)value;
    else if (k == "hyperpair_variant") ctx->hp_variant = (int)value;
    else throw status_error(PTROM_CONFIG_ERROR, "ptrom_set_tuning: unknown key '" + k + "'");
  });
}

int ptrom_synchronize(ptrom_ctx* ctx) {
  return guarded(ctx, [&] { check_device_status(ctx); });
}

int ptrom_profile_begin(ptrom_ctx* ctx) {
  return guarded(ctx, [&] {
    ctx->prof_on = true;
    ctx->prof_used = 0;
  });
}

int ptrom_profile_end(ptrom_ctx* ctx, double* total_ms, int64_t* launches) {
  return guarded(ctx, [&] {
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
    double total = 0.0;
    for (size_t k = 0; k < ctx->prof_used; ++k) {
      float ms = 0.f;
      PTROM_CUDA(cudaEventElapsedTime(&ms, ctx->prof_events[k].first, ctx->prof_events[k].second));
      total += ms;
    }
    if (total_ms) *total_ms = total;
    if (launches) *launches = (int64_t)ctx->prof_used;
    ctx->prof_on = false;
    ctx->prof_used = 0;
  });
}

// ------------------------------------------------------------ host API ---
int ptrom_pairwise_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double delta,
                                int form, const double* inflow, double* f, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_shape(n, form);
    ctx->io.reset();
    ctx->io.reserve(sizeof(double) * (size_t)(2 * n + n + (inflow ? 2 * n : 0) + 2 * n) + 4096);
    double* dx = stage_in(ctx, x, 2 * n);
    double* dg = stage_in(ctx, gamma, n);
    double* di = stage_in(ctx, inflow, inflow ? 2 * n : 0);
    validate_uploaded<double>(ctx, n, dx, dg, delta, di, "pairwise_velocity");
    double* df = ctx->io.take<double>(2 * n);
    dev_velocity_f64(ctx, n, dx, dg, delta, form, di, 0, n, df, n);
    PTROM_CUDA(cudaMemcpyAsync(f, df, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    if (n_pair_evals) *n_pair_evals = (uint64_t)n * (uint64_t)(n - 1);
  });
}

int ptrom_pairwise_velocity_f32(ptrom_ctx* ctx, int64_t n, const float* x, const float* gamma, float delta, int form,
                                const float* inflow, float* f, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_shape(n, form);
    ctx->io.reset();
    ctx->io.reserve(sizeof(float) * (size_t)(2 * n + n + (inflow ? 2 * n : 0) + 2 * n) + 4096);
    float* dx = stage_in(ctx, x, 2 * n);
    float* dg = stage_in(ctx, gamma, n);
    float* di = stage_in(ctx, inflow, inflow ? 2 * n : 0);
    validate_uploaded<float>(ctx, n, dx, dg, delta, di, "pairwise_velocity");
    float* df = ctx->io.take<float>(2 * n);
    dev_velocity_f32(ctx, n, dx, dg, delta, form, di, 0, n, df, n);
    PTROM_CUDA(cudaMemcpyAsync(f, df, sizeof(float) * 2 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    if (n_pair_evals) *n_pair_evals = (uint64_t)n * (uint64_t)(n - 1);
  });
}

int ptrom_inexact_kernel_jacobian_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double delta,
                                      int form, double* jxx, double* jxy, double* jyx, double* jyy,
                                      uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_shape(n, form);
    ctx->io.reset();
    ctx->io.reserve(sizeof(double) * (size_t)(3 * n + 4 * n) + 4096);
    double* dx = stage_in(ctx, x, 2 * n);
    double* dg = stage_in(ctx, gamma, n);
    validate_uploaded<double>(ctx, n, dx, dg, delta, (const double*)nullptr, "inexact_kernel_jacobian");
    double* dj = ctx->io.take<double>(4 * n);
    dev_jacobian_f64(ctx, n, dx, dg, delta, form, 0, n, dj, dj + n, dj + 2 * n, dj + 3 * n, 0.0, nullptr);
    double* outs[4] = {jxx, jxy, jyx, jyy};
    for (int k = 0; k < 4; ++k)
      PTROM_CUDA(cudaMemcpyAsync(outs[k], dj + k * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    // kernel_pair_jacobian does not bump the reference counter (kernel.hpp:45-73)
    if (n_pair_evals) *n_pair_evals = 0;
  });
}

int ptrom_fom_simulate_f64(ptrom_ctx* ctx, int64_t n, const double* x0, const double* gamma, double delta, int form,
                           const double* inflow, double dt, int64_t n_steps, double tol, int max_iters,
                           int jacobian_refresh_period, double* snapshots, int* iterations, uint8_t* converged,
                           double* relative_residual, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    // integrators.hpp:20-23 TimeGrid::validate, 60-65 NewtonConfig::validate
    if (!(dt > 0)) config_fail("time step must be positive");
    if (n_steps < 0) config_fail("negative step count");
    if (!(tol > 0)) config_fail("Newton tolerance must be positive");
    if (max_iters < 1) config_fail("Newton max_iters must be >= 1");
    if (jacobian_refresh_period < 1) config_fail("Jacobian refresh period must be >= 1");
    validate_shape(n, form);
    ctx->io.reset();
    ctx->io.reserve(sizeof(double) * (size_t)(2 * n + n + (inflow ? 2 * n : 0)) + 4096);
    double* dx = stage_in(ctx, x0, 2 * n);
    double* dg = stage_in(ctx, gamma, n);
    double* di = stage_in(ctx, inflow, inflow ? 2 * n : 0);
    validate_uploaded<double>(ctx, n, dx, dg, delta, di, "pairwise_velocity");
    FomResult r = fom_simulate_device(ctx, n, dx, dg, delta, form, di, dt, n_steps, tol, max_iters,
                                      jacobian_refresh_period, snapshots, iterations, converged, relative_residual);
    if (n_pair_evals) *n_pair_evals = (uint64_t)r.velocity_evals * (uint64_t)n * (uint64_t)(n - 1);
  });
}

// integrators.hpp:243-272 on device-resident inputs (x0, gamma, inflow and
// the snapshot matrix in HBM); step statistics are written to host arrays.
int ptrom_dev_fom_simulate_f64(ptrom_ctx* ctx, int64_t n, const double* d_x0, const double* d_gamma, double delta,
                               int form, const double* d_inflow, double dt, int64_t n_steps, double tol, int max_iters,
                               int jacobian_refresh_period, double* d_snapshots, int* iterations, uint8_t* converged,
                               double* relative_residual, uint64_t* n_velocity_evals, uint64_t* n_jacobian_evals) {
  return guarded(ctx, [&] {
    if (!(dt > 0)) config_fail("time step must be positive");
    if (n_steps < 0) config_fail("negative step count");
    if (!(tol > 0)) config_fail("Newton tolerance must be positive");
    if (max_iters < 1) config_fail("Newton max_iters must be >= 1");
    if (jacobian_refresh_period < 1) config_fail("Jacobian refresh period must be >= 1");
    validate_shape(n, form);
    validate_uploaded<double>(ctx, n, d_x0, d_gamma, delta, d_inflow, "pairwise_velocity");
    FomResult r = fom_simulate_device(ctx, n, d_x0, d_gamma, delta, form, d_inflow, dt, n_steps, tol, max_iters,
                                      jacobian_refresh_period, d_snapshots, iterations, converged, relative_residual);
    if (n_velocity_evals) *n_velocity_evals = (uint64_t)r.velocity_evals;
    if (n_jacobian_evals) *n_jacobian_evals = (uint64_t)r.jacobian_evals;
  });
}

// kernel.hpp:174-191
int ptrom_hamiltonian_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double* out) {
  return guarded(ctx, [&] {
    validate_shape(n, PTROM_FORM_STANDARD);
    ctx->io.reset();
    ctx->io.reserve(sizeof(double) * (size_t)(3 * n + 1) + 4096);
    double* dx = stage_in(ctx, x, 2 * n);
    double* dg = stage_in(ctx, gamma, n);
    validate_uploaded<double>(ctx, n, dx, dg, 0.0, (const double*)nullptr, "hamiltonian");
    double* dh = ctx->io.take<double>(1);
    dev_hamiltonian_f64(ctx, n, dx, dg, dh);
    PTROM_CUDA(cudaMemcpyAsync(out, dh, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
  });
}

namespace {
// kernel.hpp:200-203 LatticeSpec::validate + kernel.hpp:219-222
double lattice_scale(int64_t nx, int64_t ny, double x_min, double x_max, double y_min, double y_max, double c_g,
                     double l, double gamma_bar) {
  if (nx < 2 || ny < 2) config_fail("lattice needs at least 2 points per axis");
  if (!(x_max > x_min) || !(y_max > y_min)) config_fail("degenerate lattice extents");
  if (!(gamma_bar > 0)) config_fail("velocity_field_grid: gamma_bar must be positive");
  if (!(c_g > 0) || !(l > 0)) config_fail("velocity_field_grid: characteristic length must be positive");
  return c_g * l / gamma_bar;
}
}  // namespace

// kernel.hpp:213-238; grid is ny x nx column-major (entry (j, i) at j + i*ny).
int ptrom_velocity_field_grid_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double delta,
                                  int form, double x_min, double x_max, int64_t nx, double y_min, double y_max,
                                  int64_t ny, double c_g, double l, double gamma_bar, double* grid,
                                  uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_shape(n, form);
    ctx->io.reset();
    const size_t cells = nx >= 2 && ny >= 2 ? (size_t)(nx * ny) : 0;  // lattice_scale validates below
    ctx->io.reserve(sizeof(double) * ((size_t)(3 * n) + cells) + 4096);
    double* dx = stage_in(ctx, x, 2 * n);
    double* dg = stage_in(ctx, gamma, n);
    validate_uploaded<double>(ctx, n, dx, dg, delta, (const double*)nullptr, "velocity_field_grid");
    const double scale = lattice_scale(nx, ny, x_min, x_max, y_min, y_max, c_g, l, gamma_bar);
    double* dgrid = ctx->io.take<double>((size_t)(nx * ny));
    dev_velocity_field_grid_f64(ctx, n, dx, dg, delta, form, x_min, x_max, nx, y_min, y_max, ny, scale, dgrid);
    PTROM_CUDA(cudaMemcpyAsync(grid, dgrid, sizeof(double) * nx * ny, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    if (n_pair_evals) *n_pair_evals = (uint64_t)(nx * ny) * (uint64_t)n;
  });
}

// ---------------------------------------------------------- device API ---
int ptrom_dev_hamiltonian_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma, double* d_out) {
  return guarded(ctx, [&] {
    if (n <= 0) config_fail("particle system is empty");
    dev_hamiltonian_f64(ctx, n, d_x, d_gamma, d_out);
  });
}

int ptrom_dev_velocity_field_grid_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                      double delta, int form, double x_min, double x_max, int64_t nx, double y_min,
                                      double y_max, int64_t ny, double c_g, double l, double gamma_bar,
                                      double* d_grid) {
  return guarded(ctx, [&] {
    if (n <= 0) config_fail("particle system is empty");
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    const double scale = lattice_scale(nx, ny, x_min, x_max, y_min, y_max, c_g, l, gamma_bar);
    dev_velocity_field_grid_f64(ctx, n, d_x, d_gamma, delta, form, x_min, x_max, nx, y_min, y_max, ny, scale,
                                d_grid);
  });
}

int ptrom_dev_pairwise_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma, double delta,
                                    int form, const double* d_inflow, int64_t t_begin, int64_t t_end, double* d_f,
                                    int64_t ld_f) {
  return guarded(ctx, [&] {
    check_rows(n, t_begin, t_end);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    if (ld_f < t_end - t_begin) config_fail("ld_f smaller than the row count");
    dev_velocity_f64(ctx, n, d_x, d_gamma, delta, form, d_inflow, t_begin, t_end, d_f, ld_f);
  });
}

int ptrom_dev_pairwise_velocity_f32(ptrom_ctx* ctx, int64_t n, const float* d_x, const float* d_gamma, float delta,
                                    int form, const float* d_inflow, int64_t t_begin, int64_t t_end, float* d_f,
                                    int64_t ld_f) {
  return guarded(ctx, [&] {
    check_rows(n, t_begin, t_end);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    if (ld_f < t_end - t_begin) config_fail("ld_f smaller than the row count");
    dev_velocity_f32(ctx, n, d_x, d_gamma, delta, form, d_inflow, t_begin, t_end, d_f, ld_f);
  });
}

int ptrom_dev_pairwise_velocity_peers_f64(ptrom_ctx* ctx, int64_t n, int32_t n_peers,
                                          const double* const* d_peer_blocks, const int64_t* peer_offsets,
                                          const double* d_gamma, double delta, int form, const double* d_inflow,
                                          int64_t t_begin, int64_t t_end, const double* d_local, double* d_f,
                                          int64_t ld_f) {
  return guarded(ctx, [&] {
    check_rows(n, t_begin, t_end);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    if (n_peers < 1 || n_peers > 8) config_fail("peer count outside [1, 8]");
    if (!d_peer_blocks || !peer_offsets) config_fail("null peer table");
    if (peer_offsets[0] != 0 || peer_offsets[n_peers] != n) config_fail("peer offsets must span [0, n]");
    for (int r = 0; r < n_peers; ++r) {
      if (peer_offsets[r + 1] < peer_offsets[r]) config_fail("peer offsets must be non-decreasing");
      if (!d_peer_blocks[r] && peer_offsets[r + 1] > peer_offsets[r]) config_fail("null peer block");
    }
    if (ld_f < t_end - t_begin) config_fail("ld_f smaller than the row count");
    const long long m = t_end - t_begin;
    std::vector<long long> off(peer_offsets, peer_offsets + n_peers + 1);
    dev_velocity_peers_f64(ctx, n, n_peers, d_peer_blocks, off.data(), d_gamma, delta, form, d_inflow, t_begin,
                           t_end, d_local, d_local + m, d_f, ld_f);
  });
}

// ---- CUDA IPC for the peer-memory exchange (one process per GPU) ----
int ptrom_ipc_alloc(ptrom_ctx* ctx, uint64_t bytes, void** d_ptr) {
  return guarded(ctx, [&] {
    if (!d_ptr) config_fail("null output pointer");
    PTROM_CUDA(cudaMalloc(d_ptr, std::max<uint64_t>(bytes, 8)));
  });
}
int ptrom_ipc_free(ptrom_ctx* ctx, void* d_ptr) {
  return guarded(ctx, [&] { PTROM_CUDA(cudaFree(d_ptr)); });
}
int ptrom_ipc_get_handle(ptrom_ctx* ctx, void* d_ptr, uint8_t* handle64) {
  return guarded(ctx, [&] {
    cudaIpcMemHandle_t h;
    PTROM_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
  });
}
int ptrom_ipc_open_handle(ptrom_ctx* ctx, const uint8_t* handle64, void** d_ptr) {
  return guarded(ctx, [&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    PTROM_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}
int ptrom_ipc_close_handle(ptrom_ctx* ctx, void* d_ptr) {
  return guarded(ctx, [&] { PTROM_CUDA(cudaIpcCloseMemHandle(d_ptr)); });
}
int ptrom_dev_memcpy(ptrom_ctx* ctx, void* d_dst, const void* d_src, uint64_t bytes) {
  return guarded(ctx, [&] { PTROM_CUDA(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDefault, ctx->stream)); });
}

int ptrom_dev_inexact_kernel_jacobian_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                          double delta, int form, int64_t t_begin, int64_t t_end, double* d_jxx,
                                          double* d_jxy, double* d_jyx, double* d_jyy) {
  return guarded(ctx, [&] {
    check_rows(n, t_begin, t_end);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    dev_jacobian_f64(ctx, n, d_x, d_gamma, delta, form, t_begin, t_end, d_jxx, d_jxy, d_jyx, d_jyy, 0.0, nullptr);
  });
}

int ptrom_dev_newton_blocks_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma, double delta,
                                int form, double dt, int64_t t_begin, int64_t t_end, double* d_inv) {
  return guarded(ctx, [&] {
    check_rows(n, t_begin, t_end);
    if (!(dt > 0)) config_fail("time step must be positive");
    dev_jacobian_f64(ctx, n, d_x, d_gamma, delta, form, t_begin, t_end, nullptr, nullptr, nullptr, nullptr, dt, d_inv);
  });
}

int ptrom_dev_residual_f64(ptrom_ctx* ctx, int64_t m, int64_t ld, const double* d_xi, const double* d_fxi,
                           const double* d_xprev, const double* d_fprev, double dt, double* d_r, double* d_norm2) {
  return guarded(ctx, [&] {
    if (m < 0 || ld < m) config_fail("bad residual shape");
    ctx->scratch.reset();
    ctx->scratch.reserve(residual_block_part_count() * sizeof(double) + 4096);
    double* bp = ctx->scratch.take<double>(residual_block_part_count());
    dev_residual_f64(ctx, m, ld, d_xi, d_fxi, d_xprev, d_fprev, dt, d_r, d_norm2, bp);
  });
}

int ptrom_dev_newton_update_f64(ptrom_ctx* ctx, int64_t m, int64_t ld, const double* d_inv, const double* d_r,
                                double* d_x) {
  return guarded(ctx, [&] {
    if (m < 0 || ld < m) config_fail("bad update shape");
    dev_newton_update_f64(ctx, m, ld, d_inv, d_r, d_x);
  });
}

}  // extern "C"
