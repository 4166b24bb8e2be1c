// comm.cu — multi-GPU communicator (comm.cuh) and the target-sharded FOM
// (SURVEY.md §8e row 1): ptrom_comm_*, ptrom_dev_pairwise_velocity_sharded_f64,
// ptrom_fom_simulate_sharded_f64.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed (see comm.cuh)

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "ops.cuh"

namespace ptrom {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(sym("ncclReduceScatter"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.broadcast && api.all_gather &&
             api.reduce_scatter &&
             api.group_start && api.group_end && api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw status_error(PTROM_CUDA_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

void host_check(int rc, const char* what) {
  if (rc != 0) throw status_error(PTROM_CUDA_ERROR, std::string(what) + " (host collective) failed with " +
                                                        std::to_string(rc));
}

ncclComm_t as_nccl(const ptrom_comm* c) { return static_cast<ncclComm_t>(c->nccl); }

}  // namespace

void comm_sync(ptrom_ctx* ctx, ptrom_comm*) { PTROM_CUDA(cudaStreamSynchronize(ctx->stream)); }

void comm_allgatherv(ptrom_ctx* ctx, ptrom_comm* c, void* d_buf, const std::vector<size_t>& off,
                     const std::vector<size_t>& cnt) {
  if (c->world == 1) return;
  char* b = static_cast<char*>(d_buf);
  if (c->nccl) {
    const NcclApi& api = nccl();
    nccl_check(api.group_start(), "ncclGroupStart");
    for (int r = 0; r < c->world; ++r)
      if (cnt[r]) nccl_check(api.broadcast(b + off[r], b + off[r], cnt[r], ncclUint8, r, as_nccl(c), ctx->stream),
                             "ncclBroadcast");
    nccl_check(api.group_end(), "ncclGroupEnd");
    return;
  }
  const size_t mx = *std::max_element(cnt.begin(), cnt.end());
  std::vector<char> send(std::max<size_t>(mx, 1)), recv(std::max<size_t>(mx, 1) * c->world);
  if (cnt[c->rank])
    PTROM_CUDA(cudaMemcpyAsync(send.data(), b + off[c->rank], cnt[c->rank], cudaMemcpyDeviceToHost, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  host_check(c->ops.all_gather(c->user, send.data(), recv.data(), mx), "all_gather");
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank && cnt[r])
      PTROM_CUDA(cudaMemcpyAsync(b + off[r], recv.data() + (size_t)r * mx, cnt[r], cudaMemcpyHostToDevice,
                                 ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void comm_reduce_scatter_rows(ptrom_ctx* ctx, ptrom_comm* c, const double* d_in, long long rows, long long row_len,
                              double* d_out) {
  const long long chunk = row_len / c->world;
  if (c->world == 1) {
    PTROM_CUDA(cudaMemcpyAsync(d_out, d_in, (size_t)rows * row_len * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  if (c->nccl) {  // grouped, at most 64 collectives per group
    const NcclApi& api = nccl();
    for (long long r0 = 0; r0 < rows; r0 += 64) {
      nccl_check(api.group_start(), "ncclGroupStart");
      for (long long r = r0; r < std::min(rows, r0 + 64); ++r)
        nccl_check(api.reduce_scatter(d_in + r * row_len, d_out + r * chunk, (size_t)chunk, ncclFloat64, ncclSum,
                                      as_nccl(c), ctx->stream),
                   "ncclReduceScatter");
      nccl_check(api.group_end(), "ncclGroupEnd");
    }
    return;
  }
  // host transport: gather every rank's rows, sum the own chunk in rank order
  const size_t bytes = (size_t)rows * row_len * 8;
  std::vector<double> mine((size_t)rows * row_len), all((size_t)rows * row_len * c->world);
  PTROM_CUDA(cudaMemcpyAsync(mine.data(), d_in, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  host_check(c->ops.all_gather(c->user, mine.data(), all.data(), bytes), "all_gather");
  std::vector<double> out((size_t)rows * chunk, 0.0);
  for (int q = 0; q < c->world; ++q)
    for (long long r = 0; r < rows; ++r)
      for (long long k = 0; k < chunk; ++k)
        out[r * chunk + k] += all[(size_t)q * rows * row_len + r * row_len + c->rank * chunk + k];
  PTROM_CUDA(cudaMemcpyAsync(d_out, out.data(), out.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void comm_bcast_many(ptrom_ctx* ctx, ptrom_comm* c, const std::vector<std::pair<void*, size_t>>& bufs, int root) {
  if (c->world == 1) return;
  if (c->nccl) {
    const NcclApi& api = nccl();
    nccl_check(api.group_start(), "ncclGroupStart");
    for (const auto& [p, bytes] : bufs)
      if (bytes) nccl_check(api.broadcast(p, p, bytes, ncclUint8, root, as_nccl(c), ctx->stream), "ncclBroadcast");
    nccl_check(api.group_end(), "ncclGroupEnd");
    return;
  }
  for (const auto& [p, bytes] : bufs) {
    if (!bytes) continue;
    std::vector<char> h(bytes);
    if (c->rank == root) PTROM_CUDA(cudaMemcpyAsync(h.data(), p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
    host_check(c->ops.broadcast(c->user, h.data(), bytes, root), "broadcast");
    if (c->rank != root) PTROM_CUDA(cudaMemcpyAsync(p, h.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
    PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  }
}

void comm_bcast(ptrom_ctx* ctx, ptrom_comm* c, void* d_buf, size_t bytes, int root) {
  comm_bcast_many(ctx, c, {{d_buf, bytes}}, root);
}

void comm_bcast_host(ptrom_ctx* ctx, ptrom_comm* c, void* h_buf, size_t bytes, int root) {
  if (c->world == 1 || !bytes) return;
  if (!c->nccl) {
    host_check(c->ops.broadcast(c->user, h_buf, bytes, root), "broadcast");
    return;
  }
  void* d = nullptr;
  PTROM_CUDA(cudaMallocAsync(&d, bytes, ctx->stream));
  if (c->rank == root) PTROM_CUDA(cudaMemcpyAsync(d, h_buf, bytes, cudaMemcpyHostToDevice, ctx->stream));
  comm_bcast(ctx, c, d, bytes, root);
  PTROM_CUDA(cudaMemcpyAsync(h_buf, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PTROM_CUDA(cudaFreeAsync(d, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void comm_allgather_host(ptrom_ctx* ctx, ptrom_comm* c, const void* h_send, void* h_recv, size_t bytes) {
  if (c->world == 1) {
    std::memcpy(h_recv, h_send, bytes);
    return;
  }
  if (!c->nccl) {
    host_check(c->ops.all_gather(c->user, h_send, h_recv, bytes), "all_gather");
    return;
  }
  char* d = nullptr;
  PTROM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes * (c->world + 1), ctx->stream));
  PTROM_CUDA(cudaMemcpyAsync(d, h_send, bytes, cudaMemcpyHostToDevice, ctx->stream));
  nccl_check(nccl().all_gather(d, d + bytes, bytes, ncclUint8, as_nccl(c), ctx->stream), "ncclAllGather");
  PTROM_CUDA(cudaMemcpyAsync(h_recv, d + bytes, bytes * c->world, cudaMemcpyDeviceToHost, ctx->stream));
  PTROM_CUDA(cudaFreeAsync(d, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace {

// The SoA position exchange of a target-sharded evaluation: rank r's rows
// [lo_r, hi_r) of the x half and of the y half of the 2n state.
void exchange_positions(ptrom_ctx* ctx, ptrom_comm* c, long long n, double* d_x_full) {
  std::vector<size_t> o1(c->world), c1(c->world);
  for (int r = 0; r < c->world; ++r) {
    long long lo, hi;
    shard_bounds(n, r, c->world, lo, hi);
    o1[r] = (size_t)lo * 8;
    c1[r] = (size_t)(hi - lo) * 8;
  }
  if (c->world == 1) return;
  if (c->nccl) {  // both halves in one group
    const NcclApi& api = nccl();
    nccl_check(api.group_start(), "ncclGroupStart");
    char* b = reinterpret_cast<char*>(d_x_full);
    for (int half = 0; half < 2; ++half)
      for (int r = 0; r < c->world; ++r)
        if (c1[r])
          nccl_check(api.broadcast(b + half * n * 8 + o1[r], b + half * n * 8 + o1[r], c1[r], ncclUint8, r,
                                   as_nccl(c), ctx->stream),
                     "ncclBroadcast");
    nccl_check(api.group_end(), "ncclGroupEnd");
    return;
  }
  comm_allgatherv(ctx, c, d_x_full, o1, c1);
  comm_allgatherv(ctx, c, d_x_full + n, o1, c1);
}

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

struct DevBufs {
  std::vector<void*> p;
  ptrom_ctx* ctx;
  explicit DevBufs(ptrom_ctx* c) : ctx(c) {}
  ~DevBufs() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  T* alloc(size_t count) {
    T* d = nullptr;
    PTROM_CUDA(cudaMalloc(&d, std::max<size_t>(count, 1) * sizeof(T)));
    p.push_back(d);
    return d;
  }
};

void check_comm(ptrom_ctx* ctx, const ptrom_comm* comm) {
  if (!comm) config_fail("null communicator");
  if (comm->device != ctx->device) config_fail("communicator and context are on different devices");
}

}  // namespace
}  // namespace ptrom

using namespace ptrom;

extern "C" {

int ptrom_comm_unique_id(uint8_t id_out[128]) {
  const NcclApi& api = nccl();
  if (!api.ok) return PTROM_CUDA_ERROR;
  ncclUniqueId id;
  if (api.get_unique_id(&id) != ncclSuccess) return PTROM_CUDA_ERROR;
  std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return PTROM_OK;
}

int ptrom_comm_init(ptrom_ctx* ctx, int rank, int world, const uint8_t id[128], ptrom_comm** out) {
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) config_fail("comm_init: rank outside [0, world)");
    if (!id || !out) config_fail("comm_init: null unique id or output");
    const NcclApi& api = nccl();
    if (!api.ok) throw status_error(PTROM_CUDA_ERROR, "comm_init: " + api.why);
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t nc = nullptr;
    nccl_check(api.comm_init_rank(&nc, world, uid, rank), "ncclCommInitRank");
    auto* c = new ptrom_comm;
    c->rank = rank;
    c->world = world;
    c->device = ctx->device;
    c->nccl = nc;
    *out = c;
  });
}

int ptrom_comm_init_host(ptrom_ctx* ctx, int rank, int world, const ptrom_host_collectives* ops, void* user,
                         ptrom_comm** out) {
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) config_fail("comm_init: rank outside [0, world)");
    if (!ops || !ops->all_gather || !ops->broadcast || !out) config_fail("comm_init_host: missing collectives");
    auto* c = new ptrom_comm;
    c->rank = rank;
    c->world = world;
    c->device = ctx->device;
    c->ops = *ops;
    c->user = user;
    *out = c;
  });
}

void ptrom_comm_destroy(ptrom_comm* comm) {
  if (!comm) return;
  if (comm->nccl) {
    cudaSetDevice(comm->device);
    nccl().comm_destroy(static_cast<ncclComm_t>(comm->nccl));
  }
  delete comm;
}

int ptrom_comm_transport(const ptrom_comm* comm) { return comm && comm->nccl ? 1 : 0; }

int ptrom_dev_pairwise_velocity_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* d_x_local,
                                            double* d_x_full, const double* d_gamma, double delta, int form,
                                            const double* d_inflow, double* d_f_local) {
  return guarded(ctx, [&] {
    check_comm(ctx, comm);
    if (n <= 0) config_fail("particle system is empty");
    if (form != PTROM_FORM_STANDARD && form != PTROM_FORM_DENOMINATOR_SCALED) config_fail("unknown kernel form");
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    long long lo, hi;
    shard_bounds(n, comm->rank, comm->world, lo, hi);
    const long long m = hi - lo;
    if (m > 0) {
      PTROM_CUDA(cudaMemcpyAsync(d_x_full + lo, d_x_local, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      PTROM_CUDA(cudaMemcpyAsync(d_x_full + n + lo, d_x_local + m, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    exchange_positions(ctx, comm, n, d_x_full);
    if (sym_sharded_applies(ctx, n, comm->world))  // unordered pairs + one reduce-scatter
      dev_velocity_sym_sharded_f64(ctx, comm, n, d_x_full, d_gamma, delta, form, d_inflow, d_f_local);
    else
      dev_velocity_f64(ctx, n, d_x_full, d_gamma, delta, form, d_inflow, lo, hi, d_f_local, m);
  });
}

// integrators.hpp:243-272 + FomStepper::step (integrators.hpp:126-178) over
// this rank's targets. The Newton decision needs the global |r|, so each
// iteration reads the G partials back (8·G bytes) — one host round trip per
// Newton iteration, against one all-pairs evaluation of m x n pairs (1.2 s
// per rank at config 5, G = 8).
int ptrom_fom_simulate_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* x0,
                                   const double* gamma, double delta, int form, const double* inflow, double dt,
                                   int64_t n_steps, double tol, int max_iters, int refresh,
                                   double* snapshots_local, int* iterations, uint8_t* converged,
                                   double* relative_residual, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    check_comm(ctx, comm);
    if (!(dt > 0)) config_fail("time step must be positive");
    if (n_steps < 0) config_fail("negative step count");
    if (!(tol > 0)) config_fail("Newton tolerance must be positive");
    if (max_iters < 1) config_fail("Newton max_iters must be >= 1");
    if (refresh < 1) config_fail("Jacobian refresh period must be >= 1");
    if (n <= 0) config_fail("particle system is empty");
    if (form != PTROM_FORM_STANDARD && form != PTROM_FORM_DENOMINATOR_SCALED) config_fail("unknown kernel form");
    long long lo, hi;
    shard_bounds(n, comm->rank, comm->world, lo, hi);
    const long long m = hi - lo;
    cudaStream_t st = ctx->stream;
    DevBufs mem(ctx);
    double* x_full = mem.alloc<double>(2 * n);
    double* g = mem.alloc<double>(n);
    double* inf = inflow ? mem.alloc<double>(2 * n) : nullptr;
    PTROM_CUDA(cudaMemcpyAsync(x_full, x0, 2 * n * 8, cudaMemcpyHostToDevice, st));
    PTROM_CUDA(cudaMemcpyAsync(g, gamma, n * 8, cudaMemcpyHostToDevice, st));
    if (inf) PTROM_CUDA(cudaMemcpyAsync(inf, inflow, 2 * n * 8, cudaMemcpyHostToDevice, st));
    validate_uploaded<double>(ctx, n, x_full, g, delta, inf, "pairwise_velocity");
    const size_t rows = (size_t)std::max<long long>(2 * m, 1);
    double* x_prev = mem.alloc<double>(rows);
    double* f_prev = mem.alloc<double>(rows);
    double* xi = mem.alloc<double>(rows);
    double* fxi = mem.alloc<double>(rows);
    double* r = mem.alloc<double>(rows);
    double* inv = mem.alloc<double>(2 * rows);
    double* norm2 = mem.alloc<double>(1);
    double* block_part = mem.alloc<double>(residual_block_part_count());
    PTROM_CUDA(cudaMemsetAsync(norm2, 0, 8, st));
    if (m > 0) {
      PTROM_CUDA(cudaMemcpyAsync(x_prev, x_full + lo, m * 8, cudaMemcpyDeviceToDevice, st));
      PTROM_CUDA(cudaMemcpyAsync(x_prev + m, x_full + n + lo, m * 8, cudaMemcpyDeviceToDevice, st));
    }
    long long evals = 0;
    const bool sym = sym_sharded_applies(ctx, n, comm->world);
    auto velocity = [&](double* f_out) {  // f = velocity(x_full) on the local rows (integrators.hpp:257-259)
      if (sym)
        dev_velocity_sym_sharded_f64(ctx, comm, n, x_full, g, delta, form, inf, f_out);
      else
        dev_velocity_f64(ctx, n, x_full, g, delta, form, inf, lo, hi, f_out, m);
      ++evals;
    };
    auto global_norm = [&]() -> double {  // partials all-gathered, summed in rank order
      if (m > 0) dev_residual_f64(ctx, m, m, xi, fxi, x_prev, f_prev, dt, r, norm2, block_part);
      double mine = 0.0;
      PTROM_CUDA(cudaMemcpyAsync(&mine, norm2, 8, cudaMemcpyDeviceToHost, st));
      PTROM_CUDA(cudaStreamSynchronize(st));
      check_device_status(ctx);
      std::vector<double> parts(comm->world);
      comm_allgather_host(ctx, comm, &mine, parts.data(), 8);
      double s = 0.0;
      for (double v : parts) s += v;
      return std::sqrt(s);
    };
    velocity(f_prev);
    bool have_blocks = false;
    for (long long s = 0; s < n_steps; ++s) {
      // ξ = x_prev, f_ξ = f_prev (integrators.hpp:130-131); x_full holds the gathered x_prev
      if (m > 0) {
        PTROM_CUDA(cudaMemcpyAsync(xi, x_prev, 2 * m * 8, cudaMemcpyDeviceToDevice, st));
        PTROM_CUDA(cudaMemcpyAsync(fxi, f_prev, 2 * m * 8, cudaMemcpyDeviceToDevice, st));
      }
      const bool refresh_due = (s % refresh) == 0 || !have_blocks;
      bool refreshed = false, conv = false;
      int updates = 0;
      double r0 = 0.0, rel = 0.0;
      while (true) {
        const double nr = global_norm();
        if (updates == 0) {
          r0 = nr;
          if (r0 == 0.0) {
            conv = true;
            rel = 0.0;
            break;
          }
        }
        rel = nr / r0;
        if (rel <= tol) {
          conv = true;
          break;
        }
        if (updates >= max_iters) break;
        if (refresh_due && !refreshed) {  // integrators.hpp:181-194: blocks at ξ (x_full = gathered ξ)
          if (sym)  // unordered pairs, rank share + reduce-scatter (bit-identical rows)
            dev_jacobian_sym_sharded_f64(ctx, comm, n, x_full, g, delta, form, dt, inv);
          else
            dev_jacobian_f64(ctx, n, x_full, g, delta, form, lo, hi, nullptr, nullptr, nullptr, nullptr, dt, inv);
          refreshed = have_blocks = true;
        }
        if (m > 0) dev_newton_update_f64(ctx, m, m, inv, r, xi);
        ++updates;
        if (m > 0) {
          PTROM_CUDA(cudaMemcpyAsync(x_full + lo, xi, m * 8, cudaMemcpyDeviceToDevice, st));
          PTROM_CUDA(cudaMemcpyAsync(x_full + n + lo, xi + m, m * 8, cudaMemcpyDeviceToDevice, st));
        }
        exchange_positions(ctx, comm, n, x_full);
        velocity(fxi);
      }
      std::swap(x_prev, xi);
      std::swap(f_prev, fxi);
      if (snapshots_local && m > 0)
        PTROM_CUDA(cudaMemcpyAsync(snapshots_local + (size_t)s * 2 * m, x_prev, 2 * m * 8, cudaMemcpyDeviceToHost, st));
      if (iterations) iterations[s] = updates;
      if (converged) converged[s] = conv ? 1 : 0;
      if (relative_residual) relative_residual[s] = rel;
    }
    PTROM_CUDA(cudaStreamSynchronize(st));
    check_device_status(ctx);
    if (n_pair_evals) *n_pair_evals = (uint64_t)evals * (uint64_t)m * (uint64_t)(n - 1);
  });
}

}  // extern "C"
