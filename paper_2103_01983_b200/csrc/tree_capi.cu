// tree_capi.cu — C ABI for the quadtree path (include/ptrom_b200.h "tree").
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "comm.cuh"
#include "ops.cuh"
#include "tree.cuh"

namespace ptrom {
void tree_collect(ptrom_ctx* ctx, Tree& t, int crit_kind, double crit_value, const std::vector<long long>& targets,
                  std::vector<long long>& c_off, std::vector<int>& clusters, std::vector<long long>& d_off,
                  std::vector<long long>& direct);
}

struct ptrom_tree {
  int device = 0;
  ptrom::Tree t;
  ~ptrom_tree() {
    cudaSetDevice(device);
    cudaDeviceSynchronize();  // the tree may have been used on any stream
    t.free_all(nullptr);
  }
};

using namespace ptrom;

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

// ClusterCriterion factories (quadtree.hpp:195-202)
void check_criterion(int kind, double value) {
  if (kind == PTROM_CRIT_BARNES_HUT) {
    if (!(value >= 0)) config_fail("opening ratio must be >= 0");
  } else if (kind == PTROM_CRIT_NEIGHBOR) {
    if (!(value >= 0)) config_fail("neighborhood width factor must be >= 0");
  } else {
    config_fail("unknown cluster criterion");
  }
}

// kernel.hpp:84-103 (sys.validate + check_state) for the tree evaluators.
// kernel.hpp:84-93 validate, host part (size, form); the finiteness and δ
// checks run on the uploaded copies (validate_uploaded, validate.cu).
void validate_eval_shape(long long n, int form) {
  if (n <= 0) config_fail("particle system is empty");
  if (form != PTROM_FORM_STANDARD && form != PTROM_FORM_DENOMINATOR_SCALED) config_fail("unknown kernel form");
}

struct DevBuf {
  cudaStream_t s;
  std::vector<void*> ptrs;
  template <class T>
  T* up(const T* h, size_t count) {
    if (!h) return nullptr;
    T* d;
    PTROM_CUDA(cudaMallocAsync(&d, std::max<size_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(d);
    PTROM_CUDA(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
  }
  template <class T>
  T* alloc(size_t count) {
    T* d;
    PTROM_CUDA(cudaMallocAsync(&d, std::max<size_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(d);
    return d;
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

// Shard blocks (slot order, x then y per rank block) back to particle order.
__global__ void scatter_slots_kernel(long long n, int world, const int* __restrict__ perm,
                                     const double* __restrict__ slots, double* __restrict__ f) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    // the rank block holding slot k (shard_bounds: lo_r = n·r / G)
    int r = (int)((k * world) / n);
    while (r > 0 && n * r / world > k) --r;
    while (r + 1 < world && n * (r + 1) / world <= k) ++r;
    const long long lo = n * r / world, hi = n * (r + 1) / world, m = hi - lo;
    const long long p = perm[k];
    f[p] = slots[2 * lo + (k - lo)];
    f[p + n] = slots[2 * lo + m + (k - lo)];
  }
}

}  // namespace

extern "C" {

int ptrom_dev_tree_build_f64(ptrom_ctx* ctx, int64_t n, const double* d_px, const double* d_py, const double* d_gamma,
                             int64_t leaf_capacity, ptrom_tree** out) {
  return guarded(ctx, [&] {
    if (!out) config_fail("build_tree: null output");
    auto* h = new ptrom_tree;
    h->device = ctx->device;
    try {
      tree_build(ctx, h->t, n, d_px, d_py, d_gamma, leaf_capacity, ctx->tree_seq_max);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int ptrom_tree_build_f64(ptrom_ctx* ctx, int64_t n, const double* px, const double* py, const double* gamma,
                         int64_t leaf_capacity, ptrom_tree** out) {
  return guarded(ctx, [&] {
    // quadtree.hpp:127-131 validation order
    if (n <= 0) config_fail("build_tree: no points");
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(px[i]) || !std::isfinite(py[i]) || !std::isfinite(gamma[i]))
        config_fail("build_tree: non-finite input");
    if (leaf_capacity < 1) config_fail("build_tree: leaf_capacity must be >= 1");
    DevBuf b{ctx->stream};
    const double* dx = b.up(px, n);
    const double* dy = b.up(py, n);
    const double* dg = b.up(gamma, n);
    auto* h = new ptrom_tree;
    h->device = ctx->device;
    try {
      tree_build(ctx, h->t, n, dx, dy, dg, leaf_capacity, ctx->tree_seq_max);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ptrom_tree_free(ptrom_tree* tree) { delete tree; }

int ptrom_tree_stats(ptrom_ctx* ctx, double* build_ms, double* eval_ms, uint64_t* interactions, uint64_t* prune_tests,
                     uint64_t* nodes, uint64_t* resolved_targets) {
  return guarded(ctx, [&] {
    const TreeStats& st = ctx->tree_stats;
    if (build_ms) *build_ms = st.build_ms;
    if (eval_ms) *eval_ms = st.eval_ms;
    if (interactions) *interactions = st.interactions;
    if (prune_tests) *prune_tests = st.prune_tests;
    if (nodes) *nodes = st.nodes;
    if (resolved_targets) *resolved_targets = st.resolved_targets;
  });
}

int ptrom_tree_build_info(ptrom_ctx* ctx, int* morton, int* levels) {
  return guarded(ctx, [&] {
    if (morton) *morton = ctx->tree_stats.morton;
    if (levels) *levels = (int)ctx->tree_stats.levels;
  });
}

int64_t ptrom_tree_num_nodes(const ptrom_tree* tree) { return tree ? (int64_t)tree->t.nodes.count : 0; }

int ptrom_tree_export(ptrom_ctx* ctx, const ptrom_tree* tree, double* bounds, double* width, double* centroid,
                      double* gamma_sum, int32_t* children, int64_t* begin, int64_t* end, int32_t* depth,
                      uint8_t* centroid_fallback, int64_t* perm, int64_t* slot, int32_t* leaf_node) {
  return guarded(ctx, [&] {
    if (!tree) config_fail("null tree");
    const Tree& t = tree->t;
    const size_t nn = t.nodes.count, n = (size_t)t.n;
    cudaStream_t s = ctx->stream;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst) PTROM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    d2h(bounds, t.nodes.bounds, nn * 32);
    d2h(width, t.nodes.width, nn * 8);
    d2h(centroid, t.nodes.centroid, nn * 16);
    d2h(gamma_sum, t.nodes.gamma_sum, nn * 8);
    d2h(children, t.nodes.children, nn * 16);
    d2h(depth, t.nodes.depth, nn * 4);
    d2h(centroid_fallback, t.nodes.fallback, nn);
    d2h(leaf_node, t.leaf_node, n * 4);
    std::vector<int> tmp;
    auto widen = [&](int64_t* dst, const int* src, size_t count) {
      if (!dst) return;
      tmp.resize(count);
      PTROM_CUDA(cudaMemcpyAsync(tmp.data(), src, count * 4, cudaMemcpyDeviceToHost, s));
      PTROM_CUDA(cudaStreamSynchronize(s));
      for (size_t i = 0; i < count; ++i) dst[i] = tmp[i];
    };
    widen(begin, t.nodes.begin, nn);
    widen(end, t.nodes.end, nn);
    widen(perm, t.perm, n);
    widen(slot, t.slot, n);
    PTROM_CUDA(cudaStreamSynchronize(s));
  });
}

int ptrom_collect_clusters(ptrom_ctx* ctx, ptrom_tree* tree, int crit_kind, double crit_value, int64_t n_targets,
                           const int64_t* targets, int64_t* cluster_offsets, int32_t* clusters, int64_t clusters_cap,
                           int64_t* direct_offsets, int64_t* direct, int64_t direct_cap) {
  return guarded(ctx, [&] {
    if (!tree) config_fail("null tree");
    check_criterion(crit_kind, crit_value);
    std::vector<long long> ids(targets, targets + n_targets);
    for (long long t : ids)
      if (t < 0 || t >= tree->t.n) config_fail("collect_clusters: bad target id");
    std::vector<long long> c_off, d_off, dl;
    std::vector<int> cl;
    tree_collect(ctx, tree->t, crit_kind, crit_value, ids, c_off, cl, d_off, dl);
    std::copy(c_off.begin(), c_off.end(), cluster_offsets);
    std::copy(d_off.begin(), d_off.end(), direct_offsets);
    if (clusters && clusters_cap >= (int64_t)cl.size()) std::copy(cl.begin(), cl.end(), clusters);
    if (direct && direct_cap >= (int64_t)dl.size()) std::copy(dl.begin(), dl.end(), direct);
  });
}

int ptrom_bh_velocity_f64(ptrom_ctx* ctx, ptrom_tree* tree, int64_t n, const double* x, const double* gamma,
                          double delta, int form, int crit_kind, double crit_value, const double* inflow, double* f,
                          uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_eval_shape(n, form);
    DevBuf b{ctx->stream};
    const double* dx = b.up(x, 2 * n);
    const double* dg = b.up(gamma, n);
    const double* di = b.up(inflow, inflow ? 2 * n : 0);
    validate_uploaded<double>(ctx, n, dx, dg, delta, di, "bh_velocity");
    if (!tree || tree->t.n != n) config_fail("bh_velocity: tree size mismatch");
    check_criterion(crit_kind, crit_value);
    double* df = b.alloc<double>(2 * n);
    const unsigned long long pairs =
        tree_eval(ctx, tree->t, dx, dg, delta, form, crit_kind, crit_value, di, df, nullptr, nullptr, nullptr, nullptr);
    PTROM_CUDA(cudaMemcpyAsync(f, df, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    if (n_pair_evals) *n_pair_evals = pairs;
  });
}

int ptrom_bh_jacobian_f64(ptrom_ctx* ctx, ptrom_tree* tree, int64_t n, const double* x, const double* gamma,
                          double delta, int form, int crit_kind, double crit_value, double* dfx_dx, double* dfx_dy,
                          double* dfy_dx, double* dfy_dy) {
  return guarded(ctx, [&] {
    validate_eval_shape(n, form);
    DevBuf b{ctx->stream};
    const double* dx = b.up(x, 2 * n);
    const double* dg = b.up(gamma, n);
    validate_uploaded<double>(ctx, n, dx, dg, delta, (const double*)nullptr, "bh_jacobian");
    if (!tree || tree->t.n != n) config_fail("bh_jacobian: tree size mismatch");
    check_criterion(crit_kind, crit_value);
    double* dj = b.alloc<double>(4 * n);
    tree_eval(ctx, tree->t, dx, dg, delta, form, crit_kind, crit_value, nullptr, nullptr, dj, dj + n, dj + 2 * n,
              dj + 3 * n);
    double* outs[4] = {dfx_dx, dfx_dy, dfy_dx, dfy_dy};
    for (int k = 0; k < 4; ++k)
      PTROM_CUDA(cudaMemcpyAsync(outs[k], dj + k * n, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
  });
}

int ptrom_dev_barnes_hut_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                      double delta, int form, int crit_kind, double crit_value, int64_t leaf_capacity,
                                      const double* d_inflow, double* d_f, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    check_criterion(crit_kind, crit_value);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    Tree t;
    try {
      tree_build(ctx, t, n, d_x, d_x + n, d_gamma, leaf_capacity, ctx->tree_seq_max);
      const unsigned long long pairs = tree_eval(ctx, t, d_x, d_gamma, delta, form, crit_kind, crit_value, d_inflow,
                                                 d_f, nullptr, nullptr, nullptr, nullptr);
      if (n_pair_evals) *n_pair_evals = pairs;
    } catch (...) {
      t.free_all(ctx->stream);
      throw;
    }
    t.free_all(ctx->stream);
  });
}

int ptrom_dev_barnes_hut_velocity_slots_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                            double delta, int form, int crit_kind, double crit_value,
                                            int64_t leaf_capacity, const double* d_inflow, int64_t k_begin,
                                            int64_t k_end, double* d_f_slots, int32_t* d_perm,
                                            uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    check_criterion(crit_kind, crit_value);
    if (!(delta >= 0)) config_fail("negative desingularization constant");
    if (n <= 0) config_fail("particle system is empty");
    if (k_begin < 0 || k_end > n || k_begin > k_end) config_fail("target slot range outside [0, n]");
    if (leaf_capacity < 1) config_fail("build_tree: leaf_capacity must be >= 1");
    Tree t;
    try {
      tree_build(ctx, t, n, d_x, d_x + n, d_gamma, leaf_capacity, ctx->tree_seq_max);
      const unsigned long long pairs = tree_eval(ctx, t, d_x, d_gamma, delta, form, crit_kind, crit_value, d_inflow,
                                                 nullptr, nullptr, nullptr, nullptr, nullptr, k_begin, k_end,
                                                 d_f_slots);
      if (d_perm) PTROM_CUDA(cudaMemcpyAsync(d_perm, t.perm, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
      if (n_pair_evals) *n_pair_evals = pairs;
    } catch (...) {
      t.free_all(ctx->stream);
      throw;
    }
    t.free_all(ctx->stream);
  });
}

int ptrom_barnes_hut_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double delta,
                                  int form, int crit_kind, double crit_value, int64_t leaf_capacity,
                                  const double* inflow, double* f, uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    validate_eval_shape(n, form);
    DevBuf b{ctx->stream};
    const double* dx = b.up(x, 2 * n);
    const double* dg = b.up(gamma, n);
    const double* di = b.up(inflow, inflow ? 2 * n : 0);
    validate_uploaded<double>(ctx, n, dx, dg, delta, di, "bh_velocity");
    check_criterion(crit_kind, crit_value);
    if (leaf_capacity < 1) config_fail("build_tree: leaf_capacity must be >= 1");
    double* df = b.alloc<double>(2 * n);
    Tree t;
    try {
      tree_build(ctx, t, n, dx, dx + n, dg, leaf_capacity, ctx->tree_seq_max);
      const unsigned long long pairs =
          tree_eval(ctx, t, dx, dg, delta, form, crit_kind, crit_value, di, df, nullptr, nullptr, nullptr, nullptr);
      if (n_pair_evals) *n_pair_evals = pairs;
    } catch (...) {
      t.free_all(ctx->stream);
      throw;
    }
    t.free_all(ctx->stream);
    PTROM_CUDA(cudaMemcpyAsync(f, df, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
  });
}

/* Sharded Barnes–Hut velocity (replicated build, far field
 * split by target). Every rank passes the full state, builds the same tree
 * (the build is deterministic), evaluates the contiguous tree slots
 * [r·n/G, (r+1)·n/G), and the slot blocks are all-gathered and scattered
 * back to particle order: every rank returns the full f (2n), bit-identical
 * to ptrom_barnes_hut_velocity_f64. n_pair_evals is the sum over ranks. */
int ptrom_barnes_hut_velocity_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* x,
                                          const double* gamma, double delta, int form, int crit_kind,
                                          double crit_value, int64_t leaf_capacity, const double* inflow, double* f,
                                          uint64_t* n_pair_evals) {
  return guarded(ctx, [&] {
    if (!comm) config_fail("null communicator");
    if (comm->device != ctx->device) config_fail("communicator and context are on different devices");
    validate_eval_shape(n, form);
    DevBuf b{ctx->stream};
    const double* dx = b.up(x, 2 * n);
    const double* dg = b.up(gamma, n);
    const double* di = b.up(inflow, inflow ? 2 * n : 0);
    validate_uploaded<double>(ctx, n, dx, dg, delta, di, "bh_velocity");
    check_criterion(crit_kind, crit_value);
    if (leaf_capacity < 1) config_fail("build_tree: leaf_capacity must be >= 1");
    const int G = comm->world;
    long long lo, hi;
    shard_bounds(n, comm->rank, G, lo, hi);
    double* slots = b.alloc<double>(2 * n);
    double* df = b.alloc<double>(2 * n);
    unsigned long long mine = 0;
    Tree t;
    try {
      tree_build(ctx, t, n, dx, dx + n, dg, leaf_capacity, ctx->tree_seq_max);
      if (hi > lo)
        mine = tree_eval(ctx, t, dx, dg, delta, form, crit_kind, crit_value, di, nullptr, nullptr, nullptr, nullptr,
                         nullptr, lo, hi, slots + 2 * lo);
      std::vector<size_t> off(G), cnt(G);
      for (int r = 0; r < G; ++r) {
        long long l, h;
        shard_bounds(n, r, G, l, h);
        off[r] = (size_t)(2 * l) * 8;
        cnt[r] = (size_t)(2 * (h - l)) * 8;
      }
      comm_allgatherv(ctx, comm, slots, off, cnt);
      const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)ctx->num_sms * 8);
      scatter_slots_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(n, G, t.perm, slots, df);
      PTROM_LAUNCH_CHECK();
    } catch (...) {
      t.free_all(ctx->stream);
      throw;
    }
    t.free_all(ctx->stream);
    PTROM_CUDA(cudaMemcpyAsync(f, df, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
    check_device_status(ctx);
    if (n_pair_evals) {
      std::vector<unsigned long long> all(G);
      comm_allgather_host(ctx, comm, &mine, all.data(), sizeof(mine));
      unsigned long long tot = 0;
      for (unsigned long long v : all) tot += v;
      *n_pair_evals = tot;
    }
  });
}

}  // extern "C"
