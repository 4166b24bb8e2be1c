// common.cuh — context, status latch, scratch arena and small device helpers
// shared by every translation unit of libptrom_b200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ptrom_b200.h"

#if !defined(__CUDA_ARCH__) || (__CUDA_ARCH__ >= 1000)
#else
#error "libptrom_b200 is written for sm_100a only"
#endif

namespace ptrom {

// Thrown inside the library and mapped to a status code at the C boundary.
struct status_error : std::runtime_error {
  int code;
  status_error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
[[noreturn]] inline void config_fail(const std::string& w) { throw status_error(PTROM_CONFIG_ERROR, w); }
[[noreturn]] inline void numerical_fail(const std::string& w) { throw status_error(PTROM_NUMERICAL_ERROR, w); }

#define PTROM_CUDA(call)                                                                            \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::ptrom::status_error(PTROM_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define PTROM_LAUNCH_CHECK() PTROM_CUDA(cudaGetLastError())

// Device status latch (written by kernels, read at synchronization points).
//  word[0]: 0 ok, else a status-kind code (see below)
//  word[1]: smallest offending particle index (for the reference's messages)
enum : int {
  kStatusOk = 0,
  kStatusNonFiniteVelocity = 1,  // coincident pair with zero desingularization
  kStatusSingularBlock = 2,      // integrators.hpp:187-189
  kStatusNonFiniteJacobian = 3,
  kStatusZeroClusterCirculation = 4,  // affine batch: G_A + mu G_B == 0
  kStatusCoincidentPair = 5,  // hamiltonian d² == 0; index = i·n + j (kernel.hpp:185-187)
};
struct DeviceStatus {
  int kind;
  int pad;
  long long index;
};

__device__ inline void latch_status(DeviceStatus* st, int kind, long long index) {
  const int old = atomicCAS(&st->kind, 0, kind);
  if (old == 0 || old == kind) atomicMin(&st->index, index);
}

// Growable device scratch arena owned by the context. Regions are handed out
// per call; callers never keep them across API calls.
struct Arena {
  void* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  void reset() { used = 0; }
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    if (base) cudaFree(base);
    base = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 4 + (1u << 20);
    PTROM_CUDA(cudaMalloc(&base, want));
    cap = want;
  }
  template <class T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    size_t need = off + count * sizeof(T);
    if (need > cap) throw status_error(PTROM_CUDA_ERROR, "scratch arena too small (internal sizing bug)");
    used = need;
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
  }
};

}  // namespace ptrom

namespace ptrom {
struct TreeStats {  // last tree build / evaluation on this context (ptrom_tree_stats)
  double build_ms = 0, eval_ms = 0;
  unsigned long long interactions = 0, prune_tests = 0, nodes = 0, levels = 0, resolved_targets = 0;
  int morton = 0;  // 1 when the last build used the Morton-key path
};
}  // namespace ptrom

struct ptrom_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  ptrom::DeviceStatus* d_status = nullptr;  // device latch
  ptrom::DeviceStatus* h_status = nullptr;  // pinned mirror
  ptrom::Arena scratch;                     // per-call temporaries (partials, norms)
  ptrom::Arena io;                          // host-API staging buffers
  // ptrom_profile_begin/end: events around the dominant kernel launches
  bool prof_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  long long status_pair_n = 0;
  int* h_counts = nullptr;  // pinned scratch for small D2H reads (tree level counts)
  unsigned* tile_ctr = nullptr;  // per-target-tile arrival counters of the fused chunk reduction (kept zeroed)
  size_t tile_ctr_cap = 0;  // n for decoding kStatusCoincidentPair (i·n + j)
  int allpairs_variant = 0;
  int hp_variant = 0;         // PTROM hyperpair kernel (tuning: hyperpair_variant; 1 = generic kernel)  // tuning knob (PTROM_ALLPAIRS_VARIANT), 0 = default shape
  ptrom::TreeStats tree_stats;
  int tree_seq_max = 2048;   // nodes up to this size get bit-exact sequential sums (PTROM_TREE_SEQ_MAX)
  long long reassign_big = 4096;  // clusters above this many members take reassign_big_kernel (PTROM_REASSIGN_BIG)
  int smem_optin = 232448;   // cudaDevAttrMaxSharedMemoryPerBlockOptin
  int tree_build_mode = 0;   // 0: Morton-key build (level build when it does not apply), 1: level build (PTROM_TREE_BUILD=levels)
};

namespace ptrom {

// RAII bracket recording start/stop events around one dominant-kernel launch
// when profiling is enabled on the context.
struct ProfScope {
  ptrom_ctx* ctx;
  cudaEvent_t stop = nullptr;
  explicit ProfScope(ptrom_ctx* c) : ctx(c) {
    if (!ctx->prof_on) return;
    if (ctx->prof_used == ctx->prof_events.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      ctx->prof_events.emplace_back(a, b);
    }
    auto& pr = ctx->prof_events[ctx->prof_used++];
    cudaEventRecord(pr.first, ctx->stream);
    stop = pr.second;
  }
  ~ProfScope() {
    if (stop) cudaEventRecord(stop, ctx->stream);
  }
};

// Reads and clears the device latch (synchronizes the stream). Throws a
// status_error carrying the reference's wording when something was latched.
void check_device_status(ptrom_ctx* ctx);

// Occupancy-aware split of the source range into chunks so that
// n_tiles * n_chunks fills whole waves of resident blocks.
int choose_source_chunks(ptrom_ctx* ctx, long long n_tiles, long long n_sources, int resident_per_sm,
                         long long min_chunk);

}  // namespace ptrom
