// comm.cuh — the multi-GPU communicator behind ptrom_comm.
//
// One rank per GPU. Two transports with one interface:
//  * NCCL (production): device buffers, stream-ordered on the context stream;
//    libnccl.so.2 is dlopen'ed at ptrom_comm_init (the one torch or the host
//    already loaded, else the system copy), so the library has no link-time
//    NCCL dependency.
//  * host callbacks (ptrom_host_collectives): the caller's own transport
//    (MPI, gloo, ...) on host buffers; device data is staged through the host
//    and every collective synchronizes.
#pragma once

#include <vector>

#include "common.cuh"

struct ptrom_comm {
  int rank = 0, world = 1, device = 0;
  void* nccl = nullptr;  // ncclComm_t
  ptrom_host_collectives ops{};
  void* user = nullptr;
};

namespace ptrom {

// Even contiguous split of `count` units (rank r owns [lo, hi)), the same
// rule as sharded.py's shard_bounds.
inline void shard_bounds(long long count, int rank, int world, long long& lo, long long& hi) {
  lo = count * rank / world;
  hi = count * (rank + 1) / world;
}

// Every rank r holds bytes [off[r], off[r] + cnt[r]) of d_buf; afterwards every
// rank holds all blocks (all-gather-v; NCCL: one group of in-place broadcasts).
void comm_allgatherv(ptrom_ctx* ctx, ptrom_comm* c, void* d_buf, const std::vector<size_t>& off,
                     const std::vector<size_t>& cnt);
// Device buffer broadcast from root (same local pointer role on every rank).
void comm_bcast(ptrom_ctx* ctx, ptrom_comm* c, void* d_buf, size_t bytes, int root);
// Several device broadcasts from root issued as one group.
void comm_bcast_many(ptrom_ctx* ctx, ptrom_comm* c, const std::vector<std::pair<void*, size_t>>& bufs, int root);
// Host buffer broadcast / rank-ordered all-gather (synchronous).
void comm_bcast_host(ptrom_ctx* ctx, ptrom_comm* c, void* h_buf, size_t bytes, int root);
void comm_allgather_host(ptrom_ctx* ctx, ptrom_comm* c, const void* h_send, void* h_recv, size_t bytes);
// `rows` rows of row_len doubles (row_len divisible by world): rank r gets,
// for every row, the element-wise sum over the ranks of the row's r-th
// chunk (row_len / world doubles) in d_out[row][·]. Used where every element
// has at most one non-zero contributor, so the sum is exact.
void comm_reduce_scatter_rows(ptrom_ctx* ctx, ptrom_comm* c, const double* d_in, long long rows, long long row_len,
                              double* d_out);
// Waits for the context stream (and, for NCCL, the communicator's work on it).
void comm_sync(ptrom_ctx* ctx, ptrom_comm* c);

}  // namespace ptrom
