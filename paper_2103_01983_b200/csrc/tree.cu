// tree.cu — Barnes–Hut quadtree on sm_100a: build, aggregation, traversal.
//
// Replaces quadtree.hpp:51-308 (build_tree, finish_node, split_node,
// bh_prune_check, neighbor_prune_check, collect_clusters, bh_velocity,
// bh_jacobian) and BarnesHutModel integrators.hpp:83-102.
//
// Build = MSD radix sort on the replayed midpoint path, one 2-bit digit per
// level. Level d holds the nodes created at depth d; for every node that
// splits (count > leaf_capacity and depth < 64, quadtree.hpp:74) each member
// computes its quadrant with the reference's arithmetic ((b0+b1)/2 midpoint,
// `<=` goes SW, quadtree.hpp:77-85) and the members are stably partitioned
// into SW, SE, NW, NE by a global 4-counter exclusive scan + scatter. Because
// every partition is stable and the first order is the identity, each node's
// segment is in ascending particle-id order when it is created — exactly the
// order finish_node (quadtree.hpp:51-67) sums in — and leaf members end up in
// ascending-id order inside perm like the reference's stable buckets.
//
// Preorder ids (quadtree.hpp:97-116 assign a child id then recurse): sorting
// all nodes by (begin, depth) yields preorder, so ids are the rank of that
// 64-bit key (CUB radix sort). skip[id] = first node with begin >= end is the
// stackless-DFS successor of a pruned/leaf node.
//
// Aggregation: nodes with <= kSeqMax members sum their segment sequentially
// in the reference order with _rn intrinsics (bit-identical gamma_sum and
// centroid, "exact"); larger nodes use a fixed-order block reduction (run to
// run deterministic) and carry a rigorous error bound on the centroid. A
// Barnes–Hut prune test on a non-exact node whose ratio lies within that
// bound of θ is "uncertain": the node's exact sequential sums are computed
// and the traversal is re-run, so prune decisions — and hence cluster lists
// — are always the reference's.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cfloat>
#include <climits>
#include <cmath>
#include <type_traits>
#include <vector>

#include "ops.cuh"
#include "tree.cuh"

namespace ptrom {

namespace {

constexpr int kMaxDepth = 64;  // quadtree.hpp:13
constexpr int kThreads = 256;

// All tree buffers come from the stream-ordered pool allocator (no
// cudaMalloc/cudaFree device synchronizations inside a build).
thread_local cudaStream_t g_alloc_stream = nullptr;
template <class T>
T* dalloc(size_t count) {
  T* p = nullptr;
  if (count) PTROM_CUDA(cudaMallocAsync(&p, count * sizeof(T), g_alloc_stream));
  return p;
}
inline void dfree(void* p) {
  if (p) cudaFreeAsync(p, g_alloc_stream);
}

int grid_for(ptrom_ctx* ctx, long long count, int tpb = kThreads) {
  long long g = (count + tpb - 1) / tpb;
  return (int)std::max(1LL, std::min(g, (long long)ctx->num_sms * 16));
}

struct U4Sum {
  __host__ __device__ uint4 operator()(const uint4& a, const uint4& b) const {
    return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
};

__device__ __forceinline__ unsigned comp(const uint4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}

// Quadrant prefix counters for the level partition. uint4: one-hot counts of
// all four quadrants. u64 (n + 1 < 2^21): three 21-bit counts packed into one
// word (half the scan traffic); inside a splitting node every element is
// counted, so quadrant 3 = span - (q0 + q1 + q2).
constexpr int kPackBits = 21;
__device__ __forceinline__ uint4 quad_one(int q, uint4*) {
  return make_uint4(q == 0, q == 1, q == 2, q == 3);
}
__device__ __forceinline__ unsigned long long quad_one(int q, unsigned long long*) {
  return q < 3 ? 1ull << (kPackBits * q) : 0ull;
}
__device__ __forceinline__ uint4 quad_zero(uint4*) { return make_uint4(0, 0, 0, 0); }
__device__ __forceinline__ unsigned long long quad_zero(unsigned long long*) { return 0ull; }
// count of quadrant q among positions [i0, i1) of one splitting node (a = scan[i0], b = scan[i1])
__device__ __forceinline__ unsigned quad_delta(const uint4& a, const uint4& b, int q, int) {
  return comp(b, q) - comp(a, q);
}
__device__ __forceinline__ unsigned quad_delta(unsigned long long a, unsigned long long b, int q, int span) {
  constexpr unsigned long long m = (1ull << kPackBits) - 1;
  const unsigned d0 = (unsigned)(((b >> 0) & m) - ((a >> 0) & m));
  const unsigned d1 = (unsigned)(((b >> kPackBits) & m) - ((a >> kPackBits) & m));
  const unsigned d2 = (unsigned)(((b >> (2 * kPackBits)) & m) - ((a >> (2 * kPackBits)) & m));
  return q == 0 ? d0 : q == 1 ? d1 : q == 2 ? d2 : (unsigned)span - d0 - d1 - d2;
}

// ---------------------------------------------------------------- hull ---
__global__ void hull_kernel(long long n, const double* __restrict__ px, const double* __restrict__ py,
                            double* __restrict__ block_out) {
  double xl = DBL_MAX, xh = -DBL_MAX, yl = DBL_MAX, yh = -DBL_MAX;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    xl = fmin(xl, px[i]);
    xh = fmax(xh, px[i]);
    yl = fmin(yl, py[i]);
    yh = fmax(yh, py[i]);
  }
  using BR = cub::BlockReduce<double, kThreads>;
  __shared__ typename BR::TempStorage t0, t1, t2, t3;
  xl = BR(t0).Reduce(xl, cub::Min());
  xh = BR(t1).Reduce(xh, cub::Max());
  yl = BR(t2).Reduce(yl, cub::Min());
  yh = BR(t3).Reduce(yh, cub::Max());
  if (threadIdx.x == 0) {
    block_out[4 * blockIdx.x + 0] = xl;
    block_out[4 * blockIdx.x + 1] = xh;
    block_out[4 * blockIdx.x + 2] = yl;
    block_out[4 * blockIdx.x + 3] = yh;
  }
}

__global__ void iota_copy_kernel(long long n, const double* __restrict__ px, const double* __restrict__ py,
                                 const double* __restrict__ g, int* __restrict__ ord, double* __restrict__ sx,
                                 double* __restrict__ sy, double* __restrict__ sg, int* __restrict__ pos_rec,
                                 int root_splits) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    ord[i] = (int)i;
    sx[i] = px[i];
    sy[i] = py[i];
    sg[i] = g[i];
    pos_rec[i] = root_splits ? 0 : -1;
  }
}

// ------------------------------------------------------------- levels ---
// quadtree.hpp:81-86: quadrant digit of each member of a splitting node.
template <class T>
__global__ void digit_kernel(long long n, const int* __restrict__ pos_rec, const double* __restrict__ sx,
                             const double* __restrict__ sy, const double* __restrict__ rec_mid, T* __restrict__ flags,
                             unsigned char* __restrict__ digit) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= n; k += (long long)gridDim.x * blockDim.x) {
    T f = quad_zero((T*)nullptr);
    if (k < n) {
      const int r = pos_rec[k];
      if (r >= 0) {
        const double cx = rec_mid[2 * r], cy = rec_mid[2 * r + 1];
        const int qx = sx[k] <= cx ? 0 : 1;
        const int qy = sy[k] <= cy ? 0 : 1;
        const int q = qy * 2 + qx;
        digit[k] = (unsigned char)q;
        f = quad_one(q, (T*)nullptr);
      }
    }
    flags[k] = f;
  }
}

// Per level node: child counts (from the scan) and number of children.
// Level descriptors live on the device: lv = {first record, node count,
// records so far}; the host only holds upper bounds (Lub), so several levels
// run back to back without a host round trip.
template <class T>
__global__ void child_count_kernel(const int* __restrict__ lv, int Lub, const int* __restrict__ rec_begin,
                                   const int* __restrict__ rec_end, const unsigned char* __restrict__ rec_split,
                                   const T* __restrict__ scan, int* __restrict__ nchild) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l > Lub) return;
  const int L = lv[1], r = lv[0] + l;
  int c = 0;
  if (l < L && rec_split[r]) {
    const int span = rec_end[r] - rec_begin[r];
    const T a = scan[rec_begin[r]], b = scan[rec_end[r]];
    for (int q = 0; q < 4; ++q) c += quad_delta(a, b, q, span) != 0;
  }
  nchild[l] = c;
}

// quadtree.hpp:87-116: child records in SW, SE, NW, NE order.
// lv_next = {R, C, R + C} for the children level (C = total child count).
__global__ void level_advance_kernel(const int* __restrict__ lv, const int* __restrict__ child_off, int Lub,
                                     int* __restrict__ lv_next) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int C = child_off[Lub];
    lv_next[0] = lv[2];
    lv_next[1] = C;
    lv_next[2] = lv[2] + C;
  }
}

template <class T>
__global__ void make_children_kernel(const int* __restrict__ lv, int leaf_cap, const T* __restrict__ scan,
                                     const int* __restrict__ child_off, TreeRecords rec, int* __restrict__ n_split_next) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lv[1]) return;
  const int r = lv[0] + l, next_base = lv[2];
  if (!rec.split[r]) return;
  const int span = rec.end[r] - rec.begin[r];
  const T a = scan[rec.begin[r]], b = scan[rec.end[r]];
  const double b0 = rec.bounds[4 * r], b1 = rec.bounds[4 * r + 1], b2 = rec.bounds[4 * r + 2], b3 = rec.bounds[4 * r + 3];
  const double cx = rec.mid[2 * r], cy = rec.mid[2 * r + 1];
  const double half = __ddiv_rn(rec.width[r], 2.0);
  int cursor = rec.begin[r];
  int j = 0;
  int splits = 0;
  for (int q = 0; q < 4; ++q) {
    const int cnt = (int)quad_delta(a, b, q, span);
    if (cnt == 0) continue;
    const int c = next_base + child_off[l] + (j++);
    rec.children[4 * r + q] = c;
    rec.begin[c] = cursor;
    rec.end[c] = cursor + cnt;
    cursor += cnt;
    const double cb0 = (q & 1) ? cx : b0, cb1 = (q & 1) ? b1 : cx;
    const double cb2 = (q & 2) ? cy : b2, cb3 = (q & 2) ? b3 : cy;
    rec.bounds[4 * c] = cb0;
    rec.bounds[4 * c + 1] = cb1;
    rec.bounds[4 * c + 2] = cb2;
    rec.bounds[4 * c + 3] = cb3;
    rec.mid[2 * c] = __dmul_rn(__dadd_rn(cb0, cb1), 0.5);  // (b0 + b1) / 2, exact halving
    rec.mid[2 * c + 1] = __dmul_rn(__dadd_rn(cb2, cb3), 0.5);
    rec.width[c] = half;
    rec.depth[c] = rec.depth[r] + 1;
    rec.children[4 * c] = rec.children[4 * c + 1] = rec.children[4 * c + 2] = rec.children[4 * c + 3] = -1;
    const bool sp = cnt > leaf_cap && rec.depth[r] + 1 < kMaxDepth;
    rec.split[c] = sp ? 1 : 0;
    splits += sp;
  }
  if (splits) atomicAdd(n_split_next, splits);
}

// Stable scatter of the splitting nodes' members into their children.
template <class T>
__global__ void scatter_kernel(long long n, const int* __restrict__ pos_rec, const unsigned char* __restrict__ digit,
                               const T* __restrict__ scan, TreeRecords rec, const int* __restrict__ ord,
                               const double* __restrict__ sx, const double* __restrict__ sy,
                               const double* __restrict__ sg, int* __restrict__ ord_n, double* __restrict__ sx_n,
                               double* __restrict__ sy_n, double* __restrict__ sg_n, int* __restrict__ pos_rec_n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const int r = pos_rec[k];
    long long np = k;
    int nrec = -1;
    if (r >= 0) {
      const int q = digit[k];
      const int c = rec.children[4 * r + q];
      const int b0 = rec.begin[r];
      np = rec.begin[c] + (long long)quad_delta(scan[b0], scan[k], q, (int)(k - b0));
      nrec = rec.split[c] ? c : -1;
    }
    ord_n[np] = ord[k];
    sx_n[np] = sx[k];
    sy_n[np] = sy[k];
    sg_n[np] = sg[k];
    pos_rec_n[np] = nrec;
  }
}

// quadtree.hpp:51-67 finish_node: sequential sums in the reference's order.
__device__ __forceinline__ void finish_exact(TreeRecords& rec, int r, int b, int e, double gs, double wx, double wy,
                                             double plx, double ply) {
  rec.gamma_sum[r] = gs;
  const bool fb = gs == 0.0;
  rec.fallback[r] = fb ? 1 : 0;
  const double c = (double)(e - b);
  rec.centroid[2 * r] = fb ? __ddiv_rn(plx, c) : __ddiv_rn(wx, gs);
  rec.centroid[2 * r + 1] = fb ? __ddiv_rn(ply, c) : __ddiv_rn(wy, gs);
  rec.exact[r] = 1;
  rec.cerr[r] = 0.0;
}

// Nodes [R0, R1) of one level, one lane each. Nodes with at most kLaneSum
// members are summed by their own lane (short sequential chains, all lanes
// busy — the many small nodes of the deep levels); larger ones go to the mid
// list (one warp each, sums_mid_kernel) or, above seq_max, to the large list
// (multi-CTA, certified).
constexpr int kSumWarps = kThreads / 32;
constexpr int kLaneSum = 48;
__global__ void __launch_bounds__(kThreads) sums_small_kernel(const int* __restrict__ lv, TreeRecords rec,
                                                              const double* __restrict__ sx,
                                                              const double* __restrict__ sy,
                                                              const double* __restrict__ sg, int seq_max,
                                                              int* __restrict__ large_list,
                                                              int* __restrict__ large_count,
                                                              int* __restrict__ mid_list,
                                                              int* __restrict__ mid_count) {
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= lv[1]) return;
  const int r = lv[0] + i;
  const int b = rec.begin[r], e = rec.end[r];
  const int cnt = e - b;
  if (cnt > seq_max) {
    large_list[atomicAdd(large_count, 1)] = r;
    return;
  }
  if (cnt > kLaneSum) {
    mid_list[atomicAdd(mid_count, 1)] = r;
    return;
  }
  double gs = 0.0, wx = 0.0, wy = 0.0, plx = 0.0, ply = 0.0;
#pragma unroll 4
  for (int k = b; k < e; ++k) {
    const double g = sg[k], x = sx[k], y = sy[k];
    gs = __dadd_rn(gs, g);
    wx = __dadd_rn(wx, __dmul_rn(g, x));
    wy = __dadd_rn(wy, __dmul_rn(g, y));
    plx = __dadd_rn(plx, x);
    ply = __dadd_rn(ply, y);
  }
  finish_exact(rec, r, b, e, gs, wx, wy, plx, ply);
}

// Mid-size nodes (kLaneSum < members <= seq_max): one warp per node. The
// lanes stage kMidChunk members at a time in shared memory (coalesced, 4 per
// lane) and prefetch the next chunk into registers while lane 0 runs the
// reference's sequential chain over the current one (the chain, not the
// load latency, bounds the node).
constexpr int kMidChunk = 128;
__global__ void __launch_bounds__(kThreads) sums_mid_kernel(TreeRecords rec, const double* __restrict__ sx,
                                                            const double* __restrict__ sy,
                                                            const double* __restrict__ sg,
                                                            const int* __restrict__ mid_list,
                                                            int* __restrict__ mid_count) {
  __shared__ double st[kSumWarps][2][3][kMidChunk];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int total = *mid_count;
  constexpr int PER = kMidChunk / 32;
  for (int w = blockIdx.x * kSumWarps + wib; w < total; w += gridDim.x * kSumWarps) {
    const int r = mid_list[w];
    const int b = rec.begin[r], e = rec.end[r];
    double pg[PER], px[PER], py[PER];
    auto fetch = [&](int c0) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int k = c0 + u * 32 + lane;
        pg[u] = k < e ? sg[k] : 0.0;
        px[u] = k < e ? sx[k] : 0.0;
        py[u] = k < e ? sy[k] : 0.0;
      }
    };
    auto put = [&](int buf) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        st[wib][buf][0][u * 32 + lane] = pg[u];
        st[wib][buf][1][u * 32 + lane] = px[u];
        st[wib][buf][2][u * 32 + lane] = py[u];
      }
    };
    fetch(b);
    put(0);
    __syncwarp();
    // The five chains run on lanes 0..4 (same instructions, one term each):
    // lane 0 Σg, 1 Σg·x, 2 Σg·y, 3 Σx, 4 Σy — term = a·b with b = 1 where the
    // reference adds a plain value (exact), so every chain is the reference's.
    const int ia = lane == 3 ? 1 : lane == 4 ? 2 : 0;  // operand a: g, x or y
    const int ib = lane == 1 ? 1 : lane == 2 ? 2 : -1;  // operand b: x, y or 1
    double acc = 0.0;
    int buf = 0;
    for (int c0 = b; c0 < e; c0 += kMidChunk) {
      const bool more = c0 + kMidChunk < e;
      if (more) fetch(c0 + kMidChunk);  // in flight while lanes 0..4 add
      if (lane < 5) {
        const int n = min(kMidChunk, e - c0);
        const double* A = st[wib][buf][ia];
        const double* Bv = st[wib][buf][ib < 0 ? 0 : ib];
        const double* Bp = ib < 0 ? nullptr : Bv;
        int j = 0;
        for (; j + 8 <= n; j += 8) {  // loads of 8 members issued ahead of the chain
          double a8[8], b8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            a8[u] = A[j + u];
            b8[u] = Bp ? Bp[j + u] : 1.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(a8[u], b8[u]));
        }
        for (; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(A[j], Bp ? Bp[j] : 1.0));
      }
      __syncwarp();
      if (more) put(buf ^ 1);
      __syncwarp();
      buf ^= 1;
    }
    const double gs = __shfl_sync(0xffffffffu, acc, 0), wx = __shfl_sync(0xffffffffu, acc, 1),
                 wy = __shfl_sync(0xffffffffu, acc, 2), plx = __shfl_sync(0xffffffffu, acc, 3),
                 ply = __shfl_sync(0xffffffffu, acc, 4);
    if (lane == 0) finish_exact(rec, r, b, e, gs, wx, wy, plx, ply);
  }
}

// Large-node finish: centroid from block/child-reduced sums red = {Σg, Σgx,
// Σgy, Σx, Σy, Σ|g|, Σ|gx|, Σ|gy|}, with a rigorous bound on its distance from
// the reference's sequential order (quadtree.hpp:51-67).
__device__ void finish_certified(TreeRecords& rec, int r, int b, int e, const double (&red)[8]) {
  const double m = (double)(e - b);
  const double u = 0x1p-53;
  // both orders are within (m-1)u·Σ|a| (+ product rounding) of the exact
  // sum; their difference within twice that (first order, padded).
  const double k2 = 2.05 * (m + 1.0) * u;
  const double eg = k2 * red[5], ex = k2 * (red[6] * 1.0001), ey = k2 * (red[7] * 1.0001);
  const double gs = red[0];
  rec.gamma_sum[r] = gs;
  const bool fb = gs == 0.0;
  rec.fallback[r] = fb ? 1 : 0;
  double cx, cy, err;
  if (fb) {
    cx = __ddiv_rn(red[3], m);
    cy = __ddiv_rn(red[4], m);
  } else {
    cx = __ddiv_rn(red[1], gs);
    cy = __ddiv_rn(red[2], gs);
  }
  if (fabs(gs) <= 2.0 * eg) {
    err = INFINITY;  // the fallback flag itself is uncertain
  } else {
    const double ag = fabs(gs) - eg;
    err = (ex + fabs(cx) * eg) / ag + (ey + fabs(cy) * eg) / ag + 8.0 * u * (fabs(cx) + fabs(cy));
  }
  rec.centroid[2 * r] = cx;
  rec.centroid[2 * r + 1] = cy;
  rec.exact[r] = 0;
  rec.cerr[r] = err;
}

// Large nodes (> seq_max members) in ONE launch: every CTA finds the node of
// each of its chunks (kChunk members) from the large list, reduces the chunk
// with a fixed-order block reduction; the last CTA to finish adds each
// node's chunk partials in chunk order (deterministic) and finishes the
// centroid with a rigorous bound on its distance from the reference's
// sequential order. With no large node at the level the launch is a no-op.
constexpr int kChunk = 8192;
__global__ void __launch_bounds__(kThreads) large_sums_kernel(TreeRecords rec, const double* __restrict__ sx,
                                                              const double* __restrict__ sy,
                                                              const double* __restrict__ sg,
                                                              const int* __restrict__ large_list,
                                                              int* __restrict__ large_count,
                                                              int* __restrict__ chunk_off,
                                                              double* __restrict__ part,
                                                              unsigned* __restrict__ done_ctr) {
  const int total = *large_count;
  if (total == 0) return;
  using BR = cub::BlockReduce<double, kThreads>;
  using BS = cub::BlockScan<int, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ typename BS::TempStorage stmp;
  constexpr int kMaxLarge = 4096;  // chunk offsets kept in shared memory
  __shared__ int s_off[kMaxLarge + 1];
  __shared__ bool s_last;
  __shared__ int s_carry;
  // chunk offsets of the large nodes: block-wide scan, 256 nodes per round
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int l0 = 0; l0 < total; l0 += kThreads) {
    const int li = l0 + threadIdx.x;
    int nc = 0;
    if (li < total) {
      const int r = large_list[li];
      nc = (rec.end[r] - rec.begin[r] + kChunk - 1) / kChunk;
    }
    int ex = 0, agg = 0;
    BS(stmp).ExclusiveSum(nc, ex, agg);
    const int carry = s_carry;
    if (li < total) {
      if (li < kMaxLarge) s_off[li] = carry + ex;
      if (blockIdx.x == 0) chunk_off[li] = carry + ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + agg;
    __syncthreads();
  }
  const int nchunks = s_carry;
  if (total <= kMaxLarge && threadIdx.x == 0) s_off[total] = nchunks;
  if (blockIdx.x == 0 && threadIdx.x == 0) chunk_off[total] = nchunks;
  __syncthreads();
  for (int ci = blockIdx.x; ci < nchunks; ci += gridDim.x) {
    int li = 0, base = 0;
    if (total <= kMaxLarge) {  // node of chunk ci: last li with s_off[li] <= ci
      int lo = 0, hi = total;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= ci) lo = mid;
        else hi = mid;
      }
      li = lo;
      base = s_off[lo];
    } else {  // very long lists: linear walk over the global offsets
      int acc = 0;
      for (int q = 0; q < total; ++q) {
        const int r = large_list[q];
        const int nc = (rec.end[r] - rec.begin[r] + kChunk - 1) / kChunk;
        if (ci < acc + nc) {
          li = q;
          base = acc;
          break;
        }
        acc += nc;
      }
    }
    const int r = large_list[li];
    const int b = rec.begin[r] + (ci - base) * kChunk;
    const int e = min(rec.end[r], b + kChunk);
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // gs wx wy plx ply |g| |gx| |gy|
#pragma unroll 4
    for (int k = b + threadIdx.x; k < e; k += kThreads) {
      const double g = sg[k], x = sx[k], y = sy[k];
      const double gx = __dmul_rn(g, x), gy = __dmul_rn(g, y);
      v[0] = __dadd_rn(v[0], g);
      v[1] = __dadd_rn(v[1], gx);
      v[2] = __dadd_rn(v[2], gy);
      v[3] = __dadd_rn(v[3], x);
      v[4] = __dadd_rn(v[4], y);
      v[5] = __dadd_rn(v[5], fabs(g));
      v[6] = __dadd_rn(v[6], fabs(gx));
      v[7] = __dadd_rn(v[7], fabs(gy));
    }
    for (int c = 0; c < 8; ++c) {
      const double t = BR(tmp).Sum(v[c]);
      if (threadIdx.x == 0) part[8 * (long long)ci + c] = t;
      __syncthreads();
    }
  }
  // last CTA: finish every large node
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int li = threadIdx.x; li < total; li += blockDim.x) {
    const int r = large_list[li];
    const int b = rec.begin[r], e = rec.end[r];
    double red[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int ci = chunk_off[li]; ci < chunk_off[li + 1]; ++ci)
      for (int c = 0; c < 8; ++c) red[c] = __dadd_rn(red[c], part[8 * (long long)ci + c]);
    finish_certified(rec, r, b, e, red);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *done_ctr = 0;  // ready for the next level
    *large_count = 0;
  }
}

// ------------------------------------------------------------ preorder ---
// Preorder (quadtree.hpp:97-116 numbers a child, then recurses) sorts nodes by
// (begin, depth); the nodes sharing a begin are one ancestor chain with
// consecutive depths, so id = #(nodes with a smaller begin) + depth - (the
// chain's smallest depth): a histogram over begin, one scan, no sort.
__global__ void begin_hist_kernel(int R, const int* __restrict__ rbegin, const int* __restrict__ rdepth,
                                  int* __restrict__ cnt, int* __restrict__ mind) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int b = rbegin[r];
  atomicAdd(cnt + b, 1);
  atomicMin(mind + b, rdepth[r]);
}

__global__ void preorder_ids_kernel(int R, const int* __restrict__ rbegin, const int* __restrict__ rdepth,
                                    const int* __restrict__ base, const int* __restrict__ mind,
                                    int* __restrict__ rec2id, int* __restrict__ order) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int b = rbegin[r];
  const int id = base[b] + rdepth[r] - mind[b];
  rec2id[r] = id;
  order[id] = r;
}


__global__ void emit_nodes_kernel(int R, const int* __restrict__ order, const int* __restrict__ rec2id,
                                  const int* __restrict__ begin_base, TreeRecords rec, TreeNodes nd) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= R) return;
  const int r = order[id];
  for (int k = 0; k < 4; ++k) {
    nd.bounds[4 * id + k] = rec.bounds[4 * r + k];
    const int c = rec.children[4 * r + k];
    nd.children[4 * id + k] = c >= 0 ? rec2id[c] : -1;
  }
  const int b = rec.begin[r], e = rec.end[r];
  const bool leaf = rec.children[4 * r] < 0 && rec.children[4 * r + 1] < 0 && rec.children[4 * r + 2] < 0 &&
                    rec.children[4 * r + 3] < 0;
  // skip: first node in preorder with begin >= e
  const int lo = begin_base[e];
  nd.width[id] = rec.width[r];
  nd.centroid[2 * id] = rec.centroid[2 * r];
  nd.centroid[2 * id + 1] = rec.centroid[2 * r + 1];
  nd.gamma_sum[id] = rec.gamma_sum[r];
  nd.begin[id] = b;
  nd.end[id] = e;
  nd.depth[id] = rec.depth[r];
  nd.fallback[id] = rec.fallback[r];
  nd.exact[id] = rec.exact[r];
  nd.cerr[id] = rec.cerr[r];
  nd.skip[id] = lo;
  nd.leaf[id] = leaf ? 1 : 0;
}

__global__ void particle_maps_kernel(long long n, const int* __restrict__ perm, int* __restrict__ slot) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    slot[perm[k]] = (int)k;
}

__global__ void leaf_node_kernel(int R, TreeNodes nd, const int* __restrict__ perm, int* __restrict__ leaf_node) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= R || !nd.leaf[id]) return;
  for (int k = nd.begin[id]; k < nd.end[id]; ++k) leaf_node[perm[k]] = id;
}

// Exact sequential sums for the flagged (uncertain) nodes: members in
// ascending id order are {p : begin <= slot[p] < end}.
__global__ void exact_sums_kernel(int R, long long n, TreeNodes nd, const int* __restrict__ slot,
                                  const double* __restrict__ px, const double* __restrict__ py,
                                  const double* __restrict__ g) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= R || !nd.need_exact[id] || nd.exact[id]) return;
  const int b = nd.begin[id], e = nd.end[id];
  double gs = 0.0, wx = 0.0, wy = 0.0, plx = 0.0, ply = 0.0;
  for (long long p = 0; p < n; ++p) {
    const int s = slot[p];
    if (s < b || s >= e) continue;
    const double gg = g[p], x = px[p], y = py[p];
    gs = __dadd_rn(gs, gg);
    wx = __dadd_rn(wx, __dmul_rn(gg, x));
    wy = __dadd_rn(wy, __dmul_rn(gg, y));
    plx = __dadd_rn(plx, x);
    ply = __dadd_rn(ply, y);
  }
  nd.gamma_sum[id] = gs;
  const bool fb = gs == 0.0;
  nd.fallback[id] = fb ? 1 : 0;
  const double c = (double)(e - b);
  nd.centroid[2 * id] = fb ? __ddiv_rn(plx, c) : __ddiv_rn(wx, gs);
  nd.centroid[2 * id + 1] = fb ? __ddiv_rn(ply, c) : __ddiv_rn(wy, gs);
  nd.exact[id] = 1;
  nd.cerr[id] = 0.0;
}

}  // namespace

// ---------------------------------------------------------------- build ---
void TreeRecords::alloc(size_t cap_) {
  cap = cap_;
  begin = dalloc<int>(cap);
  end = dalloc<int>(cap);
  depth = dalloc<int>(cap);
  children = dalloc<int>(4 * cap);
  split = dalloc<unsigned char>(cap);
  fallback = dalloc<unsigned char>(cap);
  exact = dalloc<unsigned char>(cap);
  bounds = dalloc<double>(4 * cap);
  mid = dalloc<double>(2 * cap);
  width = dalloc<double>(cap);
  centroid = dalloc<double>(2 * cap);
  gamma_sum = dalloc<double>(cap);
  cerr = dalloc<double>(cap);
}
void TreeRecords::free() {
  void* ps[] = {begin, end, depth, children, split, fallback, exact, bounds, mid, width, centroid, gamma_sum, cerr};
  for (void* p : ps) dfree(p);
  *this = TreeRecords{};
}
void TreeRecords::grow(size_t need, size_t used, cudaStream_t s) {
  if (need <= cap) return;
  TreeRecords n;
  n.alloc(std::max(need, cap * 2));
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) PTROM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  };
  cp(n.begin, begin, used * 4);
  cp(n.end, end, used * 4);
  cp(n.depth, depth, used * 4);
  cp(n.children, children, used * 16);
  cp(n.split, split, used);
  cp(n.fallback, fallback, used);
  cp(n.exact, exact, used);
  cp(n.bounds, bounds, used * 32);
  cp(n.mid, mid, used * 16);
  cp(n.width, width, used * 8);
  cp(n.centroid, centroid, used * 16);
  cp(n.gamma_sum, gamma_sum, used * 8);
  cp(n.cerr, cerr, used * 8);
  free();
  *this = n;
}

void TreeNodes::alloc(size_t nn) {
  count = nn;
  bounds = dalloc<double>(4 * nn);
  width = dalloc<double>(nn);
  centroid = dalloc<double>(2 * nn);
  gamma_sum = dalloc<double>(nn);
  cerr = dalloc<double>(nn);
  children = dalloc<int>(4 * nn);
  begin = dalloc<int>(nn);
  end = dalloc<int>(nn);
  depth = dalloc<int>(nn);
  skip = dalloc<int>(nn);
  fallback = dalloc<unsigned char>(nn);
  exact = dalloc<unsigned char>(nn);
  leaf = dalloc<unsigned char>(nn);
  need_exact = dalloc<unsigned char>(nn);
}
void TreeNodes::free() {
  void* ps[] = {bounds, width, centroid, gamma_sum, cerr, children, begin, end, depth, skip, fallback, exact, leaf,
                need_exact};
  for (void* p : ps) dfree(p);
  *this = TreeNodes{};
}

void Tree::free_all(cudaStream_t s) {
  g_alloc_stream = s;
  nodes.free();
  void* ps[] = {perm, slot, leaf_node, sx, sy, sg, px, py, g};
  for (void* p : ps) dfree(p);
  perm = slot = leaf_node = nullptr;
  sx = sy = sg = px = py = g = nullptr;
}

// Preorder numbering and the final tables, shared by both builds: records
// [0, R) with perm-order members (ord, sx, sy, sg become the tree's).
void finish_tree(ptrom_ctx* ctx, Tree& t, TreeRecords& rec, int R, int* ord, double* sx, double* sy, double* sg) {
  cudaStream_t s = ctx->stream;
  const long long n = t.n;
  // ---- preorder numbering
  int *cnt = dalloc<int>(n + 1), *base = dalloc<int>(n + 1), *mind = dalloc<int>(n + 1);
  int *order = dalloc<int>(R), *rec2id = dalloc<int>(R);
  PTROM_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), s));
  PTROM_CUDA(cudaMemsetAsync(mind, 0x7f, (n + 1) * sizeof(int), s));
  begin_hist_kernel<<<(R + kThreads - 1) / kThreads, kThreads, 0, s>>>(R, rec.begin, rec.depth, cnt, mind);
  PTROM_LAUNCH_CHECK();
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, base, (int)(n + 1), s);
  void* stmp = dalloc<char>(scan_bytes + 256);
  PTROM_CUDA(cub::DeviceScan::ExclusiveSum(stmp, scan_bytes, cnt, base, (int)(n + 1), s));
  preorder_ids_kernel<<<(R + kThreads - 1) / kThreads, kThreads, 0, s>>>(R, rec.begin, rec.depth, base, mind, rec2id,
                                                                         order);
  t.nodes.alloc(R);
  emit_nodes_kernel<<<(R + kThreads - 1) / kThreads, kThreads, 0, s>>>(R, order, rec2id, base, rec, t.nodes);
  PTROM_LAUNCH_CHECK();
  PTROM_CUDA(cudaMemsetAsync(t.nodes.need_exact, 0, R, s));

  t.perm = ord;
  t.sx = sx;
  t.sy = sy;
  t.sg = sg;
  t.slot = dalloc<int>(n);
  t.leaf_node = dalloc<int>(n);
  particle_maps_kernel<<<grid_for(ctx, n), kThreads, 0, s>>>(n, t.perm, t.slot);
  leaf_node_kernel<<<(R + kThreads - 1) / kThreads, kThreads, 0, s>>>(R, t.nodes, t.perm, t.leaf_node);
  PTROM_LAUNCH_CHECK();
  void* frees[] = {cnt, base, mind, order, rec2id, stmp};
  for (void* p : frees) dfree(p);
}

bool tree_build_morton(ptrom_ctx* ctx, Tree& t, long long leaf_cap, int seq_max);

// quadtree.hpp:124-162 build_tree over device points (px, py) and weights g.
void tree_build(ptrom_ctx* ctx, Tree& t, long long n, const double* d_px, const double* d_py, const double* d_g,
                long long leaf_cap, int seq_max) {
  if (n <= 0) config_fail("build_tree: no points");
  if (n >= (1LL << 30)) config_fail("build_tree: more than 2^30 points is not supported");
  if (leaf_cap < 1) config_fail("build_tree: leaf_capacity must be >= 1");
  cudaStream_t s = ctx->stream;
  g_alloc_stream = s;
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, s);
  t.free_all(s);
  t.n = n;
  t.leaf_cap = leaf_cap;
  // keep the build inputs (exact-sum fallback and collect_clusters target positions)
  t.px = dalloc<double>(n);
  t.py = dalloc<double>(n);
  t.g = dalloc<double>(n);
  PTROM_CUDA(cudaMemcpyAsync(t.px, d_px, n * 8, cudaMemcpyDeviceToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(t.py, d_py, n * 8, cudaMemcpyDeviceToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(t.g, d_g, n * 8, cudaMemcpyDeviceToDevice, s));

  ctx->tree_stats = TreeStats{};
  if (ctx->tree_build_mode == 0 && tree_build_morton(ctx, t, leaf_cap, seq_max)) {
    cudaEventRecord(ev1, s);
    PTROM_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    ctx->tree_stats.build_ms = ms;
    ctx->tree_stats.nodes = t.nodes.count;
    ctx->tree_stats.morton = 1;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return;
  }

  // ---- root: tight square hull (quadtree.hpp:139-151)
  const int hb = std::min<long long>((n + kThreads - 1) / kThreads, 256);
  double* hull = dalloc<double>(4 * hb);
  hull_kernel<<<hb, kThreads, 0, s>>>(n, t.px, t.py, hull);
  PTROM_LAUNCH_CHECK();
  std::vector<double> hh(4 * hb);
  PTROM_CUDA(cudaMemcpyAsync(hh.data(), hull, hh.size() * 8, cudaMemcpyDeviceToHost, s));
  PTROM_CUDA(cudaStreamSynchronize(s));
  dfree(hull);
  double x_lo = hh[0], x_hi = hh[1], y_lo = hh[2], y_hi = hh[3];
  for (int b = 1; b < hb; ++b) {
    x_lo = std::min(x_lo, hh[4 * b]);
    x_hi = std::max(x_hi, hh[4 * b + 1]);
    y_lo = std::min(y_lo, hh[4 * b + 2]);
    y_hi = std::max(y_hi, hh[4 * b + 3]);
  }
  if (!std::isfinite(x_lo) || !std::isfinite(x_hi) || !std::isfinite(y_lo) || !std::isfinite(y_hi))
    config_fail("build_tree: non-finite input");
  double side = std::max(x_hi - x_lo, y_hi - y_lo);
  if (side == 0.0) side = 1.0;
  t.root_width = side;
  const double cx = (x_lo + x_hi) / 2.0, cy = (y_lo + y_hi) / 2.0;
  const double rb[4] = {cx - side / 2.0, cx + side / 2.0, cy - side / 2.0, cy + side / 2.0};
  const double rmid[2] = {(rb[0] + rb[1]) / 2.0, (rb[2] + rb[3]) / 2.0};

  TreeRecords rec;
  {
    // room for the tree plus the speculative look-ahead of the level batches
    // (see run_levels) so that the records rarely need to grow
    const long long lcap = std::min<long long>(n + 1, 4 * (n / (leaf_cap + 1)) + 4);
    const long long est = (n / std::max<long long>(1, leaf_cap)) * 2 + 16;
    rec.alloc((size_t)std::max<long long>(1024, lcap > 524288 ? est : std::max(est, 5 * lcap)));
  }
  const int zero = 0, one = 1, neg[4] = {-1, -1, -1, -1};
  const int nn32 = (int)n, d0 = 0;
  const unsigned char root_split = (n > leaf_cap) ? 1 : 0;
  PTROM_CUDA(cudaMemcpyAsync(rec.begin, &zero, 4, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.end, &nn32, 4, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.depth, &d0, 4, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.children, neg, 16, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.split, &root_split, 1, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.bounds, rb, 32, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.mid, rmid, 16, cudaMemcpyHostToDevice, s));
  PTROM_CUDA(cudaMemcpyAsync(rec.width, &side, 8, cudaMemcpyHostToDevice, s));
  (void)one;

  // ---- level buffers
  int *ord = dalloc<int>(n), *ord_n = dalloc<int>(n), *pr = dalloc<int>(n), *pr_n = dalloc<int>(n);
  double *sx = dalloc<double>(n), *sy = dalloc<double>(n), *sg = dalloc<double>(n);
  double *sx_n = dalloc<double>(n), *sy_n = dalloc<double>(n), *sg_n = dalloc<double>(n);
  const bool packed = n + 1 < (1LL << kPackBits);  // u64 counters (3 x 21 bits) else uint4
  void* flags_raw = dalloc<uint4>(n + 1);
  void* scan_raw = dalloc<uint4>(n + 1);
  unsigned char* digit = dalloc<unsigned char>(n);
  int* dcount = dalloc<int>(4);  // [0] splits at next level, [1] large-node count, [2] mid-node count
  int* h_counts = ctx->h_counts;  // pinned, owned by the context
  size_t scan_tmp_bytes = 0, scan_tmp_u64 = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, scan_tmp_bytes, (uint4*)flags_raw, (uint4*)scan_raw, U4Sum(),
                                 make_uint4(0, 0, 0, 0), n + 1, s);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp_u64, (unsigned long long*)flags_raw, (unsigned long long*)scan_raw,
                                n + 1, s);
  scan_tmp_bytes = std::max(scan_tmp_bytes, scan_tmp_u64);
  size_t scan2_tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan2_tmp_bytes, (int*)nullptr, (int*)nullptr, (int)std::min<long long>(n, INT_MAX), s);
  void* tmp = dalloc<char>(std::max(scan_tmp_bytes, scan2_tmp_bytes) + 256);
  int* nchild = nullptr;
  int* child_off = nullptr;
  size_t lvl_cap = 0;
  const long long max_large = n / std::max(1, seq_max) + 2;  // nodes > seq_max at one level
  int* large_list = dalloc<int>(max_large);
  int* chunk_off = dalloc<int>(max_large + 1);
  double* large_part = dalloc<double>(8 * (n / kChunk + max_large + 1));
  unsigned* done_ctr = dalloc<unsigned>(1);
  PTROM_CUDA(cudaMemsetAsync(done_ctr, 0, sizeof(unsigned), s));
  int* mid_list = dalloc<int>(std::max<long long>(1, n));
  // level descriptors {first record, nodes, records so far}, ping-pong
  int* lv_buf = dalloc<int>(8);
  int* lv_cur = lv_buf;
  int* lv_next = lv_buf + 4;
  auto run_sums = [&](const int* lv, long long nodes_ub) {
    sums_small_kernel<<<(int)std::max<long long>(1, (nodes_ub + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        lv, rec, sx, sy, sg, seq_max, large_list, dcount + 1, mid_list, dcount + 2);
    const int mid_blocks = (int)std::min<long long>((nodes_ub + kSumWarps - 1) / kSumWarps, ctx->num_sms * 16LL);
    sums_mid_kernel<<<std::max(1, mid_blocks), kThreads, 0, s>>>(rec, sx, sy, sg, mid_list, dcount + 2);
    large_sums_kernel<<<ctx->num_sms * 2, kThreads, 0, s>>>(rec, sx, sy, sg, large_list, dcount + 1, chunk_off,
                                                            large_part, done_ctr);
    PTROM_LAUNCH_CHECK();
  };

  iota_copy_kernel<<<grid_for(ctx, n), kThreads, 0, s>>>(n, t.px, t.py, t.g, ord, sx, sy, sg, pr, root_split);
  PTROM_LAUNCH_CHECK();
  {
    const int lv0[4] = {0, 1, 1, 0};
    PTROM_CUDA(cudaMemcpyAsync(lv_cur, lv0, sizeof(lv0), cudaMemcpyHostToDevice, s));
  }
  // root sums
  PTROM_CUDA(cudaMemsetAsync(dcount, 0, 16, s));
  run_sums(lv_cur, 1);

  int R = 1;
  // Nodes per level are bounded by 4 x (splitting nodes) <= 4 n / (leaf_cap + 1):
  // levels run in batches of K on upper bounds, one host round trip per batch
  // (speculative levels past the last split are empty no-ops).
  const long long Lcap = std::min<long long>(n + 1, 4 * (n / (leaf_cap + 1)) + 4);
  const int K = Lcap > 524288 ? 1 : 4;
  auto run_levels = [&](auto* tag) {
  using T = std::remove_pointer_t<decltype(tag)>;
  T* flags = static_cast<T*>(flags_raw);
  T* scan = static_cast<T*>(scan_raw);
  long long Lub = 1, R_ub = 1;
  while (root_split) {
    for (int lvl = 0; lvl < K; ++lvl) {
      const long long Cub = std::min(Lcap, 4 * Lub);
      rec.grow((size_t)(R_ub + Cub), (size_t)R_ub, s);
      if ((size_t)(Lub + 1) > lvl_cap) {
        dfree(nchild);
        dfree(child_off);
        lvl_cap = std::max<size_t>(Lub + 1, lvl_cap * 2);
        nchild = dalloc<int>(lvl_cap);
        child_off = dalloc<int>(lvl_cap);
      }
      digit_kernel<<<grid_for(ctx, n + 1), kThreads, 0, s>>>(n, pr, sx, sy, rec.mid, flags, digit);
      PTROM_LAUNCH_CHECK();
      if constexpr (std::is_same_v<T, uint4>)
        PTROM_CUDA(cub::DeviceScan::ExclusiveScan(tmp, scan_tmp_bytes, flags, scan, U4Sum(), make_uint4(0, 0, 0, 0),
                                                  n + 1, s));
      else
        PTROM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_tmp_bytes, flags, scan, n + 1, s));
      child_count_kernel<<<(int)((Lub + 1 + kThreads - 1) / kThreads), kThreads, 0, s>>>(
          lv_cur, (int)Lub, rec.begin, rec.end, rec.split, scan, nchild);
      PTROM_LAUNCH_CHECK();
      PTROM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan2_tmp_bytes, nchild, child_off, (int)(Lub + 1), s));
      level_advance_kernel<<<1, 32, 0, s>>>(lv_cur, child_off, (int)Lub, lv_next);
      PTROM_CUDA(cudaMemsetAsync(dcount, 0, 16, s));
      make_children_kernel<<<(int)((Lub + kThreads - 1) / kThreads), kThreads, 0, s>>>(lv_cur, (int)leaf_cap, scan,
                                                                                      child_off, rec, dcount);
      PTROM_LAUNCH_CHECK();
      scatter_kernel<<<grid_for(ctx, n), kThreads, 0, s>>>(n, pr, digit, scan, rec, ord, sx, sy, sg, ord_n, sx_n,
                                                           sy_n, sg_n, pr_n);
      PTROM_LAUNCH_CHECK();
      std::swap(ord, ord_n);
      std::swap(sx, sx_n);
      std::swap(sy, sy_n);
      std::swap(sg, sg_n);
      std::swap(pr, pr_n);
      run_sums(lv_next, Cub);
      std::swap(lv_cur, lv_next);
      Lub = Cub;
      R_ub += Cub;
    }
    PTROM_CUDA(cudaMemcpyAsync(h_counts, lv_cur, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
    PTROM_CUDA(cudaStreamSynchronize(s));
    R = h_counts[2];
    if (h_counts[1] == 0) break;
    Lub = h_counts[1];
    R_ub = R;
  }
  };
  if (packed)
    run_levels((unsigned long long*)nullptr);
  else
    run_levels((uint4*)nullptr);

  finish_tree(ctx, t, rec, R, ord, sx, sy, sg);
  cudaEventRecord(ev1, s);
  PTROM_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  ctx->tree_stats.build_ms = ms;
  ctx->tree_stats.nodes = R;
  ctx->tree_stats.levels = 0;
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);

  void* frees[] = {ord_n, pr, pr_n, sx_n, sy_n, sg_n, flags_raw, scan_raw, digit, dcount, tmp, nchild, child_off, large_list,
                   chunk_off, large_part, done_ctr, mid_list, lv_buf};
  for (void* p : frees) dfree(p);
  rec.free();
}


// ========================================================= Morton build ===
// The same tree from one sort. Node bounds depend only on the path from the
// root (child bounds = parent bounds cut at the parent's midpoint,
// quadtree.hpp:87-93), so each point replays the reference's midpoint
// arithmetic down its path on its own and records the 2-bit quadrant of each
// level in a 64-bit key (level 0 in the top bits). A stable radix sort of
// (key, id) puts every node's members in one contiguous range, children in
// SW, SE, NW, NE order. Then:
//  * nodes above seq_max members (the certified-sum "large" nodes) are split
//    level by level in one cooperative launch (grid barrier per level): the
//    child boundaries are the digit changes inside the node's key range;
//  * every node of at most seq_max members whose parent is large roots a
//    subtree that one CTA finishes in shared memory: its keys, ids and
//    (Γ, x, y) are loaded once; the CTA splits it level by level, then walks
//    the levels back up: a leaf sorts its members by id (the reference's
//    bucket order, quadtree.hpp:81-105, giving perm / sx / sy / sg), an
//    internal node merges its children's ascending-id runs, and finish_node's
//    five sequential chains (quadtree.hpp:51-67) run over that order, so the
//    sums are bit-identical;
//  * the large nodes take the certified chunked reduction (large_sums_kernel).
// A split needed below the key's levels, a subtree with more local nodes than
// the CTA holds, or a record-capacity overflow makes the host rebuild with the
// level build (same tree).
namespace {

constexpr int kMortonLevels = 32;
constexpr int kSubMax = 2048;     // members of a subtree (seq_max <= kSubMax)
constexpr int kSubNodes = 1024;   // local nodes of a subtree
constexpr int kSubThreads = 256;
constexpr int kSubBig = 1024;
constexpr int kSubLevels = 64;
constexpr int kListShorts = 22016;  // ascending-id lists of all local levels, level L at L*m (shared memory)
constexpr int kThreadChain = 256;  // chains of nodes up to this size run in one thread

struct MortonState {
  int lvl_cnt[kMaxDepth + 2];  // records per level of the large-node pass (level 0 = root)
  int overflow;                // split needed below the key's levels / capacity exceeded
  int overflow_depth;          // ... because of the key's levels (a 32-level key may fix it)
  int finite;                  // hull finite
  int levels_used;
  int large_count, sub_count;
  int sub_big, sub_small;      // subtrees above / at most kSubBig members (big ones scheduled first)
  int rec_extra;               // records created by the subtree CTAs
  int sub_next;                // subtree work counter (dynamic scheduling)
  unsigned bar_count, bar_gen;
  double width;
};

__device__ __forceinline__ void grid_barrier(MortonState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &st->bar_gen;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(&st->bar_count, 1u) == gridDim.x - 1) {
      st->bar_count = 0;
      __threadfence();
      atomicAdd(&st->bar_gen, 1u);
    } else {
      while (*vgen == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Root record from the hull partials (quadtree.hpp:139-151), on the device.
__global__ void morton_root_kernel(int hb, const double* __restrict__ hull, long long n, long long leaf_cap,
                                   TreeRecords rec, MortonState* st) {
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31;
  double xl = DBL_MAX, xh = -DBL_MAX, yl = DBL_MAX, yh = -DBL_MAX;
  for (int b = lane; b < hb; b += 32) {
    xl = fmin(xl, hull[4 * b]);
    xh = fmax(xh, hull[4 * b + 1]);
    yl = fmin(yl, hull[4 * b + 2]);
    yh = fmax(yh, hull[4 * b + 3]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    xl = fmin(xl, __shfl_xor_sync(0xffffffffu, xl, o));
    xh = fmax(xh, __shfl_xor_sync(0xffffffffu, xh, o));
    yl = fmin(yl, __shfl_xor_sync(0xffffffffu, yl, o));
    yh = fmax(yh, __shfl_xor_sync(0xffffffffu, yh, o));
  }
  if (lane != 0) return;
  st->finite = isfinite(xl) && isfinite(xh) && isfinite(yl) && isfinite(yh);
  double side = fmax(__dsub_rn(xh, xl), __dsub_rn(yh, yl));
  if (side == 0.0) side = 1.0;
  const double cx = __dmul_rn(__dadd_rn(xl, xh), 0.5), cy = __dmul_rn(__dadd_rn(yl, yh), 0.5);
  const double hs = __dmul_rn(side, 0.5);
  const double b0 = __dsub_rn(cx, hs), b1 = __dadd_rn(cx, hs), b2 = __dsub_rn(cy, hs), b3 = __dadd_rn(cy, hs);
  rec.begin[0] = 0;
  rec.end[0] = (int)n;
  rec.depth[0] = 0;
  for (int q = 0; q < 4; ++q) rec.children[q] = -1;
  rec.split[0] = n > leaf_cap ? 1 : 0;
  rec.bounds[0] = b0;
  rec.bounds[1] = b1;
  rec.bounds[2] = b2;
  rec.bounds[3] = b3;
  rec.mid[0] = __dmul_rn(__dadd_rn(b0, b1), 0.5);
  rec.mid[1] = __dmul_rn(__dadd_rn(b2, b3), 0.5);
  rec.width[0] = side;
  st->width = side;
  st->lvl_cnt[0] = 1;
}

// Path key of every point: the quadrant chosen at each of `levels` levels
// with the reference's midpoint and `<=` rule (quadtree.hpp:77-85).
__global__ void morton_keys_kernel(long long n, const double* __restrict__ px, const double* __restrict__ py,
                                   const TreeRecords rec, int levels, unsigned long long* __restrict__ key,
                                   int* __restrict__ ids) {
  const double r0 = rec.bounds[0], r1 = rec.bounds[1], r2 = rec.bounds[2], r3 = rec.bounds[3];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double x = px[i], y = py[i];
    double b0 = r0, b1 = r1, b2 = r2, b3 = r3;
    unsigned long long k = 0;
    for (int l = 0; l < levels; ++l) {
      const double cx = __dmul_rn(__dadd_rn(b0, b1), 0.5), cy = __dmul_rn(__dadd_rn(b2, b3), 0.5);
      const bool qx = !(x <= cx), qy = !(y <= cy);
      k = (k << 2) | (unsigned long long)((qy ? 2 : 0) | (qx ? 1 : 0));
      if (qx) b0 = cx; else b1 = cx;
      if (qy) b2 = cy; else b3 = cy;
    }
    key[i] = k;
    ids[i] = (int)i;
  }
}

__device__ __forceinline__ int key_digit(const unsigned long long* __restrict__ skey, int k, int shift) {
  return (int)((__ldg(skey + k) >> shift) & 3ull);
}

// Child geometry of record r (quadtree.hpp:87-105) into record c for quadrant q.
__device__ __forceinline__ void morton_child_geometry(TreeRecords& rec, int r, int c, int q, int d, bool l2) {
  double b0, b1, b2, b3, cx, cy, w;
  if (l2) {  // parent written by another CTA of this launch
    b0 = __ldcg(rec.bounds + 4 * r);
    b1 = __ldcg(rec.bounds + 4 * r + 1);
    b2 = __ldcg(rec.bounds + 4 * r + 2);
    b3 = __ldcg(rec.bounds + 4 * r + 3);
    cx = __ldcg(rec.mid + 2 * r);
    cy = __ldcg(rec.mid + 2 * r + 1);
    w = __ldcg(rec.width + r);
  } else {
    b0 = rec.bounds[4 * r];
    b1 = rec.bounds[4 * r + 1];
    b2 = rec.bounds[4 * r + 2];
    b3 = rec.bounds[4 * r + 3];
    cx = rec.mid[2 * r];
    cy = rec.mid[2 * r + 1];
    w = rec.width[r];
  }
  const double cb0 = (q & 1) ? cx : b0, cb1 = (q & 1) ? b1 : cx;
  const double cb2 = (q & 2) ? cy : b2, cb3 = (q & 2) ? b3 : cy;
  rec.bounds[4 * c] = cb0;
  rec.bounds[4 * c + 1] = cb1;
  rec.bounds[4 * c + 2] = cb2;
  rec.bounds[4 * c + 3] = cb3;
  rec.mid[2 * c] = __dmul_rn(__dadd_rn(cb0, cb1), 0.5);
  rec.mid[2 * c + 1] = __dmul_rn(__dadd_rn(cb2, cb3), 0.5);
  rec.width[c] = __ddiv_rn(w, 2.0);
  rec.depth[c] = d + 1;
  rec.children[4 * c] = rec.children[4 * c + 1] = rec.children[4 * c + 2] = rec.children[4 * c + 3] = -1;
}

// Large nodes (> seq_max members), level by level (quadtree.hpp:70-116): one
// cooperative launch, a grid barrier between levels, a warp per node with a
// grouped 11-ary search for the three digit boundaries. Children of at most
// seq_max members are subtree roots for morton_subtree_kernel.
__global__ void __launch_bounds__(kThreads) morton_levels_kernel(const unsigned long long* __restrict__ skey,
                                                                 int levels, long long leaf_cap, int seq_max,
                                                                 TreeRecords rec, int rec_cap, MortonState* st,
                                                                 int* __restrict__ sub_list, int sub_half,
                                                                 int* __restrict__ large_list) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int nwarps = gridDim.x * (kThreads / 32);
  int base = 0, cnt = 1;
  int d = 0;
  for (;; ++d) {
    const int next_base = base + cnt;
    const int shift = 2 * (levels - 1 - d);
    for (int w = gwarp; w < cnt; w += nwarps) {
      const int r = base + w;
      const int b = __ldcg(rec.begin + r), e = __ldcg(rec.end + r);
      if (e - b <= seq_max) {
        if (lane == 0) {  // big subtrees at the front, the rest from sub_cap/2 on
          atomicAdd(&st->sub_count, 1);
          if (e - b > kSubBig) sub_list[atomicAdd(&st->sub_big, 1)] = r;
          else sub_list[sub_half + atomicAdd(&st->sub_small, 1)] = r;
        }
        continue;
      }
      if (lane == 0) large_list[atomicAdd(&st->large_count, 1)] = r;
      if (d >= levels) {  // a large node always splits (count > seq_max >= leaf_capacity)
        if (lane == 0) {
          st->overflow = 1;
          st->overflow_depth = 1;
        }
        continue;
      }
      const int g = lane < 11 ? 0 : (lane < 22 ? 1 : 2);
      const int g0 = g * 11, gsz = g == 2 ? 10 : 11, gl = lane - g0;
      const int q = g + 1;
      int lo = b, hi = e;  // first k in [lo, hi] with digit >= q (hi = e: none)
      while (__any_sync(0xffffffffu, hi > lo)) {
        const long long span = hi - lo;
        const int p = lo + (int)((span * gl) / gsz);
        const bool pred = hi > lo && key_digit(skey, p, shift) >= q;
        const unsigned bits = (__ballot_sync(0xffffffffu, pred) >> g0) & ((1u << gsz) - 1u);
        if (hi > lo) {
          const int J = bits ? __ffs(bits) - 1 : gsz;
          const int pJ = J < gsz ? lo + (int)((span * J) / gsz) : hi;
          const int pJm = J > 0 ? lo + (int)((span * (J - 1)) / gsz) + 1 : lo;
          lo = pJm;
          hi = pJ;
        }
      }
      const int s1 = __shfl_sync(0xffffffffu, lo, 0), s2 = __shfl_sync(0xffffffffu, lo, 11),
                s3 = __shfl_sync(0xffffffffu, lo, 22);
      if (lane == 0) {
        const int sb[5] = {b, s1, s2, s3, e};
        int nch = 0;
        for (int k = 0; k < 4; ++k) nch += sb[k + 1] > sb[k];
        const int first = next_base + atomicAdd(&st->lvl_cnt[d + 1], nch);
        if (first + nch > rec_cap) {
          st->overflow = 1;
        } else {
          int j = 0;
          for (int k = 0; k < 4; ++k) {
            if (sb[k + 1] == sb[k]) {
              rec.children[4 * r + k] = -1;
              continue;
            }
            const int c = first + (j++);
            rec.children[4 * r + k] = c;
            rec.begin[c] = sb[k];
            rec.end[c] = sb[k + 1];
            rec.split[c] = (sb[k + 1] - sb[k] > leaf_cap && d + 1 < kMaxDepth) ? 1 : 0;
            morton_child_geometry(rec, r, c, k, d, true);
          }
        }
      }
    }
    grid_barrier(st);
    const int ncnt = *(volatile int*)&st->lvl_cnt[d + 1];
    const int ovf = *(volatile int*)&st->overflow;
    base = next_base;
    cnt = ncnt;
    if (cnt == 0 || ovf || d + 1 > kMaxDepth) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->levels_used = d + 1;
}

// Shared-memory layout of one subtree CTA.
using SubIdSort = cub::BlockRadixSort<unsigned, kSubThreads, kSubMax / kSubThreads, short>;
struct SubSmem {
  union {
    unsigned long long keys[kSubMax];     // topology phase
    typename SubIdSort::TempStorage sort;  // member ids -> ascending order
    short lists[kListShorts];             // ascending-id member list of every node, level L at L*m
  } u;
  double g[kSubMax], x[kSubMax], y[kSubMax];
  int ids[kSubMax];                    // particle id of each member
  short lb[kSubNodes], le[kSubNodes];  // local node ranges (member positions in key order)
  short lfirst[kSubNodes], lpar[kSubNodes];
  unsigned char ldep[kSubNodes], lsplit[kSubNodes], lmask[kSubNodes], lq[kSubNodes];
  short lvl_start[kSubLevels + 2];
  int nloc, nlvl, base, ovf;
};

static_assert(sizeof(SubSmem) <= 112 * 1024, "two subtree CTAs per SM (228 KB shared memory)");

// One CTA per subtree root (see the section comment). Phases:
//  1. members (key, id, Γ, x, y) into shared memory;
//  2. local topology level by level (binary searches for the digit changes);
//  3. one record allocation for the subtree, records written in parallel
//     (geometry replayed from the subtree root down each node's path);
//  4. members sorted by id (bitonic, shared memory): the root's ascending-id
//     list; each level's lists are stably partitioned into the children's
//     (ballots), kept per level in global scratch `lists`;
//  5. finish_node's chains for every node over its list in one parallel pass
//     (a thread per node up to 64 members, lanes 0..4 of a warp above), and
//     the leaves' members into perm / sx / sy / sg.
__global__ void __launch_bounds__(kSubThreads, 2) morton_subtree_kernel(
    const unsigned long long* __restrict__ skey, const int* __restrict__ sid, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pg, const int* __restrict__ sub_list, int sub_half,
    MortonState* st, TreeRecords rec, int rec_cap, int levels, long long leaf_cap, int id_bits,
    int* __restrict__ perm, double* __restrict__ sx, double* __restrict__ sy,
    double* __restrict__ sg, double* __restrict__ aux, long long* __restrict__ prof) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_abs[kSubThreads / 32][3];
  SubSmem& S = *reinterpret_cast<SubSmem*>(smem_raw);
#define SUBPROF(ph)                                                          \
  if (prof && tid == 0) prof[(long long)si * 10 + (ph)] = clock64();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarp = kSubThreads / 32;
  __shared__ int s_top, s_skip;
  if (tid == 0) {  // records of the large-node pass come first
    int t = 0;
    for (int d = 0; d <= kMaxDepth + 1; ++d) t += st->lvl_cnt[d];
    s_top = t;
    s_skip = st->overflow || !st->finite;
  }
  __syncthreads();
  if (s_skip) return;
  const int rec_top = s_top;
  const int n_sub = st->sub_count;
  __shared__ int s_si;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_si = atomicAdd(&st->sub_next, 1);  // CTAs take subtrees as they free up
    __syncthreads();
    const int si = s_si;
    if (si >= n_sub) break;
    const int nbig = st->sub_big;
    const int r = si < nbig ? sub_list[si] : sub_list[sub_half + (si - nbig)];
    const int b = rec.begin[r], e = rec.end[r], m = e - b;
    const int d0 = rec.depth[r];
    SUBPROF(0)
    // ---- 1. members
    {
      constexpr int IPT = kSubMax / kSubThreads;
      int v[IPT];
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int k = u * kSubThreads + tid;
        v[u] = k < m ? sid[b + k] : -1;
        if (k < m) {
          S.u.keys[k] = skey[b + k];
          S.ids[k] = v[u];
        }
      }
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int k = u * kSubThreads + tid;
        if (v[u] >= 0) {
          S.g[k] = pg[v[u]];
          S.x[k] = px[v[u]];
          S.y[k] = py[v[u]];
        }
      }
    }
    if (tid == 0) {
      S.lb[0] = 0;
      S.le[0] = (short)m;
      S.ldep[0] = 0;
      S.lsplit[0] = rec.split[r];
      S.lpar[0] = -1;
      S.lq[0] = 0;
      S.nloc = 1;
      S.nlvl = 0;
      S.lvl_start[0] = 0;
      S.lvl_start[1] = 1;
      S.ovf = 0;
    }
    __syncthreads();
    SUBPROF(1)
    // ---- 2. topology, level by level inside the subtree
    for (int L = 0;; ++L) {
      const int lo = S.lvl_start[L], hi = S.lvl_start[L + 1];
      if (lo == hi || S.ovf) break;
      for (int j = lo + tid; j < hi; j += kSubThreads) {
        S.lmask[j] = 0;
        if (!S.lsplit[j]) continue;
        const int d = d0 + S.ldep[j];
        if (d >= levels) {
          S.ovf = 1;
          st->overflow_depth = 1;
          continue;
        }
        const int shift = 2 * (levels - 1 - d);
        const int jb = S.lb[j], je = S.le[j];
        int sb[5] = {jb, jb, jb, jb, je};
#pragma unroll
        for (int q = 1; q <= 3; ++q) {
          int l = jb, h = je;
          while (l < h) {
            const int md = (l + h) >> 1;
            if ((int)((S.u.keys[md] >> shift) & 3ull) >= q) h = md;
            else l = md + 1;
          }
          sb[q] = l;
        }
        int nch = 0;
        unsigned char mask = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (sb[q + 1] > sb[q]) {
            ++nch;
            mask |= (unsigned char)(1u << q);
          }
        const int first = atomicAdd(&S.nloc, nch);
        if (first + nch > kSubNodes) {
          S.ovf = 1;
          continue;
        }
        S.lfirst[j] = (short)first;
        S.lmask[j] = mask;
        int c = first;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!(mask & (1u << q))) continue;
          const int cnt = sb[q + 1] - sb[q];
          S.lb[c] = (short)sb[q];
          S.le[c] = (short)sb[q + 1];
          S.ldep[c] = (unsigned char)(S.ldep[j] + 1);
          S.lsplit[c] = (cnt > leaf_cap && d + 1 < kMaxDepth) ? 1 : 0;
          S.lpar[c] = (short)j;
          S.lq[c] = (unsigned char)q;
          ++c;
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int nn = min(S.nloc, kSubNodes);
        S.lvl_start[L + 2] = (short)nn;
        S.nlvl = L + 1;
        if (L + 2 > kSubLevels || (long long)(L + 2) * m > kListShorts) S.ovf = 1;
      }
      __syncthreads();
    }
    SUBPROF(2)
    // ---- 3. records
    if (tid == 0 && !S.ovf) {
      const int extra = S.nloc - 1;
      S.base = extra ? rec_top + atomicAdd(&st->rec_extra, extra) : 0;
      if (S.base + extra > rec_cap) S.ovf = 1;
    }
    __syncthreads();
    if (S.ovf) {
      if (tid == 0) st->overflow = 1;
      __syncthreads();
      continue;
    }
    const int nloc = S.nloc, base = S.base;
    auto rid = [&](int j) { return j == 0 ? r : base + j - 1; };
    {
      const double r0 = rec.bounds[4 * r], r1 = rec.bounds[4 * r + 1], r2 = rec.bounds[4 * r + 2],
                   r3 = rec.bounds[4 * r + 3], rw = rec.width[r];
      for (int j = tid; j < nloc; j += kSubThreads) {
        const int me = rid(j);
        if (j > 0) {
          // path quadrants from the subtree root, then the reference's halvings
          unsigned long long path = 0;
          int depth = 0;
          for (int c = j; c > 0; c = S.lpar[c]) {
            path |= (unsigned long long)S.lq[c] << (2 * depth);
            ++depth;
          }
          double b0 = r0, b1 = r1, b2 = r2, b3 = r3, w = rw;
          for (int l = depth - 1; l >= 0; --l) {
            const int q = (int)((path >> (2 * l)) & 3ull);
            const double cx = __dmul_rn(__dadd_rn(b0, b1), 0.5), cy = __dmul_rn(__dadd_rn(b2, b3), 0.5);
            if (q & 1) b0 = cx; else b1 = cx;
            if (q & 2) b2 = cy; else b3 = cy;
            w = __ddiv_rn(w, 2.0);
          }
          rec.bounds[4 * me] = b0;
          rec.bounds[4 * me + 1] = b1;
          rec.bounds[4 * me + 2] = b2;
          rec.bounds[4 * me + 3] = b3;
          rec.mid[2 * me] = __dmul_rn(__dadd_rn(b0, b1), 0.5);
          rec.mid[2 * me + 1] = __dmul_rn(__dadd_rn(b2, b3), 0.5);
          rec.width[me] = w;
          rec.depth[me] = d0 + S.ldep[j];
          rec.begin[me] = b + S.lb[j];
          rec.end[me] = b + S.le[j];
          rec.split[me] = S.lsplit[j];
        }
        const unsigned mask = S.lsplit[j] ? S.lmask[j] : 0u;
        int c = S.lfirst[j];
#pragma unroll
        for (int q = 0; q < 4; ++q) rec.children[4 * me + q] = (mask & (1u << q)) ? rid(c++) : -1;
      }
    }
    SUBPROF(3)
    // ---- 4. ascending-id lists: radix sort of the member ids (block-wide),
    // then stable partitions level by level into the children's ranges
    {
      constexpr int IPT = kSubMax / kSubThreads;
      unsigned kk[IPT];
      short vv[IPT];
      const unsigned pad = id_bits >= 32 ? 0xffffffffu : ((1u << id_bits) - 1u);
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int k = tid * IPT + u;
        kk[u] = k < m ? (unsigned)S.ids[k] : pad;  // pads sort after every member (stable)
        vv[u] = (short)k;
      }
      __syncthreads();  // keys of the topology phase are dead
      SubIdSort(S.u.sort).Sort(kk, vv, 0, id_bits);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < IPT; ++u)
        if (tid * IPT + u < m) S.u.lists[tid * IPT + u] = vv[u];
    }
    __syncthreads();
    SUBPROF(4)
    for (int L = 0; L + 1 < S.nlvl; ++L) {
      const short* src = S.u.lists + L * m;
      short* dst = S.u.lists + (L + 1) * m;
      for (int j = S.lvl_start[L] + warp; j < S.lvl_start[L + 1]; j += nwarp) {
        if (!S.lsplit[j]) continue;
        const unsigned mask = S.lmask[j];
        int rs1 = 0, rs2 = 0, rs3 = 0, cb[4];
        {
          int c = S.lfirst[j], cur = S.lb[j];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            cb[q] = cur;
            if (mask & (1u << q)) cur = S.le[c++];
            if (q == 0) rs1 = cur;
            if (q == 1) rs2 = cur;
            if (q == 2) rs3 = cur;
          }
        }
        const int jb = S.lb[j], je = S.le[j];
        for (int t0 = jb; t0 < je; t0 += 32) {
          const int t = t0 + lane;
          const bool act = t < je;
          const int k = act ? src[t] : 0;
          const int q = (k >= rs1) + (k >= rs2) + (k >= rs3);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const unsigned bal = __ballot_sync(0xffffffffu, act && q == qq);
            if (act && q == qq) dst[cb[qq] + __popc(bal & ((1u << lane) - 1u))] = (short)k;
            cb[qq] += __popc(bal);
          }
        }
      }
      __syncthreads();
    }
    SUBPROF(5)
    // ---- 5. finish_node chains over the ascending lists: a thread per node
    // up to kThreadChain members (the five chains interleaved), lanes 0..4 of
    // a warp above; leaves' members into perm / sx / sy / sg
    for (int j = tid; j < nloc; j += kSubThreads) {
      const int jb = S.lb[j], je = S.le[j];
      if (je - jb > kThreadChain) continue;
      const short* l = S.u.lists + S.ldep[j] * m;
      const bool leaf = !S.lsplit[j];
      double gs = 0.0, wx = 0.0, wy = 0.0, plx = 0.0, ply = 0.0;
#pragma unroll 4
      for (int t = jb; t < je; ++t) {
        const int k = l[t];
        const double g = S.g[k], x = S.x[k], y = S.y[k];
        gs = __dadd_rn(gs, g);
        wx = __dadd_rn(wx, __dmul_rn(g, x));
        wy = __dadd_rn(wy, __dmul_rn(g, y));
        plx = __dadd_rn(plx, x);
        ply = __dadd_rn(ply, y);
        if (leaf) {
          perm[b + t] = S.ids[k];
          sx[b + t] = x;
          sy[b + t] = y;
          sg[b + t] = g;
        }
      }
      finish_exact(rec, rid(j), b + jb, b + je, gs, wx, wy, plx, ply);
      if (j == 0) {  // subtree root: raw sums for the large nodes above
        aux[8 * r] = gs;
        aux[8 * r + 1] = wx;
        aux[8 * r + 2] = wy;
        aux[8 * r + 3] = plx;
        aux[8 * r + 4] = ply;
      }
    }
    {
      const double* A = lane == 3 ? S.x : lane == 4 ? S.y : S.g;
      const double* B = lane == 1 ? S.x : lane == 2 ? S.y : nullptr;
      for (int j = warp; j < nloc; j += nwarp) {
        const int jb = S.lb[j], je = S.le[j];
        if (je - jb <= kThreadChain) continue;
        const short* l = S.u.lists + S.ldep[j] * m;
        double acc = 0.0;
        if (lane < 5) {
          int t = jb;
          for (; t + 8 <= je; t += 8) {
            double a8[8], b8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int k = l[t + u];
              a8[u] = A[k];
              b8[u] = B ? B[k] : 1.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(a8[u], b8[u]));
          }
          for (; t < je; ++t) {
            const int k = l[t];
            acc = __dadd_rn(acc, __dmul_rn(A[k], B ? B[k] : 1.0));
          }
        }
        const double gs = __shfl_sync(0xffffffffu, acc, 0), wx = __shfl_sync(0xffffffffu, acc, 1),
                     wy = __shfl_sync(0xffffffffu, acc, 2), plx = __shfl_sync(0xffffffffu, acc, 3),
                     ply = __shfl_sync(0xffffffffu, acc, 4);
        if (lane == 0) {
          finish_exact(rec, rid(j), b + jb, b + je, gs, wx, wy, plx, ply);
          if (j == 0) {
            aux[8 * r] = gs;
            aux[8 * r + 1] = wx;
            aux[8 * r + 2] = wy;
            aux[8 * r + 3] = plx;
            aux[8 * r + 4] = ply;
          }
        }
      }
    }
    __syncthreads();
    SUBPROF(6)
    // Σ|Γ|, Σ|Γx|, Σ|Γy| of the subtree (any fixed order: they only bound
    // the rounding of the large nodes' sums)
    {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int k = tid; k < m; k += kSubThreads) {
        const double g = S.g[k];
        a0 += fabs(g);
        a1 += fabs(__dmul_rn(g, S.x[k]));
        a2 += fabs(__dmul_rn(g, S.y[k]));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        a0 += __shfl_down_sync(0xffffffffu, a0, off);
        a1 += __shfl_down_sync(0xffffffffu, a1, off);
        a2 += __shfl_down_sync(0xffffffffu, a2, off);
      }
      if (lane == 0) {
        s_abs[warp][0] = a0;
        s_abs[warp][1] = a1;
        s_abs[warp][2] = a2;
      }
      __syncthreads();
      if (tid < 3) {
        double t = 0.0;
        for (int w = 0; w < nwarp; ++w) t += s_abs[w][tid];
        aux[8 * r + 5 + tid] = t;
      }
      __syncthreads();
    }
    SUBPROF(7)
    if (prof && tid == 0) {
      prof[(long long)si * 10 + 8] = m;
      prof[(long long)si * 10 + 9] = (long long)S.nloc * 100 + S.nlvl;
    }
  }
#undef SUBPROF
}

// Large nodes (> seq_max members) bottom-up from their children's raw sums,
// one CTA, deepest large level first. Any summation order is within
// (m-1)u·Σ|a| of the exact sum, as is the reference's sequential order, so the
// node carries the same certified centroid bound as large_sums_kernel.
__global__ void __launch_bounds__(1024) morton_large_kernel(TreeRecords rec, const MortonState* __restrict__ st,
                                                            int seq_max, double* __restrict__ aux) {
  __shared__ int base[kMaxDepth + 3];
  if (st->overflow || !st->finite) return;
  if (threadIdx.x == 0) {
    base[0] = 0;
    for (int d = 0; d <= kMaxDepth + 1; ++d) base[d + 1] = base[d] + st->lvl_cnt[d];
  }
  __syncthreads();
  for (int d = st->levels_used - 1; d >= 0; --d) {
    for (int r = base[d] + threadIdx.x; r < base[d + 1]; r += blockDim.x) {
      const int b = rec.begin[r], e = rec.end[r];
      if (e - b <= seq_max) continue;
      double red[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = 0; q < 4; ++q) {
        const int c = rec.children[4 * r + q];
        if (c < 0) continue;
        for (int k = 0; k < 8; ++k) red[k] = __dadd_rn(red[k], aux[8 * c + k]);
      }
      for (int k = 0; k < 8; ++k) aux[8 * r + k] = red[k];
      finish_certified(rec, r, b, e, red);
    }
    __syncthreads();
  }
}

}  // namespace

// Returns false (nothing built) when the Morton path does not apply or
// overflowed; the caller then runs the level build.
int tree_build_morton_levels(ptrom_ctx* ctx, Tree& t, long long leaf_cap, int seq_max, const int levels);
bool tree_build_morton(ptrom_ctx* ctx, Tree& t, long long leaf_cap, int seq_max) {
  const long long n = t.n;
  // leaf_capacity < 4 gives subtrees with more local nodes than a CTA holds
  // (kSubNodes): the level build, without a wasted attempt
  if (leaf_cap > 32 || leaf_cap < 4 || seq_max > kSubMax || seq_max < leaf_cap) return false;
  // key depth: the uniform-density depth plus a margin (fewer radix passes);
  // a tree that needs more levels is rebuilt once with all 32
  int lg4 = 0;
  while (lg4 < kMortonLevels && (1LL << (2 * lg4)) * leaf_cap < n) ++lg4;
  const int levels = std::min(kMortonLevels, std::max(8, lg4 + 8));
  const int r = tree_build_morton_levels(ctx, t, leaf_cap, seq_max, levels);
  if (r == 0) return true;
  // only a key-depth overflow can be fixed by more levels; a capacity
  // overflow (subtree nodes, list storage, records) goes to the level build
  return r == 1 && levels < kMortonLevels && tree_build_morton_levels(ctx, t, leaf_cap, seq_max, kMortonLevels) == 0;
}

// 0: built; 1: a split was needed below the key's levels; 2: another capacity overflow.
int tree_build_morton_levels(ptrom_ctx* ctx, Tree& t, long long leaf_cap, int seq_max, const int levels) {
  const long long n = t.n;
  cudaStream_t s = ctx->stream;

  // ---- root (device-side hull finish, no host round trip)
  const int hb = std::min<long long>((n + kThreads - 1) / kThreads, 256);
  double* hull = dalloc<double>(4 * hb);
  hull_kernel<<<hb, kThreads, 0, s>>>(n, t.px, t.py, hull);
  PTROM_LAUNCH_CHECK();
  const long long est = 4 * ((2 * n) / std::max<long long>(1, leaf_cap) + 64);
  const int rec_cap = (int)std::min<long long>(est, INT_MAX / 8);
  TreeRecords rec;
  rec.alloc((size_t)rec_cap);
  MortonState* st = dalloc<MortonState>(1);
  PTROM_CUDA(cudaMemsetAsync(st, 0, sizeof(MortonState), s));
  morton_root_kernel<<<1, 32, 0, s>>>(hb, hull, n, leaf_cap, rec, st);
  PTROM_LAUNCH_CHECK();

  // ---- keys and the stable sort
  unsigned long long *key = dalloc<unsigned long long>(n), *skey = dalloc<unsigned long long>(n);
  int *ids = dalloc<int>(n), *sid = dalloc<int>(n);
  morton_keys_kernel<<<grid_for(ctx, n), kThreads, 0, s>>>(n, t.px, t.py, rec, levels, key, ids);
  PTROM_LAUNCH_CHECK();
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, skey, ids, sid, (int)n, 0, 2 * levels, s);
  void* stmp = dalloc<char>(sort_bytes + 256);
  PTROM_CUDA(cub::DeviceRadixSort::SortPairs(stmp, sort_bytes, key, skey, ids, sid, (int)n, 0, 2 * levels, s));

  // ---- large nodes level by level
  const long long max_large = (long long)(kMaxDepth + 1) * (n / std::max(1, seq_max) + 2);
  const int sub_half = (int)std::min<long long>(rec_cap, 4 * max_large + 4);
  int* sub_list = dalloc<int>(2 * (size_t)sub_half);
  int* large_list = dalloc<int>(max_large);
  {
    int occ = 0;
    PTROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, morton_levels_kernel, kThreads, 0));
    // few large nodes per level: a small grid keeps the grid barrier cheap
    const int grid = std::min(ctx->num_sms * std::max(1, occ), 32);
    void* args[] = {(void*)&skey, (void*)&levels, (void*)&leaf_cap, (void*)&seq_max, (void*)&rec,
                    (void*)&rec_cap, (void*)&st, (void*)&sub_list, (void*)&sub_half, (void*)&large_list};
    PTROM_CUDA(cudaLaunchCooperativeKernel((void*)morton_levels_kernel, grid, kThreads, args, 0, s));
  }
  double* aux = nullptr;
  MortonState* h_st = reinterpret_cast<MortonState*>(ctx->h_counts);
  static_assert(sizeof(MortonState) <= 512, "pinned scratch");
  auto read_state = [&]() {
    PTROM_CUDA(cudaMemcpyAsync(h_st, st, sizeof(MortonState), cudaMemcpyDeviceToHost, s));
    PTROM_CUDA(cudaStreamSynchronize(s));
    return *h_st;
  };
  auto release = [&]() {
    void* frees[] = {hull, st, key, skey, ids, sid, stmp, sub_list, large_list, aux};
    for (void* p : frees) dfree(p);
  };

  // ---- subtrees of at most seq_max members: topology, leaf order, exact
  // sums (no host round trip: the kernels read the level counts on the device)
  int* perm = dalloc<int>(n);
  double *sx = dalloc<double>(n), *sy = dalloc<double>(n), *sg = dalloc<double>(n);
  aux = dalloc<double>(8 * (size_t)rec_cap);  // raw sums of the subtree roots and large nodes
  {
    // per call: the attribute belongs to the current device's context
    PTROM_CUDA(cudaFuncSetAttribute(morton_subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(SubSmem)));
    const int nb = ctx->num_sms * 2;
    int id_bits = 1;
    while (id_bits < 31 && (1LL << id_bits) <= n) ++id_bits;
    // PTROM_SUBTREE_PROFILE=<csv path>: per-subtree phase clocks (tools/, not the product path)
    static const char* sub_prof_path = std::getenv("PTROM_SUBTREE_PROFILE");
    const bool sub_prof = sub_prof_path != nullptr;
    const int max_sub = (int)std::min<long long>(rec_cap, 4 * max_large + 4);
    long long* prof = sub_prof ? dalloc<long long>((size_t)max_sub * 10) : nullptr;
    morton_subtree_kernel<<<nb, kSubThreads, sizeof(SubSmem), s>>>(skey, sid, t.px, t.py, t.g, sub_list, sub_half, st, rec,
                                                                   rec_cap, levels, leaf_cap, id_bits, perm,
                                                                   sx, sy, sg, aux, prof);
    PTROM_LAUNCH_CHECK();
    if (prof) {
      const MortonState h1 = read_state();
      std::vector<long long> hp((size_t)h1.sub_count * 10);
      PTROM_CUDA(cudaMemcpyAsync(hp.data(), prof, hp.size() * 8, cudaMemcpyDeviceToHost, s));
      PTROM_CUDA(cudaStreamSynchronize(s));
      if (FILE* f = std::fopen(sub_prof_path, "w")) {
        for (int i = 0; i < h1.sub_count; ++i) {
          for (int k = 0; k < 10; ++k) std::fprintf(f, "%lld%c", hp[10 * i + k], k == 9 ? '\n' : ',');
        }
        std::fclose(f);
      }
      dfree(prof);
    }
  }
  morton_large_kernel<<<1, 1024, 0, s>>>(rec, st, seq_max, aux);
  PTROM_LAUNCH_CHECK();
  const MortonState hs = read_state();
  if (!hs.finite) {
    dfree(perm);
    dfree(sx);
    dfree(sy);
    dfree(sg);
    release();
    rec.free();
    config_fail("build_tree: non-finite input");
  }
  if (hs.overflow) {
    dfree(perm);
    dfree(sx);
    dfree(sy);
    dfree(sg);
    release();
    rec.free();
    return hs.overflow_depth ? 1 : 2;
  }
  int R = hs.rec_extra;
  for (int d = 0; d <= kMaxDepth + 1; ++d) R += hs.lvl_cnt[d];
  t.root_width = hs.width;
  finish_tree(ctx, t, rec, R, perm, sx, sy, sg);
  ctx->tree_stats.levels = hs.levels_used;
  release();
  rec.free();
  return 0;
}

// Computes exact sums for nodes flagged need_exact; returns how many.
int tree_resolve_uncertain(ptrom_ctx* ctx, Tree& t, const int* d_flag_count) {
  int h = 0;
  PTROM_CUDA(cudaMemcpyAsync(&h, d_flag_count, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PTROM_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h == 0) return 0;
  const int R = (int)t.nodes.count;
  exact_sums_kernel<<<(R + 127) / 128, 128, 0, ctx->stream>>>(R, t.n, t.nodes, t.slot, t.px, t.py, t.g);
  PTROM_LAUNCH_CHECK();
  return h;
}

}  // namespace ptrom
