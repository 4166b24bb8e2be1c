// tree.cuh — device-side quadtree representation (quadtree.hpp:15-47).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace ptrom {

// Build-time node records (level order).
struct TreeRecords {
  size_t cap = 0;
  int *begin = nullptr, *end = nullptr, *depth = nullptr, *children = nullptr;
  unsigned char *split = nullptr, *fallback = nullptr, *exact = nullptr;
  double *bounds = nullptr, *mid = nullptr, *width = nullptr, *centroid = nullptr, *gamma_sum = nullptr,
         *cerr = nullptr;
  void alloc(size_t cap);
  void free();
  void grow(size_t need, size_t used, cudaStream_t s);
};

// Final node table in preorder (the reference's node ids).
struct TreeNodes {
  size_t count = 0;
  double* bounds = nullptr;     // 4 per node: x_min, x_max, y_min, y_max
  double* width = nullptr;
  double* centroid = nullptr;   // 2 per node
  double* gamma_sum = nullptr;
  double* cerr = nullptr;       // centroid error bound vs the reference order (0 when exact)
  int* children = nullptr;      // 4 per node, SW SE NW NE, -1 when empty
  int* begin = nullptr;
  int* end = nullptr;
  int* depth = nullptr;
  int* skip = nullptr;          // preorder successor after this node's subtree
  unsigned char* fallback = nullptr;
  unsigned char* exact = nullptr;       // sums bit-identical to the reference's sequential order
  unsigned char* leaf = nullptr;
  unsigned char* need_exact = nullptr;  // set by traversals hitting an uncertain prune test
  void alloc(size_t nn);
  void free();
};

struct Tree {
  long long n = 0;
  long long leaf_cap = 0;
  double root_width = 0.0;  // node widths are root_width / 2^depth (depth <= 64)
  TreeNodes nodes;
  int* perm = nullptr;       // particle ids grouped by node slices
  int* slot = nullptr;       // perm^-1
  int* leaf_node = nullptr;  // leaf id per particle
  double *sx = nullptr, *sy = nullptr, *sg = nullptr;  // build points / weights in perm order
  double *px = nullptr, *py = nullptr, *g = nullptr;   // build points / weights by particle id
  void free_all(cudaStream_t s);  // stream-ordered release on s
};

}  // namespace ptrom
