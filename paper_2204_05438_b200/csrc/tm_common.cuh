// tm_common.cuh -- device-side half-edge algebra and status reporting shared by
// the sm_100a kernels of the mesh -> polygons path.
//
// Half-edge convention (reference mesh_core.py:1-14, 104-129): h = 3t + j is the
// edge of triangle t opposite corner j; origin = corner (j+1)%3, target =
// corner (j+2)%3, interior on the left (CCW triangles).
//
// Device layout:
//   xy        double2[n]            vertex coordinates
//   tri       int32[3T]             corners
//   hw        int32[3T]             packed half-edge word: (twin << 1) | frontier.
//                                   Border half-edges hold -1 (twin -1, frontier 1).
//                                   One dependent 4-byte load per rotation step.
//   max_edge  int8[T]               longest-edge slot (labeling.py:46-62)
//   seed      uint8[T]              seed flag (labeling.py:65-89)
//   trivertex int32[n]              lowest incident triangle (mesh_core.py:171-178)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmb {

constexpr int kNumSMs = 148;

// ---- defect / error kinds (first eight mirror mesh_core.ValidationReport kinds)
enum Kind : int {
  K_INDEX_RANGE = 0,
  K_ORIENTATION = 1,
  K_DEGENERATE = 2,
  K_DUPLICATE = 3,
  K_RECIPROCITY = 4,
  K_EDGE_COUNT = 5,
  K_TRIVERTEX = 6,
  K_NEIGHBORS = 7,         // caller-supplied neighbors disagree with the twin build
  K_WALK = 8,              // boundary walk did not terminate (traversal.py:337-341)
  K_NO_FRONTIER = 9,       // BFS found no frontier edge (traversal.py:192)
  K_NO_CONVERGE = 10,      // tip removal did not converge (reparation.py:361-364)
  K_SPLIT_LAW = 11,        // strict split broke |pa|+|pb| == |P|+2 (reparation.py:221-225)
  K_POOL = 12,             // repair scratch pool exhausted (capacity, retried by host)
  K_BARRIER = 13,          // barrier edge not found around tip (reparation.py:137-139)
  K_NO_INTERNAL = 14,      // tip vertex has no internal edge (reparation.py:143-144)
  K_STRUCT = 15,           // other structural failure (fan does not close, border promotion ...)
  K_NUM = 16
};

struct DevStatus {
  unsigned long long first[K_NUM];  // smallest element index reporting this kind
  unsigned int count[K_NUM];
};

__device__ __forceinline__ void report(DevStatus* st, int kind, long long idx) {
  atomicAdd(&st->count[kind], 1u);
  atomicMin(&st->first[kind], (unsigned long long)idx);
}

// ---- half-edge algebra
__device__ __forceinline__ int32_t he_next(int32_t h) { return (h % 3 == 2) ? h - 2 : h + 1; }
__device__ __forceinline__ int32_t he_prev(int32_t h) { return (h % 3 == 0) ? h + 2 : h - 1; }
__device__ __forceinline__ int32_t he_origin(const int32_t* __restrict__ tri, int32_t h) { return __ldg(tri + he_next(h)); }
__device__ __forceinline__ int32_t he_target(const int32_t* __restrict__ tri, int32_t h) { return __ldg(tri + he_prev(h)); }

__device__ __forceinline__ int32_t hw_twin(int32_t w) { return w >> 1; }     // -1 for border
__device__ __forceinline__ bool hw_front(int32_t w) { return (w & 1) != 0; }

// Boundary successor (traversal.py:195-217 / _advance 242-261): from frontier
// half-edge h rotate clockwise around target(h) across non-frontier edges to the
// next frontier half-edge.  One dependent load of the packed word per crossing.
// Returns -1 if the rotation exceeds `limit` crossings.
__device__ __forceinline__ int32_t walk_next(const int32_t* hw, int32_t h, long long limit) {
  int32_t c = he_next(h);
  int32_t w = hw[c];
  long long spins = 0;
  while (!hw_front(w)) {
    c = he_next(hw_twin(w));
    w = hw[c];
    if (++spins > limit) return -1;
  }
  return c;
}

// smallest-slot frontier half-edge of triangle t, or -1
__device__ __forceinline__ int32_t min_frontier_slot(const int32_t* hw, int32_t t) {
  int32_t b = 3 * t;
  if (hw_front(hw[b])) return b;
  if (hw_front(hw[b + 1])) return b + 1;
  if (hw_front(hw[b + 2])) return b + 2;
  return -1;
}

// ---- fans (reparation.py:82-124).  rot_ccw(h) = twin(prev(h)); rot_cw(h) = next(twin(h)).
__device__ __forceinline__ int32_t rot_ccw(const int32_t* hw, int32_t h) { return hw_twin(hw[he_prev(h)]); }
__device__ __forceinline__ int32_t rot_cw(const int32_t* hw, int32_t h) {
  int32_t w = hw_twin(hw[h]);
  return w < 0 ? -1 : he_next(w);
}

// Cyclic successor in the reference fan order (_fan_around: the CCW ring from g0
// followed by the reversed CW run), which is CCW rotation with a wrap from the
// CCW-most half-edge to the CW-most one across a border gap.  Independent of g0.
__device__ __forceinline__ int32_t fan_step(const int32_t* hw, int32_t g, int guard) {
  int32_t w = rot_ccw(hw, g);
  if (w >= 0) return w;
  int32_t c = g;
  for (int i = 0; i < guard; i++) {
    int32_t d = rot_cw(hw, c);
    if (d < 0) return c;
    c = d;
  }
  return -1;
}

// Half-edge of triangle t with origin v (reparation.py:74-79), -1 if none.
__device__ __forceinline__ int32_t he_with_origin(const int32_t* tri, int32_t t, int32_t v) {
  for (int j = 0; j < 3; j++)
    if (he_origin(tri, 3 * t + j) == v) return 3 * t + j;
  return -1;
}

}  // namespace tmb
