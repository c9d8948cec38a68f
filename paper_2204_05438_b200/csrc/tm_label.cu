// tm_label.cu -- K0 (half-edge twin build) fused with K1 (LabelMax) and K2
// (LabelSeed + LabelFrontier).
//
// Replaces: mesh_core.compute_trivertex (mesh_core.py:171-178), the neighbor
// back-slot searches of labeling.py:84,110, and labeling.label_max /
// label_seeds / label_frontiers (labeling.py:46-115).  The reference receives
// `neighbors` from Qhull; here adjacency is derived from the triangle list.
//
// Pass A (per triangle, HBM-bound gather): corners -> tri32, three fp64 squared
//   lengths computed UNFUSED (__dmul_rn/__dadd_rn; numpy's ((b-c)**2).sum is
//   dx*dx + dy*dy with two roundings), first-max argmax -> max_edge;
//   signed-area validation; atomicMin trivertex; and insertion of the three
//   undirected edge keys into an open-addressing hash table of int32 half-edge
//   ids (linear probing, load <= 0.5).  The second arrival of a key claims the
//   slot with a MATCHED bit and writes both twins.  A third arrival is an
//   edge shared by >2 triangles (validate's "edge_count"); equal direction is a
//   reciprocity/orientation defect.
// Pass B (per triangle): frontier / seed from max_edge of both sides, written
//   as packed words hw = (twin << 1) | frontier (in place over the twin array).
#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint32_t kMatched = 0x80000000u;

__device__ __forceinline__ uint64_t mix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ double sqlen(double2 p, double2 q) {
  double dx = __dsub_rn(p.x, q.x);
  double dy = __dsub_rn(p.y, q.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// numpy argmax over (l0, l1, l2): first NaN wins, otherwise the first maximum.
__device__ __forceinline__ int argmax3(double l0, double l1, double l2) {
  if (isnan(l0)) return 0;
  double best = l0;
  int m = 0;
  if (!(l1 <= best)) {
    best = l1;
    m = 1;
    if (isnan(best)) return 1;
  }
  if (!(l2 <= best)) m = 2;
  return m;
}

template <typename TI>
__device__ __forceinline__ int32_t corner(const TI* tri, int64_t s) { return (int32_t)__ldg(tri + s); }

template <typename TI>
__device__ __forceinline__ void insert_edge(const TI* __restrict__ tri, uint32_t* __restrict__ slots,
                                            uint64_t cap, int32_t* __restrict__ twin, DevStatus* st,
                                            int32_t h, int32_t o, int32_t g) {
  uint32_t lo = (uint32_t)min(o, g), hi = (uint32_t)max(o, g);
  uint64_t key = ((uint64_t)lo << 32) | hi;
  uint64_t i = __umul64hi(mix64(key), cap);
  for (uint64_t probe = 0; probe < cap; probe++) {
    uint32_t cur = slots[i];
    if (cur == kEmpty) {
      uint32_t prev = atomicCAS(slots + i, kEmpty, (uint32_t)h);
      if (prev == kEmpty) return;
      cur = prev;
    }
    int32_t hc = (int32_t)(cur & ~kMatched);
    int64_t tc = hc / 3, jc = hc % 3;
    int32_t oc = corner(tri, 3 * tc + (jc + 1) % 3);
    int32_t gc = corner(tri, 3 * tc + (jc + 2) % 3);
    if ((uint32_t)min(oc, gc) == lo && (uint32_t)max(oc, gc) == hi) {
      if (cur & kMatched) { report(st, K_EDGE_COUNT, h / 3); return; }
      if (oc != g || gc != o) { report(st, K_RECIPROCITY, h / 3); return; }
      uint32_t prev = atomicCAS(slots + i, cur, cur | kMatched);
      if (prev != cur) { report(st, K_EDGE_COUNT, h / 3); return; }
      twin[h] = hc;
      twin[hc] = h;
      return;
    }
    i = (i + 1 == cap) ? 0 : i + 1;
  }
  report(st, K_STRUCT, h / 3);  // table full: impossible at load <= 0.5
}

template <typename TI>
__global__ void __launch_bounds__(256) k_tri_pass(const double2* __restrict__ xy, int64_t n,
                                                  const TI* __restrict__ tri, int64_t T,
                                                  int32_t* __restrict__ tri32, int8_t* __restrict__ max_edge,
                                                  uint32_t* __restrict__ slots, uint64_t cap,
                                                  int32_t* __restrict__ twin, int32_t* __restrict__ tv,
                                                  int check, DevStatus* st) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = (int64_t)__ldg(tri + 3 * t), b = (int64_t)__ldg(tri + 3 * t + 1), c = (int64_t)__ldg(tri + 3 * t + 2);
    if (a < 0 || a >= n || b < 0 || b >= n || c < 0 || c >= n) {
      report(st, K_INDEX_RANGE, t);
      max_edge[t] = 0;
      continue;
    }
    if (tri32 != nullptr) {
      tri32[3 * t] = (int32_t)a;
      tri32[3 * t + 1] = (int32_t)b;
      tri32[3 * t + 2] = (int32_t)c;
    }
    double2 pa = xy[a], pb = xy[b], pc = xy[c];
    // labeling.py:55-59: edge 0 joins corners 1-2, edge 1 joins 2-0, edge 2 joins 0-1
    max_edge[t] = (int8_t)argmax3(sqlen(pb, pc), sqlen(pc, pa), sqlen(pa, pb));
    if (check) {
      // mesh_core.signed_areas (160-168), sign only, unfused
      double d = __dsub_rn(__dmul_rn(__dsub_rn(pb.x, pa.x), __dsub_rn(pc.y, pa.y)),
                           __dmul_rn(__dsub_rn(pb.y, pa.y), __dsub_rn(pc.x, pa.x)));
      if (d < 0.0) report(st, K_ORIENTATION, t);
      else if (d == 0.0) report(st, K_DEGENERATE, t);
    }
    atomicMin(tv + a, (int32_t)t);
    atomicMin(tv + b, (int32_t)t);
    atomicMin(tv + c, (int32_t)t);
    int32_t h = (int32_t)(3 * t);
    insert_edge(tri, slots, cap, twin, st, h + 0, (int32_t)b, (int32_t)c);
    insert_edge(tri, slots, cap, twin, st, h + 1, (int32_t)c, (int32_t)a);
    insert_edge(tri, slots, cap, twin, st, h + 2, (int32_t)a, (int32_t)b);
  }
}

// labeling.py:65-115 fused.  k = twin % 3 replaces the back-slot search.
// `packed` = 0: hw holds raw twins (-1 border) from the pass-A build;
// `packed` = 1: hw already holds packed words (relabel with a new max_edge).
__global__ void __launch_bounds__(256) k_label_edges(const int8_t* __restrict__ max_edge, int64_t T,
                                                     int32_t* __restrict__ hw, uint8_t* __restrict__ seed,
                                                     int packed) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int me = max_edge[t];
    uint8_t s = 0;
#pragma unroll
    for (int j = 0; j < 3; j++) {
      int32_t w = hw[3 * t + j];
      if (packed) w = hw_twin(w);
      int32_t out;
      if (w < 0) {
        out = -1;                // border: frontier, twin -1
        if (j == me) s = 1;      // border terminal edge -> seed
      } else {
        int32_t nt = w / 3, k = w - 3 * nt;
        int mn = __ldg(max_edge + nt);
        bool fr = (me != j) && (mn != k);
        out = (w << 1) | (fr ? 1 : 0);
        if (j == me && mn == k && t < nt) s = 1;
      }
      hw[3 * t + j] = out;
    }
    seed[t] = s;
  }
}

__global__ void k_trivertex_fix(int32_t* tv, int64_t n) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if (tv[v] == 0x7F7F7F7F) tv[v] = -1;
}

// Compare a caller-supplied neighbor array (reference layout, -1 border)
// against the twin build: neighbors[h] == twin[h] // 3.
template <typename TI>
__global__ void k_check_neighbors(const int32_t* __restrict__ hw, const TI* __restrict__ nb, int64_t H, DevStatus* st) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < H; h += (int64_t)gridDim.x * blockDim.x) {
    int32_t tw = hw_twin(hw[h]);
    int64_t expect = tw < 0 ? -1 : tw / 3;
    if ((int64_t)nb[h] != expect) report(st, K_NEIGHBORS, h / 3);
  }
}

__global__ void k_unpack(const int32_t* __restrict__ hw, int64_t H, int32_t* __restrict__ twin, uint8_t* __restrict__ fr) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < H; h += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = hw[h];
    if (twin) twin[h] = hw_twin(w);
    if (fr) fr[h] = hw_front(w) ? 1 : 0;
  }
}

__global__ void k_pack_frontier(int32_t* __restrict__ hw, int64_t H, const uint8_t* __restrict__ fr) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < H; h += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = hw[h];
    hw[h] = (w & ~1) | (fr[h] ? 1 : 0);
  }
}

static inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

uint64_t hash_capacity(int64_t T) {
  // at most 3T/2 + border distinct keys; capacity 3T keeps the load <= 0.5
  uint64_t c = (uint64_t)(3 * T);
  return c < 64 ? 64 : c;
}

void launch_label_a(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int check,
                    int32_t* tri32, int32_t* hw, int8_t* max_edge, int32_t* tv, uint32_t* slots, uint64_t cap,
                    DevStatus* st, cudaStream_t s) {
  cudaMemsetAsync(slots, 0xFF, cap * sizeof(uint32_t), s);
  cudaMemsetAsync(hw, 0xFF, (size_t)(3 * T) * sizeof(int32_t), s);
  if (n > 0) {
    // sentinel 0x7F7F7F7F (> any triangle index), mapped to -1 after the atomicMin pass
    cudaMemsetAsync(tv, 0x7F, (size_t)n * sizeof(int32_t), s);
  }
  if (T > 0) {
    const int B = 256;
    if (tri_is64)
      k_tri_pass<int64_t><<<grid_for(T, B), B, 0, s>>>((const double2*)xy, n, (const int64_t*)tri, T, tri32, max_edge,
                                                       slots, cap, hw, tv, check, st);
    else
      k_tri_pass<int32_t><<<grid_for(T, B), B, 0, s>>>((const double2*)xy, n, (const int32_t*)tri, T,
                                                       tri32 == tri ? nullptr : tri32, max_edge, slots, cap, hw, tv,
                                                       check, st);
    note_launch(1);
  }
}

void launch_label_b(int64_t n, int64_t T, int32_t* hw, const int8_t* max_edge, uint8_t* seed, int32_t* tv,
                    cudaStream_t s) {
  if (T > 0) {
    k_label_edges<<<grid_for(T, 256), 256, 0, s>>>(max_edge, T, hw, seed, 0);
    note_launch(1);
  }
  if (n > 0) {
    k_trivertex_fix<<<grid_for(n, 256), 256, 0, s>>>(tv, n);
    note_launch(1);
  }
}

void launch_relabel(const int8_t* max_edge, int64_t T, int32_t* hw, uint8_t* seed, cudaStream_t s) {
  if (T > 0) k_label_edges<<<grid_for(T, 256), 256, 0, s>>>(max_edge, T, hw, seed, 1), note_launch(1);
}

void launch_check_neighbors(const int32_t* hw, const void* nb, int nb_is64, int64_t T, DevStatus* st, cudaStream_t s) {
  if (T <= 0) return;
  if (nb_is64)
    k_check_neighbors<int64_t><<<grid_for(3 * T, 256), 256, 0, s>>>(hw, (const int64_t*)nb, 3 * T, st);
  else
    k_check_neighbors<int32_t><<<grid_for(3 * T, 256), 256, 0, s>>>(hw, (const int32_t*)nb, 3 * T, st);
}

void launch_unpack(const int32_t* hw, int64_t T, int32_t* twin, uint8_t* fr, cudaStream_t s) {
  if (T > 0) k_unpack<<<grid_for(3 * T, 256), 256, 0, s>>>(hw, 3 * T, twin, fr);
}

void launch_pack_frontier(int32_t* hw, int64_t T, const uint8_t* fr, cudaStream_t s) {
  if (T > 0) k_pack_frontier<<<grid_for(3 * T, 256), 256, 0, s>>>(hw, 3 * T, fr);
}

}  // namespace tmb
