// tm_traverse.cu -- K3: seed-parallel region boundary walks into a CSR polygon
// array.  Replaces traversal.build_polygon_mesh (traversal.py:303-347), the
// start-edge rule (traversal.py:325-330 + find_start_frontier 172-192) and the
// numba walk kernels _advance / _walk_lengths / _walk_write (242-300).
//
// Output order is ascending seed order with a count -> exclusive scan -> write
// layout, which reproduces the reference's SEQUENTIAL `mesh`/`positions` byte
// for byte instead of the paper's unordered AtomicAdd append.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

constexpr int kBfsCap = 48;

// Start half-edge of a seed (traversal.py:325-330): the smallest frontier slot
// of t, else the FIFO BFS of find_start_frontier (172-192) across non-frontier
// edges, slots 0,1,2 in order.  The BFS queue doubles as the seen set (every
// triangle is enqueued exactly when first seen).  Returns -2 on local overflow.
__device__ int32_t seed_start(const int32_t* __restrict__ hw, int32_t t) {
  int32_t h = min_frontier_slot(hw, t);
  if (h >= 0) return h;
  int32_t q[kBfsCap];
  int head = 0, tail = 1;
  q[0] = t;
  while (head < tail) {
    int32_t u = q[head++];
    for (int j = 0; j < 3; j++) {
      int32_t w = hw[3 * u + j];
      if (hw_front(w)) return 3 * u + j;
      int32_t nt = hw_twin(w) / 3;  // non-frontier => interior => twin exists
      bool seen = false;
      for (int i = 0; i < tail; i++) seen |= (q[i] == nt);
      if (!seen) {
        if (tail == kBfsCap) return -2;
        q[tail++] = nt;
      }
    }
  }
  return -1;
}

__global__ void __launch_bounds__(256) k_trav_start(const int32_t* __restrict__ hw, const int32_t* __restrict__ seeds,
                                                    int64_t P, int32_t* __restrict__ start,
                                                    int32_t* __restrict__ overflow, unsigned int* n_overflow,
                                                    DevStatus* st) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t t = seeds[i];
    int32_t h = seed_start(hw, t);
    if (h == -2) overflow[atomicAdd(n_overflow, 1u)] = (int32_t)i;
    else if (h < 0) report(st, K_NO_FRONTIER, t);
    start[i] = h;
  }
}

// Slow path for BFS regions larger than the register queue: one thread, a
// global FIFO and a stamp array for the seen set.  Rare (max 17 visited at 10M).
__global__ void k_bfs_slow(const int32_t* __restrict__ hw, const int32_t* __restrict__ seeds,
                           int32_t* __restrict__ start, const int32_t* __restrict__ overflow,
                           const unsigned int* n_overflow, int32_t* __restrict__ queue, int32_t* __restrict__ stamp,
                           DevStatus* st) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned int no = *n_overflow;
  for (unsigned int k = 0; k < no; k++) {
    int32_t i = overflow[k], t = seeds[i], res = -1;
    int64_t head = 0, tail = 1;
    queue[0] = t;
    stamp[t] = (int32_t)k;
    while (head < tail && res < 0) {
      int32_t u = queue[head++];
      for (int j = 0; j < 3; j++) {
        int32_t w = hw[3 * u + j];
        if (hw_front(w)) { res = 3 * u + j; break; }
        int32_t nt = hw_twin(w) / 3;
        if (stamp[nt] != (int32_t)k) { stamp[nt] = (int32_t)k; queue[tail++] = nt; }
      }
    }
    if (res < 0) report(st, K_NO_FRONTIER, t);
    start[i] = res;
  }
}

__global__ void __launch_bounds__(256) k_trav_len(const int32_t* __restrict__ hw, const int32_t* __restrict__ seeds,
                                                  const int32_t* __restrict__ start, int64_t P, long long limit,
                                                  int64_t* __restrict__ len, DevStatus* st) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t h0 = start[i], h = h0;
    long long n = 0;
    if (h0 >= 0) {
      for (;;) {
        if (++n > limit) { n = -1; break; }
        h = walk_next(hw, h, limit);
        if (h < 0) { n = -1; break; }
        if (h == h0) break;
      }
      if (n < 0) report(st, K_WALK, seeds[i]);
    }
    len[i] = n > 0 ? n : 0;
  }
}

__global__ void __launch_bounds__(256) k_trav_write(const int32_t* __restrict__ tri, const int32_t* __restrict__ hw,
                                                    const int32_t* __restrict__ start, int64_t P, long long limit,
                                                    const int64_t* __restrict__ offsets, int32_t* __restrict__ verts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = offsets[i], end = offsets[i + 1];
    int32_t h0 = start[i], h = h0;
    if (h0 < 0 || end == w) continue;
    do {
      verts[w++] = he_origin(tri, h);
      h = walk_next(hw, h, limit);
    } while (h != h0 && h >= 0 && w < end);
  }
}

static inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

size_t select_seeds_temp_bytes(int64_t T) {
  size_t bytes = 0;
  thrust::counting_iterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, bytes, it, (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr, (int)T);
  return bytes;
}

void launch_select_seeds(const uint8_t* seed, int64_t T, int32_t* seeds, int64_t* n_seeds, void* temp, size_t temp_bytes,
                         cudaStream_t s) {
  thrust::counting_iterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(temp, temp_bytes, it, seed, seeds, n_seeds, (int)T, s);
}

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)n);
  return bytes;
}

void launch_scan(const int64_t* in, int64_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, s);
}

void launch_trav_start(const int32_t* hw, const int32_t* seeds, int64_t P, int32_t* start, int32_t* overflow,
                       unsigned int* n_overflow, int32_t* queue, int32_t* stamp, DevStatus* st, cudaStream_t s) {
  if (P <= 0) return;
  k_trav_start<<<grid_for(P, 256), 256, 0, s>>>(hw, seeds, P, start, overflow, n_overflow, st);
  note_launch(1);
  k_bfs_slow<<<1, 32, 0, s>>>(hw, seeds, start, overflow, n_overflow, queue, stamp, st);
  note_launch(1);
}

void launch_trav_len(const int32_t* hw, const int32_t* seeds, const int32_t* start, int64_t P, int64_t T,
                     int64_t* len, DevStatus* st, cudaStream_t s) {
  if (P <= 0) return;
  k_trav_len<<<grid_for(P, 256), 256, 0, s>>>(hw, seeds, start, P, 3 * T + 3, len, st);
  note_launch(1);
}

void launch_trav_write(const int32_t* tri, const int32_t* hw, const int32_t* start, int64_t P, int64_t T,
                       const int64_t* offsets, int32_t* verts, cudaStream_t s) {
  if (P <= 0) return;
  k_trav_write<<<grid_for(P, 256), 256, 0, s>>>(tri, hw, start, P, 3 * T + 3, offsets, verts);
  note_launch(1);
}

}  // namespace tmb
