// tm_scan.cu -- device-count scans and stream compaction used between the
// phases, so no host round trip is needed to size a launch (the whole path is
// one CUDA graph).  Three-pass tile scheme: per-tile reduce, single-block scan
// of the tile sums, per-tile scan + scatter.  Element counts are read from
// device memory; the host only supplies an upper bound for the grid.
#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;  // 2048

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T x, T* total) {
  __shared__ T warp_sums[kScanThreads / 32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < kScanThreads / 32 ? warp_sums[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  T r = inc - x + warp_sums[wid];
  __syncthreads();
  return r;
}

// ---- exclusive sum over in[0..n] where element n contributes 0: out[n] = total
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int64_t* __restrict__ in,
                                                              const int64_t* __restrict__ n_dev,
                                                              int64_t* __restrict__ tile_sums) {
  int64_t n = *n_dev;
  int64_t base = (int64_t)blockIdx.x * kTile;
  int64_t s = 0;
  if (base <= n) {
    for (int k = 0; k < kScanItems; k++) {
      int64_t i = base + k * kScanThreads + threadIdx.x;
      if (i < n) s += in[i];
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ int64_t ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; w++) t += ws[w];
    tile_sums[blockIdx.x] = t;
  }
}

// single block: exclusive scan of the tile sums in place (count from n_dev)
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(int64_t* __restrict__ tile_sums,
                                                             const int64_t* __restrict__ n_dev, int64_t extra) {
  int64_t n = (n_dev ? *n_dev : 0) + extra;  // elements covered
  int64_t nt = (n + kTile - 1) / kTile;
  int64_t carry = 0;
  __shared__ int64_t tot;
  for (int64_t b = 0; b < nt; b += kScanThreads) {
    int64_t i = b + threadIdx.x;
    int64_t x = i < nt ? tile_sums[i] : 0;
    int64_t ex = block_exclusive_scan<int64_t>(x, &tot);
    if (i < nt) tile_sums[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_final(const int64_t* __restrict__ in,
                                                             const int64_t* __restrict__ n_dev,
                                                             const int64_t* __restrict__ tile_sums,
                                                             int64_t* __restrict__ out) {
  int64_t n = *n_dev;
  int64_t base = (int64_t)blockIdx.x * kTile;
  if (base > n) return;
  // each thread owns kScanItems consecutive elements
  int64_t first = base + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = first + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  __shared__ int64_t tot;
  int64_t ex = block_exclusive_scan<int64_t>(s, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = first + k;
    if (i <= n) out[i] = ex;
    ex += v[k];
  }
}

// ---- ascending indices base_index + t with flag[t] != 0 (seed compaction), count -> *n_out
__global__ void __launch_bounds__(kScanThreads) k_flag_reduce(const uint8_t* __restrict__ flag, int64_t n,
                                                              int64_t* __restrict__ tile_sums) {
  int64_t base = (int64_t)blockIdx.x * kTile;
  int64_t first = base + (int64_t)threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) s += (first + k < n) ? (flag[first + k] != 0) : 0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ int ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; w++) t += ws[w];
    tile_sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_flag_scatter(const uint8_t* __restrict__ flag, int64_t n,
                                                               const int64_t* __restrict__ tile_sums,
                                                               int32_t* __restrict__ out, int64_t* n_out,
                                                               int64_t base_index) {
  int64_t base = (int64_t)blockIdx.x * kTile;
  int64_t first = base + (int64_t)threadIdx.x * kScanItems;
  uint8_t f[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    f[k] = (first + k < n) ? (flag[first + k] != 0) : 0;
    s += f[k];
  }
  __shared__ int64_t tot;
  int64_t pos = block_exclusive_scan<int64_t>(s, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; k++)
    if (f[k]) out[pos++] = (int32_t)(base_index + first + k);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) *n_out = pos;
}

static inline int tiles_for(int64_t n) { return (int)((n + kTile) / kTile); }  // covers n+1 elements

size_t scan_scratch_elems(int64_t n_cap) { return (size_t)tiles_for(n_cap) + 1; }

void launch_scan_dev(const int64_t* in, int64_t* out, const int64_t* n_dev, int64_t n_cap, int64_t* tile_sums,
                     cudaStream_t s) {
  int nt = tiles_for(n_cap);
  k_scan_reduce<<<nt, kScanThreads, 0, s>>>(in, n_dev, tile_sums);
  k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile_sums, n_dev, 1);
  k_scan_final<<<nt, kScanThreads, 0, s>>>(in, n_dev, tile_sums, out);
  note_launch(3);
}

void launch_select_flags(const uint8_t* flag, int64_t n, int32_t* out, int64_t* n_out, int64_t* tile_sums,
                         cudaStream_t s, int64_t base_index) {
  int nt = (int)((n + kTile - 1) / kTile);
  if (nt < 1) nt = 1;
  k_flag_reduce<<<nt, kScanThreads, 0, s>>>(flag, n, tile_sums);
  k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile_sums, nullptr, n);
  k_flag_scatter<<<nt, kScanThreads, 0, s>>>(flag, n, tile_sums, out, n_out, base_index);
  note_launch(3);
}

__global__ void k_gather_at(const int64_t* __restrict__ arr, const int64_t* __restrict__ idx, int64_t* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *dst = arr[*idx];
}

// *dst = arr[*idx] on the device (no host round trip)
void launch_gather_at(const int64_t* arr, const int64_t* idx, int64_t* dst, cudaStream_t s) {
  k_gather_at<<<1, 32, 0, s>>>(arr, idx, dst);
  note_launch(1);
}

// offsets[i] += delta for i in [0, n] (stitching a rank's CSR into the global one)
__global__ void k_shift(int64_t* __restrict__ a, int64_t n, int64_t delta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] += delta;
}

void launch_shift(int64_t* a, int64_t n, int64_t delta, cudaStream_t s) {
  int64_t g = (n + 1 + 255) / 256;
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  k_shift<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(a, n, delta);
  note_launch(1);
}

}  // namespace tmb
