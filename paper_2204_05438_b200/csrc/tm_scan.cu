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
  // kScanItems consecutive tile sums per thread: one pass per 2048 tiles, the
  // thread's loads all in flight (one tile per thread per pass cost a dependent
  // load per 256 tiles: 35 us for the 9.8 k tiles of a 20M-triangle selection)
  for (int64_t b = 0; b < nt; b += kTile) {
    const int64_t first = b + (int64_t)threadIdx.x * kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
      v[k] = first + k < nt ? tile_sums[first + k] : 0;
      s += v[k];
    }
    int64_t ex = carry + block_exclusive_scan<int64_t>(s, &tot);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
      if (first + k < nt) tile_sums[first + k] = ex;
      ex += v[k];
    }
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

// ---- single-pass exclusive scan of one or two int64 arrays over in[0..n]
// (element n contributes 0, so out[n] = total; n read from the device),
// decoupled look-back: each tile publishes its aggregate, then its inclusive
// prefix; a tile's warp 0 sums predecessors' aggregates 32 at a time until it
// meets a published prefix.  Tiles are numbered in launch order by an atomic
// counter, so every predecessor is resident or done (no deadlock).
struct ScanTotals {
  int64_t* tot0 = nullptr;     // out0[n]
  int64_t* tot1 = nullptr;     // out1[n]
  int64_t* csr_end = nullptr;  // csr_end[out0[n]] = out1[n] (final CSR offset)
};

struct ScanState {
  unsigned int* counter;  // [1 + ntiles]: tile counter, then per-tile flags (0 none, 1 aggregate, 2 prefix)
  int64_t* agg;           // [2][ntiles] aggregates
  int64_t* pre;           // [2][ntiles] inclusive prefixes
  int64_t ntiles;
};

template <int NV>
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const int64_t* __restrict__ in0,
                                                                const int64_t* __restrict__ in1,
                                                                int64_t* __restrict__ out0, int64_t* __restrict__ out1,
                                                                const int64_t* __restrict__ n_dev, ScanState ss,
                                                                ScanTotals tt) {
  __shared__ unsigned int s_tile;
  __shared__ int64_t s_pre[NV], s_tot[NV];
  const int64_t n = *n_dev;
  // persistent blocks take tiles in counter order until past the data (the grid is
  // sized by a host bound; tiles beyond the data never publish: nobody looks that far)
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(ss.counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kTile;
  if (base > n) break;
  volatile unsigned int* flags = ss.counter + 1;
  const int64_t first = base + (int64_t)threadIdx.x * kScanItems;
  const int64_t* in[2] = {in0, in1};
  int64_t v[NV][kScanItems], ex[NV];
#pragma unroll
  for (int a = 0; a < NV; a++) {
    int64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
      const int64_t i = first + k;
      v[a][k] = i < n ? in[a][i] : 0;
      sum += v[a][k];
    }
    ex[a] = block_exclusive_scan<int64_t>(sum, &s_tot[a]);
  }
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    int64_t tot[NV];
#pragma unroll
    for (int a = 0; a < NV; a++) tot[a] = s_tot[a];
    if (lane == 0) {
#pragma unroll
      for (int a = 0; a < NV; a++) {
        if (tile == 0) ss.pre[a * ss.ntiles] = tot[a];
        else ss.agg[a * ss.ntiles + tile] = tot[a];
      }
      __threadfence();
      flags[tile] = tile == 0 ? 2u : 1u;
    }
    int64_t prefix[NV] = {};
    for (int64_t t_hi = tile - 1; t_hi >= 0; t_hi -= 32) {
      const int64_t idx = t_hi - lane;  // lane 0 = nearest predecessor
      unsigned f = idx >= 0 ? flags[idx] : 2u;
      while (__any_sync(0xffffffffu, f == 0u))
        if (f == 0u) f = flags[idx];
      __threadfence();
      const unsigned done = __ballot_sync(0xffffffffu, f == 2u);
      const int stop = done ? __ffs(done) - 1 : 32;  // nearest predecessor with a prefix
#pragma unroll
      for (int a = 0; a < NV; a++) {
        int64_t x = 0;
        if (idx >= 0 && lane < stop) x = __ldcg(ss.agg + a * ss.ntiles + idx);
        if (idx >= 0 && lane == stop) x = __ldcg(ss.pre + a * ss.ntiles + idx);
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        prefix[a] += x;
      }
      if (done) break;
    }
    if (lane == 0) {
      if (tile > 0) {
#pragma unroll
        for (int a = 0; a < NV; a++) ss.pre[a * ss.ntiles + tile] = prefix[a] + tot[a];
        __threadfence();
        flags[tile] = 2u;
      }
#pragma unroll
      for (int a = 0; a < NV; a++) s_pre[a] = prefix[a];
    }
  }
  __syncthreads();
  int64_t* out[2] = {out0, out1};
  int64_t total[NV];
#pragma unroll
  for (int a = 0; a < NV; a++) {
    int64_t run = s_pre[a] + ex[a];
    total[a] = -1;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
      const int64_t i = first + k;
      if (i <= n) out[a][i] = run;
      if (i == n) total[a] = run;
      run += v[a][k];
    }
  }
  if (total[0] >= 0) {  // the thread holding element n: totals (and the CSR end) without extra launches
    if (tt.tot0) *tt.tot0 = total[0];
    if (NV > 1 && tt.tot1) *tt.tot1 = total[NV - 1];
    if (NV > 1 && tt.csr_end) tt.csr_end[total[0]] = total[NV - 1];
  }
  __syncthreads();  // s_tile / s_pre / s_tot are reused by the next tile
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

size_t scan_lookback_bytes(int64_t n_cap) {
  const int64_t nt = n_cap / kTile + 2;
  return (size_t)(nt + 2) * sizeof(unsigned int) + 4 * (size_t)nt * sizeof(int64_t) + 64;
}

void launch_scan_lookback(const int64_t* in0, const int64_t* in1, int64_t* out0, int64_t* out1,
                          const int64_t* n_dev, int64_t n_cap, void* scratch, cudaStream_t s, int64_t* tot0,
                          int64_t* tot1, int64_t* csr_end) {
  const int64_t nt = n_cap / kTile + 2;  // tiles covering n_cap + 1 elements
  ScanState ss;
  ss.counter = static_cast<unsigned int*>(scratch);
  const size_t head = (((size_t)(nt + 2) * sizeof(unsigned int)) + 63) & ~(size_t)63;
  ss.agg = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + head);
  ss.pre = ss.agg + 2 * nt;
  ss.ntiles = nt;
  cudaMemsetAsync(ss.counter, 0, (size_t)(nt + 1) * sizeof(unsigned int), s);
  ScanTotals tt;
  tt.tot0 = tot0;
  tt.tot1 = tot1;
  tt.csr_end = csr_end;
  const int grid = (int)(nt < (int64_t)kNumSMs * 4 ? nt : (int64_t)kNumSMs * 4);
  if (in1)
    k_scan_lookback<2><<<grid, kScanThreads, 0, s>>>(in0, in1, out0, out1, n_dev, ss, tt);
  else
    k_scan_lookback<1><<<grid, kScanThreads, 0, s>>>(in0, nullptr, out0, nullptr, n_dev, ss, tt);
  note_launch(1);
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
