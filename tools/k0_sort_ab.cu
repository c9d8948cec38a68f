// k0_sort_ab.cu -- measurement only (not part of the library): the north
// star's sort-based twin build (K0) for comparison with the hash-table K0 of
// tm_label.cu.  Keys (min << 32) | max of every half-edge, CUB radix sort of
// (key, half-edge) pairs, adjacent equal keys are twins.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/_k0_sort_ab.so tools/k0_sort_ab.cu
//   python tools/k0_sort_ab.py u10m
#include <cstdint>
#include <cub/device/device_radix_sort.cuh>

namespace {

__global__ void k_keys(const int64_t* __restrict__ tri, int64_t T, int b, unsigned long long* __restrict__ keys,
                       int32_t* __restrict__ vals) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < 3 * T; h += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = h / 3;
    const int j = (int)(h - 3 * t);
    const uint32_t o = (uint32_t)tri[3 * t + (j + 1) % 3], g = (uint32_t)tri[3 * t + (j + 2) % 3];
    keys[h] = ((unsigned long long)min(o, g) << b) | max(o, g);  // packed (min, max): 2b significant bits
    vals[h] = (int32_t)h;
  }
}

__global__ void k_pairs(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ vals, int64_t H,
                        int32_t* __restrict__ twin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const bool prev = i > 0 && keys[i - 1] == k, next = i + 1 < H && keys[i + 1] == k;
    twin[vals[i]] = next ? vals[i + 1] : (prev ? vals[i - 1] : -1);
  }
}

}  // namespace

extern "C" {

// device buffers from the caller; returns milliseconds of the three stages (keys, sort, pairs)
int k0_sort(const int64_t* d_tri, int64_t T, int64_t n, int32_t* d_twin, void* d_tmp, size_t tmp_bytes, float* ms3) {
  int b = 1;
  while ((1ll << b) < n) b++;
  const int64_t H = 3 * T;
  unsigned long long *k_in = nullptr, *k_out = nullptr;
  int32_t *v_in = nullptr, *v_out = nullptr;
  cudaMalloc(&k_in, H * 8);
  cudaMalloc(&k_out, H * 8);
  cudaMalloc(&v_in, H * 4);
  cudaMalloc(&v_out, H * 4);
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, k_in, k_out, v_in, v_out, (int)H, 0, 2 * b);
  void* tmp = d_tmp;
  bool own = false;
  if (need > tmp_bytes) {
    cudaMalloc(&tmp, need);
    own = true;
  }
  cudaEvent_t e[4];
  for (auto& x : e) cudaEventCreate(&x);
  cudaEventRecord(e[0]);
  k_keys<<<148 * 16, 256>>>(d_tri, T, b, k_in, v_in);
  cudaEventRecord(e[1]);
  cub::DeviceRadixSort::SortPairs(tmp, need, k_in, k_out, v_in, v_out, (int)H, 0, 2 * b);
  cudaEventRecord(e[2]);
  k_pairs<<<148 * 16, 256>>>(k_out, v_out, H, d_twin);
  cudaEventRecord(e[3]);
  cudaEventSynchronize(e[3]);
  for (int k = 0; k < 3; k++) cudaEventElapsedTime(ms3 + k, e[k], e[k + 1]);
  for (auto& x : e) cudaEventDestroy(x);
  if (own) cudaFree(tmp);
  cudaFree(k_in);
  cudaFree(k_out);
  cudaFree(v_in);
  cudaFree(v_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
