// tm_post.cu -- device kernels around the mesh -> polygons path: input
// validation that does not fall out of the twin build (trivertex), the
// polygon-mesh analytics the reference computes for its statistics, and the
// canonical output form.
//
// Replaces (paths relative to /root/reference/pkg/src/termesh):
//   mesh_core.validate, trivertex rule           mesh_core.py:268-283
//   traversal.tip_flags                          traversal.py:112-124
//   traversal.repeated_vertex_flags              traversal.py:127-137
//   traversal.extra_vertex_visits                traversal.py:140-147
//   traversal.unique_vertices                    traversal.py:150-153
//   traversal.boundary_edge_count                traversal.py:156-166
//   traversal.enclosed_signed_areas              traversal.py:94-109
//   oracle.canonicalize / _min_rotation          oracle.py:124-141
//
// Canonical order without a comparison sort: every polygon is rotated to its
// smallest rotation, whose first element is the polygon's minimum vertex m.
// Python tuple order sorts by that first element first, so a counting sort
// over m (histogram over the n vertices + exclusive scan + scatter) leaves only
// the polygons sharing a minimum vertex to be ordered among themselves -- a
// handful per bucket (the fan of m) -- which one thread per bucket does with a
// full lexicographic comparison (shorter prefix first, as tuples compare).
#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

static inline int grid_of(int64_t n, int block, int per_sm = 16) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ------------------------------------------------------------ trivertex rule
template <typename TI>
__global__ void k_mark_referenced(const TI* __restrict__ tri, int64_t n3, int64_t n, uint32_t* __restrict__ bits) {
  GRID_STRIDE(s, n3) {
    const int64_t v = (int64_t)tri[s];
    if (v >= 0 && v < n) atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

// mesh_core.py:268-283: tv[v] in [-1, T); -1 only for an unreferenced vertex;
// otherwise triangle tv[v] must contain v.
template <typename TI>
__global__ void k_check_trivertex(const int64_t* __restrict__ tv, int64_t n, const TI* __restrict__ tri, int64_t T,
                                  const uint32_t* __restrict__ bits, DevStatus* st) {
  GRID_STRIDE(v, n) {
    const int64_t t = tv[v];
    const bool referenced = (bits[v >> 5] >> (v & 31)) & 1u;
    bool bad = t < -1 || t >= T || (t == -1 && referenced);
    if (!bad && t >= 0)
      bad = !((int64_t)tri[3 * t] == v || (int64_t)tri[3 * t + 1] == v || (int64_t)tri[3 * t + 2] == v);
    if (bad) report(st, K_TRIVERTEX, v);
  }
}

void launch_check_trivertex(const void* tri, int tri_is64, int64_t T, const int64_t* tv, int64_t n, uint32_t* bits,
                            DevStatus* st, cudaStream_t s) {
  if (n <= 0) return;
  cudaMemsetAsync(bits, 0, (size_t)((n + 31) / 32) * sizeof(uint32_t), s);
  if (tri_is64) {
    if (T > 0) k_mark_referenced<int64_t><<<grid_of(3 * T, 256), 256, 0, s>>>((const int64_t*)tri, 3 * T, n, bits);
    k_check_trivertex<int64_t><<<grid_of(n, 256), 256, 0, s>>>(tv, n, (const int64_t*)tri, T, bits, st);
  } else {
    if (T > 0) k_mark_referenced<int32_t><<<grid_of(3 * T, 256), 256, 0, s>>>((const int32_t*)tri, 3 * T, n, bits);
    k_check_trivertex<int32_t><<<grid_of(n, 256), 256, 0, s>>>(tv, n, (const int32_t*)tri, T, bits, st);
  }
  note_launch(T > 0 ? 2 : 1);
}

// largest vertex id of a CSR (callers that do not know the vertex count)
__global__ void k_max_vertex(const int32_t* __restrict__ v, int64_t F, int* out) {
  int m = -1;
  GRID_STRIDE(k, F) m = max(m, v[k]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

void launch_max_vertex(const int32_t* v, int64_t F, int* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0xFF, sizeof(int), s);  // -1
  if (F > 0) k_max_vertex<<<grid_of(F, 256), 256, 0, s>>>(v, F, out), note_launch(1);
}

// ------------------------------------------------------------ analytics
// one flag byte per vertex id in [0, n) used by the CSR; out-of-range ids are
// reported (K_INDEX_RANGE, slot index)
__global__ void k_mark_vertices(const int32_t* __restrict__ v, int64_t F, int64_t n, uint8_t* __restrict__ flag,
                                DevStatus* st) {
  GRID_STRIDE(k, F) {
    const int32_t x = v[k];
    if (x < 0 || x >= n) report(st, K_INDEX_RANGE, k);
    else flag[x] = 1;
  }
}

void launch_mark_vertices(const int32_t* v, int64_t F, int64_t n, uint8_t* flag, DevStatus* st, cudaStream_t s) {
  if (n > 0) cudaMemsetAsync(flag, 0, (size_t)n, s);
  if (F > 0) k_mark_vertices<<<grid_of(F, 256), 256, 0, s>>>(v, F, n, flag, st), note_launch(1);
}

// Distinct undirected boundary edges (traversal.py:156-166): every slot's
// (v[k], v[next]) pair as key (lo << 32) | hi into an open-addressing set;
// a successful insert counts one edge (warp-aggregated).
__global__ void k_edge_set(const int64_t* __restrict__ off, int64_t P, const int32_t* __restrict__ v,
                           unsigned long long* __restrict__ table, uint64_t mask, unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  // one thread per polygon slot range would serialise long polygons; a
  // grid-stride loop over polygons with lanes over their slots keeps it simple
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < P; i += nw) {
    const int64_t a = off[i], L = off[i + 1] - a;
    for (int64_t k0 = 0; k0 < L; k0 += 32) {
      const int64_t k = k0 + lane;
      bool fresh = false;
      if (k < L) {
        const uint32_t x = (uint32_t)v[a + k], y = (uint32_t)v[a + (k + 1 == L ? 0 : k + 1)];
        const unsigned long long key = ((unsigned long long)min(x, y) << 32) | max(x, y);
        uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> 20;
        for (;;) {
          h &= mask;
          const unsigned long long prev = atomicCAS(table + h, ~0ull, key);
          if (prev == ~0ull) { fresh = true; break; }
          if (prev == key) break;
          h++;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, fresh);
      if (lane == 0 && m) atomicAdd(count, (unsigned long long)__popc(m));
    }
  }
}

void launch_edge_set(const int64_t* off, int64_t P, const int32_t* v, unsigned long long* table, int64_t table_slots,
                     unsigned long long* count, cudaStream_t s) {
  cudaMemsetAsync(table, 0xFF, (size_t)table_slots * sizeof(unsigned long long), s);
  if (P > 0) k_edge_set<<<grid_of(32 * P, 256), 256, 0, s>>>(off, P, v, table, (uint64_t)(table_slots - 1), count),
      note_launch(1);
}

// Per polygon: tip flag (traversal.py:112-124: some cyclic triple a, b, a --
// also for the index wrap of 1- and 2-slot walks), repeated flag and extra
// visits (length - distinct vertices).  Short polygons in registers/local
// compares on one thread; polygons longer than kShortPoly are left to
// k_poly_flags_long (list).
constexpr int kShortPoly = 64;

__global__ void k_poly_flags(const int64_t* __restrict__ off, int64_t P, const int32_t* __restrict__ v,
                             uint8_t* __restrict__ tip, uint8_t* __restrict__ rep, unsigned long long* extra,
                             int32_t* __restrict__ long_list, unsigned int* n_long) {
  unsigned long long ex = 0;
  GRID_STRIDE(i, P) {
    const int64_t a = off[i], L = off[i + 1] - a;
    bool t = false;
    for (int64_t k = 0; k < L && !t; k++) {
      const int64_t pk = k == 0 ? L - 1 : k - 1, nk = k == L - 1 ? 0 : k + 1;
      t = v[a + pk] == v[a + nk];
    }
    tip[i] = t;
    if (L > kShortPoly) {
      long_list[atomicAdd(n_long, 1u)] = (int32_t)i;
      continue;
    }
    int dup = 0;
    for (int64_t k = 1; k < L; k++) {
      const int32_t x = v[a + k];
      bool seen = false;
      for (int64_t j = 0; j < k && !seen; j++) seen = v[a + j] == x;
      dup += seen;
    }
    rep[i] = dup > 0;
    ex += dup;
  }
  for (int o = 16; o > 0; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
  if ((threadIdx.x & 31) == 0 && ex) atomicAdd(extra, ex);
}

// Long polygons, one block, one polygon at a time: stamp[x] = min slot of x
// (stamp entries are INT_MAX between polygons); slot k is a repeat iff
// stamp[v[k]] != k.  Sequential over polygons, so polygons sharing vertices
// never race on the stamps.
__global__ void __launch_bounds__(1024) k_poly_flags_long(const int64_t* __restrict__ off,
                                                          const int32_t* __restrict__ v,
                                                          const int32_t* __restrict__ list, const unsigned int* n_list,
                                                          int32_t* __restrict__ stamp, uint8_t* __restrict__ rep,
                                                          unsigned long long* extra) {
  __shared__ unsigned long long s_dup;
  const unsigned int m = *n_list;
  for (unsigned int q = 0; q < m; q++) {
    const int32_t i = list[q];
    const int64_t a = off[i], L = off[i + 1] - a;
    if (threadIdx.x == 0) s_dup = 0;
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) atomicMin(stamp + v[a + k], (int32_t)k);
    __syncthreads();
    unsigned long long d = 0;
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) d += stamp[v[a + k]] != (int32_t)k;
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0 && d) atomicAdd(&s_dup, d);
    __syncthreads();
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) stamp[v[a + k]] = 0x7FFFFFFF;
    if (threadIdx.x == 0) {
      rep[i] = s_dup > 0;
      if (s_dup) atomicAdd(extra, s_dup);
    }
    __syncthreads();
  }
}

void launch_poly_flags(const int64_t* off, int64_t P, const int32_t* v, uint8_t* tip, uint8_t* rep,
                       unsigned long long* extra, int32_t* long_list, unsigned int* n_long, int32_t* stamp,
                       cudaStream_t s) {
  if (P <= 0) return;
  k_poly_flags<<<grid_of(P, 256), 256, 0, s>>>(off, P, v, tip, rep, extra, long_list, n_long);
  k_poly_flags_long<<<1, 1024, 0, s>>>(off, v, long_list, n_long, stamp, rep, extra);
  note_launch(2);
}

// Shoelace area per polygon in numpy's order (traversal.py:94-109):
// cross_k = x_k*y_{k+1} - x_{k+1}*y_k, each product rounded (no FMA), and
// np.add.reduceat over the polygon = cross_0 + pairwise_sum(cross_1..L-1)
// (numpy's pairwise summation: < 8 terms sequential from 0.0, up to 128 in
// eight interleaved accumulators, longer halves recursively).
__device__ __forceinline__ double cross_at(const double2* __restrict__ xy, const int32_t* __restrict__ v, int64_t a,
                                           int64_t L, int64_t k) {
  const double2 p = xy[v[a + k]], q = xy[v[a + (k + 1 == L ? 0 : k + 1)]];
  return __dsub_rn(__dmul_rn(p.x, q.y), __dmul_rn(q.x, p.y));
}

__device__ double pairwise_block(const double2* xy, const int32_t* v, int64_t a, int64_t L, int64_t k0, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r = __dadd_rn(r, cross_at(xy, v, a, L, k0 + i));
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; j++) r[j] = cross_at(xy, v, a, L, k0 + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], cross_at(xy, v, a, L, k0 + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, cross_at(xy, v, a, L, k0 + i));
  return res;
}

// numpy pairwise_sum with an explicit stack (blocks of <= 128 are leaves)
__device__ double pairwise_sum(const double2* xy, const int32_t* v, int64_t a, int64_t L, int64_t k0, int64_t n) {
  if (n <= 128) return pairwise_block(xy, v, a, L, k0, n);
  struct Fr { int64_t k0, n; int state; double left; };
  Fr st[40];
  int sp = 0;
  st[0] = {k0, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Fr& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_block(xy, v, a, L, f.k0, f.n);
      sp--;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.k0, n2, 0, 0.0};
      sp++;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.k0 + n2, f.n - n2, 0, 0.0};
      sp++;
    } else {
      ret = __dadd_rn(f.left, ret);
      sp--;
    }
  }
  return ret;
}

__global__ void k_poly_areas(const int64_t* __restrict__ off, int64_t P, const int32_t* __restrict__ v,
                             const double2* __restrict__ xy, double* __restrict__ area) {
  GRID_STRIDE(i, P) {
    const int64_t a = off[i], L = off[i + 1] - a;
    double s = 0.0;
    if (L > 0) s = __dadd_rn(cross_at(xy, v, a, L, 0), pairwise_sum(xy, v, a, L, 1, L - 1));
    area[i] = __dmul_rn(0.5, s);
  }
}

void launch_poly_areas(const int64_t* off, int64_t P, const int32_t* v, const double* xy, double* area,
                       cudaStream_t s) {
  if (P > 0) k_poly_areas<<<grid_of(P, 128), 128, 0, s>>>(off, P, v, (const double2*)xy, area), note_launch(1);
}

// ------------------------------------------------------------ canonicalize
// rot[i]: start slot of the smallest rotation (oracle.py:124-132); bucket of
// polygon i = its minimum vertex + 1 (0 for an empty polygon); hist counts.
__device__ __forceinline__ int cmp_rot(const int32_t* __restrict__ v, int64_t a, int64_t L, int64_t r1, int64_t r2) {
  for (int64_t k = 0; k < L; k++) {
    const int64_t i1 = r1 + k < L ? r1 + k : r1 + k - L, i2 = r2 + k < L ? r2 + k : r2 + k - L;
    const int32_t x = v[a + i1], y = v[a + i2];
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}

__global__ void k_canon_rot(const int64_t* __restrict__ off, int64_t P, const int32_t* __restrict__ v, int64_t n,
                            int32_t* __restrict__ rot, int32_t* __restrict__ bucket,
                            unsigned long long* __restrict__ hist, DevStatus* st) {
  GRID_STRIDE(i, P) {
    const int64_t a = off[i], L = off[i + 1] - a;
    int64_t best = 0;
    int32_t m = 0x7FFFFFFF;
    int cnt = 0;
    for (int64_t k = 0; k < L; k++) {
      const int32_t x = v[a + k];
      if (x < m) { m = x; best = k; cnt = 1; }
      else if (x == m) cnt++;
    }
    if (cnt > 1) {  // repeated minimum (non-simple polygon): compare its rotations
      for (int64_t k = best + 1; k < L; k++)
        if (v[a + k] == m && cmp_rot(v, a, L, k, best) < 0) best = k;
    }
    if (L > 0 && (m < 0 || m >= n)) {
      report(st, K_INDEX_RANGE, i);
      m = 0;
    }
    const int32_t b = L > 0 ? m + 1 : 0;
    rot[i] = (int32_t)best;
    bucket[i] = b;
    atomicAdd(hist + b, 1ull);
  }
}

__global__ void k_canon_scatter(int64_t P, const int32_t* __restrict__ bucket, unsigned long long* __restrict__ cursor,
                                int32_t* __restrict__ order) {
  GRID_STRIDE(i, P) order[atomicAdd(cursor + bucket[i], 1ull)] = (int32_t)i;
}

// tuple order of two rotated polygons (shorter prefix first)
__device__ __forceinline__ int cmp_poly(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                        const int32_t* __restrict__ rot, int32_t p, int32_t q) {
  const int64_t a = off[p], La = off[p + 1] - a, b = off[q], Lb = off[q + 1] - b;
  const int64_t ra = rot[p], rb = rot[q];
  const int64_t K = La < Lb ? La : Lb;
  for (int64_t k = 0; k < K; k++) {
    const int64_t ia = ra + k < La ? ra + k : ra + k - La, ib = rb + k < Lb ? rb + k : rb + k - Lb;
    const int32_t x = v[a + ia], y = v[b + ib];
    if (x != y) return x < y ? -1 : 1;
  }
  return La < Lb ? -1 : (La > Lb ? 1 : 0);
}

// one thread per bucket: insertion sort of its polygons (start = exclusive
// scan of the histogram; buckets hold the polygons of one minimum vertex)
__global__ void k_canon_bucket_sort(const int64_t* __restrict__ start, int64_t nb, const int64_t* __restrict__ off,
                                    const int32_t* __restrict__ v, const int32_t* __restrict__ rot,
                                    int32_t* __restrict__ order) {
  GRID_STRIDE(b, nb) {
    const int64_t s0 = start[b], s1 = start[b + 1];
    if (s1 - s0 < 2) continue;
    for (int64_t i = s0 + 1; i < s1; i++) {
      const int32_t x = order[i];
      int64_t j = i - 1;
      while (j >= s0 && cmp_poly(off, v, rot, order[j], x) > 0) {
        order[j + 1] = order[j];
        j--;
      }
      order[j + 1] = x;
    }
  }
}

__global__ void k_canon_lengths(const int32_t* __restrict__ order, int64_t P, const int64_t* __restrict__ off,
                                int64_t* __restrict__ len) {
  GRID_STRIDE(j, P) {
    const int32_t i = order[j];
    len[j] = off[i + 1] - off[i];
  }
}

// warp per output polygon: copy the rotated vertex run
__global__ void k_canon_write(const int32_t* __restrict__ order, int64_t P, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ v, const int32_t* __restrict__ rot,
                              const int64_t* __restrict__ off_out, int32_t* __restrict__ v_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < P; j += nw) {
    const int32_t i = order[j];
    const int64_t a = off[i], L = off[i + 1] - a, r = rot[i], o = off_out[j];
    for (int64_t k = lane; k < L; k += 32) {
      const int64_t src = r + k < L ? r + k : r + k - L;
      v_out[o + k] = v[a + src];
    }
  }
}

void launch_canon_rot(const int64_t* off, int64_t P, const int32_t* v, int64_t n, int32_t* rot, int32_t* bucket,
                      unsigned long long* hist, DevStatus* st, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, (size_t)(n + 2) * sizeof(unsigned long long), s);
  if (P > 0) k_canon_rot<<<grid_of(P, 256), 256, 0, s>>>(off, P, v, n, rot, bucket, hist, st), note_launch(1);
}

void launch_canon_sort(int64_t P, int64_t n, const int64_t* off, const int32_t* v, const int32_t* rot,
                       const int32_t* bucket, const int64_t* start, unsigned long long* cursor, int32_t* order,
                       cudaStream_t s) {
  if (P <= 0) return;
  cudaMemcpyAsync(cursor, start, (size_t)(n + 2) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  k_canon_scatter<<<grid_of(P, 256), 256, 0, s>>>(P, bucket, cursor, order);
  k_canon_bucket_sort<<<grid_of(n + 1, 256), 256, 0, s>>>(start, n + 1, off, v, rot, order);
  note_launch(2);
}

void launch_canon_lengths(const int32_t* order, int64_t P, const int64_t* off, int64_t* len, cudaStream_t s) {
  if (P > 0) k_canon_lengths<<<grid_of(P, 256), 256, 0, s>>>(order, P, off, len), note_launch(1);
}

void launch_canon_write(const int32_t* order, int64_t P, const int64_t* off, const int32_t* v, const int32_t* rot,
                        const int64_t* off_out, int32_t* v_out, cudaStream_t s) {
  if (P > 0) k_canon_write<<<grid_of(32 * P, 256), 256, 0, s>>>(order, P, off, v, rot, off_out, v_out), note_launch(1);
}

}  // namespace tmb
