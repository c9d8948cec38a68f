// tm_traverse.cu -- K3: seed-parallel region boundary walks into a CSR polygon
// array.  Replaces traversal.build_polygon_mesh (traversal.py:303-347), the
// start-edge rule (traversal.py:325-330 + find_start_frontier 172-192) and the
// numba walk kernels _advance / _walk_lengths / _walk_write (242-300).
//
// Output order is ascending seed order with a count -> exclusive scan -> write
// layout, which reproduces the reference's SEQUENTIAL `mesh`/`positions` byte
// for byte instead of the paper's unordered AtomicAdd append.
//
// The walks are split at "rulers" so no thread walks a whole long polygon
// (hull-sliver regions reach 902 boundary vertices at 1M, 3210 at 10M): the
// rulers are every seed's start half-edge plus a hash-sampled 1/8 of all
// frontier half-edges.  (1) every ruler walks to the next ruler (expected 8
// boundary steps); (2) every seed follows its ruler chain (L/8 links) for the
// polygon length and the ruler offsets; (3) scan; (4) every ruler on a seed
// cycle writes its run.  Critical path ~ max ruler gap + L/8 instead of L.
#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

constexpr int kBfsCap = 48;

// Start half-edge of a seed (traversal.py:325-330): the smallest frontier slot
// of t, else the FIFO BFS of find_start_frontier (172-192) across non-frontier
// edges, slots 0,1,2 in order.  The BFS queue doubles as the seen set (every
// triangle is enqueued exactly when first seen).  Returns -2 on local overflow.
__device__ int32_t seed_start(const int32_t* __restrict__ hw, int32_t t, int cap = kBfsCap) {
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
        if (tail == cap) return -2;
        q[tail++] = nt;
      }
    }
  }
  return -1;
}

__device__ __forceinline__ void mark_start(uint32_t* bits, int32_t h) { atomicOr(bits + (h >> 5), 1u << (h & 31)); }
__device__ __forceinline__ bool is_start(const uint32_t* bits, int32_t h) { return (__ldg(bits + (h >> 5)) >> (h & 31)) & 1u; }
// 1 in 8 half-edges, by a multiplicative hash of the id
__device__ __forceinline__ bool sampled(int32_t h) { return ((uint32_t)h * 0x9E3779B1u) < (1u << 29); }
// Rulers of this run: the start half-edges of its seeds, plus the sampled
// half-edges of its own half-edge range [hb, he) (the whole mesh on one GPU;
// a rank's triangle range when the seeds are partitioned, so the ruler walks
// are partitioned too and other ranks' rulers never end a walk).
struct RulerSet {
  const uint32_t* bits;
  int32_t hb, he;
};
__device__ __forceinline__ bool is_ruler(const RulerSet& rs, int32_t h) {
  return (sampled(h) && h >= rs.hb && h < rs.he) || is_start(rs.bits, h);
}

__global__ void __launch_bounds__(256) k_trav_start(const int32_t* __restrict__ hw, const int32_t* __restrict__ seeds,
                                                    const int64_t* __restrict__ Pp, int32_t* __restrict__ start,
                                                    int32_t* __restrict__ overflow, unsigned int* n_overflow,
                                                    uint32_t* __restrict__ bits, DevStatus* st, int bfs_cap) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t t = seeds[i];
    int32_t h = seed_start(hw, t, bfs_cap);
    if (h == -2) overflow[atomicAdd(n_overflow, 1u)] = (int32_t)i;
    else if (h < 0) report(st, K_NO_FRONTIER, t);
    else mark_start(bits, h);
    start[i] = h;
  }
}

// Slow path for BFS regions larger than the register queue: one thread, a
// global FIFO and a stamp array for the seen set.  Rare (max 17 visited at 10M).
// The stamps are all -1 between runs: set once at allocation, restored here.
__global__ void k_bfs_slow(const int32_t* __restrict__ hw, const int32_t* __restrict__ seeds,
                           int32_t* __restrict__ start, const int32_t* __restrict__ overflow,
                           const unsigned int* n_overflow, int32_t* __restrict__ queue, int32_t* __restrict__ stamp,
                           uint32_t* __restrict__ bits, DevStatus* st) {
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
    else mark_start(bits, res);
    start[i] = res;
    for (int64_t j = 0; j < tail; j++) stamp[queue[j]] = -1;  // leave the stamps clean (no per-run memset)
  }
}

// (1) every ruler walks to the next ruler: R[h] = {next ruler, run length, previous ruler}
// indexed by half-edge id, one 16-byte record (the chain passes read a ruler's
// successor and distance, or predecessor and distance, with one sector each)
__device__ __forceinline__ void set_next(RulerRec* R, int32_t h, int32_t g, int32_t d) {
  *reinterpret_cast<int2*>(R + h) = make_int2(g, d);
}
__device__ __forceinline__ int4 ld_rec(const RulerRec* R, int32_t h) {
  return __ldg(reinterpret_cast<const int4*>(R + h));
}
// Runs longer than kMaxRun boundary steps are cut by "virtual" rulers (marked
// in the start bitmap, which only later kernels read): the gap between two
// hash-sampled rulers is geometric with a ~100-step tail, and the write pass
// walks each run on one thread, so bounding runs bounds its tail.  A virtual
// ruler lies inside a gap that exactly one walk covers.
constexpr int kMaxRun = 24;
__device__ __forceinline__ void walk_ruler(const int32_t* __restrict__ hw, const RulerSet& rs, int32_t h,
                                           long long limit, RulerRec* __restrict__ R,
                                           uint32_t* __restrict__ vbits, DevStatus* st) {
  int32_t cur = h, g = h;
  long long d = 0, total = 0;
  for (;;) {
    d++;
    total++;
    g = walk_next(hw, g, limit);
    if (g < 0 || total > limit) { report(st, K_WALK, h / 3); g = h; break; }
    if (is_ruler(rs, g)) break;
    if (d == kMaxRun) {
      mark_start(vbits, g);
      set_next(R, cur, g, (int32_t)d);
      R[g].prev = cur;
      cur = g;
      d = 0;
    }
  }
  set_next(R, cur, g, (int32_t)d);
  R[g].prev = cur;  // every ruler is the successor of exactly one ruler of its cycle
}

// About one half-edge in nine starts a walk, so a warp first gathers the rulers
// of a 256-half-edge tile into a shared queue and then walks them on all lanes
// (a thread-per-half-edge loop keeps ~3 of 32 lanes walking).
constexpr int kWalkTile = 8;  // 32-wide chunks per warp tile
__global__ void __launch_bounds__(256) k_ruler_walk(const int32_t* __restrict__ hw, RulerSet rs, long long limit,
                                                    RulerRec* __restrict__ R, uint32_t* vbits, DevStatus* st) {
  __shared__ int32_t s_q[8][32 * kWalkTile];
  const int lane = threadIdx.x & 31;
  int32_t* q = s_q[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1u;
  const int64_t tile = 32 * kWalkTile;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = rs.hb + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * tile; base < rs.he;
       base += nwarps * tile) {
    int n = 0;
#pragma unroll
    for (int c = 0; c < kWalkTile; c++) {
      const int64_t h = base + c * 32 + lane;
      const bool r = h < rs.he && hw_front(hw[h]) && is_ruler(rs, (int32_t)h);
      const unsigned m = __ballot_sync(0xffffffffu, r);
      if (r) q[n + __popc(m & lt)] = (int32_t)h;
      n += __popc(m);
    }
    __syncwarp();
    for (int k = lane; k < n; k += 32) walk_ruler(hw, rs, q[k], limit, R, vbits, st);
    __syncwarp();
  }
}

// partitioned runs: the start rulers that lie outside the own half-edge range
__global__ void __launch_bounds__(256) k_ruler_walk_starts(const int32_t* __restrict__ hw, RulerSet rs,
                                                           const int32_t* __restrict__ start,
                                                           const int64_t* __restrict__ Pp, long long limit,
                                                           RulerRec* __restrict__ R, uint32_t* vbits,
                                                           DevStatus* st) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t h = start[i];
    if (h < 0 || (h >= rs.hb && h < rs.he)) continue;
    walk_ruler(hw, rs, h, limit, R, vbits, st);
  }
}

// (2a) polygon length and ruler count per seed (traversal.py:264-281).  Two
// walkers per cycle -- forward over next, backward over prev -- consume the
// rulers from both ends, so the longest cycle costs half as many dependent hops.
__global__ void __launch_bounds__(256) k_chain_count(const int32_t* __restrict__ seeds, const int32_t* __restrict__ start,
                                                     const int64_t* __restrict__ Pp, long long limit,
                                                     const RulerRec* __restrict__ R,
                                                     int64_t* __restrict__ len, int64_t* __restrict__ nrul,
                                                     int32_t* __restrict__ long_list, unsigned int* n_long,
                                                     int4* __restrict__ cc, int64_t cc_cap, DevStatus* st) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t h0 = start[i];
    long long L = 0, cnt = 0;
    int4 c0 = make_int4(0, 0, 0, 0), c1 = c0;  // the first four visits (f0, df0, b0, db0), (f1, df1, b1, db1)
    if (h0 >= 0) {
      int32_t f = h0, b = R[h0].prev;  // next ruler to consume going forward / backward
      for (;;) {
        // both walkers' records loaded together: one memory round trip per step of the pair
        const int4 rf = ld_rec(R, f), rb = ld_rec(R, b);
        const int32_t df = rf.y, nf = rf.x, db = rb.y, pb = rb.z;
        if (cnt == 0) c0.x = f, c0.y = df;
        else if (cnt == 2) c1.x = f, c1.y = df;
        L += df;
        cnt++;
        if (f == b) break;
        f = nf;
        if (cnt == 1) c0.z = b, c0.w = db;
        else if (cnt == 3) c1.z = b, c1.w = db;
        L += db;
        cnt++;
        if (b == f) break;
        b = pb;
        if (L > limit) { report(st, K_WALK, seeds[i]); L = 0; cnt = 0; break; }
      }
    }
    len[i] = L;
    nrul[i] = cnt;
    // chains of <= 4 rulers (most polygons) hand their visits to k_chain_emit,
    // which then reads 32 coalesced bytes per seed instead of re-walking R
    if (cc != nullptr && i < cc_cap && cnt <= 4) {
      cc[2 * i] = c0;
      cc[2 * i + 1] = c1;
    }
    // whole path: the long polygons go to the early long-item repair (k_classify_long)
    if (long_list && L > kClassifyShort) long_list[atomicAdd(n_long, 1u)] = (int32_t)i;
  }
}

// (2b) emit (ruler, absolute output offset) entries in chain order, from both ends
__global__ void __launch_bounds__(256) k_chain_emit(const int32_t* __restrict__ start, const int64_t* __restrict__ Pp,
                                                    const RulerRec* __restrict__ R,
                                                    const int64_t* __restrict__ offsets, const int64_t* __restrict__ eoff,
                                                    int32_t* __restrict__ ent_r, int64_t* __restrict__ ent_base,
                                                    int64_t ecap, const int4* __restrict__ cc, int64_t cc_cap,
                                                    DevStatus* st) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t h0 = start[i];
    int64_t kf = eoff[i], kb = eoff[i + 1] - 1;
    if (h0 < 0 || kb < kf) continue;
    if (kb >= ecap) { report(st, K_STRUCT, i); continue; }
    int64_t pf = offsets[i], pb = offsets[i + 1];  // forward start / backward end offsets
    const int64_t cnt = kb - kf + 1;
    if (cc != nullptr && i < cc_cap && cnt <= 4) {  // replay k_chain_count's visits: f0, b0, f1, b1
      const int4 c0 = __ldg(cc + 2 * i), c1 = __ldg(cc + 2 * i + 1);
      ent_r[kf] = c0.x;
      ent_base[kf] = pf;
      if (cnt >= 2) { pb -= c0.w; ent_r[kb] = c0.z; ent_base[kb] = pb; }
      if (cnt >= 3) { pf += c0.y; ent_r[kf + 1] = c1.x; ent_base[kf + 1] = pf; }
      if (cnt >= 4) { pb -= c1.w; ent_r[kb - 1] = c1.z; ent_base[kb - 1] = pb; }
      continue;
    }
    int32_t f = h0, b = R[h0].prev;
    for (;;) {
      const int4 rf = ld_rec(R, f), rb = ld_rec(R, b);
      const int32_t df = rf.y, nf = rf.x, db = rb.y, nb = rb.z;
      ent_r[kf] = f;
      ent_base[kf] = pf;
      pf += df;
      kf++;
      if (f == b) break;
      f = nf;
      pb -= db;
      ent_r[kb] = b;
      ent_base[kb] = pb;
      kb--;
      if (b == f) break;
      b = nb;
    }
  }
}

// (4) every ruler run writes origin(h) for its boundary half-edges (traversal.py:284-300)
__global__ void __launch_bounds__(256) k_ruler_write(const int32_t* __restrict__ tri, const int32_t* __restrict__ hw,
                                                     const int64_t* __restrict__ n_entries,
                                                     const int32_t* __restrict__ ent_r,
                                                     const int64_t* __restrict__ ent_base,
                                                     const RulerRec* __restrict__ R, long long limit,
                                                     int64_t ecap, int32_t* __restrict__ verts,
                                                     int32_t* __restrict__ hv) {
  int64_t E = *n_entries;
  if (E > ecap) E = ecap;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t g = ent_r[k];
    int64_t w = ent_base[k];
    int d = R[g].dist;
    for (int s = 0; s < d; s++) {
      verts[w + s] = he_origin(tri, g);
      if (hv) hv[w + s] = g;  // the boundary half-edge of each slot (fan starts for repair)
      g = walk_next(hw, g, limit);
    }
  }
}

// the runs of the listed polygons (one block per polygon, one thread per run)
__global__ void __launch_bounds__(128) k_ruler_write_list(const int32_t* __restrict__ tri,
                                                          const int32_t* __restrict__ hw,
                                                          const int32_t* __restrict__ list, const unsigned int* n_list,
                                                          const int64_t* __restrict__ eoff,
                                                          const int32_t* __restrict__ ent_r,
                                                          const int64_t* __restrict__ ent_base,
                                                          const RulerRec* __restrict__ R, long long limit,
                                                          int32_t* __restrict__ verts, int32_t* __restrict__ hv) {
  const unsigned int nl = *n_list;
  for (unsigned int w = blockIdx.x; w < nl; w += gridDim.x) {
    const int32_t i = list[w];
    for (int64_t k = eoff[i] + threadIdx.x; k < eoff[i + 1]; k += blockDim.x) {
      int32_t g = ent_r[k];
      const int64_t b = ent_base[k];
      const int d = R[g].dist;
      for (int s = 0; s < d; s++) {
        verts[b + s] = he_origin(tri, g);
        if (hv) hv[b + s] = g;
        g = walk_next(hw, g, limit);
      }
    }
  }
}

static inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// Pp: device polygon (seed) count; Pcap: host upper bound used for the grid.
void launch_trav_start(const int32_t* hw, const int32_t* seeds, const int64_t* Pp, int64_t Pcap, int32_t* start,
                       int32_t* overflow, unsigned int* n_overflow, int32_t* queue, int32_t* stamp, uint32_t* bits,
                       DevStatus* st, cudaStream_t s) {
  static int bfs_cap = -1;
  if (bfs_cap < 0) {  // testing hook: TERMESH_BFS_CAP sends more seeds to the BFS slow path
    const char* e = getenv("TERMESH_BFS_CAP");
    bfs_cap = (e && *e) ? atoi(e) : kBfsCap;
    if (bfs_cap < 1 || bfs_cap > kBfsCap) bfs_cap = kBfsCap;
  }
  k_trav_start<<<grid_for(Pcap, 256), 256, 0, s>>>(hw, seeds, Pp, start, overflow, n_overflow, bits, st, bfs_cap);
  k_bfs_slow<<<1, 32, 0, s>>>(hw, seeds, start, overflow, n_overflow, queue, stamp, bits, st);
  note_launch(2);
}

void launch_ruler_walk(const int32_t* hw, uint32_t* bits, int64_t T, int64_t t_begin, int64_t t_end,
                       const int32_t* start, const int64_t* Pp, int64_t Pcap, RulerRec* R, DevStatus* st,
                       cudaStream_t s) {
  if (T <= 0) return;
  RulerSet rs{bits, (int32_t)(3 * t_begin), (int32_t)(3 * t_end)};
  k_ruler_walk<<<grid_for(3 * (t_end - t_begin), 256), 256, 0, s>>>(hw, rs, 3 * T + 3, R, bits, st);
  note_launch(1);
  if (t_begin > 0 || t_end < T) {
    k_ruler_walk_starts<<<grid_for(Pcap, 256), 256, 0, s>>>(hw, rs, start, Pp, 3 * T + 3, R, bits, st);
    note_launch(1);
  }
}

void launch_chain_count(const int32_t* seeds, const int32_t* start, const int64_t* Pp, int64_t Pcap, int64_t T,
                        const RulerRec* R, int64_t* len, int64_t* nrul,
                        int32_t* long_list, unsigned int* n_long, int4* cc, int64_t cc_cap, DevStatus* st,
                        cudaStream_t s) {
#ifdef TM_NO_CHAIN_CACHE  // A/B: k_chain_emit re-walks every chain
  cc = nullptr;
#endif
  k_chain_count<<<grid_for(Pcap, 256), 256, 0, s>>>(seeds, start, Pp, 3 * T + 3, R, len, nrul,
                                                    long_list, n_long, cc, cc_cap, st);
  note_launch(1);
}

void launch_chain_emit(const int32_t* start, const int64_t* Pp, int64_t Pcap, const RulerRec* R,
                       const int64_t* offsets, const int64_t* eoff,
                       int32_t* ent_r, int64_t* ent_base, int64_t ecap, const int4* cc, int64_t cc_cap, DevStatus* st,
                       cudaStream_t s) {
#ifdef TM_NO_CHAIN_CACHE
  cc = nullptr;
#endif
  k_chain_emit<<<grid_for(Pcap, 256), 256, 0, s>>>(start, Pp, R, offsets, eoff, ent_r, ent_base,
                                                   ecap, cc, cc_cap, st);
  note_launch(1);
}

void launch_ruler_write(const int32_t* tri, const int32_t* hw, const int64_t* n_entries, const int32_t* ent_r,
                        const int64_t* ent_base, const RulerRec* R, int64_t T, int64_t ecap, int32_t* verts,
                        int32_t* hv, cudaStream_t s) {
  k_ruler_write<<<kNumSMs * 16, 256, 0, s>>>(tri, hw, n_entries, ent_r, ent_base, R, 3 * T + 3, ecap, verts, hv);
  note_launch(1);
}

void launch_ruler_write_list(const int32_t* tri, const int32_t* hw, const int32_t* list, const unsigned int* n_list,
                             const int64_t* eoff, const int32_t* ent_r, const int64_t* ent_base, const RulerRec* R,
                             int64_t T, int64_t Pcap, int32_t* verts, int32_t* hv, cudaStream_t s) {
  k_ruler_write_list<<<kNumSMs, 128, 0, s>>>(tri, hw, list, n_list, eoff, ent_r, ent_base, R, 3 * T + 3, verts, hv);
  note_launch(1);
}

}  // namespace tmb
