// tm_repair.cu -- K4: barrier-edge tip removal and pinch splitting, plus the
// CSR stitch.  Replaces reparation.repair_all (reparation.py:343-377) and its
// helpers: find_barrier_tip (59-71), the fan rotations (82-124),
// middle_internal_edge (127-145), _pinch_candidates / _wedge_internal_edges
// (148-205), _split_polygon (208-229) and the round driver (232-340).
//
// Schedule: one work item per non-simple input polygon.  The
// item replays the reference's rounds on its own piece list (round r splits
// every piece that still has a tip, pa before pb), which is exactly the
// reference's global round schedule restricted to that polygon: distinct
// polygons have disjoint interiors, so their frontier mutations never
// interact.  Leaves come out in the reference's raw order.
//
// Tip splits do not re-walk the mesh: the two pieces are arcs
// of the parent cycle cut at the tip v and at the occurrence j of u = target(e)
// whose boundary wedge contains twin(e); each piece is then rotated to start at
// origin(h0), h0 = smallest frontier slot of e/3 (resp. twin(e)/3), which is
// where the reference's re-walk (poly_construction) starts.  If the wedge or
// rotation search fails the split falls back to the re-walk.  Pinch trial splits
// (rare) always re-walk, with revert on a broken length law.
//
// Piece records live in a device pool: {offset, len|flags}.  Each warp
// allocates from its own arena (one global atomic per arena, not per piece),
// so the bump counter is not a serialisation point.  A pool overflow is
// reported; the host restores the pre-repair frontier bits and retries with a
// larger pool.
#include <cstdlib>

#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kLongMin = 96;    // items longer than this go to k_repair_tips_long first
constexpr int kHugeMin = 512;   // ... and the longest ones are dequeued first
constexpr uint32_t F_TIP = 1u << 30;
constexpr uint32_t F_REP = 1u << 31;
constexpr uint32_t F_FAIL = 1u << 29;
constexpr uint32_t LEN_MASK = (1u << 29) - 1;

struct RepairCtx {
  const int32_t* tri;
  int32_t* hw;
  const int32_t* tv;  // a triangle incident to each polygon vertex: fan starts (tip fans are rotation-invariant)
  int64_t T;
  int32_t* pool;
  unsigned long long pool_cap;
  unsigned long long* pool_top;
  int32_t* undo;
  unsigned long long* undo_top;
  unsigned long long undo_cap;
  DevStatus* st;
  int tv_exact;       // tv is the reference trivertex (lowest incident triangle, mesh_core.py:171-178)
  unsigned long long* dbg;  // debug counters (tm_ctx_debug), may be null
};

__device__ __forceinline__ int64_t palloc(const RepairCtx& c, int64_t n) {
  unsigned long long o = atomicAdd(c.pool_top, (unsigned long long)n);
  if (o + (unsigned long long)n > c.pool_cap) return -1;
  return (int64_t)o;
}

// The packed word is (twin << 1) | frontier and the twins are known, so a
// promotion is two plain stores -- no load, nothing to wait for.
__device__ __forceinline__ void promote(const RepairCtx& c, int32_t e, int32_t te) {
  c.hw[e] = (te << 1) | 1;
  c.hw[te] = (e << 1) | 1;
}

// Per-warp bump arena carved from the pool (state held by lane 0).
struct WarpArena {
  long long cur = 0, end = 0;
};

// Warp-uniform allocation of n slots; returns -1 when the pool is exhausted.
__device__ __forceinline__ long long warp_alloc(const RepairCtx& c, WarpArena& a, long long n, long long refill,
                                                int lane) {
  long long o = 0;
  if (lane == 0) {
    if (a.cur + n > a.end) {
      long long want = n > refill ? n : refill;
      long long base = palloc(c, want);
      if (base < 0) {
        o = -1;
      } else {
        a.cur = base;
        a.end = base + want;
      }
    }
    if (o == 0) {
      o = a.cur;
      a.cur += n;
    }
  }
  return __shfl_sync(0xffffffffu, o, 0);
}

__device__ __forceinline__ void demote(const RepairCtx& c, int32_t e, int32_t te) {
  c.hw[e] = te << 1;
  c.hw[te] = e << 1;
}

// ------------------------------------------------------------ classify
// Per input polygon: tip flag, repeated flag, extra visits.  Work items are the
// polygons with a repeated vertex (a tip implies one).
// (len - distinct) of a polygon of n <= N vertices held in registers
template <int N>
__device__ __forceinline__ int extra_visits_reg(const int32_t* __restrict__ s, int n) {
  int32_t r[N];
#pragma unroll
  for (int k = 0; k < N; k++) r[k] = k < n ? __ldg(s + k) : (int32_t)(0x80000000u + (uint32_t)k);
  int ex = 0;
#pragma unroll
  for (int k = 1; k < N; k++) {
    bool dup = false;
#pragma unroll
    for (int q = 0; q < k; q++) dup |= r[q] == r[k];
    ex += dup;
  }
  return ex;
}

__device__ __forceinline__ int lane_id() { return (int)(threadIdx.x & 31); }

// (n - distinct) of s[0..n), n <= 64, one warp: lane l holds s[l] and s[32 + l];
// unused lanes hold distinct negatives (and are masked from the count).  The
// matches run on every lane (warp-uniform code, full mask).
__device__ __forceinline__ int warp_extra_64(const int32_t* __restrict__ s, int n, int lane) {
  const int32_t x0 = lane < n ? __ldg(s + lane) : -1 - lane;
  const int32_t x1 = lane + 32 < n ? __ldg(s + lane + 32) : -33 - lane;
  const int f0 = __ffs(__match_any_sync(kFull, x0)) - 1;
  const unsigned m1x = __match_any_sync(kFull, x1);
  int f1 = -1;
  if (n > 32)
    for (int q = 0; q < 32; q++)
      if (__shfl_sync(kFull, x0, q) == x1 && f1 < 0) f1 = q;
  if (f1 < 0) f1 = 32 + __ffs(m1x) - 1;
  return __popc(__ballot_sync(kFull, lane < n && f0 < lane)) +
         __popc(__ballot_sync(kFull, lane + 32 < n && f1 < lane + 32));
}

// Block-aggregated append: one global atomic per block and list instead of
// one per element (a single hot counter serialises thousands of returning
// atomics).  All threads of the block must call it.
__device__ __forceinline__ int block_append(bool want, unsigned int* counter, int* s_cnt, unsigned int* s_base) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(kFull, want);
  int wbase = 0;
  if (lane == 0 && m) wbase = atomicAdd(s_cnt, __popc(m));
  wbase = __shfl_sync(kFull, wbase, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int c = *s_cnt;
    *s_cnt = 0;  // ready for the next call (its adds follow the barrier below)
    *s_base = c ? atomicAdd(counter, (unsigned)c) : 0u;
  }
  __syncthreads();
  return want ? (int)*s_base + wbase + __popc(m & ((1u << lane) - 1u)) : -1;
}

__global__ void __launch_bounds__(256) k_classify(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                  const int64_t* __restrict__ Pp, int32_t* __restrict__ item_of,
                                                  int32_t* __restrict__ items, unsigned int* n_items,
                                                  int32_t* __restrict__ long_list, unsigned int* n_long,
                                                  unsigned long long* stats, const int32_t* __restrict__ hv,
                                                  int32_t* __restrict__ tv, int append_long,
                                                  int32_t* __restrict__ item_state) {
  __shared__ int s_cnt;
  __shared__ unsigned int s_base;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int64_t P = *Pp;
  unsigned long long extra_sum = 0, rep_cnt = 0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < P; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool is_long = false, is_item = false, mid = false;
    int64_t b = 0, n = 0, ex = 0;
    if (i < P) {
      b = off[i];
      n = off[i + 1] - b;
      if (n > kClassifyShort) {
        is_long = append_long;  // k_classify_long sets item_of[i]
      } else {
        item_of[i] = -1;
        // registers: all loads in flight at once, compares without reloads
        if (n <= 16) ex = extra_visits_reg<16>(v + b, (int)n);
        else mid = true;
      }
    }
    // 16 < n <= 48 (6% of the polygons, but in 85% of the warps): the whole warp
    // per polygon, first occurrences by __match_any_sync / shuffles, instead of
    // every lane of such a warp running the 48-wide quadratic compare
    for (unsigned mm = __ballot_sync(kFull, mid); mm; mm &= mm - 1) {
      const int src = __ffs(mm) - 1;
      const int64_t bb = __shfl_sync(kFull, b, src);
      const int nn = (int)__shfl_sync(kFull, n, src);
      const int e = warp_extra_64(v + bb, nn, lane_id());
      if ((int)(threadIdx.x & 31) == src) ex = e;
    }
    if (i < P && n <= kClassifyShort && ex > 0) {
      extra_sum += ex;
      rep_cnt++;
      is_item = true;
    }
    const int pl = block_append(is_long, n_long, &s_cnt, &s_base);
    if (is_long) long_list[pl] = (int32_t)i;
    const int pi = block_append(is_item, n_items, &s_cnt, &s_base);
    if (is_item) {
      items[pi] = (int32_t)i;
      item_state[pi] = 0;  // (no per-run memset of the state array)
      item_of[i] = pi;
      if (hv) {  // whole path: fan start of every vertex of the work item (any incident triangle)
        const int64_t b = off[i], e = off[i + 1];
        for (int64_t k = b; k < e; k++) tv[v[k]] = hv[k] / 3;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    extra_sum += __shfl_xor_sync(kFull, extra_sum, o);
    rep_cnt += __shfl_xor_sync(kFull, rep_cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (extra_sum) atomicAdd(stats + 2, extra_sum);
    if (rep_cnt) atomicAdd(stats + 6, rep_cnt);
  }
}

// long polygons: one block each; distinct vertices counted with an
// open-addressing set -- in shared memory (len <= kSetCap/2), else in a
// block-private region bump-allocated from the repair pool (the polygon of the
// hull sliver reaches ~10^4 vertices at 100M points), else (pool exhausted)
// a block-parallel quadratic scan.
constexpr int kSetCap = 8192;
__global__ void __launch_bounds__(256) k_classify_long(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                       const int32_t* __restrict__ long_list,
                                                       const unsigned int* n_long, int32_t* __restrict__ item_of,
                                                       int32_t* __restrict__ items, unsigned int* n_items,
                                                       unsigned long long* stats, LongQueue q,
                                                       const int32_t* __restrict__ hv, int32_t* __restrict__ tv,
                                                       int32_t* __restrict__ item_state, int32_t* pool,
                                                       unsigned long long* pool_top, unsigned long long pool_cap,
                                                       int32_t* __restrict__ item_depth) {
  __shared__ int32_t s_tab[kSetCap];
  __shared__ unsigned int dups;
  __shared__ long long s_gbase;
  unsigned int nl = *n_long;
  for (unsigned int w = blockIdx.x; w < nl; w += gridDim.x) {
    int32_t i = long_list[w];
    int64_t b = off[i];
    int n = (int)(off[i + 1] - b);
    const int32_t* s = v + b;
    int cap = 64;
    while (cap < 2 * n) cap <<= 1;
    if (threadIdx.x == 0) {
      dups = 0;
      s_gbase = -1;
      if (cap > kSetCap) {
        const unsigned long long o = atomicAdd(pool_top, (unsigned long long)cap);
        if (o + (unsigned long long)cap <= pool_cap) s_gbase = (long long)o;
      }
    }
    __syncthreads();
    unsigned int my = 0;
    if (cap <= kSetCap || s_gbase >= 0) {
      int32_t* tab = cap <= kSetCap ? s_tab : pool + s_gbase;
      for (int k = threadIdx.x; k < cap; k += blockDim.x) tab[k] = -1;
      __syncthreads();
      for (int p = threadIdx.x; p < n; p += blockDim.x) {
        int32_t x = s[p];
        uint32_t slot = ((uint32_t)x * 0x9E3779B1u) >> (32 - __ffs(cap) + 1);
        for (;;) {
          int32_t prev = atomicCAS(&tab[slot], -1, x);
          if (prev == -1) break;
          if (prev == x) { my++; break; }
          slot = (slot + 1) & (cap - 1);
        }
      }
    } else {
      __syncthreads();
      for (int p = threadIdx.x; p < n; p += blockDim.x) {
        int32_t x = s[p];
        bool dup = false;
        for (int q = 0; q < p && !dup; q++) dup = s[q] == x;
        my += dup;
      }
    }
    atomicAdd(&dups, my);
    __syncthreads();
    if (dups > 0 && hv)
      for (int p = threadIdx.x; p < n; p += blockDim.x) tv[s[p]] = hv[b + p] / 3;
    if (threadIdx.x == 0 && dups == 0) item_of[i] = -1;
    if (threadIdx.x == 0 && dups > 0) {
      unsigned int k = atomicAdd(n_items, 1u);
      items[k] = i;
      item_state[k] = 0;
      item_depth[k] = (int32_t)dups;  // hint for k_repair_tips_seg: ~ the item's splits (pool-region blocks above gm_dups)
      item_of[i] = (int32_t)k;
      atomicAdd(stats + 2, (unsigned long long)dups);
      atomicAdd(stats + 6, 1ull);
      if (n > kHugeMin) q.huge[atomicAdd(q.n_huge, 1u)] = (int32_t)k;
      else if (n > kLongMin) q.longq[atomicAdd(q.n_long, 1u)] = (int32_t)k;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ mesh helpers
// reparation.py:127-145.  The fan order is cyclic (fan_step), so starting at
// the barrier half-edge enumerates fan[barrier_at:] + fan[:barrier_at].
__device__ int32_t middle_internal_edge(const RepairCtx& c, int32_t v, int32_t barrier, int32_t poly) {
  int32_t t0 = c.tv[v];
  int32_t g0 = t0 < 0 ? -1 : he_with_origin(c.tri, t0, v);
  if (g0 < 0) { report(c.st, K_STRUCT, poly); return -1; }
  int guard = (int)(3 * c.T + 3 < (1LL << 30) ? 3 * c.T + 3 : (1LL << 30));
  int32_t g = g0, gb = -1;
  int k = 0, deg = 0;
  do {
    int32_t w = c.hw[g];
    if (gb < 0 && hw_front(w) && he_target(c.tri, g) == barrier) gb = g;
    if (!hw_front(w)) k++;
    deg++;
    g = fan_step(c.hw, g, guard);
    if (g < 0 || deg > guard) { report(c.st, K_STRUCT, poly); return -1; }
  } while (g != g0);
  if (gb < 0) { report(c.st, K_BARRIER, poly); return -1; }
  if (k == 0) { report(c.st, K_NO_INTERNAL, poly); return -1; }
  int want = (k - 1) / 2, cnt = 0;
  g = gb;
  for (int s = 0; s < deg; s++) {
    if (!hw_front(c.hw[g])) {
      if (cnt == want) return g;
      cnt++;
    }
    g = fan_step(c.hw, g, guard);
  }
  report(c.st, K_STRUCT, poly);
  return -1;
}

__device__ long long walk_len(const RepairCtx& c, int32_t h0) {
  long long limit = 3 * c.T + 3, guard = 2 * 3 * c.T + 3, n = 0;
  int32_t h = h0;
  do {
    if (++n > guard) return -1;
    h = walk_next(c.hw, h, limit);
    if (h < 0) return -1;
  } while (h != h0);
  return n;
}

__device__ void walk_write(const RepairCtx& c, int32_t h0, int32_t* out) {
  long long limit = 3 * c.T + 3;
  int32_t h = h0;
  do {
    *out++ = he_origin(c.tri, h);
    h = walk_next(c.hw, h, limit);
  } while (h != h0 && h >= 0);
}


// ------------------------------------------------------------ warp helpers
// One warp cooperates on one piece.  Lanes split O(len) scans and copies; the
// sequential mesh rotations run on one or two lanes and are broadcast.  All
// control flow below is warp-uniform.
constexpr int kFanCap = 64;
constexpr int kTipWarps = 4;  // warps per block of k_repair_tips

__device__ __forceinline__ int wrap_idx(int x, int n) { return x >= n ? x - n : (x < 0 ? x + n : x); }

// Smallest p in [0, n) with pred(p), or -1.  kScanUnroll 32-wide chunks per
// round (their loads in flight together).  1, not 8: k_repair_tips is
// instruction-fetch bound (ncu at 10M: "no instruction" is the top stall, 28%
// of the samples) and every unrolled copy of an inlined predicate adds code;
// 8 -> 2 cut its SASS from 7.3 k to 5.2 k instructions and the 10M step by
// 0.24 ms, 2 -> 1 another 0.05 ms (tools/ab_lib.sh).
#ifndef TM_SCAN_UNROLL
#define TM_SCAN_UNROLL 1
#endif
constexpr int kScanUnroll = TM_SCAN_UNROLL;
template <typename Pred>
__device__ __forceinline__ int warp_find_first(int n, int lane, Pred pred) {
  for (int base = 0; base < n; base += 32 * kScanUnroll) {
    bool hit[kScanUnroll];
#pragma unroll
    for (int c = 0; c < kScanUnroll; c++) {
      int p = base + c * 32 + lane;
      hit[c] = p < n && pred(p);
    }
#pragma unroll
    for (int c = 0; c < kScanUnroll; c++) {
      unsigned m = __ballot_sync(kFull, hit[c]);
      if (m) return base + c * 32 + __ffs(m) - 1;
    }
  }
  return -1;
}

// dst[k] = src(k) for k in [0, n), staged in registers (8 loads in flight per lane)
template <typename Src>
__device__ __forceinline__ void warp_copy(int32_t* dst, int n, int lane, Src src) {
  for (int base = 0; base < n; base += 32 * kScanUnroll) {
    int32_t buf[kScanUnroll];
#pragma unroll
    for (int c = 0; c < kScanUnroll; c++) {
      int k = base + c * 32 + lane;
      if (k < n) buf[c] = src(k);
    }
#pragma unroll
    for (int c = 0; c < kScanUnroll; c++) {
      int k = base + c * 32 + lane;
      if (k < n) dst[k] = buf[c];
    }
  }
}

// first position p (cyclic triple s[p-1] == s[p+1]) or -1 (reparation.py:59-71)
__device__ int warp_first_tip(const int32_t* s, int n, int lane) {
#if !defined(TM_NO_SHFL_SCAN) && !defined(TM_NO_SHFL_TIP)
  if (n <= 32) {  // one load per lane, cyclic neighbours by shuffle
    const int32_t x = lane < n ? s[lane] : 0;
    const int32_t pv = __shfl_sync(kFull, x, lane == 0 ? n - 1 : lane - 1);
    const int32_t nx = __shfl_sync(kFull, x, lane + 1 >= n ? 0 : lane + 1);
    const unsigned m = __ballot_sync(kFull, lane < n && pv == nx);
    return m ? __ffs(m) - 1 : -1;
  }
#endif
  return warp_find_first(n, lane, [&](int p) { return s[p == 0 ? n - 1 : p - 1] == s[p + 1 == n ? 0 : p + 1]; });
}

__device__ __forceinline__ uint32_t warp_tip_flag(const int32_t* s, int n, int lane) {
  return warp_first_tip(s, n, lane) >= 0 ? F_TIP : 0u;
}

// (len - distinct) of s[0..n) (traversal.py:140-147), quadratic over lanes
__device__ int warp_extra_visits(const int32_t* s, int n, int lane) {
  int extra = 0;
  for (int pb = 0; pb < n; pb += 32) {
    int p = pb + lane;
    int32_t x = p < n ? s[p] : INT32_MIN;
    bool dup = false;
    for (int qb = 0; qb <= pb; qb += 32) {
      int32_t y = qb + lane < n ? s[qb + lane] : INT32_MIN + 1;
      int qmax = min(32, n - qb);
      for (int k = 0; k < qmax; k++) {
        int32_t yk = __shfl_sync(kFull, y, k);
        dup |= (qb + k < p) && (yk == x);
      }
    }
    extra += __popc(__ballot_sync(kFull, dup && p < n));
  }
  return extra;
}

// Fan of v in the reference order (_fan_around from the trivertex half-edge
// g0, reparation.py:91-124) collected into fan[0..deg) by two walkers: lane 0
// rotates CCW from g0, lane 1 rotates CW.  A closed fan ends where the walkers
// meet; an open fan is the CCW run followed by the reversed CW run.  Half the
// dependent loads of a one-sided walk.  Returns deg, -1 on a structural
// failure, or kFanCap + 1 when the fan does not fit (caller falls back).
__device__ int warp_collect_fan(const RepairCtx& c, int32_t v, int32_t* fan, int32_t* back, int lane) {
  int32_t g0 = -1;
  __syncwarp();  // the buffers may still be read by every lane of a previous use (racecheck)
  if (lane == 0) {
    int32_t t0 = c.tv[v];
    g0 = t0 < 0 ? -1 : he_with_origin(c.tri, t0, v);
    if (g0 >= 0) fan[0] = g0;
  }
  g0 = __shfl_sync(kFull, g0, 0);
  if (g0 < 0) return -1;
  int32_t cur = g0;                 // lane 0: CCW walker, lane 1: CW walker
  bool stop = false;
  int a = 0, b = 0;                 // fan[1..a] from lane 0, back[0..b) from lane 1
  int deg = kFanCap + 1, mode = 0;  // mode 1: append the meeting element
  for (int step = 0; step < kFanCap; step++) {
    int32_t nxt = -1;
    if (lane == 0 && !stop) nxt = rot_ccw(c.hw, cur);
    if (lane == 1 && !stop) nxt = rot_cw(c.hw, cur);
    int32_t n0 = __shfl_sync(kFull, nxt, 0), n1 = __shfl_sync(kFull, nxt, 1);
    int32_t c1 = __shfl_sync(kFull, cur, 1);
    bool s0 = __shfl_sync(kFull, stop, 0), s1 = __shfl_sync(kFull, stop, 1);
    int aa = __shfl_sync(kFull, a, 0), bb = __shfl_sync(kFull, b, 1);
    if (!s0 && !s1 && n0 >= 0) {
      if (n0 == c1) { deg = 1 + aa + bb; break; }            // CCW reached the CW walker's element
      if (n0 == n1) { deg = 2 + aa + bb; mode = 1; break; }  // both stepped onto the same element
    }
    if (lane == 0 && !stop) {
      if (nxt < 0) stop = true;
      else { a++; if (a < kFanCap) fan[a] = nxt; cur = nxt; }
    }
    if (lane == 1 && !stop) {
      if (nxt < 0) stop = true;
      else { if (b < kFanCap) back[b] = nxt; b++; cur = nxt; }
    }
    s0 = __shfl_sync(kFull, stop, 0);
    s1 = __shfl_sync(kFull, stop, 1);
    aa = __shfl_sync(kFull, a, 0);
    bb = __shfl_sync(kFull, b, 1);
    if (s0 && s1) { deg = 1 + aa + bb; break; }              // open fan: both walkers at the border
    if (1 + aa + bb + 1 > kFanCap) break;
  }
  a = __shfl_sync(kFull, a, 0);
  b = __shfl_sync(kFull, b, 1);
  if (deg > kFanCap) return kFanCap + 1;
  __syncwarp();
  if (mode == 1) {
    int32_t m = -1;
    if (lane == 0) m = rot_ccw(c.hw, fan[a]);
    if (lane == 0) fan[a + 1] = m;
    a++;
  }
  __syncwarp();
  for (int k = lane; k < b; k += 32) fan[1 + a + k] = back[b - 1 - k];
  __syncwarp();
  return deg;
}

// reparation.py:127-145: the ((k-1)//2)-th non-frontier half-edge of the fan
// rotated to start at the barrier half-edge (target == barrier, frontier).
// A fan collected once can be reused while the mesh topology is unchanged (a
// promotion only flips frontier bits): `in` supplies a cached fan (global
// memory, in_deg entries), `out`/`out_deg` receive the collected one.
struct FanCache {
  const int32_t* in = nullptr;
  int in_deg = 0;
  int32_t* out = nullptr;
  int* out_deg = nullptr;
};

__device__ int32_t warp_middle_internal_edge(const RepairCtx& c, int32_t v, int32_t barrier, int32_t poly,
                                             int32_t* fan, int32_t* back, int lane, bool quiet = false,
                                             FanCache fc = FanCache()) {
  int deg;
  if (fc.in) {
    deg = fc.in_deg;
    fan = const_cast<int32_t*>(fc.in);
  } else {
    deg = warp_collect_fan(c, v, fan, back, lane);
    if (fc.out_deg) {
      if (deg >= 0 && deg <= kFanCap)
        for (int k = lane; k < deg; k += 32) fc.out[k] = fan[k];
      if (lane == 0) *fc.out_deg = (deg >= 0 && deg <= kFanCap) ? deg : -1;
    }
  }
  if (deg < 0) {
    if (lane == 0 && !quiet) report(c.st, K_STRUCT, poly);
    return -1;
  }
  if (deg > kFanCap) {
    if (quiet) return -1;  // precompute: leave it to the exact on-the-fly path
    int32_t e = -1;
    if (lane == 0) e = middle_internal_edge(c, v, barrier, poly);
    return __shfl_sync(kFull, e, 0);
  }
  unsigned long long imask = 0, bmask = 0;
  for (int base = 0; base < deg; base += 32) {
    int idx = base + lane;
    bool fr = false, in_fan = idx < deg;
    int32_t tg = -1;
    if (in_fan) {
      int32_t g = fan[idx];
      fr = hw_front(c.hw[g]);
      tg = he_target(c.tri, g);
    }
    unsigned bi = __ballot_sync(kFull, in_fan && fr && tg == barrier);
    unsigned ii = __ballot_sync(kFull, in_fan && !fr);
    bmask |= (unsigned long long)bi << base;
    imask |= (unsigned long long)ii << base;
  }
  if (bmask == 0) {
    if (lane == 0 && !quiet) report(c.st, K_BARRIER, poly);
    return -1;
  }
  if (imask == 0) {
    if (lane == 0 && !quiet) report(c.st, K_NO_INTERNAL, poly);
    return -1;
  }
  int at = __ffsll((long long)bmask) - 1;
  int k = __popcll(imask), want = (k - 1) / 2;
  unsigned long long hi = imask & (~0ull << at), lo = imask & ((1ull << at) - 1);
  unsigned long long m = hi;
  int cnt_hi = __popcll(hi);
  if (want >= cnt_hi) { m = lo; want -= cnt_hi; }
  for (int r = 0; r < want; r++) m &= m - 1;
  return fan[__ffsll((long long)m) - 1];
}

// Re-walk split (reparation.py:216-229 after promotion), warp-uniform result:
// 1 = pieces written through alloc, 0 = length law failed, -1 = error.
template <typename Alloc>
__device__ int warp_rewalk_split(const RepairCtx& c, int32_t e, int32_t te, int L, int32_t poly, Alloc alloc,
                                 int lane, int32_t** A, int* la_out, int32_t** B, int* lb_out) {
  long long la = 0, lb = 0;
  int32_t ha = -1, hb = -1;
  if (lane == 0) {
    ha = min_frontier_slot(c.hw, e / 3);
    hb = min_frontier_slot(c.hw, te / 3);
    la = walk_len(c, ha);
    lb = walk_len(c, hb);
  }
  la = __shfl_sync(kFull, la, 0);
  lb = __shfl_sync(kFull, lb, 0);
  if (la < 0 || lb < 0) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return -1;
  }
  if (la + lb != (long long)L + 2) return 0;
  int32_t* p = alloc(la + lb);
  if (p == nullptr) {
    if (lane == 0) report(c.st, K_POOL, poly);
    return -1;
  }
  if (lane == 0) {
    walk_write(c, ha, p);
    walk_write(c, hb, p + la);
  }
  __syncwarp();
  *A = p;
  *la_out = (int)la;
  *B = p + la;
  *lb_out = (int)lb;
  return 1;
}

// Everything a tip split needs from the mesh (reparation.py:127-145, 216-220):
// the promoted edge e = v->u and its twin, the incoming boundary vertex a_in of
// the visit of u whose wedge holds twin(e), and the directed boundary pairs
// (oa,ga) / (ob,gb) of h0 = smallest frontier slot of e/3 and twin(e)/3 after
// the promotion (where the reference re-walks start).
struct SplitInfo {
  int32_t e, te, u, a_in, oa, ga, ob, gb;
};

// smallest frontier slot of triangle t when slot `forced` counts as frontier
__device__ __forceinline__ int32_t min_slot_with(const int32_t* hw, int32_t t, int32_t forced) {
  int32_t b = 3 * t;
  int32_t w0 = hw[b], w1 = hw[b + 1], w2 = hw[b + 2];
  if (hw_front(w0) || forced == b) return b;
  if (hw_front(w1) || forced == b + 1) return b + 1;
  if (hw_front(w2) || forced == b + 2) return b + 2;
  return -1;
}

// Computes the split of tip vertex v (barrier b) from the current frontier.
// promote_now: also set the frontier bits of e and twin(e).  quiet: do not
// report failures (precomputation).  Warp-uniform result.
__device__ bool warp_split_info(const RepairCtx& c, int32_t v, int32_t b, int32_t poly, int32_t* fan, int32_t* back,
                                int lane, bool promote_now, bool quiet, SplitInfo* out, FanCache fc = FanCache()) {
  int32_t e = warp_middle_internal_edge(c, v, b, poly, fan, back, lane, quiet, fc);
  if (e < 0) return false;
  SplitInfo s{};
  if (lane == 0) {
    s.e = e;
    s.te = hw_twin(c.hw[e]);
    s.u = he_target(c.tri, e);
    s.a_in = -1;
    if (s.te >= 0) {
      // rotate CCW from twin(e) until the crossed edge prev(g) is frontier
      int32_t g = s.te;
      long long guard = 3 * c.T + 3;
      for (long long k = 0; k < guard; k++) {
        int32_t p = he_prev(g);
        int32_t w = c.hw[p];
        if (hw_front(w)) { s.a_in = he_origin(c.tri, p); break; }
        g = hw_twin(w);
      }
      if (promote_now) promote(c, e, s.te);
      int32_t ha = min_slot_with(c.hw, e / 3, e), hb = min_slot_with(c.hw, s.te / 3, s.te);
      s.oa = he_origin(c.tri, ha); s.ga = he_target(c.tri, ha);
      s.ob = he_origin(c.tri, hb); s.gb = he_target(c.tri, hb);
    }
  }
  __syncwarp();
  s.e = __shfl_sync(kFull, s.e, 0); s.te = __shfl_sync(kFull, s.te, 0);
  s.u = __shfl_sync(kFull, s.u, 0); s.a_in = __shfl_sync(kFull, s.a_in, 0);
  s.oa = __shfl_sync(kFull, s.oa, 0); s.ga = __shfl_sync(kFull, s.ga, 0);
  s.ob = __shfl_sync(kFull, s.ob, 0); s.gb = __shfl_sync(kFull, s.gb, 0);
  if (s.te < 0) {
    if (lane == 0 && !quiet) report(c.st, K_STRUCT, poly);
    return false;
  }
  *out = s;
  return true;
}

// Arc split of piece X at tip position pos with the (already promoted) split
// info, re-walk fallback with the strict length law.
template <typename Alloc>
__device__ bool warp_split_arcs(const RepairCtx& c, const int32_t* X, int L, int pos, const SplitInfo& s,
                                int32_t poly, int lane, Alloc alloc, int32_t** A_out, int* la_out, int32_t** B_out,
                                int* lb_out) {
  const int32_t v = X[pos], u = s.u, a_in = s.a_in;
  int j = -1;
  if (a_in >= 0)
    j = warp_find_first(L, lane, [&](int q) { return X[q] == u && X[q == 0 ? L - 1 : q - 1] == a_in; });
  if (j >= 0) {
    int la = 1 + wrap_idx(pos - j, L), lb = wrap_idx(j - pos, L) + 1;
    // pa arc: A(0) = v, A(k) = X[(j+k-1) % L]; pb arc: B(k) = X[(pos+k) % L] (k < lb-1), B(lb-1) = u
    auto A_at = [&](int k) { return k == 0 ? v : X[wrap_idx(j + k - 1, L)]; };
    auto B_at = [&](int k) { return k == lb - 1 ? u : X[wrap_idx(pos + k, L)]; };
    int ka = warp_find_first(la, lane,
                             [&](int k) { return A_at(k) == s.oa && A_at(k + 1 == la ? 0 : k + 1) == s.ga; });
    int kb = warp_find_first(lb, lane,
                             [&](int k) { return B_at(k) == s.ob && B_at(k + 1 == lb ? 0 : k + 1) == s.gb; });
    if (ka >= 0 && kb >= 0) {
      int32_t* A = alloc(la + lb);
      if (A == nullptr) {
        if (lane == 0) report(c.st, K_POOL, poly);
        return false;
      }
      int32_t* B = A + la;
      warp_copy(A, la, lane, [&](int k) { return A_at(wrap_idx(ka + k, la)); });
      warp_copy(B, lb, lane, [&](int k) { return B_at(wrap_idx(kb + k, lb)); });
      __syncwarp();
      *A_out = A; *la_out = la; *B_out = B; *lb_out = lb;
      return true;
    }
  }
  int r = warp_rewalk_split(c, s.e, s.te, L, poly, alloc, lane, A_out, la_out, B_out, lb_out);
  if (r == 0 && lane == 0) report(c.st, K_SPLIT_LAW, poly);
  return r == 1;
}

// Tip split of piece X (len L) at its first tip (reparation.py:294-312 splitter).
template <typename Alloc>
__device__ bool warp_split_tip(const RepairCtx& c, const int32_t* X, int L, int32_t poly, int32_t* fan,
                               int32_t* back, int lane, Alloc alloc, int32_t** A_out, int* la_out, int32_t** B_out,
                               int* lb_out) {
  int pos = warp_first_tip(X, L, lane);
  if (pos < 0) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return false;
  }
  int32_t v = X[pos], b = X[pos == 0 ? L - 1 : pos - 1];
  SplitInfo s;
  if (!warp_split_info(c, v, b, poly, fan, back, lane, true, false, &s)) return false;
  return warp_split_arcs(c, X, L, pos, s, poly, lane, alloc, A_out, la_out, B_out, lb_out);
}

// Duplicate scan of s[0..n) (traversal.py:140-147 and the first-repeat search
// of reparation.py:184-189), one warp: a value -> first position hash map in
// pool scratch, so long pieces cost O(n), not O(n^2).  Returns the extra
// visits (n - distinct); *p1/*p2 = the first repeated position p2 and the
// first occurrence p1 of its value (-1 when none).
constexpr int kDupCap = 512;         // per-warp shared table in k_repair_tips (pieces up to 256 vertices)
constexpr int kPinchDupCap = 4096;   // per-warp shared table in k_repair_pinch (pieces up to 2048 vertices)
__device__ int warp_dup_scan(const RepairCtx& c, const int32_t* s, int n, int lane, int* p1, int* p2,
                             int2* stab = nullptr, int scap = kDupCap) {
#if defined(TM_NO_SHFL_SCAN) || defined(TM_NO_SHFL_DUP)
  if (n <= 64) {
    int extra = 0, q2 = -1, q1 = -1;
    for (int pb = 0; pb < n; pb += 32) {
      int p = pb + lane;
      int32_t x = p < n ? s[p] : 0;
      int first = -1;
      for (int q = 0; q < n && p < n; q++)
        if (s[q] == x) { first = q; break; }
      bool dup = p < n && first < p;
      unsigned m = __ballot_sync(kFull, dup);
      extra += __popc(m);
      if (m && q2 < 0) {
        int l = __ffs(m) - 1;
        q2 = pb + l;
        q1 = __shfl_sync(kFull, first, l);
      }
    }
    if (p1) *p1 = q1;
    if (p2) *p2 = q2;
    return extra;
  }
#else
  if (n <= 64) {  // in registers: lane l holds s[l] and s[32 + l]; first occurrences by match / shuffle
    // unused lanes (>= n) lie above every used one, so they never lower a used lane's
    // first occurrence; their own flags are masked off below (a piece may hold
    // negative values, so no sentinel is safe to count on)
    const int32_t x0 = lane < n ? s[lane] : -1 - lane;
    const int32_t x1 = lane + 32 < n ? s[lane + 32] : -33 - lane;
    const int f0 = __ffs(__match_any_sync(kFull, x0)) - 1;  // first position of s[lane] (within 0..31)
    int f1 = -1;
    if (n > 32) {  // (warp-uniform; the match runs on every lane, outside the per-lane branch)
      const unsigned m1x = __match_any_sync(kFull, x1);
      for (int q = 0; q < 32; q++)
        if (__shfl_sync(kFull, x0, q) == x1 && f1 < 0) f1 = q;
      if (f1 < 0) f1 = 32 + __ffs(m1x) - 1;
    }
    const unsigned m0 = __ballot_sync(kFull, lane < n && f0 < lane);
    const unsigned m1 = __ballot_sync(kFull, lane + 32 < n && f1 < lane + 32);
    int q2 = -1, q1 = -1;
    if (m0) {
      q2 = __ffs(m0) - 1;
      q1 = __shfl_sync(kFull, f0, q2);
    } else if (m1) {
      const int l = __ffs(m1) - 1;
      q2 = 32 + l;
      q1 = __shfl_sync(kFull, f1, l);
    }
    if (p1) *p1 = q1;
    if (p2) *p2 = q2;
    return __popc(m0) + __popc(m1);
  }
#endif
  int cap = 64;
  while (cap < 2 * n) cap <<= 1;
  const bool shared = stab != nullptr && cap <= scap;
  int2* tab = stab;
  if (!shared) {
    long long o = 0;
    if (lane == 0) {
      o = palloc(c, 2 * (long long)cap + 1);
      if (o >= 0) o = (o + 1) & ~1LL;  // int2 alignment
    }
    o = __shfl_sync(kFull, o, 0);
    if (o < 0) {  // pool exhausted: quadratic fallback
      if (lane == 0) report(c.st, K_POOL, -1);
      if (p1) *p1 = -1;
      if (p2) *p2 = -1;
      return warp_extra_visits(s, n, lane);
    }
    tab = reinterpret_cast<int2*>(c.pool + o);
  }
  for (int k = lane; k < cap; k += 32) tab[k] = make_int2(-1, 0x7FFFFFFF);
  __syncwarp();
  for (int p = lane; p < n; p += 32) {
    int32_t x = s[p];
    uint32_t slot = ((uint32_t)x * 0x9E3779B1u) & (cap - 1);
    for (;;) {
      int prev = atomicCAS(&tab[slot].x, -1, x);
      if (prev == -1 || prev == x) { atomicMin(&tab[slot].y, p); break; }
      slot = (slot + 1) & (cap - 1);
    }
  }
  __syncwarp();
  __threadfence_block();
  int extra = 0, q2 = -1, q1 = -1;
  for (int pb = 0; pb < n; pb += 32) {
    int p = pb + lane, first = -1;
    if (p < n) {
      int32_t x = s[p];
      uint32_t slot = ((uint32_t)x * 0x9E3779B1u) & (cap - 1);
      for (;;) {
        int2 e = shared ? tab[slot] : __ldcg(&tab[slot]);
        if (e.x == x) { first = e.y; break; }
        slot = (slot + 1) & (cap - 1);
      }
    }
    bool dup = p < n && first < p;
    unsigned m = __ballot_sync(kFull, dup);
    extra += __popc(m);
    if (m && q2 < 0) {
      int l = __ffs(m) - 1;
      q2 = pb + l;
      q1 = __shfl_sync(kFull, first, l);
    }
  }
  if (p1) *p1 = q1;
  if (p2) *p2 = q2;
  return extra;
}

// ------------------------------------------------------------ pinch phase
// reparation.py:315-340 per item, one warp, after every item's tip phase:
// the round guard is GLOBAL (extra visits of the whole tip-phase output + 1,
// reparation.py:322) and does bind on small meshes.  Rounds follow the
// reference: every eligible piece (repeated vertex, no tip, not failed
// before) gets one candidate sweep per round; the loop ends when a round
// splits nothing or the guard is reached.  Items cut off by the guard with
// pinched pieces left are counted (TM_STAT_PINCH_TRUNCATED) so a seed-
// partitioned run can check that its local guard equals the global one.

// Trial split at candidate g with strict=False (reparation.py:326-332):
// promote, re-walk both sides (lanes 0 and 1 at once) into fresh pool slots,
// keep iff |pa| + |pb| == L + 2, else revert.  Warp-uniform result: 1 split,
// 0 reverted, -1 error.
__device__ int warp_try_pinch(const RepairCtx& c, int32_t g, int L, int32_t poly, int lane, int32_t** A, int* la,
                              int32_t** B, int* lb) {
  int32_t w = hw_twin(c.hw[g]);
  if (w < 0) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return -1;
  }
  long long o = 0;
  if (lane == 0) {
    o = palloc(c, 2 * (long long)L + 4);
    if (o >= 0) promote(c, g, w);
  }
  o = __shfl_sync(kFull, o, 0);
  if (o < 0) {
    if (lane == 0) report(c.st, K_POOL, poly);
    return -1;
  }
  __syncwarp();
  int cnt = 0, err = 0, over = 0;
  if (lane < 2) {
    int32_t* dst = c.pool + o + (lane ? L + 2 : 0);
    const int32_t h0 = min_frontier_slot(c.hw, lane ? w / 3 : g / 3);
    const long long limit = 3 * c.T + 3;
    int32_t h = h0;
    if (h0 < 0) err = 1;
    else
      do {
        if (cnt > L + 1) { over = 1; break; }
        dst[cnt++] = he_origin(c.tri, h);
        h = walk_next(c.hw, h, limit);
        if (h < 0) { err = 1; break; }
      } while (h != h0);
  }
  const int ca = __shfl_sync(kFull, cnt, 0), cb = __shfl_sync(kFull, cnt, 1);
  err = __shfl_sync(kFull, err, 0) | __shfl_sync(kFull, err, 1);
  over = __shfl_sync(kFull, over, 0) | __shfl_sync(kFull, over, 1);
  if (err) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return -1;
  }
  if (over || ca + cb != L + 2) {
    if (lane == 0) demote(c, g, w);
    __syncwarp();
    return 0;
  }
  *A = c.pool + o;
  *la = ca;
  *B = c.pool + o + L + 2;
  *lb = cb;
  return 1;
}

// incoming boundary vertex of the wedge around origin(g) that holds g: rotate
// CCW from g until the crossed edge prev(.) is frontier (pre-promotion flags)
__device__ __forceinline__ int32_t wedge_in_vertex(const RepairCtx& c, int32_t g) {
  long long guard = 3 * c.T + 3;
  for (long long k = 0; k < guard; k++) {
    int32_t p = he_prev(g);
    int32_t w = c.hw[p];
    if (hw_front(w)) return he_origin(c.tri, p);
    g = hw_twin(w);
    if (g < 0) return -1;
  }
  return -1;
}

// Arc trial of candidate g = x -> y (strict=False).  With the pre-promotion
// frontier, the visit of x whose wedge holds g and the visit of y whose wedge
// holds twin(g) cut X into exactly the two cycles the re-walks would trace
// (as for tip splits), so |pa| + |pb| = L + 2 holds by
// construction; when y is not on X the promoted edge dangles inside the
// region, both re-walks trace one cycle of length L + 2 and the law fails.
// Anything else (a wedge or rotation search that fails) takes the re-walk
// trial.  Warp-uniform: 1 split, 0 reverted / not split, -1 error.
__device__ int warp_try_pinch_arc(const RepairCtx& c, int32_t g, const int32_t* X, int L, int32_t poly, int lane,
                                  int32_t** A, int* la_out, int32_t** B, int* lb_out) {
  int32_t w = -1, x = -1, y = -1, ax = -1, ay = -1;
  if (lane == 0) {
    w = hw_twin(c.hw[g]);
    x = he_origin(c.tri, g);
    y = he_target(c.tri, g);
    if (w >= 0) {
      ax = wedge_in_vertex(c, g);
      ay = wedge_in_vertex(c, w);
    }
  }
  w = __shfl_sync(kFull, w, 0);
  x = __shfl_sync(kFull, x, 0);
  y = __shfl_sync(kFull, y, 0);
  ax = __shfl_sync(kFull, ax, 0);
  ay = __shfl_sync(kFull, ay, 0);
  if (w < 0) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return -1;
  }
  if (warp_find_first(L, lane, [&](int q) { return X[q] == y; }) < 0) return 0;  // y interior: no split
  const int pos = ax < 0 ? -1 : warp_find_first(L, lane, [&](int q) { return X[q] == x && X[q == 0 ? L - 1 : q - 1] == ax; });
  const int j = ay < 0 ? -1 : warp_find_first(L, lane, [&](int q) { return X[q] == y && X[q == 0 ? L - 1 : q - 1] == ay; });
  if (pos < 0 || j < 0) return warp_try_pinch(c, g, L, poly, lane, A, la_out, B, lb_out);
  int32_t oa = 0, ga = 0, ob = 0, gb = 0;
  if (lane == 0) {
    promote(c, g, w);
    int32_t ha = min_frontier_slot(c.hw, g / 3), hb = min_frontier_slot(c.hw, w / 3);
    oa = he_origin(c.tri, ha); ga = he_target(c.tri, ha);
    ob = he_origin(c.tri, hb); gb = he_target(c.tri, hb);
  }
  oa = __shfl_sync(kFull, oa, 0); ga = __shfl_sync(kFull, ga, 0);
  ob = __shfl_sync(kFull, ob, 0); gb = __shfl_sync(kFull, gb, 0);
  const int la = wrap_idx(pos - j, L) + 1, lb = wrap_idx(j - pos, L) + 1;
  // pa = [x, X[j .. pos-1]], pb = [X[pos .. j-1], y]
  auto A_at = [&](int k) { return k == 0 ? x : X[wrap_idx(j + k - 1, L)]; };
  auto B_at = [&](int k) { return k == lb - 1 ? y : X[wrap_idx(pos + k, L)]; };
  const int ka = warp_find_first(la, lane, [&](int k) { return A_at(k) == oa && A_at(k + 1 == la ? 0 : k + 1) == ga; });
  const int kb = warp_find_first(lb, lane, [&](int k) { return B_at(k) == ob && B_at(k + 1 == lb ? 0 : k + 1) == gb; });
  if (ka < 0 || kb < 0) {
    if (lane == 0) demote(c, g, w);
    __syncwarp();
    return warp_try_pinch(c, g, L, poly, lane, A, la_out, B, lb_out);
  }
  long long o = 0;
  if (lane == 0) o = palloc(c, (long long)la + lb);
  o = __shfl_sync(kFull, o, 0);
  if (o < 0) {
    if (lane == 0) report(c.st, K_POOL, poly);
    return -1;
  }
  int32_t* pa = c.pool + o;
  int32_t* pb = pa + la;
  warp_copy(pa, la, lane, [&](int k) { return A_at(wrap_idx(ka + k, la)); });
  warp_copy(pb, lb, lane, [&](int k) { return B_at(wrap_idx(kb + k, lb)); });
  __syncwarp();
  *A = pa; *la_out = la; *B = pb; *lb_out = lb;
  return 1;
}

// Half-edge with origin v in the reference's trivertex triangle (the lowest
// incident one, mesh_core.py:171-178): the pinch candidates iterate the fan
// from there.  Without an exact trivertex the full fan is walked
// once from any incident triangle and its minimum taken.
__device__ int32_t trivertex_he(const RepairCtx& c, int32_t v, int guard) {
  int32_t t0 = c.tv[v];
  int32_t g0 = t0 < 0 ? -1 : he_with_origin(c.tri, t0, v);
  if (g0 < 0 || c.tv_exact) return g0;
  int32_t g = g0, best = g0;
  int k = 0;
  do {
    if (g / 3 < best / 3) best = g;
    g = fan_step(c.hw, g, guard);
    if (g < 0 || ++k > guard) return -1;
  } while (g != g0);
  return best;
}

// _pinch_candidates (reparation.py:169-205) for one piece, candidates in the
// reference order, each trial-split until one keeps.  Every lane runs the
// (identical) candidate enumeration so the trials stay warp-convergent.
// Fan of v collected once (two walkers) and rotated to the reference anchor,
// the half-edge of the lowest incident triangle (_fan_at_vertex / trivertex,
// reparation.py:91-124): returns deg (fan[(anchor + i) % deg] is the i-th
// half-edge in fan_step order), or -1 when the fan does not fit kFanCap.
__device__ int warp_anchored_fan(const RepairCtx& c, int32_t v, int32_t* fan, int32_t* back, int lane, int* anchor) {
  const int deg = warp_collect_fan(c, v, fan, back, lane);
  if (deg < 1 || deg > kFanCap) return -1;
  int best_t = 0x7FFFFFFF, best_k = 0;
  for (int k = lane; k < deg; k += 32) {
    const int t = fan[k] / 3;
    if (t < best_t) { best_t = t; best_k = k; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int ot = __shfl_xor_sync(kFull, best_t, o), ok = __shfl_xor_sync(kFull, best_k, o);
    if (ot < best_t || (ot == best_t && ok < best_k)) { best_t = ot; best_k = ok; }
  }
  *anchor = best_k;
  return deg;
}

__device__ int warp_pinch_split_slow(const RepairCtx& c, const int32_t* X, int L, int32_t poly, int lane, int32_t** A,
                                     int* la, int32_t** B, int* lb, int p1, int p2);

// _pinch_candidates with the fans held in shared memory (the frontier bits are
// read per candidate sweep: a failed trial is reverted before the next one).
// Falls back to the rotation-by-rotation enumeration when a fan exceeds kFanCap.
__device__ int warp_pinch_split(const RepairCtx& c, const int32_t* X, int L, int32_t poly, int lane, int32_t** A,
                                int* la, int32_t** B, int* lb, int2* stab) {
  long long ck0 = clock64();
  int p1 = -1, p2 = -1;  // first repeated vertex (reparation.py:184-189)
  warp_dup_scan(c, X, L, lane, &p1, &p2, stab, kPinchDupCap);
  if (c.dbg && lane == 0) { atomicAdd(c.dbg + 64, (unsigned long long)(clock64() - ck0)); atomicMax(c.dbg + 70, (unsigned long long)L); }
  if (p2 < 0) return 0;
  // the duplicate table is free until the caller scans the children: fan buffers
  int32_t* fan = reinterpret_cast<int32_t*>(stab);
  int32_t* back = fan + kFanCap;
  int anc = 0;
  int deg = warp_anchored_fan(c, X[p2], fan, back, lane, &anc);
  if (deg < 0) return warp_pinch_split_slow(c, X, L, poly, lane, A, la, B, lb, p1, p2);
  __syncwarp();
  const int poss[2] = {p2, p1};
  for (int q = 0; q < 2; q++) {  // wedge internal edges at the second, then the first visit
    const int32_t outv = X[(poss[q] + 1) % L];
    const int i_out = warp_find_first(deg, lane, [&](int i) {
      const int32_t g = fan[(anc + i) % deg];
      return hw_front(c.hw[g]) && he_target(c.tri, g) == outv;
    });
    if (i_out < 0) {
      if (lane == 0) report(c.st, K_STRUCT, poly);
      return -1;
    }
    const int j = warp_find_first(deg - 1, lane, [&](int t) { return hw_front(c.hw[fan[(anc + i_out + 1 + t) % deg]]); });
    const int k = j < 0 ? deg - 1 : j;
    if (k == 0) continue;
    const int mid = (k - 1) / 2;
    for (int ord = -1; ord < k; ord++) {  // middle edge first, then the rest in order
      const int idx = ord < 0 ? mid : ord;
      if (ord == mid) continue;
      const int32_t cand = fan[(anc + i_out + 1 + idx) % deg];
      long long ckt = clock64();
      int r = warp_try_pinch_arc(c, cand, X, L, poly, lane, A, la, B, lb);
      if (c.dbg && lane == 0) { atomicAdd(c.dbg + 65, (unsigned long long)(clock64() - ckt)); atomicAdd(c.dbg + 66, 1ull); }
      if (r != 0) return r;
    }
  }
  for (int idx = p1 + 1; idx < p2; idx++) {  // internal fan edges of the inner-loop vertices
    deg = warp_anchored_fan(c, X[idx], fan, back, lane, &anc);
    if (deg < 0) return warp_pinch_split_slow(c, X, L, poly, lane, A, la, B, lb, -idx - 2, p2);  // resume at idx
    __syncwarp();
    for (int base = 0; base < deg; base += 32) {
      const int i = base + lane;
      const bool inner = i < deg && !hw_front(c.hw[fan[(anc + i) % deg]]);
      unsigned m = __ballot_sync(kFull, inner);
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int32_t g = fan[(anc + base + b) % deg];
        long long ckt = clock64();
        int r = warp_try_pinch_arc(c, g, X, L, poly, lane, A, la, B, lb);
        if (c.dbg && lane == 0) { atomicAdd(c.dbg + 65, (unsigned long long)(clock64() - ckt)); atomicAdd(c.dbg + 67, 1ull); }
        if (r != 0) return r;
      }
    }
  }
  return 0;
}

// The rotation-by-rotation enumeration (fans larger than kFanCap).  p1 < -1
// encodes a resume at inner vertex idx = -p1 - 2 (the wedges are done).
__device__ int warp_pinch_split_slow(const RepairCtx& c, const int32_t* X, int L, int32_t poly, int lane, int32_t** A,
                                     int* la, int32_t** B, int* lb, int p1, int p2) {
  int first_inner = -1;
  if (p1 < -1) {
    first_inner = -p1 - 2;
    int q1 = -1, q2 = -1;
    warp_dup_scan(c, X, L, lane, &q1, &q2);
    p1 = q1;
  }
  const int32_t v = X[p2];
  const int guard = (int)(3 * c.T + 3 < (1LL << 30) ? 3 * c.T + 3 : (1LL << 30));
  int32_t g0 = trivertex_he(c, v, guard);
  if (g0 < 0) {
    if (lane == 0) report(c.st, K_STRUCT, poly);
    return -1;
  }
  int deg = 0;
  {
    int32_t g = g0;
    do {
      deg++;
      g = fan_step(c.hw, g, guard);
      if (g < 0 || deg > guard) {
        if (lane == 0) report(c.st, K_STRUCT, poly);
        return -1;
      }
    } while (g != g0);
  }
  const int poss[2] = {p2, p1};
  for (int q = first_inner < 0 ? 0 : 2; q < 2; q++) {  // wedge internal edges at the second, then the first visit
    int32_t outv = X[(poss[q] + 1) % L];
    int32_t g = g0, gout = -1;
    for (int st = 0; st < deg; st++) {
      if (hw_front(c.hw[g]) && he_target(c.tri, g) == outv) { gout = g; break; }
      g = fan_step(c.hw, g, guard);
    }
    if (gout < 0) {
      if (lane == 0) report(c.st, K_STRUCT, poly);
      return -1;
    }
    int k = 0;
    g = fan_step(c.hw, gout, guard);
    for (int st = 1; st < deg; st++) {
      if (hw_front(c.hw[g])) break;
      k++;
      g = fan_step(c.hw, g, guard);
    }
    if (k == 0) continue;
    const int mid = (k - 1) / 2;
    for (int ord = -1; ord < k; ord++) {  // middle edge first, then the rest in order
      int idx = ord < 0 ? mid : ord;
      if (ord == mid) continue;
      int32_t cand = gout;
      for (int st = 0; st <= idx; st++) cand = fan_step(c.hw, cand, guard);
      long long ckt = clock64();
      int r = warp_try_pinch_arc(c, cand, X, L, poly, lane, A, la, B, lb);
      if (c.dbg && lane == 0) { atomicAdd(c.dbg + 65, (unsigned long long)(clock64() - ckt)); atomicAdd(c.dbg + 66, 1ull); }
      if (r != 0) return r;
    }
  }
  for (int idx = first_inner < 0 ? p1 + 1 : first_inner; idx < p2; idx++) {  // internal fan edges of the inner-loop vertices
    int32_t x = X[idx];
    int32_t gx0 = trivertex_he(c, x, guard);
    if (gx0 < 0) {
      if (lane == 0) report(c.st, K_STRUCT, poly);
      return -1;
    }
    int32_t g = gx0;
    int cnt = 0;
    do {
      if (!hw_front(c.hw[g])) {
        long long ckt = clock64();
        int r = warp_try_pinch_arc(c, g, X, L, poly, lane, A, la, B, lb);
        if (c.dbg && lane == 0) { atomicAdd(c.dbg + 65, (unsigned long long)(clock64() - ckt)); atomicAdd(c.dbg + 67, 1ull); }
        if (r != 0) return r;
      }
      g = fan_step(c.hw, g, guard);
      if (g < 0 || ++cnt > guard) {
        if (lane == 0) report(c.st, K_STRUCT, poly);
        return -1;
      }
    } while (g != gx0);
  }
  return 0;
}

// Pinch rounds of item w (record list in the pool) and its output totals.
// Rounds r0, r0+1, ... of item w under `guard`.  With `park`, guard is only a
// lower bound of the global one (the extra visits summed so far): reaching it
// with pinched pieces left parks the item (state 4, next round in item_depth)
// for the final pass instead of ending its loop.
struct PinchPark {
  int32_t* item_state = nullptr;
  int32_t* item_depth = nullptr;
  int32_t* list = nullptr;
  unsigned int* n = nullptr;
  unsigned long long* deferred = nullptr;  // counts items parked at the FINAL local guard (seed partition)
};
__device__ void warp_finish_pinch(const RepairCtx& c, int64_t w, int32_t poly, long long list, int n, int lane,
                                  int64_t* item_list, int32_t* item_n, int64_t* item_slots,
                                  unsigned long long* stats, long long guard, int2* stab, long long r0 = 0,
                                  PinchPark park = PinchPark()) {
  bool ok = true, truncated = false;
  for (long long r = r0; ok; r++) {
    int elig = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      int k = k0 + lane;
      bool e = false;
      if (k < n) {
        uint32_t rl = (uint32_t)c.pool[list + 2 * k + 1];
        e = (rl & F_REP) && !(rl & F_TIP) && !(rl & F_FAIL);
      }
      elig += __popc(__ballot_sync(kFull, e));
    }
    if (elig == 0) break;
    if (r >= guard) {
      if (park.list) {  // whether the global guard allows round r is not known yet
        // a consistent (provisional) output size for the stitch that may run
        // before the item is finished (seed partition, tm_resume_pinch follows)
        long long ps = 0;
        for (int k = lane; k < n; k += 32) ps += (uint32_t)c.pool[list + 2 * k + 1] & LEN_MASK;
        for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(kFull, ps, o);
        if (lane == 0) {
          item_slots[w] = ps;
          item_list[w] = list;
          item_n[w] = n;
          park.item_depth[w] = (int32_t)r;
          park.item_state[w] = 4;
          park.list[atomicAdd(park.n, 1u)] = (int32_t)w;
          if (park.deferred) atomicAdd(park.deferred, 1ull);
        }
        return;
      }
      truncated = true;  // the reference's loop ends here with pinched polygons left
      break;
    }
    long long nl = 0;
    if (lane == 0) nl = palloc(c, 2 * (long long)(n + elig));
    nl = __shfl_sync(kFull, nl, 0);
    if (nl < 0) {
      if (lane == 0) report(c.st, K_POOL, poly);
      ok = false;
      break;
    }
    int m = 0, did = 0;
    for (int k = 0; k < n && ok; k++) {
      uint32_t ro = (uint32_t)c.pool[list + 2 * k], rl = (uint32_t)c.pool[list + 2 * k + 1];
      if ((rl & F_REP) && !(rl & F_TIP) && !(rl & F_FAIL)) {
        int32_t *A, *B;
        int al, bl;
        long long cks = clock64();
        int res = warp_pinch_split(c, c.pool + ro, (int)(rl & LEN_MASK), poly, lane, &A, &al, &B, &bl, stab);
        if (c.dbg && lane == 0) { atomicAdd(c.dbg + 68, (unsigned long long)(clock64() - cks)); atomicAdd(c.dbg + 69, 1ull); }
        if (res < 0) { ok = false; break; }
        if (res == 1) {
          long long ckf = clock64();
          uint32_t fa = warp_tip_flag(A, al, lane) | (warp_dup_scan(c, A, al, lane, nullptr, nullptr, stab, kPinchDupCap) > 0 ? F_REP : 0u);
          uint32_t fb = warp_tip_flag(B, bl, lane) | (warp_dup_scan(c, B, bl, lane, nullptr, nullptr, stab, kPinchDupCap) > 0 ? F_REP : 0u);
          if (c.dbg && lane == 0) atomicAdd(c.dbg + 71, (unsigned long long)(clock64() - ckf));
          if (lane == 0) {
            c.pool[nl + 2 * m] = (int32_t)(A - c.pool);
            c.pool[nl + 2 * m + 1] = (int32_t)((uint32_t)al | fa);
            c.pool[nl + 2 * m + 2] = (int32_t)(B - c.pool);
            c.pool[nl + 2 * m + 3] = (int32_t)((uint32_t)bl | fb);
          }
          m += 2;
          did++;
          continue;
        }
        rl |= F_FAIL;  // a failed pinch fails identically in every later round
      }
      if (lane == 0) {
        c.pool[nl + 2 * m] = (int32_t)ro;
        c.pool[nl + 2 * m + 1] = (int32_t)rl;
      }
      m++;
    }
    __syncwarp();
    if (!ok) break;
    list = nl;
    n = m;
    if (did && lane == 0) atomicAdd(stats + 4, (unsigned long long)did);
    if (did == 0) break;
  }
  if (!ok) {
    if (lane == 0) { item_list[w] = -1; item_n[w] = 0; item_slots[w] = 0; }
    return;
  }
  long long slots = 0;
  unsigned long long unrep = 0;
  for (int k0 = 0; k0 < n; k0 += 32) {
    int k = k0 + lane;
    if (k < n) {
      uint32_t rl = (uint32_t)c.pool[list + 2 * k + 1];
      slots += rl & LEN_MASK;
      unrep += (rl & F_REP) ? 1 : 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    slots += __shfl_xor_sync(kFull, slots, o);
    unrep += __shfl_xor_sync(kFull, unrep, o);
  }
  if (lane == 0) {
    item_list[w] = list;
    item_n[w] = n;
    item_slots[w] = slots;
    if (unrep) atomicAdd(stats + 3, unrep);
    if (truncated) atomicAdd(stats + 7, 1ull);
  }
}

// ------------------------------------------------------------ tip phase, global pool
// Item states (item_state[w]): 0 = not started, 1 = finished by the shared-
// memory kernel, 2 = resume from item_list/item_n/item_depth in the pool.

// With a pinch queue (short items, k_repair_tips mode 0): an item without a
// pinch candidate (no repeated leaf; the tip phase left no tips) is complete
// here and gets its output size; the others are queued for k_repair_pinch.
__device__ void finish_item(const RepairCtx& c, int64_t w, long long list, int n, long long depth, long long splits,
                            int lane, int64_t* item_list, int32_t* item_n, unsigned long long* stats, int2* stab,
                            int64_t* item_slots = nullptr, int32_t* pq = nullptr, unsigned int* n_pq = nullptr) {
  // repeated flags and extra visits of the leaves (pinch guard, reparation.py:322)
  unsigned long long ex_sum = 0;
  long long slots = 0;
  int elig = 0;
  for (int r = 0; r < n; r++) {
    uint32_t ro = (uint32_t)c.pool[list + 2 * r], rl = (uint32_t)c.pool[list + 2 * r + 1];
    int ex = warp_dup_scan(c, c.pool + ro, (int)(rl & LEN_MASK), lane, nullptr, nullptr, stab);
    if (ex > 0 && lane == 0) c.pool[list + 2 * r + 1] = (int32_t)(rl | F_REP);
    ex_sum += ex;
    slots += rl & LEN_MASK;
    elig += (ex > 0 && !(rl & (F_TIP | F_FAIL))) ? 1 : 0;
  }
  __syncwarp();
  if (lane == 0) {
    item_list[w] = list;
    item_n[w] = n;
    if (pq) {
      if (elig == 0) item_slots[w] = slots;
      else pq[atomicAdd(n_pq, 1u)] = (int32_t)w;
    }
    if (depth > 0) atomicMax(stats + 0, (unsigned long long)depth);
    if (splits) atomicAdd(stats + 1, (unsigned long long)splits);
    if (ex_sum) atomicAdd(stats + 5, ex_sum);
  }
}

// One warp per work item.  item_list[w] = pool offset of the item's record
// list, item_n[w] = #records (leaves in the reference's raw order).
#ifndef TM_TIP_MINB
#define TM_TIP_MINB 8  // resident blocks per SM the register budget is cut for (A/B builds vary it)
#endif
__global__ void __launch_bounds__(32 * kTipWarps, TM_TIP_MINB) k_repair_tips(RepairCtx c, const int32_t* __restrict__ items,
                                                                const unsigned int* n_items,
                                                                const int64_t* __restrict__ off,
                                                                const int32_t* __restrict__ v,
                                                                int64_t* __restrict__ item_list,
                                                                int32_t* __restrict__ item_n,
                                                                const int32_t* __restrict__ item_state,
                                                                const int32_t* __restrict__ item_depth,
                                                                int64_t* __restrict__ item_slots,
                                                                unsigned long long* stats, LongQueue q, int mode) {
  __shared__ int32_t s_fan[kTipWarps][kFanCap];
  __shared__ int32_t s_back[kTipWarps][kFanCap];
  __shared__ int2 s_dup[kTipWarps][kDupCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* fan = s_fan[wib];
  int32_t* back = s_back[wib];
  const unsigned int nh = mode ? *q.n_huge : 0u;
  const unsigned int ni = mode ? nh + *q.n_long : *n_items;
  // reparation.py:354-364: at most initial + 1 rounds, initial = extra visits of mesh0
  long long max_rounds = (long long)stats[2] + 1;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // mode 0: persistent warps pull items from a counter (item costs vary by 10x)
  auto next_item = [&]() -> int64_t {
    unsigned int x = 0;
    if (lane == 0) x = atomicAdd(q.tip_next, 1u);
    return (int64_t)__shfl_sync(kFull, x, 0);
  };
  for (int64_t wq = mode ? warp : next_item(); wq < ni; wq = mode ? wq + nwarps : next_item()) {
    const int64_t w = !mode ? wq : (wq < nh ? q.huge[wq] : q.longq[wq - nh]);
    int32_t i = items[w];
    int64_t b = off[i];
    int L = (int)(off[i + 1] - b);
    int st = 0;
    if (!mode) {
      if (L > kLongMin) continue;  // k_repair_tips_long runs it concurrently
    } else {
      st = item_state[w];
      if (st != 2 && st != 3) continue;
    }
    WarpArena arena;
    auto alloc = [&](long long n) -> int32_t* {
      long long o = warp_alloc(c, arena, n, 2 * (long long)L + 512, lane);
      return o < 0 ? nullptr : c.pool + o;
    };
    long long list;
    int n, ntips = 0;
    long long depth = 0, splits = 0;
    if (st == 2) {
      list = item_list[w];
      n = item_n[w];
      depth = item_depth[w];
      for (int r = 0; r < n; r++) ntips += (((uint32_t)c.pool[list + 2 * r + 1]) & F_TIP) ? 1 : 0;
    } else {
      int32_t* P0 = alloc(L + 2);
      if (P0 == nullptr) {
        if (lane == 0) { report(c.st, K_POOL, i); item_list[w] = -1; item_n[w] = 0; item_slots[w] = 0; }
        continue;
      }
      warp_copy(P0, L, lane, [&](int k) { return v[b + k]; });
      __syncwarp();
      list = (P0 - c.pool) + L;
      uint32_t f0 = warp_tip_flag(P0, L, lane);
      if (lane == 0) {
        c.pool[list] = (int32_t)(P0 - c.pool);
        c.pool[list + 1] = (int32_t)((uint32_t)L | f0);
      }
      __syncwarp();
      n = 1;
      ntips = f0 ? 1 : 0;
    }
    bool bad = false;
    while (ntips > 0 && !bad) {
      depth++;
      if (depth > max_rounds) {
        if (lane == 0) report(c.st, K_NO_CONVERGE, i);
        bad = true;
        break;
      }
      int32_t* nlp = alloc(2 * (long long)(n + ntips));
      if (nlp == nullptr) {
        if (lane == 0) report(c.st, K_POOL, i);
        bad = true;
        break;
      }
      long long nl = nlp - c.pool;
      int m = 0, nt = 0;
      for (int r = 0; r < n; r++) {
        uint32_t ro = (uint32_t)c.pool[list + 2 * r], rl = (uint32_t)c.pool[list + 2 * r + 1];
        if (!(rl & F_TIP)) {
          if (lane == 0) {
            c.pool[nl + 2 * m] = (int32_t)ro;
            c.pool[nl + 2 * m + 1] = (int32_t)rl;
          }
          m++;
          continue;
        }
        int32_t *A, *B;
        int al, bl;
        if (!warp_split_tip(c, c.pool + ro, (int)(rl & LEN_MASK), i, fan, back, lane, alloc, &A, &al, &B, &bl)) {
          bad = true;
          break;
        }
        uint32_t fa = warp_tip_flag(A, al, lane), fb = warp_tip_flag(B, bl, lane);
        if (lane == 0) {
          c.pool[nl + 2 * m] = (int32_t)(A - c.pool);
          c.pool[nl + 2 * m + 1] = (int32_t)((uint32_t)al | fa);
          c.pool[nl + 2 * m + 2] = (int32_t)(B - c.pool);
          c.pool[nl + 2 * m + 3] = (int32_t)((uint32_t)bl | fb);
        }
        m += 2;
        nt += (fa ? 1 : 0) + (fb ? 1 : 0);
        splits++;
      }
      __syncwarp();
      list = nl;
      n = m;
      ntips = nt;
    }
    if (bad) {
      if (lane == 0) { item_list[w] = -1; item_n[w] = 0; item_slots[w] = 0; }
      continue;
    }
    if (mode) finish_item(c, w, list, n, depth, splits, lane, item_list, item_n, stats, s_dup[wib]);
    else finish_item(c, w, list, n, depth, splits, lane, item_list, item_n, stats, s_dup[wib], item_slots, q.pinchq,
                     q.n_pinch);
  }
}

// ------------------------------------------------------------ tip phase, segment pieces
// Long items (hull slivers: 902 vertices / 70 tips / 41 rounds at 1M, 3210 /
// 219 / 142 at 10M): one block each.  The item's original cycle P stays in
// shared memory and every piece is a short list of SEGMENTS -- a cyclic range
// of P or one inserted vertex -- because a tip split only cuts its parent into
// two arcs and adds one vertex to each.  All per-round queries
// run over segments instead of vertices:
//   first tip      tip bitmap of P for segment interiors, explicit checks at the
//                  (few) segment junctions;
//   cut / rotation the directed boundary pair (x, y) is unique in a piece: a
//                  hash map pair -> index of P answers it for segment interiors,
//                  junctions again explicitly.
// So a split costs O(#segments), not O(|piece|).  The mesh rotations of every
// tip of P (split edge, wedge vertex, re-walk start pairs) run up front, in
// parallel; a round reuses them unless an earlier promotion touched v or u.
// Leaves are expanded into the global pool at the end.  If the segment arena
// or the record list would overflow, the current pieces go to the pool and the
// warp kernel resumes the item (item_state = 2).
constexpr int kSegWarps = 16;
constexpr int kSegMaxL = 8192;   // longer items keep their per-item arrays in global memory (below)
// Items longer than kSegMaxL (the hull-sliver polygon passes 10^4 vertices at
// 100M points) keep P, its tip bitmap / ranks, the pair map and nexttip in a
// block-private region of the repair pool instead of shared memory (the
// segment lists and piece records stay in shared memory); longer than
// kSegMaxG: the warp kernel from scratch (state 3).  3 kSegMaxG < 2^16 keeps
// the 16-bit piece lengths and nexttip entries valid.
constexpr int kSegMaxG = 21760;
constexpr int kGPairCap = 65536;  // >= 2 kSegMaxG, power of two
constexpr int kGRec = 8192;       // piece records per round list (very long items)
constexpr int kGmBlocks = 6;      // blocks of k_repair_tips_seg that take the pool-region items (several huge hull slivers at 100M)
constexpr int kGSegCap = 262144;  // segment arena (very long items)
// pool region of a pool-region block: pair map, round lists, records, segment arena (ints)
constexpr long long kGStride = (long long)kGPairCap + 2 * (long long)kGRec + 2 * (long long)kGRec * 5 +
                               2 * (long long)kGSegCap + 64;
constexpr int kPairCap = 16384;  // pair-map slots (>= 2 kSegMaxL); reused as leaf hash sets
constexpr int kSegRec = 1024;    // piece records per round list
constexpr int kSegTips = 512;    // precomputed tips per item
constexpr int kSegTouch = 2048;  // hash set of promoted-edge endpoints (load <= 1/2)
constexpr int kSmemMax = 226 * 1024;  // dynamic; leaves room for the static __shared__ words

struct Seg {
  int32_t base;        // >= 0: P[(base + i) mod L], i < len; < 0: the vertex ~base (len 1)
  uint16_t len, loff;  // pieces are shorter than 3 kSegMaxL < 2^16
};
__device__ __forceinline__ Seg mkseg(int32_t base, int len, int loff) { Seg r; r.base = base; r.len = (uint16_t)len; r.loff = (uint16_t)loff; return r; }
struct SPiece {
  int32_t soff, nseg, len, ftip;  // segments [soff, soff + nseg), first tip position (-1: none)
  int32_t fk;                     // index in P of the first tip's vertex (-1: not a range element)
};

constexpr size_t kSegFixed = (size_t)kSegMaxL * 4 + (kSegMaxL / 32) * 4 + (size_t)kPairCap * 4 +
                             2 * (size_t)kSegRec * sizeof(SPiece) + (size_t)kSegRec * 4 +
                             2 * (size_t)kSegWarps * kFanCap * 4 + 2 * (size_t)kSegTips * 4 +
                             (size_t)kSegTips * sizeof(SplitInfo) + (size_t)kSegTouch * 4 +
                             2 * (kSegMaxL / 32 + 1) * 4 + (size_t)kSegMaxL * 2 + (size_t)kSegTips * 4 +
                             (size_t)kSegRec * 4 + 128;
constexpr int kSegCap = (int)((kSmemMax - kSegFixed) / sizeof(Seg));
size_t seg_smem_bytes() { return kSegFixed + (size_t)kSegCap * sizeof(Seg); }
// the pool-region instantiation's shared layout (P, tip bitmap / ranks, nexttip for kSegMaxG, fans, tips)
constexpr size_t kSegGFixed = (size_t)kSegMaxG * 4 + 3 * (size_t)(kSegMaxG / 32 + 1) * 4 + (size_t)kSegMaxG * 2 +
                              2 * (size_t)kSegWarps * kFanCap * 4 + 2 * (size_t)kSegTips * 4 +
                              (size_t)kSegTips * sizeof(SplitInfo) + (size_t)kSegTouch * 4 + (size_t)kSegTips * 4;
static_assert(kSegGFixed <= kSmemMax, "pool-region layout exceeds the dynamic shared memory");

struct SegView {
  const int32_t* P;
  int L;
  const uint32_t* tipbits;
  const uint16_t* nexttip;
  const int32_t* pmap;
  int pmask;
  Seg* segs;
};

__device__ __forceinline__ int wrapL(int x, int L) { return x >= L ? x - L : x; }
__device__ __forceinline__ int wrapN(int x, int n) { x %= n; return x < 0 ? x + n : x; }
__device__ __forceinline__ int32_t sval(const SegView& g, const Seg& s, int i) {
  return s.base < 0 ? ~s.base : g.P[wrapL(s.base + i, g.L)];
}
__device__ __forceinline__ uint32_t pair_hash(int32_t x, int32_t y) {
  uint32_t h = (uint32_t)x * 0x9E3779B1u ^ (uint32_t)y * 0x85EBCA77u;
  return h ^ (h >> 15);
}
// index k of P with P[k-1] == x and P[k] == y, or -1
__device__ __forceinline__ int pmap_lookup(const SegView& g, int32_t x, int32_t y) {
  uint32_t i = pair_hash(x, y) & g.pmask;
  for (int probe = 0; probe <= g.pmask; probe++) {
    int k = g.pmap[i];
    if (k < 0) return -1;
    if (g.P[k] == y && g.P[k == 0 ? g.L - 1 : k - 1] == x) return k;
    i = (i + 1) & g.pmask;
  }
  return -1;
}


// first tip of P in the cyclic index range [a, a + cnt), as an offset, or -1
// (O(1): nexttip[k] = smallest tip index >= k, 0xFFFF when none)
__device__ __forceinline__ int next_tip(const SegView& g, int a, int cnt) {
  int t = g.nexttip[a];
  if (t != 0xFFFF) {
    if (t < a + cnt) return t - a;
    return -1;
  }
  if (a + cnt <= g.L) return -1;
  t = g.nexttip[0];
  return (t != 0xFFFF && t < a + cnt - g.L) ? t + g.L - a : -1;
}

// segment of X holding local position p (warp-uniform)
__device__ __forceinline__ int seg_of(const SegView& g, const SPiece& X, int p, int lane) {
  for (int c0 = 0; c0 < X.nseg; c0 += 32) {
    int s = c0 + lane;
    bool hit = false;
    if (s < X.nseg) {
      Seg sg = g.segs[X.soff + s];
      hit = sg.loff <= p && p < sg.loff + sg.len;
    }
    unsigned m = __ballot_sync(kFull, hit);
    if (m) return c0 + __ffs(m) - 1;
  }
  return -1;
}
__device__ __forceinline__ int32_t selem(const SegView& g, const SPiece& X, int p, int lane) {
  Seg sg = g.segs[X.soff + seg_of(g, X, p, lane)];
  return sval(g, sg, p - sg.loff);
}
// one lane, linear (tiny pieces)
__device__ int32_t selem1(const SegView& g, const SPiece& X, int p) {
  for (int s = 0; s < X.nseg; s++) {
    Seg sg = g.segs[X.soff + s];
    if (sg.loff <= p && p < sg.loff + sg.len) return sval(g, sg, p - sg.loff);
  }
  return -1;
}

// reparation.py:59-71 on a segment piece: the first position p with
// s[p-1] == s[p+1] (cyclic), or -1.  Warp-uniform.
__device__ int seg_first_tip(const SegView& g, const SPiece& X, int lane, int* fk_out) {
  *fk_out = -1;
  if (X.len < 4) {
    int r = -1;
    if (lane == 0)
      for (int p = 0; p < X.len && r < 0; p++)
        if (selem1(g, X, p == 0 ? X.len - 1 : p - 1) == selem1(g, X, p + 1 == X.len ? 0 : p + 1)) r = p;
    return __shfl_sync(kFull, r, 0);
  }
  for (int c0 = 0; c0 < X.nseg; c0 += 32) {
    int s = c0 + lane, best = -1, fk = -1;
    if (s < X.nseg) {
      Seg sg = g.segs[X.soff + s];
      Seg sp = g.segs[X.soff + (s == 0 ? X.nseg - 1 : s - 1)];
      Seg sn = g.segs[X.soff + (s + 1 == X.nseg ? 0 : s + 1)];
      int32_t pv = sval(g, sp, sp.len - 1), nv = sval(g, sn, 0);
      const int l = sg.len;
      if (pv == (l >= 2 ? sval(g, sg, 1) : nv)) {
        best = sg.loff;
      } else {
        if (l >= 3) {
          int d = next_tip(g, wrapL(sg.base + 1, g.L), l - 2);
          if (d >= 0) best = sg.loff + 1 + d;
        }
        if (best < 0 && l >= 2 && sval(g, sg, l - 2) == nv) best = sg.loff + l - 1;
      }
      if (best >= 0 && sg.base >= 0) fk = wrapL(sg.base + (best - sg.loff), g.L);
    }
    unsigned m = __ballot_sync(kFull, best >= 0);
    if (m) {
      *fk_out = __shfl_sync(kFull, fk, __ffs(m) - 1);
      return __shfl_sync(kFull, best, __ffs(m) - 1);
    }
  }
  return -1;
}

// local position q of X with X[q-1] == x and X[q] == y (a directed boundary
// pair is unique in a piece), or -1.  Warp-uniform.
__device__ int seg_pairfind(const SegView& g, const SPiece& X, int32_t x, int32_t y, int lane) {
  const int k = pmap_lookup(g, x, y);
  for (int c0 = 0; c0 < X.nseg; c0 += 32) {
    int s = c0 + lane, q = -1;
    if (s < X.nseg) {
      Seg sg = g.segs[X.soff + s];
      if (k >= 0 && sg.base >= 0) {
        int i = k - sg.base;
        if (i < 0) i += g.L;
        if (i >= 1 && i < sg.len) q = sg.loff + i;
      }
      if (q < 0) {
        Seg sp = g.segs[X.soff + (s == 0 ? X.nseg - 1 : s - 1)];
        if (sval(g, sg, 0) == y && sval(g, sp, sp.len - 1) == x) q = sg.loff;
      }
    }
    unsigned m = __ballot_sync(kFull, q >= 0);
    if (m) return __shfl_sync(kFull, q, __ffs(m) - 1);
  }
  return -1;
}

// Appends X's local positions [start, start + cnt) (cyclic, cnt <= |X|) to
// out[n..] as segments with local offsets from lo; returns the new count.
// Lane s clips segment s; parts land in range order (the segment holding
// `start` first, then the following ones cyclically, then -- when the range
// wraps all the way around -- that segment's head).  X's segments are maximal
// runs of P except across X's own wrap point, so at most one pair of parts
// needs merging.  Warp-uniform.
__device__ int emit_range_warp(const SegView& g, const SPiece& X, int start, int cnt, Seg* out, int n, int lo,
                               int lane) {
  if (cnt <= 0) return n;
  const int Lx = X.len, ns = X.nseg;
  const int s0 = seg_of(g, X, start, lane);
  // X's segments are maximal runs of P except across X's own wrap point
  // (segment ns-1, then segment 0): when the range crosses local position 0
  // strictly inside and the two runs are contiguous in P, their parts merge
  // (decided up front, so the parts are written once, in place).
  const Seg sl = g.segs[X.soff + ns - 1], sf = g.segs[X.soff];
  const int rj = start == 0 ? 0 : Lx - start;  // range offset of local position 0
  const bool merge = ns > 1 && rj > 0 && rj < cnt && sl.base >= 0 && sf.base >= 0 &&
                     wrapL(sl.base + sl.len, g.L) == sf.base && sl.len + sf.len <= g.L;
  const int ia = ns - 1 - s0;  // part index of segment ns-1; the part starting at local 0 is ia + 1
  const int len0 = merge ? min(s0 == 0 ? start : (int)sf.len, cnt - rj) : 0;
  int count = 0;
  for (int c0 = 0; c0 < ns; c0 += 32) {
    const int s = c0 + lane;
    bool inc = false, tail = false;
    if (s < ns) {
      const Seg sg = g.segs[X.soff + s];
      int r0, skip;
      if (s == s0) { r0 = 0; skip = start - sg.loff; }
      else { r0 = wrapN(sg.loff - start, Lx); skip = 0; }
      if (r0 < cnt) {
        inc = true;
        int idx = s - s0;
        if (idx < 0) idx += ns;
        int len = min(sg.len - skip, cnt - r0);
        if (merge && idx == ia) len += len0;
        if (!(merge && idx == ia + 1))
          out[n + idx - (merge && idx > ia + 1 ? 1 : 0)] =
              mkseg(sg.base >= 0 ? wrapL(sg.base + skip, g.L) : sg.base, len, lo + r0);
      }
      if (s == s0 && start > sg.loff) {
        int rt = Lx - (start - sg.loff);
        if (rt < cnt) {
          tail = true;
          if (!(merge && ns == ia + 1))
            out[n + ns - (merge ? 1 : 0)] = mkseg(sg.base, min(start - sg.loff, cnt - rt), lo + rt);
        }
      }
    }
    count += __popc(__ballot_sync(kFull, inc)) + __popc(__ballot_sync(kFull, tail));
  }
  __syncwarp();
  return n + count - (merge ? 1 : 0);
}

// Arc split of piece X at tip position pos with split info si:
// the cut, the children's lengths and rotations, their segment storage; the
// edge is promoted.  Returns false without side effects when a search fails
// (the caller falls back to the re-walk).  The children are then emitted by
// seg_emit_child, pa and pb by the two warps of a pair.
struct SplitPlan {
  int j, la, lb, ka, kb, base_a, base_b;
  int32_t v, u;
};
__device__ bool seg_split_plan(const RepairCtx& c, const SegView& g, const SPiece& X, int pos, int32_t v,
                               const SplitInfo& si, int* s_stop, int seg_base, int seg_cap, int lane, SplitPlan* pl,
                               unsigned long long* prof) {
  const int Lx = X.len;
  if (si.a_in < 0) return false;
  long long c0 = clock64();
  const int j = seg_pairfind(g, X, si.a_in, si.u, lane);
  long long c1 = clock64();
  if (j < 0 || j == pos) return false;
  const int la = wrapN(pos - j, Lx) + 1, lb = wrapN(j - pos, Lx) + 1;
  // pa = [v, X[j .. pos-1]], pb = [X[pos .. j-1], u]; their re-walk start pairs
  int ka = -1, kb = -1;
  const int32_t xj = selem(g, X, j, lane), xpm = selem(g, X, wrapN(pos - 1, Lx), lane);
  const int32_t xpos = v, xjm = selem(g, X, wrapN(j - 1, Lx), lane);
  if (v == si.oa && (la >= 2 ? xj : v) == si.ga) ka = 0;
  else if (la >= 2 && xpm == si.oa && v == si.ga) ka = la - 1;
  else {
    int q = seg_pairfind(g, X, si.oa, si.ga, lane);
    if (q >= 0) {
      int d = wrapN(q - j, Lx);
      if (d >= 1 && d <= la - 2) ka = d;
    }
  }
  if (si.u == si.ob && xpos == si.gb) kb = lb - 1;
  else if (lb >= 2 && xjm == si.ob && si.u == si.gb) kb = lb - 2;
  else {
    int q = seg_pairfind(g, X, si.ob, si.gb, lane);
    if (q >= 0) {
      int d = wrapN(q - pos, Lx);
      if (d >= 1 && d <= lb - 2) kb = d - 1;
    }
  }
  if (ka < 0 || kb < 0) return false;
  int base = 0;
  const int need = 2 * (X.nseg + 4);
  if (lane == 0) base = atomicAdd(s_stop, need);
  base = __shfl_sync(kFull, base, 0);
  if (base + need > seg_cap) return false;  // (capacity is checked per round; defensive)
  base += seg_base;
  if (lane == 0) {
    promote(c, si.e, si.te);
    if (prof) {
      atomicAdd(prof + 0, (unsigned long long)(c1 - c0));
      atomicAdd(prof + 1, (unsigned long long)(clock64() - c1));
      atomicAdd(prof + 3, (unsigned long long)X.nseg);
    }
  }
  *pl = SplitPlan{j, la, lb, ka, kb, base, base + X.nseg + 4, v, si.u};
  return true;
}

// child 0 = pa = rotate([v] ++ X[j .. pos-1], ka), child 1 = pb = rotate(X[pos .. j-1] ++ [u], kb)
__device__ SPiece seg_emit_child(const SegView& g, const SPiece& X, int pos, const SplitPlan& p, int which, int lane) {
  const int Lx = X.len;
  Seg* o = g.segs + (which ? p.base_b : p.base_a);
  int nn;
  if (which == 0) {
    if (p.ka == 0) {
      if (lane == 0) o[0] = mkseg(~p.v, 1, 0);
      nn = emit_range_warp(g, X, p.j, p.la - 1, o, 1, 1, lane);
    } else {
      nn = emit_range_warp(g, X, wrapN(p.j + p.ka - 1, Lx), p.la - p.ka, o, 0, 0, lane);
      if (lane == 0) o[nn] = mkseg(~p.v, 1, p.la - p.ka);
      nn = emit_range_warp(g, X, p.j, p.ka - 1, o, nn + 1, p.la - p.ka + 1, lane);
    }
  } else {
    nn = emit_range_warp(g, X, wrapN(pos + p.kb, Lx), p.lb - 1 - p.kb, o, 0, 0, lane);
    if (lane == 0) o[nn] = mkseg(~p.u, 1, p.lb - 1 - p.kb);
    nn = emit_range_warp(g, X, pos, p.kb, o, nn + 1, p.lb - p.kb, lane);
  }
  __syncwarp();
  SPiece r{which ? p.base_b : p.base_a, nn, which ? p.lb : p.la, -1, -1};
  r.ftip = seg_first_tip(g, r, lane, &r.fk);
  return r;
}

__device__ __forceinline__ void tset_add(int32_t* set, int32_t x) {
  uint32_t h = ((uint32_t)x * 0x9E3779B1u) & (kSegTouch - 1);
  for (int k = 0; k < kSegTouch; k++) {
    int32_t prev = atomicCAS(&set[h], -1, x);
    if (prev == -1 || prev == x) return;
    h = (h + 1) & (kSegTouch - 1);
  }
}
__device__ __forceinline__ bool tset_has(const int32_t* set, int32_t x) {
  uint32_t h = ((uint32_t)x * 0x9E3779B1u) & (kSegTouch - 1);
  for (int k = 0; k < kSegTouch; k++) {
    int32_t y = set[h];
    if (y == x) return true;
    if (y == -1) return false;
    h = (h + 1) & (kSegTouch - 1);
  }
  return false;
}

// two warps of a pair meet (named barrier 1 + pair; 0 is __syncthreads); the
// warp reconverges first (bar.sync is the .aligned form)
__device__ __forceinline__ void pair_sync(int pair) {
  __syncwarp();
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
}
struct PairMsg {
  int mode;
  SplitPlan plan;
};

// G = false: items kept in shared memory; G = true: items whose P exceeds
// smem_max_l or whose classification predicts more pieces than the shared
// record list holds (extra visits > gm_dups) keep their per-item arrays,
// records and segments in a block-private pool region (the hull slivers of
// 100M-point meshes: 10^4 vertices, thousands of splits).  Two instantiations,
// so the shared-memory path keeps its shared-memory loads.
template <bool G>
__device__ __forceinline__ void seg_body(RepairCtx c, const int32_t* __restrict__ items,
                                         const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                         int64_t* __restrict__ item_list, int32_t* __restrict__ item_n,
                                         int32_t* __restrict__ item_state, int32_t* __restrict__ item_depth,
                                         int64_t* __restrict__ item_slots, unsigned long long* stats, LongQueue q,
                                         unsigned long long* dbg, unsigned int trace_qi, int seg_cap, int smem_max_l,
                                         int rec_limit, int gm_dups) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // G = false: everything in shared memory.  G = true: P, its tip bitmap /
  // ranks and nexttip in shared memory sized for kSegMaxG (the pair map,
  // piece records, round lists and segment arena move to the block's pool
  // region), so the lineage's most frequent reads stay shared.
  int32_t *P, *pmap, *tiprank, *nextw, *fans, *tipv, *tipb, *tset, *s_out, *tlist;
  uint32_t* tipbits;
  uint16_t* nexttip;
  SplitInfo* tipinfo;
  int* tipdeg;
  SPiece* recs;
  Seg* segs;
  int rec_cap, scap;
  constexpr int kMaxP = G ? kSegMaxG : kSegMaxL;
  P = reinterpret_cast<int32_t*>(smem_raw);
  tipbits = reinterpret_cast<uint32_t*>(P + kMaxP);
  if constexpr (!G) {
    pmap = reinterpret_cast<int32_t*>(tipbits + kSegMaxL / 32);
    recs = reinterpret_cast<SPiece*>(pmap + kPairCap);  // [2][kSegRec]
    s_out = reinterpret_cast<int32_t*>(recs + 2 * kSegRec);
    fans = s_out + kSegRec;
  } else {
    tiprank = reinterpret_cast<int32_t*>(tipbits + kSegMaxG / 32 + 1);
    nextw = tiprank + kSegMaxG / 32 + 1;
    nexttip = reinterpret_cast<uint16_t*>(nextw + kSegMaxG / 32 + 1);
    fans = reinterpret_cast<int32_t*>(nexttip + kSegMaxG);
    pmap = s_out = tlist = nullptr;  // in the pool region (per block, below)
    recs = nullptr;
    segs = nullptr;
  }
  tipv = fans + 2 * kSegWarps * kFanCap;  // tip vertex (or -1 when its info is unusable)
  tipb = tipv + kSegTips;                 // barrier vertex
  tipinfo = reinterpret_cast<SplitInfo*>(tipb + kSegTips);
  tset = reinterpret_cast<int32_t*>(tipinfo + kSegTips);  // promoted-edge endpoints (hash set)
  if constexpr (!G) {
    tiprank = tset + kSegTouch;                                  // tips of P before word w
    nextw = tiprank + kSegMaxL / 32 + 1;                         // first non-empty tip word >= w
    nexttip = reinterpret_cast<uint16_t*>(nextw + kSegMaxL / 32 + 1);
    tipdeg = reinterpret_cast<int*>(nexttip + kSegMaxL);  // cached fan sizes (-1: none)
    tlist = tipdeg + kSegTips;                             // tipped records of the round
    segs = reinterpret_cast<Seg*>(tlist + kSegRec);
    rec_cap = rec_limit;  // kSegRec (lower only as a testing hook)
    scap = seg_cap;
  } else {
    tipdeg = reinterpret_cast<int*>(tset + kSegTouch);
    rec_cap = kGRec;
    scap = kGSegCap;
  }
  __shared__ long long s_gscr;  // pool offset of the block's region (-1: not allocated)
  if (threadIdx.x == 0) s_gscr = -1;
  // s_ntb: tipped-record count of the next round, double-buffered by round parity
  // so the reset of one round never races with the previous round's readers
  __shared__ int s_ntip, s_ntouch, s_stop, s_fail, s_ntb[2], s_need, s_tot;
  __shared__ PairMsg pmsg[kSegWarps / 2];
  __shared__ int s_wcnt[kSegWarps], s_wneed[kSegWarps];
  __shared__ long long s_base;
  __shared__ unsigned int s_w;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* fan = fans + wib * kFanCap;
  int32_t* back = fans + (kSegWarps + wib) * kFanCap;
  // reparation.py:354-364 bounds the rounds by initial + 1, initial = extra visits
  // of mesh0: a global sum the short-item classification may still be adding to
  // when this kernel starts early.  Per item a round splits a tip (depth <= L + 1);
  // k_out_counts checks the global bound on the final maximum depth.
  const unsigned int nh = *q.n_huge, nq = nh + *q.n_long;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_w = atomicAdd(G ? q.gm_next : q.next, 1u);
    __syncthreads();
    const unsigned int qi = s_w;
    if (qi >= nq) break;
    const unsigned int w = qi < nh ? (unsigned int)q.huge[qi] : (unsigned int)q.longq[qi - nh];
    // debug timeline (tm_ctx_debug): item trace_qi's rounds in dbg[0..59],
    // slowest item in dbg[60], stale / reused split infos in dbg[61] / dbg[62],
    // re-walk fallbacks in dbg[63]
    const bool trace = qi == trace_qi && threadIdx.x == 0;
    unsigned long long t_ns, t_item;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item));
    if (trace) dbg[0] = t_item;
    const int32_t i = items[w];
    const int64_t b0 = off[i];
    const int L = (int)(off[i + 1] - b0);
    if (L < 3) {
      if (threadIdx.x == 0) item_state[w] = 3;
      continue;
    }
    // the other instantiation's item?  Pool-region blocks take P over smem_max_l,
    // more predicted pieces than the shared record list (extra visits > gm_dups),
    // and P over half of it (the shared segment arena runs out first there)
    if ((L > smem_max_l || L > smem_max_l / 2 + 1 || item_depth[w] > gm_dups) != G) continue;
    if constexpr (G) {
      if (L > kSegMaxG) {
        if (threadIdx.x == 0) item_state[w] = 3;  // the warp kernel from scratch
        continue;
      }
      if (threadIdx.x == 0 && s_gscr < 0) s_gscr = palloc(c, kGStride);
      __syncthreads();
      if (s_gscr < 0) {  // pool exhausted: the warp kernel from scratch
        if (threadIdx.x == 0) item_state[w] = 3;
        continue;
      }
      pmap = c.pool + s_gscr;
      s_out = pmap + kGPairCap;
      tlist = s_out + kGRec;
      recs = reinterpret_cast<SPiece*>(tlist + kGRec);  // [2][kGRec]
      segs = reinterpret_cast<Seg*>(recs + 2 * kGRec);
    }
    int pcap = 64;
    while (pcap < 2 * L) pcap <<= 1;
    for (int k = threadIdx.x; k < L; k += blockDim.x) P[k] = v[b0 + k];
    for (int k = threadIdx.x; k < pcap; k += blockDim.x) pmap[k] = -1;
    for (int k = threadIdx.x; k < (L + 31) / 32; k += blockDim.x) tipbits[k] = 0;
    for (int k = threadIdx.x; k < kSegTouch; k += blockDim.x) tset[k] = -1;
    if (threadIdx.x == 0) { s_ntip = 0; s_ntouch = 0; s_fail = 0; s_stop = 1; }  // segs[0]: the item
    __syncthreads();
    SegView g{P, L, tipbits, nexttip, pmap, pcap - 1, segs};
    // tips of P (bitmap) and the pair map
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      int32_t a = P[k == 0 ? L - 1 : k - 1], y = P[k];
      if (a == P[k + 1 == L ? 0 : k + 1]) atomicOr(&tipbits[k >> 5], 1u << (k & 31));
      uint32_t h = pair_hash(a, y) & (pcap - 1);
      while (atomicCAS(&pmap[h], -1, k) != -1) h = (h + 1) & (pcap - 1);
    }
    __syncthreads();
    // tip slots in P order: tip k lives at tiprank[k / 32] + (tips below k in its word)
    const int nwords = (L + 31) / 32;
    if (wib == 0) {
      int carry = 0;
      for (int base = 0; base < nwords; base += 32) {
        int wd = base + lane;
        int cnt = wd < nwords ? __popc(tipbits[wd]) : 0, inc = cnt;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (wd < nwords) tiprank[wd] = carry + inc - cnt;
        carry += __shfl_sync(kFull, inc, 31);
      }
      if (lane == 0) s_ntip = carry;
    }
    __syncthreads();
    if (wib == 1) {  // nextw: suffix scan over the tip words (first non-empty word at or after w)
      int carry = 0x7FFFFFFF;
      for (int top = ((nwords + 31) & ~31) - 32; top >= 0; top -= 32) {
        int wd = top + lane;
        int x = (wd < nwords && tipbits[wd] != 0) ? wd : 0x7FFFFFFF;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_down_sync(kFull, x, o);
          if (lane + o < 32) x = min(x, y);
        }
        x = min(x, carry);
        if (wd < nwords) nextw[wd] = x;
        carry = __shfl_sync(kFull, x, 0);
      }
    }
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      uint32_t wbits = tipbits[k >> 5];
      if ((wbits >> (k & 31)) & 1u) {
        int t = tiprank[k >> 5] + __popc(wbits & ((1u << (k & 31)) - 1u));
        if (t < kSegTips) { tipv[t] = P[k]; tipb[t] = P[k == 0 ? L - 1 : k - 1]; }
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      const int wd = k >> 5;
      const uint32_t hi = tipbits[wd] & (~0u << (k & 31));
      int t;
      if (hi) t = (wd << 5) + __ffs(hi) - 1;
      else {
        const int w2 = wd + 1 < nwords ? nextw[wd + 1] : 0x7FFFFFFF;
        t = w2 == 0x7FFFFFFF ? 0xFFFF : (w2 << 5) + __ffs(tipbits[w2]) - 1;
      }
      nexttip[k] = (uint16_t)t;
    }
    __syncthreads();
    // every tip of the item is a tip of P (an arc split only removes the split
    // tip); its split edge depends only on the frontier around v and u
    const int ntip_pre = s_ntip < kSegTips ? s_ntip : kSegTips;
    // fans of the tips, cached in the pool for the stale-info recomputes
    if (threadIdx.x == 0) s_base = palloc(c, (long long)ntip_pre * kFanCap);
    __syncthreads();
    int32_t* fcache = s_base >= 0 ? c.pool + s_base : nullptr;
    for (int k = wib; k < ntip_pre; k += kSegWarps) {
      SplitInfo si;
      FanCache fc;
      if (fcache) { fc.out = fcache + (long long)k * kFanCap; fc.out_deg = tipdeg + k; }
      else if (lane == 0) tipdeg[k] = -1;
      bool ok = warp_split_info(c, tipv[k], tipb[k], i, fan, back, lane, false, true, &si, fc);
      if (lane == 0) {
        tipinfo[k] = si;
        if (!ok) tipv[k] = -1;
      }
    }
    if (threadIdx.x == 0) segs[0] = mkseg(0, L, 0);
    __syncthreads();
    if (trace) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns)); dbg[1] = t_ns; dbg[2] = L; dbg[3] = s_ntip; }
    if (wib == 0) {
      SPiece X0{0, 1, L, -1, -1};
      X0.ftip = s_ntip > 0 ? seg_first_tip(g, X0, lane, &X0.fk) : -1;
      if (lane == 0) { recs[0] = X0; s_ntb[0] = X0.ftip >= 0 ? 1 : 0; }
    }
    __syncthreads();
    int cur = 0, n = 1, ntips = s_ntb[0], hbase = 0;
    long long depth = 0, splits = 0;
    bool bad = false, spill = false;
    while (ntips > 0) {
      if (depth + 1 > (long long)L + 1) {
        if (threadIdx.x == 0) report(c.st, K_NO_CONVERGE, i);
        bad = true;
        break;
      }
      SPiece* in = recs + cur * rec_cap;
      SPiece* out = recs + (cur ^ 1) * rec_cap;
      // output slot of every input record (prefix over tip flags) and the
      // segments the round may need
#ifdef TM_SEG_WARP0_SCAN  // A/B: warp 0 alone (n / 32 dependent steps per round)
      if (wib == 0) {
        int carry = 0, need = 0;
        for (int base = 0; base < n; base += 32) {
          int r = base + lane;
          int t = (r < n && in[r].ftip >= 0) ? 1 : 0;
          int inc = t;
          for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
          }
          if (r < n) s_out[r] = r + carry + inc - t;
          if (t) tlist[carry + inc - 1] = r;  // the tipped records, in order
          carry += __shfl_sync(kFull, inc, 31);
          int nd = t ? 2 * (in[r].nseg + 4) : 0;
          for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(kFull, nd, o);
          need += nd;
        }
        if (lane == 0) s_need = need;
      }
      if (threadIdx.x == 0) s_ntb[cur ^ 1] = 0;
      __syncthreads();
#else
      // the whole block, one record per thread per pass (the record list
      // grows with the splits: hundreds of pieces in the late rounds)
      {
        int carry = 0, need = 0;  // block-uniform
        for (int base = 0; base < n; base += blockDim.x) {
          const int r = base + threadIdx.x;
          const int t = (r < n && in[r].ftip >= 0) ? 1 : 0;
          int inc = t;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
          }
          int nd = t ? 2 * (in[r].nseg + 4) : 0;
          for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(kFull, nd, o);
          if (lane == 31) s_wcnt[wib] = inc;
          if (lane == 0) s_wneed[wib] = nd;
          __syncthreads();
          int wpre = 0, tot = 0, ntot = 0;
#pragma unroll
          for (int w2 = 0; w2 < kSegWarps; w2++) {
            const int x = s_wcnt[w2];
            wpre += w2 < wib ? x : 0;
            tot += x;
            ntot += s_wneed[w2];
          }
          const int ex = carry + wpre + inc - t;
          if (r < n) s_out[r] = r + ex;
          if (t) tlist[ex] = r;  // the tipped records, in order
          carry += tot;
          need += ntot;
          __syncthreads();  // s_wcnt / s_wneed reused by the next pass
        }
        if (threadIdx.x == 0) {
          s_need = need;
          s_ntb[cur ^ 1] = 0;
        }
        __syncthreads();
      }
#endif
      // Segments are bump-allocated in one half of the arena; when a round
      // would overflow it, the live pieces are first compacted into the other
      // half, so the arena only ever has to hold the live pieces.
      const int half = scap / 2;
      if (n + ntips > rec_cap) { spill = true; break; }  // uniform
      if (s_stop + s_need > half) {
        const int nb = hbase == 0 ? half : 0;
        __syncthreads();
        if (threadIdx.x == 0) s_stop = 0;
        __syncthreads();
        for (int r = wib; r < n; r += kSegWarps) {
          SPiece X = in[r];
          int rel = 0;
          if (lane == 0) rel = atomicAdd(&s_stop, X.nseg);
          rel = __shfl_sync(kFull, rel, 0);
          for (int k = lane; k < X.nseg; k += 32) segs[nb + rel + k] = segs[X.soff + k];
          __syncwarp();  // every lane has read in[r] before lane 0 rewrites it
          if (lane == 0) in[r].soff = nb + rel;
        }
        hbase = nb;
        __syncthreads();
        if (s_stop + s_need > half) { spill = true; break; }  // uniform
      }
      const int tb = hbase;
      depth++;
      const bool tset_ok = s_ntouch <= kSegTouch / 2;  // else: always recompute
      for (int r = threadIdx.x; r < n; r += blockDim.x)
        if (in[r].ftip < 0) out[s_out[r]] = in[r];
      // Warp pairs share a split: the lead warp computes the split info, the
      // cut and the rotations (promoting the edge), then the two warps emit
      // pa and pb and find their first tips side by side.
      const int pair = wib >> 1, hf = wib & 1;
      for (int t = pair; t < ntips; t += kSegWarps / 2) {
        const int r = tlist[t];
        const SPiece X = in[r];
        const int pos = X.ftip;
        if (hf == 0) {
          long long ck0 = clock64();
          const int32_t tv_ = selem(g, X, pos, lane), bv = selem(g, X, pos == 0 ? X.len - 1 : pos - 1, lane);
          int k = -1;
          if (X.fk >= 0) {  // the precomputed slot of this tip of P
            uint32_t wbits = tipbits[X.fk >> 5];
            k = tiprank[X.fk >> 5] + __popc(wbits & ((1u << (X.fk & 31)) - 1u));
            if (k >= ntip_pre || tipv[k] != tv_) k = -1;
          }
          SplitInfo si;
          bool use = k >= 0 && tset_ok;
          if (use) {
            si = tipinfo[k];
            use = !tset_has(tset, tv_) && !tset_has(tset, si.u);  // no promotion touched v or u
          }
          if (lane == 0) atomicAdd(dbg + (use ? 62 : 61), 1ull);
          FanCache fc;
          if (k >= 0 && fcache && tipdeg[k] >= 0) { fc.in = fcache + (long long)k * kFanCap; fc.in_deg = tipdeg[k]; }
          bool ok = use || warp_split_info(c, tv_, bv, i, fan, back, lane, false, false, &si, fc);
          SplitPlan pl;
          int mode = 0;  // 0 failed, 1 pair emission, 2 lead finished alone (re-walk fallback)
          SPiece A{0, 0, 0, -1, -1}, B{0, 0, 0, -1, -1};
          long long ck1 = clock64();
          if (ok && seg_split_plan(c, g, X, pos, tv_, si, &s_stop, tb, half, lane, &pl,
                                   qi == trace_qi ? dbg + 52 : nullptr)) {
            mode = 1;
          } else if (ok) {
            // re-walk fallback (reparation.py:216-229) with the strict length law;
            // the pieces come back as one-vertex segments
            if (lane == 0) { promote(c, si.e, si.te); atomicAdd(dbg + 63, 1ull); }
            __syncwarp();
            int32_t *pa = nullptr, *pb = nullptr;
            int la = 0, lb = 0;
            auto galloc = [&](long long m) -> int32_t* {
              long long o = 0;
              if (lane == 0) o = palloc(c, m);
              o = __shfl_sync(kFull, o, 0);
              return o < 0 ? nullptr : c.pool + o;
            };
            int rr = warp_rewalk_split(c, si.e, si.te, X.len, i, galloc, lane, &pa, &la, &pb, &lb);
            if (rr == 0 && lane == 0) report(c.st, K_SPLIT_LAW, i);
            if (rr == 1) {
              int sb = 0;
              if (lane == 0) sb = atomicAdd(&s_stop, la + lb);
              sb = __shfl_sync(kFull, sb, 0);
              if (sb + la + lb > half) {
                if (lane == 0) report(c.st, K_STRUCT, i);
              } else {
                sb += tb;
                for (int x = lane; x < la; x += 32) segs[sb + x] = mkseg(~pa[x], 1, x);
                for (int x = lane; x < lb; x += 32) segs[sb + la + x] = mkseg(~pb[x], 1, x);
                __syncwarp();
                A = SPiece{sb, la, la, -1, -1};
                B = SPiece{sb + la, lb, lb, -1, -1};
                A.ftip = seg_first_tip(g, A, lane, &A.fk);
                B.ftip = seg_first_tip(g, B, lane, &B.fk);
                mode = 2;
              }
            }
          }
          if (mode == 0 && lane == 0) atomicCAS(&s_fail, 0, 1);
          if (mode != 0 && lane == 0) {
            atomicAdd(&s_ntouch, 2);
            tset_add(tset, tv_);
            tset_add(tset, si.u);
          }
          if (lane == 0) {
            pmsg[pair].mode = mode;
            pmsg[pair].plan = pl;
          }
          if (mode == 2 && lane == 0) {
            const int o = s_out[r];
            out[o] = A;
            out[o + 1] = B;
            atomicAdd(&s_ntb[cur ^ 1], (A.ftip >= 0 ? 1 : 0) + (B.ftip >= 0 ? 1 : 0));
          }
          if (qi == trace_qi && lane == 0) {
            atomicAdd(dbg + 56, (unsigned long long)(ck1 - ck0));
            atomicAdd(dbg + 57, (unsigned long long)(clock64() - ck1));
            atomicAdd(dbg + 59, 1ull);
          }
        }
        pair_sync(pair);  // the lead's message is ready
        const int mode = pmsg[pair].mode;
        if (mode == 1) {
          const SplitPlan pl = pmsg[pair].plan;
          const long long ck2 = clock64();
          const SPiece C = seg_emit_child(g, X, pos, pl, hf, lane);
          if (lane == 0) {
            out[s_out[r] + hf] = C;
            if (C.ftip >= 0) atomicAdd(&s_ntb[cur ^ 1], 1);
            if (hf == 0 && qi == trace_qi) atomicAdd(dbg + 58, (unsigned long long)(clock64() - ck2));
          }
        }
        pair_sync(pair);  // message slot free again
      }
      __syncthreads();
      splits += ntips;
      n += ntips;
      ntips = s_ntb[cur ^ 1];
      cur ^= 1;
      if (trace && depth < 48) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns)); dbg[4 + depth] = t_ns; }
      if (s_fail) {
        bad = true;
        break;
      }
    }
    if (bad) {
      if (threadIdx.x == 0) { item_state[w] = 1; item_list[w] = -1; item_n[w] = 0; item_slots[w] = 0; }
      continue;
    }
    // leaves (or the pieces before an unsplit round) -> global pool
    const SPiece* fin = recs + cur * rec_cap;
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int r = 0; r < n; r++) tot += fin[r].len;
      s_tot = tot;
      s_base = palloc(c, tot + 2 * (long long)n);
    }
    __syncthreads();
    if (s_base < 0) {
      if (threadIdx.x == 0) { report(c.st, K_POOL, i); item_state[w] = 1; item_list[w] = -1; item_n[w] = 0; item_slots[w] = 0; }
      continue;
    }
    const long long list = s_base + s_tot;
    if (wib == 0) {
      int carry = 0;
      for (int base = 0; base < n; base += 32) {
        int r = base + lane;
        int ln = r < n ? fin[r].len : 0;
        int inc = ln;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (r < n) {
          c.pool[list + 2 * r] = (int32_t)(s_base + carry + inc - ln);
          c.pool[list + 2 * r + 1] = (int32_t)((uint32_t)ln | (fin[r].ftip >= 0 ? F_TIP : 0u));
        }
        carry += __shfl_sync(kFull, inc, 31);
      }
    }
    __syncthreads();
    for (int r = wib; r < n; r += kSegWarps) {
      int32_t* dst = c.pool + (uint32_t)c.pool[list + 2 * r];
      const SPiece X = fin[r];
      for (int s = 0; s < X.nseg; s++) {
        Seg sg = segs[X.soff + s];
        for (int x = lane; x < sg.len; x += 32) dst[sg.loff + x] = sval(g, sg, x);
      }
    }
    __syncthreads();
    if (spill) {
      // record list or segment arena too small: the warp kernel continues
      // (debug counters: spills of the shared / pool-region bodies, the last
      // spilled item's length, pieces and depth)
      if (threadIdx.x == 0) {
        atomicAdd(dbg + (G ? 73 : 72), 1ull);
        dbg[74] = ((unsigned long long)L << 40) | ((unsigned long long)(n & 0xFFFFF) << 20) | (depth & 0xFFFFF);
      }
      if (threadIdx.x == 0) { item_state[w] = 2; item_list[w] = list; item_n[w] = n; item_depth[w] = (int)depth; }
      if (threadIdx.x == 0 && splits) atomicAdd(stats + 1, (unsigned long long)splits);
      continue;
    }
    // repeated flags and extra visits of the leaves (pinch guard,
    // reparation.py:322): per-warp hash sets in the (now free) pair map
    __shared__ unsigned long long s_ex;
    if (threadIdx.x == 0) s_ex = 0;
    __syncthreads();
    int32_t* set = pmap + wib * (kPairCap / kSegWarps);
    for (int r = wib; r < n; r += kSegWarps) {
      const uint32_t ro = (uint32_t)c.pool[list + 2 * r];
      const int ln = fin[r].len;
      const int32_t* s = c.pool + ro;
      int ex;
      if (2 * ln <= kPairCap / kSegWarps) {
        int cap = 64;
        while (cap < 2 * ln) cap <<= 1;
        for (int x = lane; x < cap; x += 32) set[x] = -1;
        __syncwarp();
        int mine = 0;
        for (int x = lane; x < ln; x += 32) {
          int32_t val = s[x];
          uint32_t slot = ((uint32_t)val * 0x9E3779B1u) & (cap - 1);
          for (;;) {
            int32_t prev = atomicCAS(&set[slot], -1, val);
            if (prev == -1) break;
            if (prev == val) { mine++; break; }
            slot = (slot + 1) & (cap - 1);
          }
        }
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
        ex = mine;
        __syncwarp();
      } else {
        ex = warp_dup_scan(c, s, ln, lane, nullptr, nullptr);
      }
      if (lane == 0 && ex > 0) {
        c.pool[list + 2 * r + 1] = (int32_t)((uint32_t)c.pool[list + 2 * r + 1] | F_REP);
        atomicAdd(&s_ex, (unsigned long long)ex);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      item_state[w] = 1;
      item_list[w] = list;
      item_n[w] = n;
      if (depth > 0) atomicMax(stats + 0, (unsigned long long)depth);
      if (splits) atomicAdd(stats + 1, (unsigned long long)splits);
      if (s_ex) atomicAdd(stats + 5, s_ex);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns));
      unsigned long long dur = (t_ns - t_item) / 100;  // 0.1 us units
      atomicMax(dbg + 60, (dur << 32) | ((unsigned long long)(depth & 0xFFFF) << 16) | (qi & 0xFFFF));
    }
  }
}

__global__ void __launch_bounds__(32 * kSegWarps, 1) k_repair_tips_seg(
    RepairCtx c, const int32_t* __restrict__ items, const int64_t* __restrict__ off, const int32_t* __restrict__ v,
    int64_t* __restrict__ item_list, int32_t* __restrict__ item_n, int32_t* __restrict__ item_state,
    int32_t* __restrict__ item_depth, int64_t* __restrict__ item_slots, unsigned long long* stats, LongQueue q,
    unsigned long long* dbg, unsigned int trace_qi, int seg_cap, int smem_max_l, int rec_limit, int gm_dups,
    int gm_blocks) {
  if ((int)blockIdx.x < gm_blocks)
    seg_body<true>(c, items, off, v, item_list, item_n, item_state, item_depth, item_slots, stats, q, dbg, trace_qi,
                   seg_cap, smem_max_l, rec_limit, gm_dups);
  else
    seg_body<false>(c, items, off, v, item_list, item_n, item_state, item_depth, item_slots, stats, q, dbg, trace_qi,
                    seg_cap, smem_max_l, rec_limit, gm_dups);
}

// ------------------------------------------------------------ pinch pass
__global__ void __launch_bounds__(128) k_repair_pinch(RepairCtx c, const int32_t* __restrict__ items,
                                                      const unsigned int* n_items, const int64_t* __restrict__ off,
                                                      int64_t* __restrict__ item_list, int32_t* __restrict__ item_n,
                                                      int64_t* __restrict__ item_slots,
                                                      int32_t* __restrict__ item_state,
                                                      int32_t* __restrict__ item_depth, LongQueue q,
                                                      unsigned long long* stats, int mode) {
  extern __shared__ int2 s_pdup[];  // [4][kPinchDupCap]
  const int lane = threadIdx.x & 31;
  int2* stab = s_pdup + (threadIdx.x >> 5) * kPinchDupCap;
  // reparation.py:322: guard = extra visits of the tip-phase output + 1.  stats[5]
  // sums this context's items; stats[8] adds the other ranks' share (seed
  // partition, host-set before the resume pass, mode 3).
  long long guard = (long long)*(volatile unsigned long long*)(stats + 5) + 1 +
                    (long long)*(volatile unsigned long long*)(stats + 8);
  // testing hook (seed partitions only, TERMESH_PINCH_GUARD_CAP): a smaller local
  // guard parks more items, so tm_resume_pinch's path runs on small meshes
  const long long cap = (long long)*(volatile unsigned long long*)(stats + 11);
  if (cap > 0 && mode != 3 && guard > cap) guard = cap;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (mode == 0) {
    PinchPark park{item_state, item_depth, q.parked, q.n_parked};
    // the short items finish_item queued (the rest are complete or failed)
    const unsigned int np = *q.n_pinch;
    for (int64_t k = warp; k < np; k += nwarps) {
      const int64_t w = q.pinchq[k];
      warp_finish_pinch(c, w, items[w], item_list[w], item_n[w], lane, item_list, item_n, item_slots, stats, guard,
                        stab, 0, park);
    }
    return;
  }
  const unsigned int nh = *q.n_huge, nl = *q.n_long;
  if (mode == 2) {
    // right after the shared-memory kernel, on its stream: the long items it finished
    // (state 1), under the guard known so far; items that reach it are parked
    PinchPark park{item_state, item_depth, q.parked, q.n_parked};
    for (int64_t k = warp; k < nh + nl; k += nwarps) {
      const int64_t w = k < nh ? q.huge[k] : q.longq[k - nh];
      if (item_state[w] != 1) continue;  // handed back to k_repair_tips (states 2, 3)
      const long long list = item_list[w];
      if (list < 0) {
        if (lane == 0) item_slots[w] = 0;
        continue;
      }
      warp_finish_pinch(c, w, items[w], list, item_n[w], lane, item_list, item_n, item_slots, stats, guard, stab, 0,
                        park);
    }
    return;
  }
  const unsigned int np = *q.n_parked;
  if (mode == 3) {
    // seed partition, resume under the GLOBAL guard: the items the final local
    // guard parked (state 4; the parked list may hold an item twice, the CAS claims it once)
    for (int64_t k = warp; k < np; k += nwarps) {
      const int64_t w = q.parked[k];
      int claimed = 0;
      if (lane == 0) claimed = atomicCAS(item_state + w, 4, 1) == 4;
      if (!__shfl_sync(kFull, claimed, 0)) continue;
      warp_finish_pinch(c, w, items[w], item_list[w], item_n[w], lane, item_list, item_n, item_slots, stats, guard,
                        stab, item_depth[w]);
    }
    return;
  }
  // mode 1, final (local) guard: the long items k_repair_tips resumed, then every
  // parked item.  Seed partition (stats[9] != 0): the global guard is not known
  // yet, so an item reaching the local one is parked again for mode 3 instead of
  // being cut off.
  const bool defer = *(volatile unsigned long long*)(stats + 9) != 0;
  PinchPark park;
  if (defer) park = PinchPark{item_state, item_depth, q.parked, q.n_parked, stats + 10};
  for (int64_t k = warp; k < nh + nl + np; k += nwarps) {
    const int64_t w = k < nh ? q.huge[k] : k < nh + nl ? q.longq[k - nh] : q.parked[k - nh - nl];
    const bool parked = k >= nh + nl;
    if (!parked && item_state[w] != 2 && item_state[w] != 3) continue;  // done by mode 2 (or parked)
    if (parked) {
      int claimed = 0;
      if (lane == 0) claimed = atomicCAS(item_state + w, 4, 1) == 4;
      if (!__shfl_sync(kFull, claimed, 0)) continue;
    }
    const long long list = item_list[w];
    if (list < 0) {
      if (lane == 0) item_slots[w] = 0;
      continue;
    }
    warp_finish_pinch(c, w, items[w], list, item_n[w], lane, item_list, item_n, item_slots, stats, guard, stab,
                      parked ? item_depth[w] : 0, park);
  }
}

// ------------------------------------------------------------ stitch
__global__ void __launch_bounds__(256) k_out_counts(const int64_t* __restrict__ off, const int64_t* __restrict__ Pp,
                                                    const int32_t* __restrict__ item_of, const int32_t* __restrict__ item_n,
                                                    const int64_t* __restrict__ item_slots, int64_t* __restrict__ cnt,
                                                    int64_t* __restrict__ slots, const unsigned long long* stats,
                                                    DevStatus* st) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= P; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == P) {
      cnt[i] = 0;
      slots[i] = 0;
      if (stats && stats[0] > stats[2] + 1) report(st, K_NO_CONVERGE, P);  // rounds > initial + 1
      continue;
    }
    int32_t it = item_of[i];
    if (it < 0) { cnt[i] = 1; slots[i] = off[i + 1] - off[i]; }
    else { cnt[i] = item_n[it]; slots[i] = item_slots[it]; }
  }
}

// untouched polygons: one thread each, up to 16 independent loads in flight
__device__ __forceinline__ void stitch_plain(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                             const int64_t* __restrict__ Pp, const int32_t* __restrict__ item_of,
                                             const int64_t* __restrict__ pbase, const int64_t* __restrict__ sbase,
                                             int64_t* __restrict__ off_out, int32_t* __restrict__ v_out, int64_t blk,
                                             int64_t nblk) {
  const int64_t P = *Pp;
  for (int64_t i = blk * blockDim.x + threadIdx.x; i < P; i += nblk * blockDim.x) {
    if (item_of[i] >= 0) continue;
    int64_t b = off[i], n = off[i + 1] - b, sb = sbase[i];
    off_out[pbase[i]] = sb;
    for (int64_t k0 = 0; k0 < n; k0 += 16) {
      int32_t buf[16];
#pragma unroll
      for (int k = 0; k < 16; k++)
        if (k0 + k < n) buf[k] = v[b + k0 + k];
#pragma unroll
      for (int k = 0; k < 16; k++)
        if (k0 + k < n) v_out[sb + k0 + k] = buf[k];
    }
  }
}

// repaired polygons: one warp per work item, leaves flattened across lanes
__device__ __forceinline__ void stitch_items(const int32_t* __restrict__ items, const unsigned int* n_items,
                                             const int64_t* __restrict__ item_list, const int32_t* __restrict__ item_n,
                                             const int32_t* __restrict__ pool, const int64_t* __restrict__ pbase,
                                             const int64_t* __restrict__ sbase, int64_t* __restrict__ off_out,
                                             int32_t* __restrict__ v_out, int64_t blk, int64_t nblk) {
  const int lane = threadIdx.x & 31;
  const unsigned int ni = *n_items;
  int64_t warp = (blk * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (nblk * blockDim.x) >> 5;
  for (int64_t w = warp; w < ni; w += nwarps) {
    int32_t i = items[w];
    int64_t list = item_list[w];
    int n = item_n[w];
    if (list < 0) continue;
    int64_t pb = pbase[i], sb = sbase[i];
    for (int c = 0; c < n; c += 32) {
      int r = c + lane;
      uint32_t ro = 0;
      int ln = 0;
      if (r < n) {
        ro = (uint32_t)pool[list + 2 * r];
        ln = (int)((uint32_t)pool[list + 2 * r + 1] & LEN_MASK);
      }
      int inc = ln;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int start = inc - ln, total = __shfl_sync(0xffffffffu, inc, 31);
      if (r < n) off_out[pb + r] = sb + start;
      for (int kb = 0; kb < total; kb += 32) {
        int k = kb + lane;  // all lanes stay converged for the shuffles
        // leaf owning flattened element k: last leaf whose start <= k
        int lo = 0;
        for (int step = 16; step > 0; step >>= 1) {
          int cand = lo + step;
          int cs = __shfl_sync(0xffffffffu, start, cand < 32 ? cand : 31);
          if (cand < 32 && cand + c < n && cs <= k) lo = cand;
        }
        uint32_t lro = __shfl_sync(0xffffffffu, ro, lo);
        int ls = __shfl_sync(0xffffffffu, start, lo);
        if (k < total) v_out[sb + k] = pool[lro + (k - ls)];
      }
      sb += total;
    }
  }
}

// The final CSR in one launch: every third block copies repaired items (one
// warp per item), the others untouched polygons (one thread each) -- the two
// parts are independent, and one after the other they were both on the tail
// of the step.
__global__ void __launch_bounds__(256) k_stitch(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                const int64_t* __restrict__ Pp, const int32_t* __restrict__ item_of,
                                                const int32_t* __restrict__ items, const unsigned int* n_items,
                                                const int64_t* __restrict__ item_list,
                                                const int32_t* __restrict__ item_n, const int32_t* __restrict__ pool,
                                                const int64_t* __restrict__ pbase, const int64_t* __restrict__ sbase,
                                                int64_t* __restrict__ off_out, int32_t* __restrict__ v_out) {
  const int64_t b = blockIdx.x, g = gridDim.x;
  if (b % 3 == 2)
    stitch_items(items, n_items, item_list, item_n, pool, pbase, sbase, off_out, v_out, b / 3, g / 3);
  else
    stitch_plain(off, v, Pp, item_of, pbase, sbase, off_out, v_out, b - (b + 1) / 3, g - g / 3);
}

// ---- the final CSR by UNITS.  In polygon order the untouched polygons come in
// runs between work items, and a run keeps its order and moves by one shift:
// unit k = the run before the k-th work item (polygon order) + that item's
// pieces; unit K = the trailing run.  So the per-unit counts, the scan and the
// copy cost O(items) + a coalesced copy of the runs, not a count, scan and
// per-polygon copy over every polygon.

// polygons holding a work item (ordered compaction input); the item set is
// final after classification
__global__ void __launch_bounds__(256) k_item_flags(const int32_t* __restrict__ item_of, const int64_t* __restrict__ Pp,
                                                    int64_t n, uint8_t* __restrict__ flag) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i < P && item_of[i] >= 0) ? 1 : 0;
}

// unit k: run [rs, re) of untouched polygons, then (k < K) the item of polygon re
__device__ __forceinline__ void unit_range(const int32_t* __restrict__ srt, int64_t K, int64_t P, int64_t k,
                                           int64_t* rs, int64_t* re) {
  *rs = k == 0 ? 0 : (int64_t)srt[k - 1] + 1;
  *re = k < K ? (int64_t)srt[k] : P;
}

__global__ void __launch_bounds__(256) k_unit_counts(const int64_t* __restrict__ off, const int64_t* __restrict__ Pp,
                                                     const int32_t* __restrict__ srt, const int64_t* __restrict__ Kp,
                                                     const int32_t* __restrict__ item_of,
                                                     const int32_t* __restrict__ item_n,
                                                     const int64_t* __restrict__ item_slots, int64_t* __restrict__ cnt,
                                                     int64_t* __restrict__ slots, int64_t* __restrict__ n_units,
                                                     const unsigned long long* stats, DevStatus* st) {
  const int64_t P = *Pp, K = *Kp;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= K + 1; k += (int64_t)gridDim.x * blockDim.x) {
    if (k == K + 1) {  // the scan reads one element past the count
      cnt[k] = 0;
      slots[k] = 0;
      *n_units = K + 1;
      if (stats && stats[0] > stats[2] + 1) report(st, K_NO_CONVERGE, P);  // rounds > initial + 1
      continue;
    }
    int64_t rs, re;
    unit_range(srt, K, P, k, &rs, &re);
    int64_t c = re - rs, s = off[re] - off[rs];
    if (k < K) {
      const int32_t it = item_of[re];
      c += item_n[it];
      s += item_slots[it];
    }
    cnt[k] = c;
    slots[k] = s;
  }
}

// one warp per unit: the run's offsets and vertices as coalesced copies (4
// loads in flight per lane), then the item's pieces flattened across lanes.
// (Measured: batching 32 unit headers per warp with the runs flattened across
// lanes and items in a separate half of the grid was slower -- 0.31 vs 0.21 ms
// at 10M: the per-element owner search is instruction-bound.)
#ifndef TM_STITCH_MINB
#define TM_STITCH_MINB 1
#endif
__global__ void __launch_bounds__(256, TM_STITCH_MINB) k_stitch_units(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                      const int64_t* __restrict__ Pp, const int32_t* __restrict__ srt,
                                                      const int64_t* __restrict__ Kp,
                                                      const int32_t* __restrict__ item_of,
                                                      const int64_t* __restrict__ item_list,
                                                      const int32_t* __restrict__ item_n,
                                                      const int32_t* __restrict__ pool,
                                                      const int64_t* __restrict__ pbase,
                                                      const int64_t* __restrict__ sbase, int64_t* __restrict__ off_out,
                                                      int32_t* __restrict__ v_out) {
  const int lane = threadIdx.x & 31;
  const int64_t P = *Pp, K = *Kp;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k <= K; k += nw) {
    int64_t rs, re;
    unit_range(srt, K, P, k, &rs, &re);
    int64_t pb = pbase[k], sb = sbase[k];
    const int64_t o0 = off[rs], o1 = off[re];
    for (int64_t i0 = rs; i0 < re; i0 += 128) {
      int64_t b[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t i = i0 + q * 32 + lane;
        if (i < re) b[q] = off[i];
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t i = i0 + q * 32 + lane;
        if (i < re) off_out[pb + (i - rs)] = sb + (b[q] - o0);
      }
    }
    for (int64_t j0 = o0; j0 < o1; j0 += 128) {
      int32_t b[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t j = j0 + q * 32 + lane;
        if (j < o1) b[q] = v[j];
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t j = j0 + q * 32 + lane;
        if (j < o1) v_out[sb + (j - o0)] = b[q];
      }
    }
    if (k == K) continue;
    pb += re - rs;
    sb += o1 - o0;
    const int32_t w = item_of[re];
    const int64_t list = item_list[w];
    const int n = item_n[w];
    if (list < 0) continue;
    for (int c = 0; c < n; c += 32) {  // the item's pieces, flattened across lanes
      const int r = c + lane;
      uint32_t ro = 0;
      int ln = 0;
      if (r < n) {
        ro = (uint32_t)pool[list + 2 * r];
        ln = (int)((uint32_t)pool[list + 2 * r + 1] & LEN_MASK);
      }
      int inc = ln;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int start = inc - ln, total = __shfl_sync(0xffffffffu, inc, 31);
      if (r < n) off_out[pb + r] = sb + start;
      for (int kb = 0; kb < total; kb += 32) {
        const int e = kb + lane;
        int lo = 0;
        for (int step = 16; step > 0; step >>= 1) {
          const int cand = lo + step;
          const int cs = __shfl_sync(0xffffffffu, start, cand < 32 ? cand : 31);
          if (cand < 32 && cand + c < n && cs <= e) lo = cand;
        }
        const uint32_t lro = __shfl_sync(0xffffffffu, ro, lo);
        const int ls = __shfl_sync(0xffffffffu, start, lo);
        if (e < total) v_out[sb + e] = pool[lro + (e - ls)];
      }
      sb += total;
    }
  }
}

__global__ void k_finalize(const int64_t* __restrict__ Pp, const int64_t* __restrict__ pbase,
                           const int64_t* __restrict__ sbase, int64_t* __restrict__ off_out, int64_t* p_out,
                           int64_t* f_out) {
  if (threadIdx.x || blockIdx.x) return;
  int64_t P = *Pp;
  off_out[pbase[P]] = sbase[P];
  *p_out = pbase[P];
  *f_out = sbase[P];
}

__global__ void k_undo(int32_t* hw, const int32_t* undo, const unsigned long long* undo_top, unsigned long long cap) {
  unsigned long long n = *undo_top;
  if (n > cap) n = cap;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    int32_t e = undo[k];
    int32_t te = hw_twin(hw[e]);
    hw[e] &= ~1;
    if (te >= 0) hw[te] &= ~1;
  }
}

static inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

__global__ void __launch_bounds__(256) k_tv_items(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                  const int32_t* __restrict__ hv, const int32_t* __restrict__ items,
                                                  const unsigned int* n_items, int32_t* __restrict__ tv) {
  const int lane = threadIdx.x & 31;
  const unsigned int ni = *n_items;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < ni;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t i = items[w];
    const int64_t b = off[i], e = off[i + 1];
    for (int64_t k = b + lane; k < e; k += 32) tv[v[k]] = hv[k] / 3;
  }
}

void launch_tv_items(const int64_t* off, const int32_t* v, const int32_t* hv, const int32_t* items,
                     const unsigned int* n_items, int64_t Pcap, int32_t* tv, cudaStream_t s) {
  k_tv_items<<<kNumSMs * 8, 256, 0, s>>>(off, v, hv, items, n_items, tv);
  note_launch(1);
}

void launch_classify(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, int32_t* item_of,
                     int32_t* items, unsigned int* n_items, int32_t* long_list, unsigned int* n_long,
                     unsigned long long* stats, LongQueue q, const int32_t* hv, int32_t* tv, int which,
                     int32_t* item_state, int32_t* pool, unsigned long long* pool_top, unsigned long long pool_cap,
                     int32_t* item_depth, cudaStream_t s) {
  if (which != 2) {  // short polygons (and with which == 0 the list of the long ones)
    k_classify<<<grid_for(Pcap, 256), 256, 0, s>>>(off, v, Pp, item_of, items, n_items, long_list, n_long, stats, hv,
                                                   tv, which == 0, item_state);
    note_launch(1);
  }
  if (which == 1) return;
  k_classify_long<<<kNumSMs * 4, 256, 0, s>>>(off, v, long_list, n_long, item_of, items, n_items, stats, q, hv, tv,
                                              item_state, pool, pool_top, pool_cap, item_depth);
  note_launch(1);
}

void launch_repair_tips_long(const RepairArgs& a, cudaStream_t s) {
  RepairCtx c{a.tri, a.hw, a.tv, a.T, a.pool, a.pool_cap, a.pool_top, a.undo, a.undo_top, a.undo_cap, a.st, a.tv_exact,
              a.dbg};
  static bool attr = false;
  size_t smem = seg_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_repair_tips_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  static int trace_qi = -1;
  if (trace_qi < 0) {  // debug: which long item's rounds are timestamped
    const char* e = getenv("TERMESH_TRACE_QI");
    trace_qi = (e && *e) ? atoi(e) : 0;
  }
  static int seg_cap = -1;
  if (seg_cap < 0) {  // testing hook: TERMESH_SEG_CAP shrinks the segment arena to exercise spills
    const char* e = getenv("TERMESH_SEG_CAP");
    seg_cap = (e && *e) ? atoi(e) : kSegCap;
    if (seg_cap > kSegCap) seg_cap = kSegCap;
  }
  // Blocks of this kernel fill an SM's shared memory, so every SM it holds is
  // closed to the short-item kernel running beside it.  The long items are few
  // (~17 per 1M triangles) and the longest runs first, so a small grid keeps the
  // lineage on time and leaves the other SMs to the short items: 24 blocks up
  // to 20M triangles (measured best at 1M and 10M, 16-24), proportionally more above.
  static int env_blk = -1;
  if (env_blk < 0) {  // tuning hook: TERMESH_SEG_BLOCKS
    const char* e = getenv("TERMESH_SEG_BLOCKS");
    env_blk = (e && *e) ? atoi(e) : 0;
  }
  static int smem_max_l = -1;
  if (smem_max_l < 0) {  // testing hook: TERMESH_SEG_SMEM_MAXL sends shorter items to the global-memory mode
    const char* e = getenv("TERMESH_SEG_SMEM_MAXL");
    smem_max_l = (e && *e) ? atoi(e) : kSegMaxL;
    if (smem_max_l > kSegMaxL) smem_max_l = kSegMaxL;
  }
  static int rec_limit = -1;
  if (rec_limit < 0) {  // testing hook: TERMESH_SEG_REC_CAP moves items to the pool region after fewer pieces
    const char* e = getenv("TERMESH_SEG_REC_CAP");
    rec_limit = (e && *e) ? atoi(e) : kSegRec;
    if (rec_limit > kSegRec || rec_limit < 8) rec_limit = kSegRec;
  }
  static int gm_dups = -1;
  if (gm_dups < 0) {  // items with more extra visits than this go to the pool-region blocks
    const char* e = getenv("TERMESH_SEG_GM_DUPS");
    gm_dups = (e && *e) ? atoi(e) : 3 * kSegRec / 4;
  }
  long long nblk = env_blk > 0 ? env_blk : 24 * (a.T / 20000000 + 1);
  if (nblk > kNumSMs - kGmBlocks) nblk = kNumSMs - kGmBlocks;
  nblk += kGmBlocks;  // blocks [0, kGmBlocks) take the pool-region items
  k_repair_tips_seg<<<(int)nblk, 32 * kSegWarps, smem, s>>>(c, a.items, a.off, a.v, a.item_list, a.item_n,
                                                           a.item_state, a.item_depth, a.item_slots, a.stats, a.q,
                                                           a.dbg,
                                                           (unsigned int)trace_qi, seg_cap, smem_max_l, rec_limit,
                                                           gm_dups, kGmBlocks);
  note_launch(1);
}

void launch_repair_tips(const RepairArgs& a, int mode, cudaStream_t s) {
  RepairCtx c{a.tri, a.hw, a.tv, a.T, a.pool, a.pool_cap, a.pool_top, a.undo, a.undo_top, a.undo_cap, a.st, a.tv_exact,
              a.dbg};
  static int resident = 0;
  if (!resident) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_repair_tips, 32 * kTipWarps, 0);
    if (resident < 1) resident = 1;
  }
  k_repair_tips<<<mode ? kNumSMs : kNumSMs * resident, 32 * kTipWarps, 0, s>>>(
      c, a.items, a.n_items, a.off, a.v, a.item_list, a.item_n, a.item_state, a.item_depth, a.item_slots, a.stats,
      a.q, mode);
  note_launch(1);
}

void launch_repair_pinch(const RepairArgs& a, int mode, cudaStream_t s) {
  RepairCtx c{a.tri, a.hw, a.tv, a.T, a.pool, a.pool_cap, a.pool_top, a.undo, a.undo_top, a.undo_cap, a.st, a.tv_exact,
              a.dbg};
  static bool attr = false;
  const size_t smem = 4 * kPinchDupCap * sizeof(int2);
  if (!attr) {
    cudaFuncSetAttribute(k_repair_pinch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // mode 2 runs beside the short-item kernels: a few blocks (128 KB of shared memory each)
  static int p2 = -1;
  if (p2 < 0) {  // tuning hook: TERMESH_PINCH2_BLOCKS
    const char* e = getenv("TERMESH_PINCH2_BLOCKS");
    p2 = (e && *e) ? atoi(e) : 16;
    if (p2 < 1) p2 = 16;
  }
  k_repair_pinch<<<mode == 2 ? p2 : mode ? kNumSMs : kNumSMs * 2, 128, smem, s>>>(c, a.items, a.n_items, a.off, a.item_list, a.item_n,
                                                                  a.item_slots, a.item_state, a.item_depth, a.q,
                                                                  a.stats, mode);
  note_launch(1);
}

void launch_out_counts(const int64_t* off, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                       const int32_t* item_n, const int64_t* item_slots, int64_t* cnt, int64_t* slots,
                       const unsigned long long* stats, DevStatus* st, cudaStream_t s) {
  k_out_counts<<<grid_for(Pcap + 1, 256), 256, 0, s>>>(off, Pp, item_of, item_n, item_slots, cnt, slots, stats, st);
  note_launch(1);
}

void launch_stitch(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                   const int32_t* items, const unsigned int* n_items, const int64_t* item_list, const int32_t* item_n,
                   const int32_t* pool, const int64_t* pbase, const int64_t* sbase, int64_t* off_out, int32_t* v_out,
                   cudaStream_t s) {
  k_stitch<<<kNumSMs * 12, 256, 0, s>>>(off, v, Pp, item_of, items, n_items, item_list, item_n, pool, pbase, sbase,
                                        off_out, v_out);
  note_launch(1);
}

void launch_item_sort(const int32_t* item_of, const int64_t* Pp, int64_t Pcap, uint8_t* flag, int32_t* srt,
                      int64_t* n_srt, int64_t* tiles, cudaStream_t s) {
  k_item_flags<<<grid_for(Pcap, 256), 256, 0, s>>>(item_of, Pp, Pcap, flag);
  note_launch(1);
  launch_select_flags(flag, Pcap, srt, n_srt, tiles, s, 0);
}

void launch_unit_counts(const int64_t* off, const int64_t* Pp, int64_t Pcap, const int32_t* srt, const int64_t* n_srt,
                        const int32_t* item_of, const int32_t* item_n, const int64_t* item_slots, int64_t* cnt,
                        int64_t* slots, int64_t* n_units, const unsigned long long* stats, DevStatus* st,
                        cudaStream_t s) {
  k_unit_counts<<<grid_for(Pcap / 8 + 2, 256), 256, 0, s>>>(off, Pp, srt, n_srt, item_of, item_n, item_slots, cnt,
                                                             slots, n_units, stats, st);
  note_launch(1);
}

void launch_stitch_units(const int64_t* off, const int32_t* v, const int64_t* Pp, const int32_t* srt,
                         const int64_t* n_srt, const int32_t* item_of, const int64_t* item_list, const int32_t* item_n,
                         const int32_t* pool, const int64_t* pbase, const int64_t* sbase, int64_t* off_out,
                         int32_t* v_out, cudaStream_t s) {
  k_stitch_units<<<kNumSMs * 8, 256, 0, s>>>(off, v, Pp, srt, n_srt, item_of, item_list, item_n, pool, pbase, sbase,
                                             off_out, v_out);
  note_launch(1);
}

void launch_finalize(const int64_t* Pp, const int64_t* pbase, const int64_t* sbase, int64_t* off_out,
                     int64_t* p_out, int64_t* f_out, cudaStream_t s) {
  k_finalize<<<1, 32, 0, s>>>(Pp, pbase, sbase, off_out, p_out, f_out);
  note_launch(1);
}

__global__ void k_stamp(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

// debug timeline (TERMESH_STAMPS): the time a stream reaches this point
void launch_stamp(unsigned long long* slot, cudaStream_t s) { k_stamp<<<1, 1, 0, s>>>(slot); }

void launch_undo(int32_t* hw, const int32_t* undo, const unsigned long long* undo_top, unsigned long long cap,
                 cudaStream_t s) {
  k_undo<<<kNumSMs, 256, 0, s>>>(hw, undo, undo_top, cap);
  note_launch(1);
}

}  // namespace tmb
