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

constexpr int kLongMin = 96;    // items longer than this go to k_repair_tips_long first
constexpr int kHugeMin = 512;   // ... and the longest ones are dequeued first
constexpr uint32_t F_TIP = 1u << 30;
constexpr uint32_t F_REP = 1u << 31;
constexpr uint32_t F_FAIL = 1u << 29;
constexpr uint32_t LEN_MASK = (1u << 29) - 1;

struct RepairCtx {
  const int32_t* tri;
  int32_t* hw;
  const int32_t* tv;
  int64_t T;
  int32_t* pool;
  unsigned long long pool_cap;
  unsigned long long* pool_top;
  int32_t* undo;
  unsigned long long* undo_top;
  unsigned long long undo_cap;
  DevStatus* st;
};

__device__ __forceinline__ int64_t palloc(const RepairCtx& c, int64_t n) {
  unsigned long long o = atomicAdd(c.pool_top, (unsigned long long)n);
  if (o + (unsigned long long)n > c.pool_cap) return -1;
  return (int64_t)o;
}

__device__ __forceinline__ void promote(const RepairCtx& c, int32_t e, int32_t te) {
  c.hw[e] |= 1;
  c.hw[te] |= 1;
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
  c.hw[e] &= ~1;
  c.hw[te] &= ~1;
}

// traversal.py:112-124 for one polygon
__device__ bool poly_has_tip(const int32_t* s, int64_t n) {
  for (int64_t pos = 0; pos < n; pos++) {
    int64_t a = pos == 0 ? n - 1 : pos - 1, b = pos + 1 == n ? 0 : pos + 1;
    if (s[a] == s[b]) return true;
  }
  return false;
}

// reparation.py:59-71
__device__ int64_t first_tip(const int32_t* s, int64_t n) {
  for (int64_t pos = 0; pos < n; pos++) {
    int64_t a = pos == 0 ? n - 1 : pos - 1, b = pos + 1 == n ? 0 : pos + 1;
    if (s[a] == s[b]) return pos;
  }
  return -1;
}

// (len - distinct) of one polygon (traversal.py:140-147).  Small polygons use a
// quadratic scan; long ones an in-place heap sort of a scratch copy.
__device__ void sift(int32_t* a, int64_t root, int64_t n) {
  for (;;) {
    int64_t ch = 2 * root + 1;
    if (ch >= n) return;
    if (ch + 1 < n && a[ch + 1] > a[ch]) ch++;
    if (a[root] >= a[ch]) return;
    int32_t t = a[root];
    a[root] = a[ch];
    a[ch] = t;
    root = ch;
  }
}

__device__ int64_t extra_visits(const int32_t* s, int64_t n, int32_t* scratch) {
  if (n <= 48 || scratch == nullptr) {
    int64_t extra = 0;
    for (int64_t i = 1; i < n; i++) {
      bool dup = false;
      for (int64_t j = 0; j < i && !dup; j++) dup = s[j] == s[i];
      extra += dup;
    }
    return extra;
  }
  for (int64_t i = 0; i < n; i++) scratch[i] = s[i];
  for (int64_t r = n / 2 - 1; r >= 0; r--) sift(scratch, r, n);
  for (int64_t e = n - 1; e > 0; e--) {
    int32_t t = scratch[0];
    scratch[0] = scratch[e];
    scratch[e] = t;
    sift(scratch, 0, e);
  }
  int64_t extra = 0;
  for (int64_t i = 1; i < n; i++) extra += scratch[i] == scratch[i - 1];
  return extra;
}

// ------------------------------------------------------------ classify
// Per input polygon: tip flag, repeated flag, extra visits.  Work items are the
// polygons with a repeated vertex (a tip implies one).
__global__ void __launch_bounds__(256) k_classify(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                  const int64_t* __restrict__ Pp, int32_t* __restrict__ item_of,
                                                  int32_t* __restrict__ items, unsigned int* n_items,
                                                  int32_t* __restrict__ long_list, unsigned int* n_long,
                                                  unsigned long long* stats) {
  const int64_t P = *Pp;
  unsigned long long extra_sum = 0, rep_cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = off[i], n = off[i + 1] - b;
    item_of[i] = -1;
    if (n > 48) {
      long_list[atomicAdd(n_long, 1u)] = (int32_t)i;
      continue;
    }
    int64_t ex = extra_visits(v + b, n, nullptr);
    if (ex > 0) {
      extra_sum += ex;
      rep_cnt++;
      unsigned int k = atomicAdd(n_items, 1u);
      items[k] = (int32_t)i;
      item_of[i] = (int32_t)k;
    }
  }
  if (extra_sum) atomicAdd(stats + 2, extra_sum);
  if (rep_cnt) atomicAdd(stats + 6, rep_cnt);
}

// long polygons: one block each; distinct vertices counted with a shared-memory
// open-addressing set (len <= kSetCap/2), else a block-parallel quadratic scan.
constexpr int kSetCap = 8192;
__global__ void __launch_bounds__(256) k_classify_long(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                       const int32_t* __restrict__ long_list,
                                                       const unsigned int* n_long, int32_t* __restrict__ item_of,
                                                       int32_t* __restrict__ items, unsigned int* n_items,
                                                       unsigned long long* stats, LongQueue q) {
  __shared__ int32_t tab[kSetCap];
  __shared__ unsigned int dups;
  unsigned int nl = *n_long;
  for (unsigned int w = blockIdx.x; w < nl; w += gridDim.x) {
    int32_t i = long_list[w];
    int64_t b = off[i];
    int n = (int)(off[i + 1] - b);
    const int32_t* s = v + b;
    if (threadIdx.x == 0) dups = 0;
    unsigned int my = 0;
    if (2 * n <= kSetCap) {
      int cap = 64;
      while (cap < 2 * n) cap <<= 1;
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
    if (threadIdx.x == 0 && dups > 0) {
      unsigned int k = atomicAdd(n_items, 1u);
      items[k] = i;
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

// Re-walk split (reparation.py:216-229 after promotion).  Returns 1 on success
// (pieces written), 0 when the length law fails (caller decides strictness),
// -1 on error/capacity.
__device__ int rewalk_split(const RepairCtx& c, int32_t e, int32_t te, int64_t plen, int32_t poly,
                            int64_t* pa_off, int64_t* pa_len, int64_t* pb_off, int64_t* pb_len) {
  int32_t ha = min_frontier_slot(c.hw, e / 3), hb = min_frontier_slot(c.hw, te / 3);
  long long la = walk_len(c, ha), lb = walk_len(c, hb);
  if (la < 0 || lb < 0) { report(c.st, K_STRUCT, poly); return -1; }
  if (la + lb != plen + 2) return 0;
  int64_t o = palloc(c, la + lb);
  if (o < 0) { report(c.st, K_POOL, poly); return -1; }
  walk_write(c, ha, c.pool + o);
  walk_write(c, hb, c.pool + o + la);
  *pa_off = o; *pa_len = la; *pb_off = o + la; *pb_len = lb;
  return 1;
}

// ------------------------------------------------------------ warp helpers
// One warp cooperates on one piece.  Lanes split O(len) scans and copies; the
// sequential mesh rotations run on one or two lanes and are broadcast.  All
// control flow below is warp-uniform.
constexpr unsigned kFull = 0xffffffffu;
constexpr int kFanCap = 64;
constexpr int kTipWarps = 4;  // warps per block of k_repair_tips

__device__ __forceinline__ int wrap_idx(int x, int n) { return x >= n ? x - n : (x < 0 ? x + n : x); }

// Smallest p in [0, n) with pred(p), or -1.  Eight 32-wide chunks per round
// so their loads are in flight together (one memory round trip per 256).
constexpr int kScanUnroll = 8;
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
__device__ int32_t warp_middle_internal_edge(const RepairCtx& c, int32_t v, int32_t barrier, int32_t poly,
                                             int32_t* fan, int32_t* back, int lane, bool quiet = false) {
  int deg = warp_collect_fan(c, v, fan, back, lane);
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
                                int lane, bool promote_now, bool quiet, SplitInfo* out) {
  int32_t e = warp_middle_internal_edge(c, v, b, poly, fan, back, lane, quiet);
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

// ------------------------------------------------------------ tip phase, global pool
// Item states (item_state[w]): 0 = not started, 1 = finished by the shared-
// memory kernel, 2 = resume from item_list/item_n/item_depth in the pool.

__device__ void finish_item(const RepairCtx& c, int64_t w, long long list, int n, long long depth, long long splits,
                            int lane, int64_t* item_list, int32_t* item_n, unsigned long long* stats) {
  // repeated flags and extra visits of the leaves (pinch guard, reparation.py:322)
  unsigned long long ex_sum = 0;
  for (int r = 0; r < n; r++) {
    uint32_t ro = (uint32_t)c.pool[list + 2 * r], rl = (uint32_t)c.pool[list + 2 * r + 1];
    int ex = warp_extra_visits(c.pool + ro, (int)(rl & LEN_MASK), lane);
    if (ex > 0 && lane == 0) c.pool[list + 2 * r + 1] = (int32_t)(rl | F_REP);
    ex_sum += ex;
  }
  __syncwarp();
  if (lane == 0) {
    item_list[w] = list;
    item_n[w] = n;
    if (depth > 0) atomicMax(stats + 0, (unsigned long long)depth);
    if (splits) atomicAdd(stats + 1, (unsigned long long)splits);
    if (ex_sum) atomicAdd(stats + 5, ex_sum);
  }
}

// One warp per work item.  item_list[w] = pool offset of the item's record
// list, item_n[w] = #records (leaves in the reference's raw order).
__global__ void __launch_bounds__(32 * kTipWarps) k_repair_tips(RepairCtx c, const int32_t* __restrict__ items,
                                                                const unsigned int* n_items,
                                                                const int64_t* __restrict__ off,
                                                                const int32_t* __restrict__ v,
                                                                int64_t* __restrict__ item_list,
                                                                int32_t* __restrict__ item_n,
                                                                const int32_t* __restrict__ item_state,
                                                                const int32_t* __restrict__ item_depth,
                                                                unsigned long long* stats) {
  __shared__ int32_t s_fan[kTipWarps][kFanCap];
  __shared__ int32_t s_back[kTipWarps][kFanCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* fan = s_fan[wib];
  int32_t* back = s_back[wib];
  unsigned int ni = *n_items;
  // reparation.py:354-364: at most initial + 1 rounds, initial = extra visits of mesh0
  long long max_rounds = (long long)stats[2] + 1;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < ni; w += nwarps) {
    int st = item_state[w];
    if (st == 1) continue;
    int32_t i = items[w];
    int64_t b = off[i];
    int L = (int)(off[i + 1] - b);
    if (st == 0 && L > kLongMin) continue;  // handled by k_repair_tips_long (state 1/2/3)
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
        if (lane == 0) { report(c.st, K_POOL, i); item_list[w] = -1; item_n[w] = 0; }
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
      if (lane == 0) { item_list[w] = -1; item_n[w] = 0; }
      continue;
    }
    finish_item(c, w, list, n, depth, splits, lane, item_list, item_n, stats);
  }
}

// ------------------------------------------------------------ tip phase, shared memory
// Long items (hull slivers: 902 vertices / 70 tips / 41 rounds at 1M): one
// block each, pieces in a shared-memory bump arena, the tipped pieces of a
// round split concurrently by the block's warps (distinct pieces have
// disjoint interiors).  Scans run at shared-memory latency; only the mesh
// rotations touch global memory.  If the arena or the record list fills up,
// the current pieces are written to the global pool and the warp kernel
// resumes the item (item_state = 2).
constexpr int kLongWarps = 8;
constexpr int kLongArena = 32 * 1024;  // ints (128 KiB)
constexpr int kLongRec = 1024;         // records per list
constexpr int kMaxTips = 1024;         // precomputed tips per item
constexpr int kMaxTouch = 2048;        // promoted-edge endpoints per item
size_t long_smem_bytes() {
  return (size_t)kLongArena * 4 + 2 * (size_t)kLongRec * 8 + 2 * (size_t)kLongWarps * kFanCap * 4 +
         (size_t)kMaxTips * 4 * 2 + (size_t)kMaxTips * sizeof(SplitInfo) + (size_t)kMaxTouch * 4 + 64;
}

__global__ void __launch_bounds__(32 * kLongWarps) k_repair_tips_long(RepairCtx c, const int32_t* __restrict__ items,
                                                                      const unsigned int* n_items,
                                                                      const int64_t* __restrict__ off,
                                                                      const int32_t* __restrict__ v,
                                                                      int64_t* __restrict__ item_list,
                                                                      int32_t* __restrict__ item_n,
                                                                      int32_t* __restrict__ item_state,
                                                                      int32_t* __restrict__ item_depth,
                                                                      unsigned long long* stats, int arena_cap,
                                                                      LongQueue q, unsigned long long* dbg) {
  extern __shared__ __align__(16) int32_t smem[];
  int32_t* arena = smem;
  int2* recs = reinterpret_cast<int2*>(arena + kLongArena);  // [2][kLongRec] {offset, len|flags}
  int32_t* fans = reinterpret_cast<int32_t*>(recs + 2 * kLongRec);
  int32_t* tipv = fans + 2 * kLongWarps * kFanCap;  // tip vertex (or -1 when its info is unusable)
  int32_t* tipb = tipv + kMaxTips;                  // barrier vertex
  SplitInfo* tipinfo = reinterpret_cast<SplitInfo*>(tipb + kMaxTips);
  int32_t* touched = reinterpret_cast<int32_t*>(tipinfo + kMaxTips);
  __shared__ int s_ntip, s_ntouch;
  __shared__ int s_top, s_fail, s_ntips;
  __shared__ int s_out[kLongRec];  // output index of each input record
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* fan = fans + wib * kFanCap;
  int32_t* back = fans + (kLongWarps + wib) * kFanCap;
  (void)n_items;
  long long max_rounds = (long long)stats[2] + 1;
  // dynamic queue, longest class first (the hull-sliver lineage sets the critical path)
  const unsigned int nh = *q.n_huge, nq = nh + *q.n_long;
  __shared__ unsigned int s_w;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_w = atomicAdd(q.next, 1u);
    __syncthreads();
    unsigned int qi = s_w;
    if (qi >= nq) break;
    unsigned int w = qi < nh ? (unsigned int)q.huge[qi] : (unsigned int)q.longq[qi - nh];
    const bool trace = qi == 0 && threadIdx.x == 0;
    unsigned long long t_ns;
    if (trace) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns)); dbg[0] = t_ns; }
    int32_t i = items[w];
    int64_t b = off[i];
    int L = (int)(off[i + 1] - b);
    if (L + 2 > arena_cap) {  // does not fit: the warp kernel does it from scratch
      if (threadIdx.x == 0) item_state[w] = 3;
      continue;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L; k += blockDim.x) arena[k] = v[b + k];
    if (threadIdx.x == 0) { s_top = L; s_fail = 0; }
    __syncthreads();
    int cur = 0, n = 1;
    if (threadIdx.x == 0) { s_ntip = 0; s_ntouch = 0; }
    __syncthreads();
    // Every tip of the item is a tip of its initial polygon (an arc split only
    // removes the split tip), and its split edge depends only on the frontier
    // around v and u.  So the mesh rotations for all tips run up front, in
    // parallel; a round reuses them unless an earlier promotion touched v or u.
    for (int p = threadIdx.x; p < L; p += blockDim.x) {
      int32_t a = arena[p == 0 ? L - 1 : p - 1];
      if (a == arena[p + 1 == L ? 0 : p + 1]) {
        int k = atomicAdd(&s_ntip, 1);
        if (k < kMaxTips) { tipv[k] = arena[p]; tipb[k] = a; }
      }
    }
    __syncthreads();
    const int ntip_pre = s_ntip < kMaxTips ? s_ntip : kMaxTips;
    for (int k = wib; k < ntip_pre; k += kLongWarps) {
      SplitInfo si;
      bool ok = warp_split_info(c, tipv[k], tipb[k], i, fan, back, lane, false, true, &si);
      if (lane == 0) {
        tipinfo[k] = si;
        if (!ok) tipv[k] = -1;
      }
    }
    __syncthreads();
    if (trace) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns)); dbg[1] = t_ns; dbg[2] = L; dbg[3] = s_ntip; }
    if (wib == 0) {
      uint32_t f0 = s_ntip > 0 ? F_TIP : 0u;
      if (lane == 0) { recs[0] = make_int2(0, (int)((uint32_t)L | f0)); s_ntips = f0 ? 1 : 0; }
    }
    __syncthreads();
    int ntips = s_ntips;
    long long depth = 0, splits = 0;
    bool bad = false, spill = false;
    while (ntips > 0) {
      if (depth + 1 > max_rounds) {
        if (threadIdx.x == 0) report(c.st, K_NO_CONVERGE, i);
        bad = true;
        break;
      }
      int2* in = recs + cur * kLongRec;
      int2* out = recs + (cur ^ 1) * kLongRec;
      // output slot of every input record (prefix over tip flags) and the arena
      // the round needs (a split writes |piece| + 2 slots), warp 0
      __shared__ int s_need;
      if (wib == 0) {
        int carry = 0, need = 0;
        for (int base = 0; base < n; base += 32) {
          int r = base + lane;
          int t = (r < n && ((uint32_t)in[r].y & F_TIP)) ? 1 : 0;
          int inc = t;
          for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
          }
          if (r < n) s_out[r] = r + carry + inc - t;
          carry += __shfl_sync(kFull, inc, 31);
          int nd = t ? (int)((uint32_t)in[r].y & LEN_MASK) + 2 : 0;
          for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(kFull, nd, o);
          need += nd;
        }
        if (lane == 0) s_need = need;
      }
      if (threadIdx.x == 0) s_ntips = 0;
      __syncthreads();
      if (n + ntips > kLongRec || s_top + s_need > arena_cap) { spill = true; break; }  // uniform
      depth++;
      const int ntouch0 = s_ntouch < kMaxTouch ? s_ntouch : -1;  // -1: overflowed, always recompute
      __syncthreads();
      // untouched records are pointer copies; tipped ones are split by a warp each
      for (int r = threadIdx.x; r < n; r += blockDim.x)
        if (!((uint32_t)in[r].y & F_TIP)) out[s_out[r]] = in[r];
      int t_idx = 0;
      for (int r = 0; r < n; r++) {
        if (!((uint32_t)in[r].y & F_TIP)) continue;
        int mine = (t_idx++ % kLongWarps) == wib;
        if (!mine) continue;
        auto alloc = [&](long long m) -> int32_t* {
          int o = 0;
          if (lane == 0) o = atomicAdd(&s_top, (int)m);
          o = __shfl_sync(kFull, o, 0);
          if (o + m > arena_cap) return nullptr;
          return arena + o;
        };
        int32_t *A, *B;
        int al, bl;
        const int32_t* X = arena + in[r].x;
        const int Lr = (int)((uint32_t)in[r].y & LEN_MASK);
        bool ok = false;
        int pos = warp_first_tip(X, Lr, lane);
        if (pos < 0) {
          if (lane == 0) report(c.st, K_STRUCT, i);
        } else {
          int32_t v = X[pos], bv = X[pos == 0 ? Lr - 1 : pos - 1];
          int k = warp_find_first(ntip_pre, lane, [&](int q) { return tipv[q] == v; });
          SplitInfo si;
          bool use = k >= 0 && ntouch0 >= 0;
          if (use) {
            si = tipinfo[k];
            bool stale = warp_find_first(ntouch0, lane, [&](int q) {
                           int32_t x = touched[q];
                           return x == v || x == si.u;
                         }) >= 0;
            use = !stale;
          }
          if (use) {
            if (lane == 0) promote(c, si.e, si.te);
            __syncwarp();
            ok = true;
          } else {
            ok = warp_split_info(c, v, bv, i, fan, back, lane, true, false, &si);
          }
          if (ok) {
            if (lane == 0) {
              int tk = atomicAdd(&s_ntouch, 2);
              if (tk + 2 <= kMaxTouch) { touched[tk] = v; touched[tk + 1] = si.u; }
            }
            ok = warp_split_arcs(c, X, Lr, pos, si, i, lane, alloc, &A, &al, &B, &bl);
          }
        }
        if (!ok) {
          if (lane == 0) atomicCAS(&s_fail, 0, 1);
          continue;
        }
        uint32_t fa = warp_tip_flag(A, al, lane), fb = warp_tip_flag(B, bl, lane);
        if (lane == 0) {
          int o = s_out[r];
          out[o] = make_int2((int)(A - arena), (int)((uint32_t)al | fa));
          out[o + 1] = make_int2((int)(B - arena), (int)((uint32_t)bl | fb));
          atomicAdd(&s_ntips, (fa ? 1 : 0) + (fb ? 1 : 0));
        }
      }
      __syncthreads();
      splits += ntips;
      n += ntips;
      ntips = s_ntips;
      cur ^= 1;
      if (trace && depth < 56) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns)); dbg[4 + depth] = t_ns; }
      if (s_fail) {
        bad = true;  // (the arena cannot overflow: capacity was checked before the round)
        break;
      }
    }
    if (bad) {
      if (threadIdx.x == 0) { item_state[w] = 1; item_list[w] = -1; item_n[w] = 0; }
      continue;
    }
    // leaves (or the state before an unsplit round) -> global pool
    int2* fin = recs + cur * kLongRec;
    __shared__ long long s_base;
    __shared__ int s_tot;
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int r = 0; r < n; r++) tot += (int)((uint32_t)fin[r].y & LEN_MASK);
      s_tot = tot;
      s_base = palloc(c, tot + 2 * (long long)n);
    }
    __syncthreads();
    if (s_base < 0) {
      if (threadIdx.x == 0) { report(c.st, K_POOL, i); item_state[w] = 1; item_list[w] = -1; item_n[w] = 0; }
      continue;
    }
    long long list = s_base + s_tot;
    if (wib == 0) {
      int carry = 0;
      for (int base = 0; base < n; base += 32) {
        int r = base + lane;
        int ln = r < n ? (int)((uint32_t)fin[r].y & LEN_MASK) : 0;
        int inc = ln;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (r < n) {
          c.pool[list + 2 * r] = (int32_t)(s_base + carry + inc - ln);
          c.pool[list + 2 * r + 1] = fin[r].y;
        }
        carry += __shfl_sync(kFull, inc, 31);
      }
    }
    __syncthreads();
    for (int r = wib; r < n; r += kLongWarps) {
      uint32_t ro = (uint32_t)c.pool[list + 2 * r];
      int ln = (int)((uint32_t)fin[r].y & LEN_MASK);
      const int32_t* src = arena + fin[r].x;
      warp_copy(c.pool + ro, ln, lane, [&](int k) { return src[k]; });
    }
    __syncthreads();
    if (spill) {
      // record list too long for shared memory: the warp kernel continues
      if (threadIdx.x == 0) { item_state[w] = 2; item_list[w] = list; item_n[w] = n; item_depth[w] = (int)depth; }
      if (threadIdx.x == 0 && splits) atomicAdd(stats + 1, (unsigned long long)splits);
      continue;
    }
    if (wib == 0) {
      // leaf flags from shared memory (fast), then the common epilogue
      unsigned long long ex_sum = 0;
      for (int r = 0; r < n; r++) {
        int ln = (int)((uint32_t)fin[r].y & LEN_MASK);
        int ex = warp_extra_visits(arena + fin[r].x, ln, lane);
        if (ex > 0 && lane == 0) c.pool[list + 2 * r + 1] = (int32_t)((uint32_t)fin[r].y | F_REP);
        ex_sum += ex;
      }
      if (lane == 0) {
        item_state[w] = 1;
        item_list[w] = list;
        item_n[w] = n;
        if (depth > 0) atomicMax(stats + 0, (unsigned long long)depth);
        if (splits) atomicAdd(stats + 1, (unsigned long long)splits);
        if (ex_sum) atomicAdd(stats + 5, ex_sum);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ pinch phase
// Trial-split candidate g (reparation.py:326-332 with strict=False).
__device__ int try_pinch(const RepairCtx& c, int32_t g, int64_t L, int32_t poly, int64_t* ao, int64_t* al,
                         int64_t* bo, int64_t* bl) {
  int32_t w = hw_twin(c.hw[g]);
  if (w < 0) { report(c.st, K_STRUCT, poly); return -1; }
  promote(c, g, w);
  int r = rewalk_split(c, g, w, L, poly, ao, al, bo, bl);
  if (r != 1) demote(c, g, w);
  return r;
}

// _pinch_candidates (reparation.py:169-205) for one piece; returns 1 split, 0 none, -1 error
__device__ int pinch_split(const RepairCtx& c, const int32_t* X, int64_t L, int32_t poly, int64_t* ao, int64_t* al,
                           int64_t* bo, int64_t* bl) {
  int32_t v = -1;
  int64_t p1 = 0, p2 = 0;
  for (int64_t idx = 1; idx < L && v < 0; idx++)
    for (int64_t q = 0; q < idx; q++)
      if (X[q] == X[idx]) { v = X[idx]; p1 = q; p2 = idx; break; }
  if (v < 0) return 0;
  int guard = (int)(3 * c.T + 3 < (1LL << 30) ? 3 * c.T + 3 : (1LL << 30));
  int32_t t0 = c.tv[v];
  int32_t g0 = t0 < 0 ? -1 : he_with_origin(c.tri, t0, v);
  if (g0 < 0) { report(c.st, K_STRUCT, poly); return -1; }
  int deg = 0;
  {
    int32_t g = g0;
    do {
      deg++;
      g = fan_step(c.hw, g, guard);
      if (g < 0 || deg > guard) { report(c.st, K_STRUCT, poly); return -1; }
    } while (g != g0);
  }
  int64_t poss[2] = {p2, p1};
  for (int q = 0; q < 2; q++) {
    int32_t outv = X[(poss[q] + 1) % L];
    int32_t g = g0, gout = -1;
    for (int s = 0; s < deg; s++) {
      if (hw_front(c.hw[g]) && he_target(c.tri, g) == outv) { gout = g; break; }
      g = fan_step(c.hw, g, guard);
    }
    if (gout < 0) { report(c.st, K_STRUCT, poly); return -1; }
    int k = 0;
    g = fan_step(c.hw, gout, guard);
    for (int s = 1; s < deg; s++) {
      if (hw_front(c.hw[g])) break;
      k++;
      g = fan_step(c.hw, g, guard);
    }
    if (k == 0) continue;
    int mid = (k - 1) / 2;
    for (int ord = -1; ord < k; ord++) {
      int idx = ord < 0 ? mid : ord;
      if (ord == mid) continue;
      int32_t cand = gout;
      for (int s = 0; s <= idx; s++) cand = fan_step(c.hw, cand, guard);
      int r = try_pinch(c, cand, L, poly, ao, al, bo, bl);
      if (r != 0) return r;
    }
  }
  for (int64_t idx = p1 + 1; idx < p2; idx++) {
    int32_t x = X[idx];
    int32_t tx = c.tv[x];
    int32_t gx0 = tx < 0 ? -1 : he_with_origin(c.tri, tx, x);
    if (gx0 < 0) { report(c.st, K_STRUCT, poly); return -1; }
    int32_t g = gx0;
    int cnt = 0;
    do {
      if (!hw_front(c.hw[g])) {
        int r = try_pinch(c, g, L, poly, ao, al, bo, bl);
        if (r != 0) return r;
      }
      g = fan_step(c.hw, g, guard);
      if (g < 0 || ++cnt > guard) { report(c.st, K_STRUCT, poly); return -1; }
    } while (g != gx0);
  }
  return 0;
}

__device__ uint32_t piece_flags(const RepairCtx& c, const int32_t* s, int64_t n, int32_t poly, bool* ok) {
  uint32_t f = poly_has_tip(s, n) ? F_TIP : 0u;
  int32_t* scratch = nullptr;
  if (n > 48) {
    int64_t so = palloc(c, n);
    if (so < 0) { report(c.st, K_POOL, poly); *ok = false; return 0; }
    scratch = c.pool + so;
  }
  if (extra_visits(s, n, scratch) > 0) f |= F_REP;
  return f;
}

// Runs for every item: pinch rounds (bounded by the global guard, reparation.py:322-323),
// then the item's output totals (#leaves, #slots, #unrepaired).
__global__ void __launch_bounds__(128) k_repair_pinch(RepairCtx c, const int32_t* __restrict__ items,
                                                      const unsigned int* n_items, int64_t* __restrict__ item_list,
                                                      int32_t* __restrict__ item_n, int64_t* __restrict__ item_slots,
                                                      unsigned long long* stats) {
  unsigned int ni = *n_items;
  long long guard = (long long)stats[5] + 1;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ni; w += (int64_t)gridDim.x * blockDim.x) {
    int32_t i = items[w];
    int64_t list = item_list[w];
    int n = item_n[w];
    item_slots[w] = 0;
    if (list < 0) continue;
    int n0 = n;
    bool ok = true;
    for (long long r = 0; r < guard && ok; r++) {
      int elig = 0;
      for (int k = 0; k < n; k++) {
        uint32_t rl = (uint32_t)c.pool[list + 2 * k + 1];
        elig += (rl & F_REP) && !(rl & F_TIP) && !(rl & F_FAIL);
      }
      if (elig == 0) break;
      int64_t nl = palloc(c, 2 * (int64_t)(n + elig));
      if (nl < 0) { report(c.st, K_POOL, i); ok = false; break; }
      int m = 0, did = 0;
      for (int k = 0; k < n && ok; k++) {
        uint32_t ro = (uint32_t)c.pool[list + 2 * k], rl = (uint32_t)c.pool[list + 2 * k + 1];
        if ((rl & F_REP) && !(rl & F_TIP) && !(rl & F_FAIL)) {
          int64_t ao, al, bo, bl;
          int res = pinch_split(c, c.pool + ro, rl & LEN_MASK, i, &ao, &al, &bo, &bl);
          if (res < 0) { ok = false; break; }
          if (res == 1) {
            uint32_t fa = piece_flags(c, c.pool + ao, al, i, &ok);
            uint32_t fb = piece_flags(c, c.pool + bo, bl, i, &ok);
            c.pool[nl + 2 * m] = (int32_t)ao;
            c.pool[nl + 2 * m + 1] = (int32_t)((uint32_t)al | fa);
            c.pool[nl + 2 * m + 2] = (int32_t)bo;
            c.pool[nl + 2 * m + 3] = (int32_t)((uint32_t)bl | fb);
            m += 2;
            did++;
            continue;
          }
          rl |= F_FAIL;  // a failed pinch fails identically in every later round
        }
        c.pool[nl + 2 * m] = (int32_t)ro;
        c.pool[nl + 2 * m + 1] = (int32_t)rl;
        m++;
      }
      list = nl;
      n = m;
      if (did == 0) break;
    }
    if (!ok) continue;
    unsigned long long unrep = 0;
    int64_t slots = 0;
    for (int k = 0; k < n; k++) {
      uint32_t rl = (uint32_t)c.pool[list + 2 * k + 1];
      slots += rl & LEN_MASK;
      unrep += (rl & F_REP) ? 1 : 0;
    }
    item_list[w] = list;
    item_n[w] = n;
    item_slots[w] = slots;
    if (unrep) atomicAdd(stats + 3, unrep);
    if (n != n0) atomicAdd(stats + 4, (unsigned long long)(n - n0));
  }
}

// ------------------------------------------------------------ stitch
__global__ void __launch_bounds__(256) k_out_counts(const int64_t* __restrict__ off, const int64_t* __restrict__ Pp,
                                                    const int32_t* __restrict__ item_of, const int32_t* __restrict__ item_n,
                                                    const int64_t* __restrict__ item_slots, int64_t* __restrict__ cnt,
                                                    int64_t* __restrict__ slots) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= P; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == P) { cnt[i] = 0; slots[i] = 0; continue; }
    int32_t it = item_of[i];
    if (it < 0) { cnt[i] = 1; slots[i] = off[i + 1] - off[i]; }
    else { cnt[i] = item_n[it]; slots[i] = item_slots[it]; }
  }
}

// untouched polygons: one thread each, up to 16 independent loads in flight
__global__ void __launch_bounds__(256) k_stitch_plain(const int64_t* __restrict__ off, const int32_t* __restrict__ v,
                                                      const int64_t* __restrict__ Pp,
                                                      const int32_t* __restrict__ item_of,
                                                      const int64_t* __restrict__ pbase,
                                                      const int64_t* __restrict__ sbase,
                                                      int64_t* __restrict__ off_out, int32_t* __restrict__ v_out) {
  const int64_t P = *Pp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
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
__global__ void __launch_bounds__(256) k_stitch_items(const int32_t* __restrict__ items,
                                                      const unsigned int* n_items,
                                                      const int64_t* __restrict__ item_list,
                                                      const int32_t* __restrict__ item_n,
                                                      const int32_t* __restrict__ pool,
                                                      const int64_t* __restrict__ pbase,
                                                      const int64_t* __restrict__ sbase,
                                                      int64_t* __restrict__ off_out, int32_t* __restrict__ v_out) {
  const int lane = threadIdx.x & 31;
  const unsigned int ni = *n_items;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
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

void launch_classify(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, int32_t* item_of,
                     int32_t* items, unsigned int* n_items, int32_t* long_list, unsigned int* n_long,
                     unsigned long long* stats, LongQueue q, cudaStream_t s) {
  k_classify<<<grid_for(Pcap, 256), 256, 0, s>>>(off, v, Pp, item_of, items, n_items, long_list, n_long, stats);
  note_launch(1);
  k_classify_long<<<kNumSMs * 4, 256, 0, s>>>(off, v, long_list, n_long, item_of, items, n_items, stats, q);
  note_launch(1);
}

void launch_repair_tips(const RepairArgs& a, cudaStream_t s) {
  RepairCtx c{a.tri, a.hw, a.tv, a.T, a.pool, a.pool_cap, a.pool_top, a.undo, a.undo_top, a.undo_cap, a.st};
  static bool attr = false;
  size_t smem = long_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_repair_tips_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  static int arena_cap = -1;
  if (arena_cap < 0) {  // testing hook: TERMESH_LONG_ARENA shrinks the shared arena to exercise spills
    const char* e = getenv("TERMESH_LONG_ARENA");
    arena_cap = (e && *e) ? atoi(e) : kLongArena;
    if (arena_cap > kLongArena) arena_cap = kLongArena;
  }
  k_repair_tips_long<<<kNumSMs, 32 * kLongWarps, smem, s>>>(c, a.items, a.n_items, a.off, a.v, a.item_list,
                                                             a.item_n, a.item_state, a.item_depth, a.stats,
                                                             arena_cap, a.q, a.dbg);
  k_repair_tips<<<kNumSMs * 8, 32 * kTipWarps, 0, s>>>(c, a.items, a.n_items, a.off, a.v, a.item_list, a.item_n,
                                                       a.item_state, a.item_depth, a.stats);
  note_launch(2);
}

void launch_repair_pinch(const RepairArgs& a, cudaStream_t s) {
  RepairCtx c{a.tri, a.hw, a.tv, a.T, a.pool, a.pool_cap, a.pool_top, a.undo, a.undo_top, a.undo_cap, a.st};
  k_repair_pinch<<<kNumSMs * 4, 128, 0, s>>>(c, a.items, a.n_items, a.item_list, a.item_n, a.item_slots, a.stats);
  note_launch(1);
}

void launch_out_counts(const int64_t* off, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                       const int32_t* item_n, const int64_t* item_slots, int64_t* cnt, int64_t* slots,
                       cudaStream_t s) {
  k_out_counts<<<grid_for(Pcap + 1, 256), 256, 0, s>>>(off, Pp, item_of, item_n, item_slots, cnt, slots);
  note_launch(1);
}

void launch_stitch(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                   const int32_t* items, const unsigned int* n_items, const int64_t* item_list, const int32_t* item_n,
                   const int32_t* pool, const int64_t* pbase, const int64_t* sbase, int64_t* off_out, int32_t* v_out,
                   cudaStream_t s) {
  k_stitch_plain<<<grid_for(Pcap, 256), 256, 0, s>>>(off, v, Pp, item_of, pbase, sbase, off_out, v_out);
  k_stitch_items<<<kNumSMs * 8, 256, 0, s>>>(items, n_items, item_list, item_n, pool, pbase, sbase, off_out, v_out);
  note_launch(2);
}

void launch_finalize(const int64_t* Pp, const int64_t* pbase, const int64_t* sbase, int64_t* off_out,
                     int64_t* p_out, int64_t* f_out, cudaStream_t s) {
  k_finalize<<<1, 32, 0, s>>>(Pp, pbase, sbase, off_out, p_out, f_out);
  note_launch(1);
}

void launch_undo(int32_t* hw, const int32_t* undo, const unsigned long long* undo_top, unsigned long long cap,
                 cudaStream_t s) {
  k_undo<<<kNumSMs, 256, 0, s>>>(hw, undo, undo_top, cap);
  note_launch(1);
}

}  // namespace tmb
