// tm_label.cu -- K0 (half-edge twin build) fused with K1 (LabelMax) and K2
// (LabelSeed + LabelFrontier).
//
// Replaces: mesh_core.compute_trivertex (mesh_core.py:171-178), the neighbor
// back-slot searches of labeling.py:84,110, and labeling.label_max /
// label_seeds / label_frontiers (labeling.py:46-115).  The reference receives
// `neighbors` from Qhull; here adjacency is derived from the triangle list.
//
// Two passes over the triangles, no sort:
// Pass A (per triangle): corners -> tri32, three fp64 squared lengths computed
//   UNFUSED (__dmul_rn/__dadd_rn; numpy's ((b-c)**2).sum is dx*dx + dy*dy with
//   two roundings), first-max argmax -> max_edge; signed-area
//   validation; atomicMin trivertex; and insertion of every ASCENDING
//   half-edge (origin < target) into an open-addressing table keyed by the
//   packed (min, max) vertex pair (u64 keys, u32 half-edge values, linear
//   probing, load <= 0.75).  One CAS per undirected edge, no contention: in a
//   valid mesh each key has exactly one ascending half-edge.
// Pass B (per triangle): every DESCENDING half-edge looks its partner up
//   (read-only probes) and writes the packed words hw = (twin << 1) | frontier
//   of both half-edges plus the seed flags of both triangles, so K0's twin
//   build and K2's labels finish in the same pass.
#include "tm_common.cuh"
#include "tm_internal.h"

#include <utility>

namespace tmb {

// ---------------------------------------------------------------- twin table
// Bucketed open addressing with quotienting.  The undirected edge key
// (lo << b) | hi (K = 2b bits) goes through an invertible K-bit mix x; the top
// q bits of x pick the home bucket, the low R = K - q bits ("remainder") plus
// the bucket displacement d identify the key exactly, so a slot holds the
// whole entry in 64 bits:  [ remainder | d (kDispBits) | half-edge | L ], where L
// says the half-edge is its triangle's longest edge (pass B then needs no
// gather of the partner's max_edge).
// A bucket is 4 slots = one 32-byte sector, so a probe is one sector load.
// Slots of a bucket fill in order and are never cleared, so a lookup may stop
// at the first bucket with an empty slot.
constexpr unsigned long long kEmptySlot = ~0ull;
constexpr unsigned long long kClaimBit = 1ull << 63;
constexpr int kDispBits = 5;
constexpr int kMaxDisp = (1 << kDispBits) - 1;

struct TwinTable {
  unsigned long long* slots;  // 4 * nb
  uint64_t nb_mask;           // nb - 1 (nb = 2^q buckets)
  int K, b, R, hb;
  unsigned int* ovf;          // shrunken table: displacement overflow flag (host retries at full size)
};

__device__ __forceinline__ uint64_t mixK(uint64_t x, int K) {
  const uint64_t M = (K >= 64) ? ~0ull : ((1ull << K) - 1);
  const int s = (K + 1) >> 1;
  x = (x * 0x9E3779B97F4A7C15ull) & M;
  x ^= x >> s;
  x = (x * 0xD6E8FEB86659FD93ull) & M;
  x ^= x >> s;
  return x;
}

struct Probe {
  uint64_t home;
  uint64_t tag;  // (remainder << kDispBits) at displacement 0
};

__device__ __forceinline__ Probe probe_of(const TwinTable& tb, int32_t lo, int32_t hi) {
  uint64_t key = ((uint64_t)(uint32_t)lo << tb.b) | (uint32_t)hi;
  uint64_t x = mixK(key, tb.K);
  Probe p;
  p.home = (x >> tb.R) & tb.nb_mask;
  p.tag = (x & ((1ull << tb.R) - 1)) << kDispBits;
  return p;
}

// A bucket's 4 slots as two 16-byte loads into registers (no local-memory
// array: the slot loops below are fully unrolled over named values).
struct Bucket {
  unsigned long long s0, s1, s2, s3;
  __device__ __forceinline__ unsigned long long at(int k) const {
    return k == 0 ? s0 : k == 1 ? s1 : k == 2 ? s2 : s3;  // k is a compile-time constant after unrolling
  }
};

__device__ __forceinline__ Bucket load_bucket_cg(const unsigned long long* s) {
  const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2*>(s));
  const ulonglong2 b = __ldcg(reinterpret_cast<const ulonglong2*>(s) + 1);
  return Bucket{a.x, a.y, b.x, b.y};
}

__device__ __forceinline__ Bucket load_bucket_nc(const unsigned long long* s) {
  const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(s));
  const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(s) + 1);
  return Bucket{a.x, a.y, b.x, b.y};
}

// Insert ascending half-edge h = lo -> hi.  In a valid mesh each key has one
// ascending half-edge; a second one is an orientation / reciprocity defect.
// Slots fill in order and are never cleared: an empty slot is claimed with a
// CAS; a lost race leaves the slot occupied by the winner, which is then
// examined like any occupied slot.
__device__ __forceinline__ void table_insert(const TwinTable& tb, DevStatus* st, int32_t hl, int32_t lo, int32_t hi) {
  const int32_t h = hl >> 1;  // hl = (h << 1) | L
  Probe p = probe_of(tb, lo, hi);
  for (int d = 0; d <= kMaxDisp; d++) {
    unsigned long long* bk = tb.slots + 4 * ((p.home + d) & tb.nb_mask);
    const uint64_t tag = p.tag | (uint64_t)d;
    const unsigned long long mine = (tag << tb.hb) | (uint32_t)hl;
#ifdef TM_CAS_FIRST  // A/B: claim slot 0 of the home bucket without reading the bucket first
    Bucket b;
    if (d == 0) {
      const unsigned long long c0 = atomicCAS(bk, kEmptySlot, mine);
      if (c0 == kEmptySlot) return;
      b = load_bucket_cg(bk);
      b.s0 = c0;
    } else {
      b = load_bucket_cg(bk);
    }
#else
    const Bucket b = load_bucket_cg(bk);
#endif
#pragma unroll
    for (int k = 0; k < 4; k++) {
      unsigned long long cur = b.at(k);
      if (cur == kEmptySlot) {
        cur = atomicCAS(bk + k, kEmptySlot, mine);
        if (cur == kEmptySlot) return;
      }
      if (((cur & ~kClaimBit) >> tb.hb) == tag) {
        report(st, K_RECIPROCITY, h / 3);
        return;
      }
    }
  }
  // displacement overflow (> 31 buckets; the half-size table without Qhull
  // locality, or adversarial keys): the host reruns the call with a table twice
  // the size
  if (tb.ovf) atomicOr(tb.ovf, 1u);
  else report(st, K_STRUCT, h / 3);
}

// Partner of descending half-edge o -> g (key (g, o)) as (h << 1) | L; -1 when border.
__device__ __forceinline__ int32_t table_lookup(const TwinTable& tb, DevStatus* st, int check, int32_t lo, int32_t hi,
                                                int64_t elem) {
  Probe p = probe_of(tb, lo, hi);
  const uint64_t hmask = (1ull << tb.hb) - 1;
  for (int d = 0; d <= kMaxDisp; d++) {
    unsigned long long* bk = tb.slots + 4 * ((p.home + d) & tb.nb_mask);
    const uint64_t tag = p.tag | (uint64_t)d;
    const Bucket b = load_bucket_nc(bk);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const unsigned long long cur = b.at(k);
      if (cur == kEmptySlot) return -1;
      if (((cur & ~kClaimBit) >> tb.hb) == tag) {
        if (check) {  // a second descending partner: edge shared by > 2 triangles
          unsigned long long old = atomicOr(bk + k, kClaimBit);
          if (old & kClaimBit) report(st, K_EDGE_COUNT, elem);
        }
        return (int32_t)(cur & hmask);
      }
    }
  }
  return -1;
}

// label the edge pair h (own triangle tt, own longest-edge flag `own`) + hc
// (partner, its longest-edge flag `other`): labeling.py:65-115
__device__ __forceinline__ void label_pair(int32_t* __restrict__ hw, uint8_t* __restrict__ seed, int32_t h, bool own,
                                           int32_t hc, bool other) {
  const int32_t tt = h / 3, tc = hc / 3;
  const int32_t fr = (!own && !other) ? 1 : 0;
  hw[h] = (hc << 1) | fr;
  hw[hc] = (h << 1) | fr;
  if (own) seed[tt] = (other && tt < tc) ? 1 : 0;
  if (other) seed[tc] = (own && tc < tt) ? 1 : 0;
}

// Single-pass rendezvous (unchecked labels): the two half-edges of an edge both
// probe under the undirected key (lo, hi).  The first to arrive claims an empty
// slot with its (h << 1) | L; the second finds it, marks the slot paired
// (claim bit, a fire-and-forget RED) and labels both sides at once.  Two
// arrivals racing for the same empty slot: the CAS loser reads the winner's
// entry, i.e. its partner.  Entries left unpaired are border half-edges
// (k_border_scan).  A third half-edge on one key finds a paired slot: edge_count.
__device__ __forceinline__ void table_meet(const TwinTable& tb, DevStatus* st, int32_t* __restrict__ hw,
                                           uint8_t* __restrict__ seed, int32_t hl, int32_t lo, int32_t hi) {
  Probe p = probe_of(tb, lo, hi);
  const uint64_t hmask = (1ull << tb.hb) - 1;
  for (int d = 0; d <= kMaxDisp; d++) {
    unsigned long long* bk = tb.slots + 4 * ((p.home + d) & tb.nb_mask);
    const uint64_t tag = p.tag | (uint64_t)d;
    const unsigned long long mine = (tag << tb.hb) | (uint32_t)hl;
    const Bucket b = load_bucket_cg(bk);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      unsigned long long cur = b.at(k);
      if (cur == kEmptySlot) {
        cur = atomicCAS(bk + k, kEmptySlot, mine);
        if (cur == kEmptySlot) return;
      }
      if (((cur & ~kClaimBit) >> tb.hb) == tag) {
        if (cur & kClaimBit) {
          report(st, K_EDGE_COUNT, (hl >> 1) / 3);
          return;
        }
        atomicOr(bk + k, kClaimBit);
        const int32_t pl = (int32_t)(cur & hmask);
        label_pair(hw, seed, hl >> 1, (hl & 1) != 0, pl >> 1, (pl & 1) != 0);
        return;
      }
    }
  }
  if (tb.ovf) atomicOr(tb.ovf, 1u);
  else report(st, K_STRUCT, (hl >> 1) / 3);
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

// ---- single-precision prefilter of LabelMax.  The three squared lengths
// are first computed from an fp32 copy of the coordinates (8 bytes per vertex
// instead of 16: the copy of a 10M-point mesh stays mostly in L2), each with a
// bound on its distance to the exact squared length; when the largest one
// exceeds every other by more than their bounds, the fp64 argmax (any
// rounding of the reference's dx*dx + dy*dy) has the same winner.  Otherwise
// (near-ties, exact ties, non-finite values) the fp64 coordinates are read and
// the reference formula decides.
//   x32 = x(1+e), |e| <= u = 2^-24; dx32 = (x32a - x32b)(1+e'):
//   |dx32 - dx| <= u (|xa| + |xb| + |dx|)(1 + u) =: d, |dx32^2 - dx^2| <= d (2|dx| + d),
//   and two more roundings (square, sum) of at most u each.
struct Sq32 {
  float L, E;
};
__device__ __forceinline__ Sq32 sqlen32(float2 p, float2 q) {
  const float u = 5.9604645e-08f;  // 2^-24
  const float dx = __fsub_rn(p.x, q.x), dy = __fsub_rn(p.y, q.y);
  const float L = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
  const float ax = fabsf(p.x) + fabsf(q.x) + fabsf(dx), ay = fabsf(p.y) + fabsf(q.y) + fabsf(dy);
  const float dxe = 1.01f * u * ax, dye = 1.01f * u * ay;  // |dx32 - dx|, |dy32 - dy| bounds (with slack)
  // 2 (safety) x [first-order + second-order + the roundings of the square and the sum]
  const float E = 2.0f * (dxe * (2.0f * fabsf(dx) + dxe) + dye * (2.0f * fabsf(dy) + dye) + 3.0f * u * L) + 1e-37f;
  return Sq32{L, E};
}
// winner of numpy's first-max argmax when the fp32 bounds separate it, else -1
__device__ __forceinline__ int argmax3_32(float2 a, float2 b, float2 c) {
  const Sq32 l0 = sqlen32(b, c), l1 = sqlen32(c, a), l2 = sqlen32(a, b);
  if (!(isfinite(l0.L + l0.E) && isfinite(l1.L + l1.E) && isfinite(l2.L + l2.E))) return -1;
  int m = 0;
  Sq32 best = l0;
  if (l1.L > best.L) { best = l1; m = 1; }
  if (l2.L > best.L) { best = l2; m = 2; }
  const float lo = best.L - best.E;
  if (m != 0 && !(lo > l0.L + l0.E)) return -1;
  if (m != 1 && !(lo > l1.L + l1.E)) return -1;
  if (m != 2 && !(lo > l2.L + l2.E)) return -1;
  return m;
}

__global__ void k_xy32(const double2* __restrict__ xy, int64_t n, float2* __restrict__ xy32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    xy32[i] = make_float2(__double2float_rn(p.x), __double2float_rn(p.y));
  }
}

constexpr int kLabelThreads = 256;
constexpr int kLabelWarps = kLabelThreads / 32;

// Per-warp compaction of up to 96 half-edge items (3 per lane) so the table
// probes run on dense lanes: lane l's items with flag bit j set get queue
// positions in (slot j, lane) order.  Returns the item count.
__device__ __forceinline__ int warp_compact3(unsigned flags, int lane, int32_t* q_h, int32_t* q_o, int32_t* q_g,
                                             const int32_t (&h)[3], const int32_t (&o)[3], const int32_t (&g)[3]) {
  const unsigned lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int j = 0; j < 3; j++) {
    unsigned m = __ballot_sync(0xffffffffu, (flags >> j) & 1u);
    if ((flags >> j) & 1u) {
      int pos = base + __popc(m & lt);
      q_h[pos] = h[j];
      q_o[pos] = o[j];
      q_g[pos] = g[j];
    }
    base += __popc(m);
  }
  __syncwarp();
  return base;
}

// Block-local twin matching (pass A).  Qhull emits the facets of one cone
// together, so most twins sit a few indices apart (1M uniform: median distance
// 4; 57% of the pairs inside one aligned 256-triangle block).  Each block
// matches its own half-edges in a shared-memory table first and labels those
// pairs on the spot; only the rest go through the global table.
constexpr int kLocalBits = 10;
constexpr int kLocalSlots = 1 << kLocalBits;  // >= 2 x the block's ascending half-edges (<= 2 per triangle)
constexpr int32_t kLocalMatched = (int32_t)0x80000000;

__device__ __forceinline__ uint32_t local_slot(int32_t lo, int32_t hi) {
  return ((uint32_t)lo * 0x9E3779B1u + (uint32_t)hi * 0x85EBCA77u) >> (32 - kLocalBits);
}


// Pass A (K1 + first half of K0), one thread per triangle: corners -> tri32,
// fp64 longest edge -> max_edge, orientation check, trivertex (atomicMin, a
// fire-and-forget RED), provisional labels (hw = border, seed = 1); the
// block-local pairs are matched and labelled (not in check mode, where every
// ascending half-edge goes to the global table so that the claim bits see all
// partners); then the warp's remaining ascending half-edges (origin < target)
// go into the twin table on dense lanes.
#ifndef TM_TRI_MINB
#define TM_TRI_MINB 4
#endif
#ifndef TM_PAIR_MINB
#define TM_PAIR_MINB 6
#endif
// A/B switches (measured and rejected): software-pipelined
// chunks -- the extra live registers cost a resident block per SM and the
// passes are bound by random-sector throughput, not by a chunk's chain.
#ifndef TM_TRI_PF
#define TM_TRI_PF 0
#endif
#ifndef TM_PAIR_PF
#define TM_PAIR_PF 0
#endif
template <typename TI, bool ONE>
__global__ void __launch_bounds__(kLabelThreads, TM_TRI_MINB) k_tri_pass(const double2* __restrict__ xy,
                                                            const float2* __restrict__ xy32, int64_t n,
                                                            const TI* __restrict__ tri, int64_t t_begin,
                                                            int64_t T,
                                                            int32_t* __restrict__ tri32, int8_t* __restrict__ max_edge,
                                                            TwinTable tb, int32_t* __restrict__ hw,
                                                            uint8_t* __restrict__ seed, int32_t* __restrict__ tv,
                                                            int check, DevStatus* st) {
  __shared__ int32_t sq[kLabelWarps][3][96];
  __shared__ int32_t lown[kLocalSlots];  // 0 = free, else the claiming (thread, slot j) + 1
  __shared__ uint32_t lklo[kLocalSlots], lkhi[kLocalSlots];
  __shared__ int32_t lval[kLocalSlots];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool local = !check;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t base = t_begin + blockIdx.x * (int64_t)blockDim.x;
#if TM_TRI_PF >= 1
  // Software pipeline over the grid-stride chunks: the next chunk's corners
  // (and, TM_TRI_PF >= 2, its three coordinate records) are requested while the
  // current chunk does its shared-memory matching and table inserts, so a
  // chunk's dependent chain is bucket load -> CAS instead of corners -> coordinates
  // -> bucket load -> CAS.
  int64_t na = 0, nb = 0, nc = 0;
  if (base + threadIdx.x < T) {
    const int64_t t0 = base + threadIdx.x;
    na = (int64_t)__ldg(tri + 3 * t0), nb = (int64_t)__ldg(tri + 3 * t0 + 1), nc = (int64_t)__ldg(tri + 3 * t0 + 2);
  }
#endif
#if TM_TRI_PF >= 2
  const bool pf_xy = xy32 == nullptr;
  double2 qa = make_double2(0.0, 0.0), qb = qa, qc = qa;
  if (pf_xy && base + threadIdx.x < T && (uint64_t)na < (uint64_t)n && (uint64_t)nb < (uint64_t)n &&
      (uint64_t)nc < (uint64_t)n) {
    qa = xy[na], qb = xy[nb], qc = xy[nc];
  }
#endif
  for (; base < T; base += stride) {
    const int64_t t = base + threadIdx.x;
    if (local) {
      for (int i = threadIdx.x; i < kLocalSlots; i += kLabelThreads) lown[i] = 0;
      __syncthreads();
    }
    unsigned flags = 0, desc = 0;
    int me0 = -1;
    int32_t hh[3], oo[3], gg[3];
#if TM_TRI_PF >= 2
    const double2 ca = qa, cb = qb, cc = qc;  // this chunk's coordinates (valid when its corners are in range)
#endif
    if (t < T) {
#if TM_TRI_PF >= 1
      const int64_t a = na, b = nb, c = nc;
      if (t + stride < T) {
        const int64_t tn = t + stride;
        na = (int64_t)__ldg(tri + 3 * tn), nb = (int64_t)__ldg(tri + 3 * tn + 1), nc = (int64_t)__ldg(tri + 3 * tn + 2);
      }
#else
      int64_t a = (int64_t)__ldg(tri + 3 * t), b = (int64_t)__ldg(tri + 3 * t + 1), c = (int64_t)__ldg(tri + 3 * t + 2);
#endif
      const bool bad = a < 0 || a >= n || b < 0 || b >= n || c < 0 || c >= n;
      if (!ONE || bad) {  // provisional border labels (ONE: every half-edge is labelled by whoever resolves it)
        hw[3 * t] = -1;
        hw[3 * t + 1] = -1;
        hw[3 * t + 2] = -1;
        seed[t] = 1;
      }
      if (bad) {
        report(st, K_INDEX_RANGE, t);
        max_edge[t] = 0;
        if (tri32 != nullptr) tri32[3 * t] = tri32[3 * t + 1] = tri32[3 * t + 2] = -1;
      } else {
        if (tri32 != nullptr) {
          tri32[3 * t] = (int32_t)a;
          tri32[3 * t + 1] = (int32_t)b;
          tri32[3 * t + 2] = (int32_t)c;
        }
        // labeling.py:55-59: edge 0 joins corners 1-2, edge 1 joins 2-0, edge 2 joins 0-1
        me0 = -1;
        if (xy32 != nullptr) me0 = argmax3_32(xy32[a], xy32[b], xy32[c]);
        if (me0 < 0) {
#ifdef TM_AB_NO_XY  // A/B timing builds only (wrong labels): what the coordinate gathers cost
          me0 = (int)(t % 3);
#elif TM_TRI_PF >= 2
          double2 pa = ca, pb = cb, pc = cc;
          if (!pf_xy) pa = xy[a], pb = xy[b], pc = xy[c];
          me0 = argmax3(sqlen(pb, pc), sqlen(pc, pa), sqlen(pa, pb));
#else
          const double2 pa = xy[a], pb = xy[b], pc = xy[c];
          me0 = argmax3(sqlen(pb, pc), sqlen(pc, pa), sqlen(pa, pb));
#endif
        }
        max_edge[t] = (int8_t)me0;
        if (check) {
#if TM_TRI_PF >= 2
          double2 pa = ca, pb = cb, pc = cc;
          if (!pf_xy) pa = xy[a], pb = xy[b], pc = xy[c];
#else
          const double2 pa = xy[a], pb = xy[b], pc = xy[c];
#endif
          // mesh_core.signed_areas (160-168), sign only, unfused
          double d = __dsub_rn(__dmul_rn(__dsub_rn(pb.x, pa.x), __dsub_rn(pc.y, pa.y)),
                               __dmul_rn(__dsub_rn(pb.y, pa.y), __dsub_rn(pc.x, pa.x)));
          if (d < 0.0) report(st, K_ORIENTATION, t);
          else if (d == 0.0) report(st, K_DEGENERATE, t);
        }
        if (tv != nullptr) {  // phase API only; the whole path derives fan starts from the polygons
          atomicMin(tv + a, (int32_t)t);
          atomicMin(tv + b, (int32_t)t);
          atomicMin(tv + c, (int32_t)t);
        }
        // half-edge j: origin corner (j+1)%3, target corner (j+2)%3; queued as (h << 1) | longest
        const int32_t cv[3] = {(int32_t)a, (int32_t)b, (int32_t)c};
#pragma unroll
        for (int j = 0; j < 3; j++) {
          hh[j] = (int32_t)(((3 * t + j) << 1) | (me0 == j ? 1 : 0));
          oo[j] = cv[(j + 1) % 3];
          gg[j] = cv[(j + 2) % 3];
          if (oo[j] < gg[j]) flags |= 1u << j;
          else if (oo[j] > gg[j]) desc |= 1u << j;
          else if (ONE) {  // a zero-length edge (o == g) has no partner: border
            hw[3 * t + j] = -1;
            if (me0 == j) seed[t] = 1;
          }
        }
      }
    }
    if (local) {
      int lslot[3] = {-1, -1, -1};
#pragma unroll
      for (int j = 0; j < 3; j++) {
        if (!((flags >> j) & 1u)) continue;
        uint32_t sl = local_slot(oo[j], gg[j]);
        const int me = (int)threadIdx.x * 4 + j + 1;
        for (;;) {
          if (atomicCAS(&lown[sl], 0, me) == 0) {
            lklo[sl] = (uint32_t)oo[j];
            lkhi[sl] = (uint32_t)gg[j];
            lval[sl] = hh[j];
            lslot[j] = (int)sl;
            break;
          }
          sl = (sl + 1) & (kLocalSlots - 1);
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 3; j++) {
        if (!((desc >> j) & 1u)) continue;
        uint32_t sl = local_slot(gg[j], oo[j]);
        for (;;) {
          if (lown[sl] == 0) break;
          if (lklo[sl] == (uint32_t)gg[j] && lkhi[sl] == (uint32_t)oo[j]) {
            const int32_t pl = atomicOr(&lval[sl], kLocalMatched);
            if (!(pl & kLocalMatched)) label_pair(hw, seed, (int32_t)(3 * t + j), me0 == j, pl >> 1, (pl & 1) != 0);
            else if (ONE) report(st, K_EDGE_COUNT, t);
            if (ONE) desc &= ~(1u << j);  // resolved here: not sent to the table
            break;
          }
          sl = (sl + 1) & (kLocalSlots - 1);
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 3; j++)
        if (lslot[j] >= 0 && (lval[lslot[j]] & kLocalMatched)) flags &= ~(1u << j);
    }
    if (ONE) {  // descending half-edges still unpaired meet their partner in the table too, under (g, o)
#pragma unroll
      for (int j = 0; j < 3; j++)
        if ((desc >> j) & 1u) {
          const int32_t x = oo[j];
          oo[j] = gg[j];
          gg[j] = x;
        }
      flags |= desc;
    }
#if TM_TRI_PF >= 2
    if (pf_xy && t + stride < T && (uint64_t)na < (uint64_t)n && (uint64_t)nb < (uint64_t)n &&
        (uint64_t)nc < (uint64_t)n) {
      qa = xy[na], qb = xy[nb], qc = xy[nc];  // next chunk's coordinates, in flight during the inserts
    }
#endif
    int m = warp_compact3(flags, lane, sq[wid][0], sq[wid][1], sq[wid][2], hh, oo, gg);
#ifndef TM_AB_NO_TABLE  // A/B timing builds only (wrong labels): what the table inserts cost
    for (int i = lane; i < m; i += 32) {
      if (ONE) table_meet(tb, st, hw, seed, sq[wid][0][i], sq[wid][1][i], sq[wid][2][i]);
      else table_insert(tb, st, sq[wid][0][i], sq[wid][1][i], sq[wid][2][i]);
    }
#endif
    __syncwarp();
    if (local) __syncthreads();  // lkey/lval are reset at the top of the next chunk
  }
}

// Pass B (second half of K0 + K2), one thread per triangle (and per vertex for
// the trivertex sentinel).  The warp's descending half-edges h = o -> g
// (o > g) look their ascending partner up under key (g, o) on dense lanes and
// label the edge pair from both sides at once: frontier = neither side's
// longest edge (labeling.py:92-115), terminal = both (labeling.py:65-89, seed
// on the lower triangle).  k = twin % 3 replaces the reference's back-slot
// searches.  A half-edge without a partner stays border as pass A wrote it
// (an ascending one keeps its provisional seed flag).
__global__ void __launch_bounds__(kLabelThreads, TM_PAIR_MINB) k_pair_pass(const int32_t* __restrict__ tri32, int64_t t_begin,
                                                             int64_t T,
                                                             const int8_t* __restrict__ max_edge, TwinTable tb,
                                                             int32_t* __restrict__ hw, uint8_t* __restrict__ seed,
                                                             int32_t* __restrict__ tv, int64_t n, int check,
                                                             DevStatus* st) {
  __shared__ int32_t sq[kLabelWarps][3][96];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#if TM_PAIR_PF
  // the next chunk's corners and packed words are requested before this chunk's
  // lookups (descending entries -- the only ones tested -- are written by their
  // own thread alone, so the early read sees their final pass-A value)
  int32_t nv0 = 0, nv1 = 0, nv2 = 0, nw0 = 0, nw1 = 0, nw2 = 0;
  {
    const int64_t t0 = t_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t0 < T) {
      nv0 = __ldg(tri32 + 3 * t0), nv1 = __ldg(tri32 + 3 * t0 + 1), nv2 = __ldg(tri32 + 3 * t0 + 2);
      nw0 = hw[3 * t0], nw1 = hw[3 * t0 + 1], nw2 = hw[3 * t0 + 2];
    }
  }
#endif
  for (int64_t t = t_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t - lane < T; t += stride) {
    unsigned flags = 0;
    int32_t hh[3], oo[3], gg[3];
    if (t < T) {
#if TM_PAIR_PF
      const int32_t cv[3] = {nv0, nv1, nv2};
      const int32_t w[3] = {nw0, nw1, nw2};
      if (t + stride < T) {
        const int64_t tn = t + stride;
        nv0 = __ldg(tri32 + 3 * tn), nv1 = __ldg(tri32 + 3 * tn + 1), nv2 = __ldg(tri32 + 3 * tn + 2);
        nw0 = hw[3 * tn], nw1 = hw[3 * tn + 1], nw2 = hw[3 * tn + 2];
      }
#else
      const int32_t cv[3] = {__ldg(tri32 + 3 * t), __ldg(tri32 + 3 * t + 1), __ldg(tri32 + 3 * t + 2)};
#endif
      if ((uint32_t)cv[0] < (uint32_t)n && (uint32_t)cv[1] < (uint32_t)n && (uint32_t)cv[2] < (uint32_t)n) {
        // a descending half-edge pass A already paired inside its block is no longer border
#if !TM_PAIR_PF
        const int32_t w[3] = {hw[3 * t], hw[3 * t + 1], hw[3 * t + 2]};
#endif
#pragma unroll
        for (int j = 0; j < 3; j++) {
          hh[j] = (int32_t)(3 * t + j);
          oo[j] = cv[(j + 1) % 3];
          gg[j] = cv[(j + 2) % 3];
          if (oo[j] > gg[j] && w[j] == -1) flags |= 1u << j;
        }
      }
    }
    int m = warp_compact3(flags, lane, sq[wid][0], sq[wid][1], sq[wid][2], hh, oo, gg);
    for (int i = lane; i < m; i += 32) {
      const int32_t h = sq[wid][0][i];
      const int32_t pl = table_lookup(tb, st, check, sq[wid][2][i], sq[wid][1][i], h / 3);
      if (pl < 0) continue;  // border
      const int32_t tt = h / 3, j = h - 3 * tt;
      label_pair(hw, seed, h, __ldg(max_edge + tt) == j, pl >> 1, (pl & 1) != 0);
    }
    __syncwarp();
  }
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (tv != nullptr && tv[v] == 0x7F7F7F7F) tv[v] = -1;
}

// Pass B of the single-pass labels: the table entries left unpaired are the
// border half-edges (twin -1, frontier; a border longest edge seeds its
// triangle, labeling.py:76-80), plus the trivertex sentinel.  One sequential
// read of the table.
__global__ void __launch_bounds__(256) k_border_scan(TwinTable tb, int32_t* __restrict__ hw, uint8_t* __restrict__ seed,
                                                     int32_t* __restrict__ tv, int64_t n) {
  const uint64_t hmask = (1ull << tb.hb) - 1;
  const int64_t nb = (int64_t)tb.nb_mask + 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const ulonglong2* sl = reinterpret_cast<const ulonglong2*>(tb.slots);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * nb; i += stride) {
    const ulonglong2 q = __ldcs(sl + i);
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const unsigned long long cur = k ? q.y : q.x;
      if (!(cur & kClaimBit)) {  // occupied (empty = all ones) and never paired
        const int32_t pl = (int32_t)(cur & hmask), h = pl >> 1;
        hw[h] = -1;
        if (pl & 1) seed[h / 3] = 1;
      }
    }
  }
  if (tv != nullptr)
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
      if (tv[v] == 0x7F7F7F7F) tv[v] = -1;
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

// Single-pass labels (`one`, unchecked only): both half-edges of a far edge
// meet in pass A (table_meet) and pass B is a scan of the table
// (k_border_scan).  Used where pass A overlaps the triangle upload (the
// host-array entry): the table work then hides under PCIe and only the scan
// follows the last chunk.  Device-resident runs keep insert (pass A) + lookup
// (pass B): measured 2.04 vs 2.11 ms of label time at 10M (the lookups' read-only
// probes are cheaper than the second arrivals' coherent ones).  Checked labels
// always use two passes: the claim bits must see every partner.
static inline bool single_pass(int one, int check) {
#ifdef TM_TWO_PASS  // A/B: insert + lookup passes everywhere
  return false;
#else
  return one && !check;
#endif
}

// Grid of a grid-stride label kernel: exactly the resident blocks (occupancy x
// SMs) when the work spans more, so no partial last wave -- at 10M the former
// 16-per-SM grid ran k_tri_pass in 3.2 waves of 5 resident blocks (the last
// 0.2 wave at one block per SM) and k_pair_pass in 2.67 of 6.
template <typename K>
static int resident_grid(K* fn, int64_t n, int block) {
#ifdef TM_GRID16  // A/B: the former grid
  return grid_for(n, block);
#endif
  static thread_local std::pair<const void*, int> cache[8];
  int per_sm = 0;
  for (auto& c : cache)
    if (c.first == (const void*)fn) per_sm = c.second;
  if (per_sm == 0) {
#ifdef TM_CARVEOUT  // A/B: maximum shared-memory carveout (measured: halves L1 and slows both passes ~50%)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#endif
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, 0) != cudaSuccess || per_sm < 1) per_sm = 4;
    for (auto& c : cache)
      if (c.first == nullptr) {
        c = {(const void*)fn, per_sm};
        break;
      }
  }
  const int64_t need = (n + block - 1) / block, cap = (int64_t)kNumSMs * per_sm;
  return (int)(need < 1 ? 1 : need < cap ? need : cap);
}

static int bit_length(uint64_t v) {
  int b = 0;
  while (v) { b++; v >>= 1; }
  return b;
}

// Geometry of the twin table for a mesh of n vertices / T triangles.
// shrink = s scales the bucket count by 2^-s.  s = 1 (whole path): half the
// buckets -- block-local matching pairs ~57% of the edges before the table
// (Qhull order), so the inserted keys load the half table to ~0.3; a mesh
// without that locality overflows it, which sets *ovf and the host reruns the
// call with s - 1 (full size, then 2x, 4x, 8x).
static TwinTable table_geometry(int64_t n, int64_t T, void* mem, int shrink = 0, unsigned int* ovf = nullptr,
                                int64_t keyT = -1) {
  // keyT: triangles whose keys go in (a rank's range), T: half-edge ids < 3T
  TwinTable tb{};
  tb.b = bit_length((uint64_t)(n > 1 ? n - 1 : 1));
  tb.K = 2 * tb.b;
  // payload (h << 1) | L; 2^(hb-1) > 3T, so the all-ones field is never a half-edge
  tb.hb = bit_length((uint64_t)(3 * (T > 0 ? T : 1))) + 1;
  // ascending half-edges <= 3T/2 + border; 4-slot buckets at load in [0.35, 0.7)
  // (measured: a fuller table costs more in probe/CAS conflicts than it saves in L2)
  const int64_t KT = keyT >= 0 ? keyT : T;
  uint64_t keys = (uint64_t)(3 * (KT > 0 ? KT : 1)) / 2 + 64;
  int q = bit_length((keys * 10 / 28) | 1);
  if (shrink > 0) q = q - shrink > 8 ? q - shrink : (q > 8 ? 8 : q);
  if (shrink < 0) q -= shrink;
  if (q > tb.K) q = tb.K;
  while (tb.K - q + kDispBits + tb.hb > 63 && q < tb.K) q++;  // the slot must hold remainder|d|h|L in 63 bits
  tb.R = tb.K - q;
  tb.nb_mask = (1ull << q) - 1;
  tb.slots = static_cast<unsigned long long*>(mem);
  tb.ovf = ovf;
  return tb;
}

size_t hash_bytes(int64_t n, int64_t T, int shrink) {
  TwinTable tb = table_geometry(n, T, nullptr, shrink < 0 ? shrink : 0);
  return (size_t)(tb.nb_mask + 1) * 4 * sizeof(unsigned long long);
}

void launch_label_a_prepare(int64_t n, int64_t T, int32_t* tv, void* table, cudaStream_t s, int shrink) {
  const TwinTable tb = table_geometry(n, T, nullptr, shrink);
  cudaMemsetAsync(table, 0xFF, (size_t)(tb.nb_mask + 1) * 4 * sizeof(unsigned long long), s);
  if (n > 0 && tv != nullptr) {
    // sentinel 0x7F7F7F7F (> any triangle index), mapped to -1 by pass B
    cudaMemsetAsync(tv, 0x7F, (size_t)n * sizeof(int32_t), s);
  }
}

void launch_xy32(const double* xy, int64_t n, float* xy32, cudaStream_t s) {
  if (n > 0) k_xy32<<<grid_for(n, 256), 256, 0, s>>>((const double2*)xy, n, (float2*)xy32), note_launch(1);
}

void launch_label_a_range(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int64_t t_begin,
                          int64_t t_end, int check, int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed,
                          int32_t* tv, void* table, DevStatus* st, cudaStream_t s, int shrink, unsigned int* ovf,
                          const float* xy32, int one) {
  TwinTable tb = table_geometry(n, T, table, shrink, ovf);
  if (t_end > t_begin) {
    const int B = kLabelThreads;
    const int64_t m = t_end - t_begin;
    const int g = single_pass(one, check)
                      ? (tri_is64 ? resident_grid(k_tri_pass<int64_t, true>, m, B)
                                  : resident_grid(k_tri_pass<int32_t, true>, m, B))
                      : (tri_is64 ? resident_grid(k_tri_pass<int64_t, false>, m, B)
                                  : resident_grid(k_tri_pass<int32_t, false>, m, B));
    const double2* p = (const double2*)xy;
    const float2* p32 = (const float2*)xy32;
    int32_t* t32 = tri_is64 || tri32 != tri ? tri32 : nullptr;
    if (single_pass(one, check)) {
      if (tri_is64)
        k_tri_pass<int64_t, true><<<g, B, 0, s>>>(p, p32, n, (const int64_t*)tri, t_begin, t_end, t32, max_edge, tb,
                                                  hw, seed, tv, 0, st);
      else
        k_tri_pass<int32_t, true><<<g, B, 0, s>>>(p, p32, n, (const int32_t*)tri, t_begin, t_end, t32, max_edge, tb,
                                                  hw, seed, tv, 0, st);
    } else if (tri_is64) {
      k_tri_pass<int64_t, false><<<g, B, 0, s>>>(p, p32, n, (const int64_t*)tri, t_begin, t_end, t32, max_edge, tb, hw,
                                                 seed, tv, check, st);
    } else {
      k_tri_pass<int32_t, false><<<g, B, 0, s>>>(p, p32, n, (const int32_t*)tri, t_begin, t_end, t32, max_edge, tb, hw,
                                                 seed, tv, check, st);
    }
    note_launch(1);
  }
}

void launch_label_a(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int check,
                    int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed, int32_t* tv, void* table,
                    DevStatus* st, cudaStream_t s, int shrink, unsigned int* ovf, float* xy32, int one) {
  launch_label_a_prepare(n, T, tv, table, s, shrink);
  if (xy32 && !check) launch_xy32(xy, n, xy32, s);
  launch_label_a_range(xy, n, tri, tri_is64, T, 0, T, check, tri32, hw, max_edge, seed, tv, table, st, s, shrink, ovf,
                       check ? nullptr : xy32, one);
}

void launch_label_b(const int32_t* tri32, int64_t n, int64_t T, int32_t* hw, const int8_t* max_edge, uint8_t* seed,
                    int32_t* tv, void* table, int check, DevStatus* st, cudaStream_t s, int shrink, int one) {
  TwinTable tb = table_geometry(n, T, table, shrink);
  if (single_pass(one, check)) {
    const int64_t m = (int64_t)(tb.nb_mask + 1) * 2;
    k_border_scan<<<grid_for(m > n ? m : n, 256), 256, 0, s>>>(tb, hw, seed, tv, n);
    note_launch(1);
    return;
  }
  int64_t m = (T > n || tv == nullptr) ? T : n;
  if (m > 0) {
    k_pair_pass<<<resident_grid(k_pair_pass, m, kLabelThreads), kLabelThreads, 0, s>>>(tri32, 0, T, max_edge, tb, hw, seed, tv, n,
                                                                     check, st);
    note_launch(1);
  }
}

// ------------------------------------------------------------ seed-partitioned labels
// A rank labels its triangle range [b, e) with a range-local twin table
// (passes A and B restricted to the range); half-edges still unpaired are
// either true border or have their partner in another rank's range: they are
// listed as boundary entries (key (lo << 32) | hi, value (h << 1) | longest)
// for the exchange, after which k_boundary_insert / k_boundary_match label the cross pairs.
size_t hash_bytes_range(int64_t n, int64_t T, int64_t keyT) {
  TwinTable tb = table_geometry(n, T, nullptr, 0, nullptr, keyT);
  return (size_t)(tb.nb_mask + 1) * 4 * sizeof(unsigned long long);
}

void launch_label_range(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int64_t b, int64_t e,
                        int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed, void* table, DevStatus* st,
                        unsigned int* ovf, cudaStream_t s) {
  const TwinTable tb = table_geometry(n, T, table, 0, ovf, e - b);
  cudaMemsetAsync(table, 0xFF, (size_t)(tb.nb_mask + 1) * 4 * sizeof(unsigned long long), s);
  if (e <= b) return;
  const int g = tri_is64 ? resident_grid(k_tri_pass<int64_t, false>, e - b, kLabelThreads)
                         : resident_grid(k_tri_pass<int32_t, false>, e - b, kLabelThreads);
  if (tri_is64)
    k_tri_pass<int64_t, false><<<g, kLabelThreads, 0, s>>>((const double2*)xy, nullptr, n, (const int64_t*)tri, b, e, tri32,
                                                    max_edge, tb, hw, seed, nullptr, 0, st);
  else
    k_tri_pass<int32_t, false><<<g, kLabelThreads, 0, s>>>((const double2*)xy, nullptr, n, (const int32_t*)tri, b, e,
                                                    tri32 == tri ? nullptr : tri32, max_edge, tb, hw, seed, nullptr, 0,
                                                    st);
  k_pair_pass<<<resident_grid(k_pair_pass, e - b, kLabelThreads), kLabelThreads, 0, s>>>(tri32, b, e, max_edge, tb, hw, seed, nullptr, n, 0, st);
  note_launch(2);
}

template <typename TI>
__global__ void k_tri32(const TI* __restrict__ tri, int64_t n3, int32_t* __restrict__ tri32) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n3; k += (int64_t)gridDim.x * blockDim.x)
    tri32[k] = (int32_t)tri[k];
}

void launch_tri32(const void* tri, int tri_is64, int64_t T, int32_t* tri32, cudaStream_t s) {
  if (T <= 0) return;
  if (tri_is64) k_tri32<int64_t><<<grid_for(3 * T, 256), 256, 0, s>>>((const int64_t*)tri, 3 * T, tri32);
  else k_tri32<int32_t><<<grid_for(3 * T, 256), 256, 0, s>>>((const int32_t*)tri, 3 * T, tri32);
  note_launch(1);
}

__global__ void k_boundary_extract(const int32_t* __restrict__ tri32, const int8_t* __restrict__ max_edge,
                                   const int32_t* __restrict__ hw, int64_t b, int64_t e,
                                   unsigned long long* __restrict__ keys, int32_t* __restrict__ vals,
                                   unsigned long long* count, int64_t cap) {
  const int lane = threadIdx.x & 31;
  for (int64_t h0 = 3 * b + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane); h0 < 3 * e;
       h0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = h0 + lane;
    bool want = false;
    unsigned long long key = 0;
    int32_t val = 0;
    if (h < 3 * e && hw[h] == -1) {
      const int64_t t = h / 3;
      const int j = (int)(h - 3 * t);
      const uint32_t o = (uint32_t)tri32[3 * t + (j + 1) % 3], g = (uint32_t)tri32[3 * t + (j + 2) % 3];
      key = ((unsigned long long)min(o, g) << 32) | max(o, g);
      val = (int32_t)((h << 1) | (max_edge[t] == j ? 1 : 0));
      want = true;
    }
    const unsigned m = __ballot_sync(0xffffffffu, want);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (want) {
      const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
      if ((int64_t)k < cap) {
        keys[k] = key;
        vals[k] = val;
      }
    }
  }
}

void launch_boundary_extract(const int32_t* tri32, const int8_t* max_edge, const int32_t* hw, int64_t b, int64_t e,
                             unsigned long long* keys, int32_t* vals, unsigned long long* count, int64_t cap,
                             cudaStream_t s) {
  if (e > b)
    k_boundary_extract<<<grid_for(3 * (e - b), 256), 256, 0, s>>>(tri32, max_edge, hw, b, e, keys, vals, count, cap),
        note_launch(1);
}

__device__ __forceinline__ uint64_t bhash(unsigned long long key, uint64_t mask) {
  return ((key * 0x9E3779B97F4A7C15ull) >> 17) & mask;
}

// own entries [own0, own1) go into a small table (this rank's share); every
// other rank's entry probes it, and a hit labels this side of the pair
// (labeling.py:65-115).  Reads of a small table instead of every rank
// inserting every entry.
__global__ void k_boundary_insert(const unsigned long long* __restrict__ keys, int64_t own0, int64_t own1,
                                  int32_t* __restrict__ tab, uint64_t mask) {
  for (int64_t k = own0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < own1;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (keys[k] == ~0ull) continue;  // padding of a fixed-size all-gather
    uint64_t h = bhash(keys[k], mask);
    while (atomicCAS(tab + h, -1, (int32_t)k) != -1) h = (h + 1) & mask;
  }
}

__global__ void k_boundary_match(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ vals,
                                 int64_t n_all, int64_t own0, int64_t own1, const int32_t* __restrict__ tab,
                                 uint64_t mask, int32_t* __restrict__ hw, uint8_t* __restrict__ seed) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_all; k += (int64_t)gridDim.x * blockDim.x) {
    if (k >= own0 && k < own1) continue;
    const unsigned long long key = keys[k];
    if (key == ~0ull) continue;
    uint64_t h = bhash(key, mask);
    int32_t mine = -1;
    for (;;) {
      const int32_t x = tab[h];
      if (x < 0) break;
      if (keys[x] == key) { mine = x; break; }
      h = (h + 1) & mask;
    }
    if (mine < 0) continue;
    const int32_t me = vals[mine], pv = vals[k];
    const int32_t he = me >> 1, hp = pv >> 1;
    const bool own = me & 1, other = pv & 1;
    hw[he] = (hp << 1) | ((!own && !other) ? 1 : 0);
    if (own) {
      const int32_t tt = he / 3, tc = hp / 3;
      seed[tt] = (other && tt < tc) ? 1 : 0;
    }
  }
}

void launch_boundary_resolve(const unsigned long long* keys, const int32_t* vals, int64_t n_all, int64_t own0,
                             int64_t own1, int32_t* tab, int64_t tab_slots, int32_t* hw, uint8_t* seed,
                             cudaStream_t s) {
  cudaMemsetAsync(tab, 0xFF, (size_t)tab_slots * sizeof(int32_t), s);
  if (own1 > own0)
    k_boundary_insert<<<grid_for(own1 - own0, 256), 256, 0, s>>>(keys, own0, own1, tab, (uint64_t)(tab_slots - 1));
  if (n_all > own1 - own0)
    k_boundary_match<<<grid_for(n_all, 256), 256, 0, s>>>(keys, vals, n_all, own0, own1, tab,
                                                          (uint64_t)(tab_slots - 1), hw, seed);
  note_launch(2);
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
