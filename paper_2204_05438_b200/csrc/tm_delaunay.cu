// tm_delaunay.cu -- Delaunay triangulation of a point set on the GPU (input
// generation; the reference calls Qhull through
// scipy.spatial.Delaunay, io_formats.py:351-388).
//
// Local stars with certificates.  The Delaunay star of a point p -- its
// neighbours in CCW order -- is found by gift wrapping over the points of the
// grid cells around p: from the nearest neighbour q0 (always a Delaunay
// neighbour), the next neighbour after q is the point r left of p->q whose
// circle through (p, q, r) contains no other candidate.  A triangle is
// CERTIFIED when its circumdisk, clipped to the points' box, lies inside the
// scanned cells: no point outside them can be in it, so it is a triangle of
// the global triangulation.  A point whose star does not close certified
// with a 5x5 neighbourhood retries with 9x9 and 17x17; points still open (the
// hull region, whose triangles have huge circles along the sides) are
// returned to the host, which triangulates the boundary band (one Qhull call
// on a few percent of the points) for the triangles they own.
//
// Every triangle is written once, by its smallest-index vertex (the owner);
// the output is grouped by the owners' grid cells (spatially coherent).
//
// Predicates are exact: a floating-point filter (Shewchuk's static error
// bounds) and, when it cannot decide, integer arithmetic on the coordinates
// scaled by 2^53 (exact for points on the 2^-53 grid of [0, 1) -- numpy's
// uniform draws; the host checks this before calling).
#include <cstdint>

#include "tm_common.cuh"
#include "tm_internal.h"

namespace tmb {

namespace {

// ------------------------------------------------------------ exact integer arithmetic
struct I128 {
  unsigned long long lo, hi;  // two's complement
};
__device__ __forceinline__ I128 mul64s(long long a, long long b) {  // |a|, |b| < 2^63
  I128 r;
  r.lo = (unsigned long long)a * (unsigned long long)b;
  r.hi = (unsigned long long)__mul64hi(a, b);
  return r;
}
__device__ __forceinline__ I128 sub128(I128 a, I128 b) {
  I128 r;
  r.lo = a.lo - b.lo;
  r.hi = a.hi - b.hi - (a.lo < b.lo ? 1ull : 0ull);
  return r;
}
__device__ __forceinline__ int sign128(I128 a) {
  if ((long long)a.hi < 0) return -1;
  return (a.hi | a.lo) ? 1 : 0;
}

struct I256 {
  unsigned long long w[4];  // little-endian limbs, two's complement
};
__device__ __forceinline__ I256 neg256(I256 a) {
  I256 r;
  unsigned long long carry = 1;
  for (int k = 0; k < 4; k++) {
    const unsigned long long x = ~a.w[k] + carry;
    carry = (carry && x == 0) ? 1ull : 0ull;
    r.w[k] = x;
  }
  return r;
}
__device__ __forceinline__ I256 add256(I256 a, I256 b) {
  I256 r;
  unsigned long long c = 0;
  for (int k = 0; k < 4; k++) {
    const unsigned long long s = a.w[k] + b.w[k];
    const unsigned long long c1 = s < a.w[k] ? 1ull : 0ull;
    r.w[k] = s + c;
    const unsigned long long c2 = r.w[k] < s ? 1ull : 0ull;
    c = c1 | c2;
  }
  return r;
}
// signed 128 x unsigned 128 (< 2^127 each in magnitude) -> signed 256
__device__ I256 mul_s128_u128(I128 a, unsigned long long blo, unsigned long long bhi) {
  const bool neg = (long long)a.hi < 0;
  unsigned long long alo = a.lo, ahi = a.hi;
  if (neg) {  // |a|
    alo = ~alo + 1;
    ahi = ~ahi + (alo == 0 ? 1ull : 0ull);
  }
  // schoolbook 2x2 limbs
  unsigned long long p[4] = {0, 0, 0, 0};
  const unsigned long long A[2] = {alo, ahi}, B[2] = {blo, bhi};
  for (int i = 0; i < 2; i++) {
    unsigned long long carry = 0;
    for (int j = 0; j < 2; j++) {
      const unsigned long long lo = A[i] * B[j], hi = __umul64hi(A[i], B[j]);
      unsigned long long s = p[i + j] + lo;
      unsigned long long c = s < lo ? 1ull : 0ull;
      s += carry;
      c += s < carry ? 1ull : 0ull;
      p[i + j] = s;
      carry = hi + c;
    }
    p[i + 2] += carry;
  }
  I256 r{{p[0], p[1], p[2], p[3]}};
  return neg ? neg256(r) : r;
}
__device__ __forceinline__ int sign256(I256 a) {
  if ((long long)a.w[3] < 0) return -1;
  return (a.w[0] | a.w[1] | a.w[2] | a.w[3]) ? 1 : 0;
}

constexpr double kScale = 9007199254740992.0;  // 2^53
__device__ __forceinline__ long long ix(double x) { return (long long)(x * kScale); }

// ------------------------------------------------------------ predicates
constexpr double kEps = 1.1102230246251565e-16;             // 2^-53
constexpr double kCcwErr = (3.0 + 16.0 * kEps) * kEps;      // Shewchuk ccwerrboundA
constexpr double kIccErr = (10.0 + 96.0 * kEps) * kEps;     // Shewchuk iccerrboundA

// > 0: c left of a->b (CCW)
__device__ int orient(double ax, double ay, double bx, double by, double cx, double cy) {
  const double l = (bx - ax) * (cy - ay), r = (by - ay) * (cx - ax);
  const double det = l - r;
  const double bound = kCcwErr * (fabs(l) + fabs(r));
  if (det > bound) return 1;
  if (-det > bound) return -1;
  const long long Ax = ix(ax), Ay = ix(ay);
  const I128 L = mul64s(ix(bx) - Ax, ix(cy) - Ay), R = mul64s(ix(by) - Ay, ix(cx) - Ax);
  return sign128(sub128(L, R));
}

// > 0: d strictly inside the circle through a, b, c (a, b, c CCW)
__device__ int incircle(double ax, double ay, double bx, double by, double cx, double cy, double dx, double dy) {
  const double adx = ax - dx, ady = ay - dy, bdx = bx - dx, bdy = by - dy, cdx = cx - dx, cdy = cy - dy;
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy, alift = adx * adx + ady * ady;
  const double cdxady = cdx * ady, adxcdy = adx * cdy, blift = bdx * bdx + bdy * bdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady, clift = cdx * cdx + cdy * cdy;
  const double det = alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
  const double perm = (fabs(bdxcdy) + fabs(cdxbdy)) * alift + (fabs(cdxady) + fabs(adxcdy)) * blift +
                      (fabs(adxbdy) + fabs(bdxady)) * clift;
  const double bound = kIccErr * perm;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  // exact: coordinates relative to d (54-bit), lifts (109-bit), crosses (109-bit)
  const long long Dx = ix(dx), Dy = ix(dy);
  const long long Ax = ix(ax) - Dx, Ay = ix(ay) - Dy, Bx = ix(bx) - Dx, By = ix(by) - Dy, Cx = ix(cx) - Dx,
                  Cy = ix(cy) - Dy;
  auto lift = [](long long x, long long y, unsigned long long* lo, unsigned long long* hi) {
    const unsigned long long ux = (unsigned long long)(x < 0 ? -x : x), uy = (unsigned long long)(y < 0 ? -y : y);
    unsigned long long l1 = ux * ux, h1 = __umul64hi(ux, ux), l2 = uy * uy, h2 = __umul64hi(uy, uy);
    *lo = l1 + l2;
    *hi = h1 + h2 + (*lo < l1 ? 1ull : 0ull);
  };
  unsigned long long al, ah, bl, bh, cl, ch;
  lift(Ax, Ay, &al, &ah);
  lift(Bx, By, &bl, &bh);
  lift(Cx, Cy, &cl, &ch);
  const I128 bc = sub128(mul64s(Bx, Cy), mul64s(Cx, By));
  const I128 ca = sub128(mul64s(Cx, Ay), mul64s(Ax, Cy));
  const I128 ab = sub128(mul64s(Ax, By), mul64s(Bx, Ay));
  I256 s = mul_s128_u128(bc, al, ah);
  s = add256(s, mul_s128_u128(ca, bl, bh));
  s = add256(s, mul_s128_u128(ab, cl, ch));
  return sign256(s);
}

struct Grid {
  double x0, y0, cw, ch;  // box origin, cell size
  double x1, y1;          // box end
  int G;                  // G x G cells
};

__device__ __forceinline__ int cell_coord(double v, double v0, double c, int G) {
  int k = (int)floor((v - v0) / c);
  return k < 0 ? 0 : (k >= G ? G - 1 : k);
}

}  // namespace

__global__ void k_cell_hist(const double2* __restrict__ xy, int64_t n, Grid g, int32_t* __restrict__ cell,
                            unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    const int c = cell_coord(p.y, g.y0, g.ch, g.G) * g.G + cell_coord(p.x, g.x0, g.cw, g.G);
    cell[i] = c;
    atomicAdd(hist + c, 1ull);
  }
}

__global__ void k_cell_scatter(const double2* __restrict__ xy, int64_t n, const int32_t* __restrict__ cell,
                               unsigned long long* __restrict__ cursor, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ids[atomicAdd(cursor + cell[i], 1ull)] = (int32_t)i;
}

// ids of one cell in ascending order (deterministic output), sorted coordinates
__global__ void k_cell_sort(const int64_t* __restrict__ start, int64_t ncell, int32_t* __restrict__ ids,
                            const double2* __restrict__ xy, double2* __restrict__ sxy) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = start[c], b = start[c + 1];
    for (int64_t i = a + 1; i < b; i++) {
      const int32_t x = ids[i];
      int64_t j = i - 1;
      while (j >= a && ids[j] > x) {
        ids[j + 1] = ids[j];
        j--;
      }
      ids[j + 1] = x;
    }
    for (int64_t i = a; i < b; i++) sxy[i] = xy[ids[i]];
  }
}

constexpr int kStarCap = 48;  // neighbours per star (Delaunay degrees of random points stay below ~20)

// Star of the point at sorted position k with a (2R+1)^2-cell neighbourhood.
// Returns the degree (> 0, closed certified star in nb[]), or 0 (not certified
// at this R / open: hull region), or -1 (degenerate: cocircular / collinear ties).
__device__ int star_of(int64_t k, int R, const int64_t* __restrict__ start, const int32_t* __restrict__ ids,
                       const double2* __restrict__ sxy, const Grid& g, int32_t* nb) {
  const double2 p = sxy[k];
  const int32_t pid = ids[k];
  const int cx = cell_coord(p.x, g.x0, g.cw, g.G), cy = cell_coord(p.y, g.y0, g.ch, g.G);
  const int ax = max(cx - R, 0), bx = min(cx + R, g.G - 1), ay = max(cy - R, 0), by = min(cy + R, g.G - 1);
  // the scanned region; sides on the box boundary are open (no points beyond)
  const double rx0 = ax == 0 ? -1e300 : g.x0 + ax * g.cw, rx1 = bx == g.G - 1 ? 1e300 : g.x0 + (bx + 1) * g.cw;
  const double ry0 = ay == 0 ? -1e300 : g.y0 + ay * g.ch, ry1 = by == g.G - 1 ? 1e300 : g.y0 + (by + 1) * g.ch;
  // nearest neighbour (ties: lowest id)
  double best = 1e300;
  int32_t q0 = -1;
  double q0x = 0, q0y = 0;
  for (int yy = ay; yy <= by; yy++)
    for (int64_t s = start[(int64_t)yy * g.G + ax]; s < start[(int64_t)yy * g.G + bx + 1]; s++) {
      if (s == k) continue;
      const double2 q = sxy[s];
      const double d = (q.x - p.x) * (q.x - p.x) + (q.y - p.y) * (q.y - p.y);
      const int32_t qid = ids[s];
      if (d < best || (d == best && qid < q0)) { best = d; q0 = qid; q0x = q.x; q0y = q.y; }
    }
  if (q0 < 0) return 0;
  {
    const double r = sqrt(best) * (1.0 + 1e-9) + 1e-300;
    if (p.x - r < rx0 || p.x + r > rx1 || p.y - r < ry0 || p.y + r > ry1) return 0;
  }
  int deg = 0;
  int32_t q = q0;
  double qx = q0x, qy = q0y;
  for (;;) {
    int32_t r = -1;
    double rx = 0, ry = 0;
    for (int yy = ay; yy <= by; yy++)
      for (int64_t s = start[(int64_t)yy * g.G + ax]; s < start[(int64_t)yy * g.G + bx + 1]; s++) {
        if (s == k) continue;
        const int32_t sid = ids[s];
        if (sid == q) continue;
        const double2 c = sxy[s];
        const int o = orient(p.x, p.y, qx, qy, c.x, c.y);
        if (o <= 0) {
          if (o == 0 && (c.x - p.x) * (qx - p.x) + (c.y - p.y) * (qy - p.y) > 0) return -1;  // on the ray p->q
          continue;
        }
        if (r < 0) { r = sid; rx = c.x; ry = c.y; continue; }
        const int ic = incircle(p.x, p.y, qx, qy, rx, ry, c.x, c.y);
        if (ic > 0) { r = sid; rx = c.x; ry = c.y; }
        else if (ic == 0) return -1;  // four cocircular points: no unique triangulation
      }
    if (r < 0) return 0;  // nothing left of p->q in the region: hull edge or region too small
    // certificate: circumdisk inside the region (bounding box, inflated)
    {
      const double bx_ = qx - p.x, by_ = qy - p.y, cx_ = rx - p.x, cy_ = ry - p.y;
      const double d = 2.0 * (bx_ * cy_ - by_ * cx_);
      const double b2 = bx_ * bx_ + by_ * by_, c2 = cx_ * cx_ + cy_ * cy_;
      const double ux = (cy_ * b2 - by_ * c2) / d, uy = (bx_ * c2 - cx_ * b2) / d;
      const double rad = sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1e-300;
      const double ox = p.x + ux, oy = p.y + uy;
      if (!(isfinite(rad) && ox - rad >= rx0 && ox + rad <= rx1 && oy - rad >= ry0 && oy + rad <= ry1)) return 0;
    }
    if (deg >= kStarCap) return 0;
    nb[deg++] = r;
    if (r == q0) return deg;  // the star closed
    q = r;
    qx = rx;
    qy = ry;
  }
}

// mode 0: count the triangles each point owns (cnt[k]); mode 1: write them at
// off[k] (exclusive scan of cnt).  Points that no R certifies are listed.
__global__ void __launch_bounds__(128) k_stars(const int64_t* __restrict__ start, const int32_t* __restrict__ ids,
                                               const double2* __restrict__ sxy, int64_t n, Grid g, int mode,
                                               int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
                                               int32_t* __restrict__ tri, int32_t* __restrict__ open_list,
                                               unsigned int* n_open, unsigned int* n_degenerate) {
  int32_t nb[kStarCap];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pid = ids[k];
    int deg = 0;
    for (int R = 2; R <= 8 && deg == 0; R *= 2) {
      deg = star_of(k, R, start, ids, sxy, g, nb);
      if (deg < 0) break;
    }
    if (deg <= 0) {
      if (mode == 0) {
        cnt[k] = 0;
        if (deg < 0) atomicAdd(n_degenerate, 1u);
        open_list[atomicAdd(n_open, 1u)] = pid;
      }
      continue;
    }
    // triangles (p, nb[i], nb[i+1]) are CCW; p owns those where it is the smallest index
    int64_t w = mode ? off[k] : 0;
    int64_t c = 0;
    for (int i = 0; i < deg; i++) {
      const int32_t a = nb[i], b = nb[i + 1 == deg ? 0 : i + 1];
      if (pid < a && pid < b) {
        if (mode) {
          tri[3 * w] = pid;
          tri[3 * w + 1] = a;
          tri[3 * w + 2] = b;
          w++;
        }
        c++;
      }
    }
    if (!mode) cnt[k] = c;
  }
}

void launch_delaunay_cells(const double* xy, int64_t n, double x0, double y0, double x1, double y1, int G,
                           int32_t* cell, unsigned long long* hist, cudaStream_t s) {
  Grid g{x0, y0, (x1 - x0) / G, (y1 - y0) / G, x1, y1, G};
  cudaMemsetAsync(hist, 0, (size_t)((int64_t)G * G + 2) * sizeof(unsigned long long), s);
  if (n > 0) k_cell_hist<<<kNumSMs * 8, 256, 0, s>>>((const double2*)xy, n, g, cell, hist), note_launch(1);
}

void launch_delaunay_scatter(const double* xy, int64_t n, int G, const int32_t* cell, const int64_t* start,
                             unsigned long long* cursor, int32_t* ids, double* sxy, cudaStream_t s) {
  const int64_t nc = (int64_t)G * G;
  cudaMemcpyAsync(cursor, start, (size_t)(nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  if (n > 0) k_cell_scatter<<<kNumSMs * 8, 256, 0, s>>>((const double2*)xy, n, cell, cursor, ids);
  k_cell_sort<<<kNumSMs * 8, 256, 0, s>>>(start, nc, ids, (const double2*)xy, (double2*)sxy);
  note_launch(2);
}

void launch_delaunay_stars(const int64_t* start, const int32_t* ids, const double* sxy, int64_t n, double x0,
                           double y0, double x1, double y1, int G, int mode, int64_t* cnt, const int64_t* off,
                           int32_t* tri, int32_t* open_list, unsigned int* n_open, unsigned int* n_degenerate,
                           cudaStream_t s) {
  Grid g{x0, y0, (x1 - x0) / G, (y1 - y0) / G, x1, y1, G};
  if (n > 0)
    k_stars<<<kNumSMs * 16, 128, 0, s>>>(start, ids, (const double2*)sxy, n, g, mode, cnt, off, tri, open_list, n_open,
                                         n_degenerate),
        note_launch(1);
}

}  // namespace tmb
