"""Exact Delaunay triangulation of large uniform point sets, tile-parallel.

The 100M-point config (BASELINE.json configs[3]) cannot go through one Qhull
call on the GPU host (an hour, ~150 GB).  This builds THE Delaunay
triangulation of the same points (unique for points in general position) from
independent Qhull runs on overlapping tiles, using only a local certificate:

  A triangle of the Delaunay triangulation of the points in a box H is a
  triangle of the global one when its circumdisk, clipped to the unit square
  (where all points live), lies inside H: the disk is empty locally, and no
  point outside H can be in it.

* The square is cut into G x G tiles; tile t runs Qhull on the points of its
  core box extended by a margin on each side (clipped to the square), keeps
  the triangles it certifies and owns (centroid in its core).
* The hull region, where triangles have huge circumdisks reaching along the
  sides, is done by one more Qhull run on the points within `band` of the
  square's boundary; a band triangle is certified when its clipped disk
  misses the inner square, and kept when its owner tile cannot certify it
  (a pure geometric predicate, no cross-process lookup).
* Completeness is checked, not assumed: T == 2n - 2 - h (h = hull vertices)
  and every interior edge is shared by exactly two triangles (the GPU twin
  build); a gap (an interior disk wider than the margin) raises.

Certificates use the bounding box of the circumdisk inflated by a relative
1e-9, so rounding can only make them more conservative.  The triangle order
is tile-major and Qhull order inside a tile (cone-local like a global Qhull
run); triangles are CCW.

    python tools/tiled_delaunay.py N [--grid G] [--workers W] [--check-qhull]
"""
import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

_PTS = None  # fork-inherited point array


def circum(pts, tri):
    """circumcenters and radii (float64) of triangles tri[k] = (a, b, c)"""
    a, b, c = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    bx, by = b[:, 0] - a[:, 0], b[:, 1] - a[:, 1]
    cx, cy = c[:, 0] - a[:, 0], c[:, 1] - a[:, 1]
    d = 2.0 * (bx * cy - by * cx)
    with np.errstate(divide="ignore", invalid="ignore"):
        b2, c2 = bx * bx + by * by, cx * cx + cy * cy
        ux = (cy * b2 - by * c2) / d
        uy = (bx * c2 - cx * b2) / d
    r = np.sqrt(ux * ux + uy * uy)
    bad = ~np.isfinite(r)
    r[bad] = np.inf
    ux[bad] = 0.0
    uy[bad] = 0.0
    return a[:, 0] + ux, a[:, 1] + uy, r * (1.0 + 1e-9) + 1e-12


def box_certified(cx, cy, r, box):
    """clipped circumdisk inside box (x0, y0, x1, y1) -- bounding-box test;
    box sides on the unit square's boundary are open to the outside"""
    x0, y0, x1, y1 = box
    ok = np.isfinite(r)
    ok &= (cx - r >= x0) | (x0 <= 0.0)
    ok &= (cx + r <= x1) | (x1 >= 1.0)
    ok &= (cy - r >= y0) | (y0 <= 0.0)
    ok &= (cy + r <= y1) | (y1 >= 1.0)
    # the clipped disk must also stay inside the square's part of the box:
    # a box side at the square's boundary only helps when the disk's part
    # inside the square is what matters -- the points are all in the square
    return ok


def tile_box(i, j, G, margin):
    x0, x1 = i / G, (i + 1) / G
    y0, y1 = j / G, (j + 1) / G
    return (max(0.0, x0 - margin), max(0.0, y0 - margin), min(1.0, x1 + margin), min(1.0, y1 + margin))


def owner_of(x, y, G):
    i = np.minimum((x * G).astype(np.int64), G - 1)
    j = np.minimum((y * G).astype(np.int64), G - 1)
    return i, j


def _ccw(pts, t):
    a, b, c = pts[t[:, 0]], pts[t[:, 1]], pts[t[:, 2]]
    area2 = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    cw = area2 < 0
    t[cw] = t[cw][:, [0, 2, 1]]
    return t


def run_tile(args):
    i, j, G, margin, idx_path = args
    from scipy.spatial import Delaunay
    pts = _PTS
    bx = tile_box(i, j, G, margin)
    sel = np.flatnonzero((pts[:, 0] >= bx[0]) & (pts[:, 0] <= bx[2]) & (pts[:, 1] >= bx[1]) & (pts[:, 1] <= bx[3]))
    local = pts[sel]
    d = Delaunay(local)
    if d.coplanar.size:
        raise RuntimeError(f"tile {i},{j}: Qhull dropped points")
    # global ids in ascending order: every run computes a triangle's
    # certificate and owner from the same floating-point operations
    t = np.sort(sel[d.simplices.astype(np.int64)], axis=1)
    cx, cy, r = circum(pts, t)
    cert = box_certified(cx, cy, r, bx)
    g = pts[t].mean(axis=1)
    oi, oj = owner_of(g[:, 0], g[:, 1], G)
    keep = cert & (oi == i) & (oj == j)
    out = _ccw(pts, t[keep])
    np.save(idx_path, out)
    return i, j, int(keep.sum()), int(sel.size)


def run_band(G, margin, band, path):
    from scipy.spatial import Delaunay
    pts = _PTS
    inner = (pts[:, 0] > band) & (pts[:, 0] < 1 - band) & (pts[:, 1] > band) & (pts[:, 1] < 1 - band)
    sel = np.flatnonzero(~inner)
    local = pts[sel]
    d = Delaunay(local)
    if d.coplanar.size:
        raise RuntimeError("band: Qhull dropped points")
    t = np.sort(sel[d.simplices.astype(np.int64)], axis=1)
    hull = np.unique(d.convex_hull.ravel())
    cx, cy, r = circum(pts, t)
    # certified by the band: the clipped disk misses the open inner square
    lo, hi = band, 1.0 - band
    dx = np.maximum(np.maximum(lo - cx, cx - hi), 0.0)
    dy = np.maximum(np.maximum(lo - cy, cy - hi), 0.0)
    inside_inner = (cx > lo) & (cx < hi) & (cy > lo) & (cy < hi)
    dist = np.where(inside_inner, -np.minimum(np.minimum(cx - lo, hi - cx), np.minimum(cy - lo, hi - cy)),
                    np.sqrt(dx * dx + dy * dy))
    cert = np.isfinite(r) & (dist >= r)
    # ... and not certifiable by its owner tile (that one keeps it)
    g = pts[t].mean(axis=1)
    oi, oj = owner_of(g[:, 0], g[:, 1], G)
    x0 = np.maximum(0.0, oi / G - margin)
    x1 = np.minimum(1.0, (oi + 1) / G + margin)
    y0 = np.maximum(0.0, oj / G - margin)
    y1 = np.minimum(1.0, (oj + 1) / G + margin)
    tile_ok = np.isfinite(r) & (((cx - r) >= x0) | (x0 <= 0)) & (((cx + r) <= x1) | (x1 >= 1)) & \
        (((cy - r) >= y0) | (y0 <= 0)) & (((cy + r) <= y1) | (y1 >= 1))
    keep = cert & ~tile_ok
    out = _ccw(pts, t[keep])
    np.save(path, out)
    return int(keep.sum()), int(sel.size), int(hull.size)


def tiled_delaunay(pts, grid=None, workers=None, margin=None, band=None, tmpdir="/tmp/tiled_delaunay"):
    """Triangles int64[T, 3] (CCW) of the Delaunay triangulation of pts in [0,1]^2."""
    global _PTS
    n = pts.shape[0]
    spacing = 1.0 / np.sqrt(n)
    grid = grid or max(1, int(np.sqrt(n / 400_000)))
    margin = margin or 40 * spacing
    band = band or max(60 * spacing, 2 * margin)
    workers = workers or min(os.cpu_count() or 1, 16)
    os.makedirs(tmpdir, exist_ok=True)
    _PTS = pts
    jobs = [(i, j, grid, margin, os.path.join(tmpdir, f"t{i}_{j}.npy")) for j in range(grid) for i in range(grid)]
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        band_res = pool.apply_async(run_band, (grid, margin, band, os.path.join(tmpdir, "band.npy")))
        res = pool.map(run_tile, jobs, chunksize=1)
        nb, nband, h = band_res.get()
    parts = [np.load(j[4]) for j in jobs] + [np.load(os.path.join(tmpdir, "band.npy"))]
    tri = np.concatenate(parts)
    for j in jobs:
        os.remove(j[4])
    os.remove(os.path.join(tmpdir, "band.npy"))
    T = tri.shape[0]
    info = {"n": n, "grid": grid, "margin": margin, "band": band, "workers": workers, "T": T, "hull": h,
            "band_kept": nb, "band_points": nband, "seconds": round(time.time() - t0, 1),
            "expected_T": 2 * n - 2 - h}
    if T != 2 * n - 2 - h:
        raise RuntimeError(f"tiled Delaunay incomplete: {info}")
    return tri, info


def uniform_points(n, seed=0):
    """The reference generator's draw (io_formats.py:351-388, bbox (0,0,1,1))."""
    return np.random.default_rng(seed).uniform((0.0, 0.0), (1.0, 1.0), (n, 2))


def triangulation(n, seed=0, **kw):
    """A Triangulation (reference layout) of n uniform points: tiled Delaunay,
    then neighbors and trivertex from the device twin build (tm_label), checked
    for a closed edge structure (every interior edge shared by two triangles)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2204_05438_b200 import Triangulation
    from paper_2204_05438_b200.device import DeviceMesh
    pts = uniform_points(n, seed)
    tri, info = tiled_delaunay(pts, **kw)
    t = Triangulation(pts.ravel(), tri.ravel(), np.full(tri.size, -1, np.int64))
    dm = DeviceMesh.upload(t, check=True, use_trivertex=False)  # validation: orientation, edge counts
    tw = dm.twin_host().astype(np.int64)
    nb = np.where(tw >= 0, tw // 3, -1)
    t.neighbors = nb
    t.trivertex = dm.trivertex_host()
    border = int((nb < 0).sum())
    if border != info["hull"]:
        raise RuntimeError(f"border edges {border} != hull vertices {info['hull']}")
    info["border_edges"] = border
    return t, info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--check-qhull", action="store_true", help="compare the triangle set with one Qhull run")
    a = ap.parse_args()
    pts = uniform_points(a.n)
    tri, info = tiled_delaunay(pts, grid=a.grid, workers=a.workers)
    print(info, flush=True)
    if a.check_qhull:
        from scipy.spatial import Delaunay
        ref = np.sort(Delaunay(pts).simplices.astype(np.int64), axis=1)
        got = np.sort(tri, axis=1)
        key = lambda t: (t[:, 0] * a.n + t[:, 1]) * a.n + t[:, 2]  # noqa: E731
        same = np.array_equal(np.sort(key(ref)), np.sort(key(got)))
        print("same triangle set as Qhull:", same, flush=True)
        sys.exit(0 if same else 1)


if __name__ == "__main__":
    main()
