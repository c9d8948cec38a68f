"""Delaunay input generation on the GPU.

The reference triangulates its synthetic inputs with Qhull
(io_formats.generate_random_delaunay, io_formats.py:351-388): ~20 us per
point on one host core (4 min at 10M points, about an hour and ~150 GB at
100M).  Here the interior of the point set is triangulated by tm_delaunay
(csrc/tm_delaunay.cu): one certified local star per point, exact predicates;
the hull region -- the points tm_delaunay could not certify, a thin band
along the box sides where hull triangles have huge circumcircles -- goes
through one Qhull call on the band points, keeping the triangles those points
own (smallest vertex index) whose circumdisk, clipped to the box, stays in
the band (certified the same way).  The result is THE Delaunay triangulation
(unique for points in general position): checked by T == 2n - 2 - h and the
device twin build (every interior edge shared by exactly two triangles,
border edges = hull edges).

Triangles are CCW and grouped by the grid cell of their owner, so the
triangle order is spatially coherent (unlike Qhull's); the vertex order is
the input order.
"""

import ctypes

import numpy as np

from . import _capi
from .mesh_core import Triangulation


def _on_grid(pts):
    """tm_delaunay's exact fallback needs points on the 2^-53 grid of [0, 1)."""
    if pts.size == 0:
        return True
    if pts.min() < 0.0 or pts.max() >= 1.0:
        return False
    s = pts * 9007199254740992.0
    return bool(np.all(s == np.floor(s)))


def _circum(pts, t):
    a, b, c = pts[t[:, 0]], pts[t[:, 1]], pts[t[:, 2]]
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


def _ccw(pts, t):
    a, b, c = pts[t[:, 0]], pts[t[:, 1]], pts[t[:, 2]]
    area2 = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    cw = area2 < 0
    t[cw] = t[cw][:, [0, 2, 1]]
    return t


def _band(pts, box, open_ids, width):
    """Qhull on the points within `width` of the box sides: the triangles the
    open points own, each certified (clipped circumdisk misses the inner box).
    Returns (triangles or None if a certificate fails, hull vertex count)."""
    from scipy.spatial import Delaunay
    x0, y0, x1, y1 = box
    lo_x, hi_x, lo_y, hi_y = x0 + width, x1 - width, y0 + width, y1 - width
    inner = (pts[:, 0] > lo_x) & (pts[:, 0] < hi_x) & (pts[:, 1] > lo_y) & (pts[:, 1] < hi_y)
    if inner[open_ids].any():
        return None, 0
    sel = np.flatnonzero(~inner)
    d = Delaunay(pts[sel])
    if d.coplanar.size:
        raise ValueError("a point was dropped by Qhull (coplanar)")
    t = np.sort(sel[d.simplices.astype(np.int64)], axis=1)
    h = int(np.unique(d.convex_hull.ravel()).size)
    is_open = np.zeros(pts.shape[0], dtype=bool)
    is_open[open_ids] = True
    t = t[is_open[t[:, 0]]]  # owned by an open point (t[:, 0] is the smallest index)
    cx, cy, r = _circum(pts, t)
    dx = np.maximum(np.maximum(lo_x - cx, cx - hi_x), 0.0)
    dy = np.maximum(np.maximum(lo_y - cy, cy - hi_y), 0.0)
    inside = (cx > lo_x) & (cx < hi_x) & (cy > lo_y) & (cy < hi_y)
    dist = np.where(inside, -1.0, np.sqrt(dx * dx + dy * dy))
    if not bool(np.all(np.isfinite(r) & (dist >= r))):
        return None, h
    return _ccw(pts, t), h


def delaunay_gpu(pts, box=(0.0, 0.0, 1.0, 1.0), device=None):
    """Delaunay triangles (int64[T, 3], CCW) of pts (float64[n, 2] on the 2^-53
    grid of [0, 1)) and an info dict.  Raises if the points are not in general
    position or the result fails its completeness checks."""
    import torch
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    n = pts.shape[0]
    if not _on_grid(pts):
        raise ValueError("delaunay_gpu needs points on the 2^-53 grid of [0, 1) (numpy uniform draws)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    xy = torch.from_numpy(pts.ravel()).to(dev)
    cap = 2 * n + 16
    tri = torch.empty(3 * cap, dtype=torch.int32, device=dev)
    opn = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    bx = (ctypes.c_double * 4)(*box)
    nt, no, nd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_delaunay(ctx.ptr, _capi.ptr(xy), n, bx, _capi.ptr(tri), cap, ctypes.byref(nt), _capi.ptr(opn),
                                 ctypes.byref(no), ctypes.byref(nd), _capi.stream_ptr(dev))
    ctx.check(rc)
    if nd.value:
        raise ValueError(f"{nd.value} point(s) in degenerate position (cocircular / collinear ties)")
    t_gpu = tri[: 3 * nt.value].view(-1, 3).cpu().numpy().astype(np.int64)
    open_ids = np.sort(opn[: no.value].cpu().numpy().astype(np.int64))
    # band width: the open points plus the reach of their triangles
    x0, y0, x1, y1 = box
    depth = np.minimum(np.minimum(pts[open_ids, 0] - x0, x1 - pts[open_ids, 0]),
                       np.minimum(pts[open_ids, 1] - y0, y1 - pts[open_ids, 1])) if open_ids.size else np.zeros(1)
    cell = (x1 - x0) / max(1.0, np.floor(np.sqrt(n / 2.0)))
    width = float(depth.max()) + 12 * cell
    t_band, h = None, 0
    while True:
        t_band, h = _band(pts, box, open_ids, width)
        if t_band is not None and t_gpu.shape[0] + t_band.shape[0] == 2 * n - 2 - h:
            break
        if width >= 0.5 * min(x1 - x0, y1 - y0):
            raise RuntimeError(f"GPU Delaunay incomplete (open points {open_ids.size}, width {width})")
        width *= 2
    out = np.concatenate([t_gpu, t_band])
    info = {"n": n, "T": int(out.shape[0]), "gpu_triangles": int(t_gpu.shape[0]), "open_points": int(open_ids.size),
            "band_triangles": int(t_band.shape[0]), "band_width": width, "hull": h}
    return out, info


def generate_random_delaunay_gpu(n: int, seed: int = 0):
    """The reference generator's points (uniform in the unit square,
    default_rng(seed), io_formats.py:351-388) triangulated on the GPU; the
    returned Triangulation carries neighbors and trivertex from the device
    twin build and passed its validation."""
    from .device import DeviceMesh
    pts = np.random.default_rng(seed).uniform((0.0, 0.0), (1.0, 1.0), (n, 2))
    t, info = delaunay_gpu(pts)
    tri = Triangulation(pts.ravel(), t.ravel(), np.full(t.size, -1, dtype=np.int64))
    dm = DeviceMesh.upload(tri, check=True, use_trivertex=False)
    tw = dm.twin_host().astype(np.int64)
    tri.neighbors = np.where(tw >= 0, tw // 3, -1)
    tri.trivertex = dm.trivertex_host()
    border = int((tri.neighbors < 0).sum())
    if border != info["hull"]:
        raise RuntimeError(f"border edges {border} != hull vertices {info['hull']}")
    return tri, info
