"""Region boundary walks on the GPU (drop-in for the reference traversal.py).

build_polygon_mesh (traversal.py:303-347) calls tm_traverse: start edges
(smallest frontier slot, else the reference BFS), walk lengths, exclusive scan
in ascending seed order, walk write.  The result is device CSR; the
reference's length-prefixed `mesh` / `positions` layout (traversal.py:30-45)
is materialised on first access and equals the reference SEQUENTIAL output
byte for byte.

The polygon analytics (tip_flags, repeated_vertex_flags, extra_vertex_visits,
unique_vertices, boundary_edge_count, enclosed_signed_areas) are untimed
statistics in the reference (pipeline.py:150-171); here they are device
kernels (tm_polygon_stats / tm_polygon_areas) over the device CSR.
"""

import ctypes

import numpy as np

from . import _capi
from .backend import SEQUENTIAL, Backend
from .mesh_core import Triangulation


class PolygonMesh:
    """Packed polygon storage (traversal.py:30-73).

    mesh: int64 runs [length, v0, ..., v_{length-1}]; positions: int64 offset
    of each polygon's length slot; count: number of polygons.  Internally a
    CSR pair (offsets int64[P+1], verts int32) that may live on the device.
    """

    def __init__(self, mesh=None, positions=None, count=None, *, offsets=None, verts=None):
        self._mesh = None if mesh is None else np.asarray(mesh, dtype=np.int64)
        self._positions = None if positions is None else np.asarray(positions, dtype=np.int64)
        self._d_off = offsets
        self._d_verts = verts
        self._h_off = None
        self._h_verts = None
        if count is None:
            count = (offsets.numel() - 1) if offsets is not None else len(self._positions)
        self.count = int(count)

    # ------------------------------------------------------------ CSR access
    def csr(self):
        """Host CSR (offsets int64[P+1], verts int64)."""
        if self._h_off is None:
            if self._d_off is not None:
                self._h_off = self._d_off.to("cpu").numpy()
                self._h_verts = self._d_verts.to("cpu").numpy().astype(np.int64)
            else:
                lens = self._mesh[self._positions] if self.count else np.empty(0, np.int64)
                off = np.zeros(self.count + 1, dtype=np.int64)
                np.cumsum(lens, out=off[1:])
                idx = np.repeat(self._positions + 1 - off[:-1], lens) + np.arange(int(off[-1]))
                self._h_off, self._h_verts = off, self._mesh[idx]
        return self._h_off, self._h_verts

    def device_csr(self):
        """Device CSR (offsets int64[P+1], verts int32)."""
        if self._d_off is None:
            import torch
            off, v = self.csr()
            self._d_off = torch.from_numpy(off).to("cuda")
            self._d_verts = torch.from_numpy(v.astype(np.int32)).to("cuda")
        return self._d_off, self._d_verts

    @property
    def mesh(self) -> np.ndarray:
        if self._mesh is None:
            off, v = self.csr()
            P = self.count
            out = np.empty(int(off[-1]) + P, dtype=np.int64)
            pos = off[:-1] + np.arange(P, dtype=np.int64)
            out[pos] = np.diff(off)
            mask = np.ones(out.size, dtype=bool)
            mask[pos] = False
            out[mask] = v
            self._mesh, self._positions = out, pos
        return self._mesh

    @property
    def positions(self) -> np.ndarray:
        if self._positions is None:
            _ = self.mesh
        return self._positions

    def polygon(self, i: int) -> np.ndarray:
        off, v = self.csr()
        return v[off[i]:off[i + 1]]

    def polygons(self):
        for i in range(self.count):
            yield self.polygon(i)

    def lengths(self) -> np.ndarray:
        off, _ = self.csr()
        return np.diff(off)

    def same_as(self, other: "PolygonMesh") -> bool:
        a, b = self.csr(), other.csr()
        return self.count == other.count and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

    @classmethod
    def from_polygons(cls, polys) -> "PolygonMesh":
        lens = np.fromiter((len(p) for p in polys), dtype=np.int64, count=len(polys))
        off = np.zeros(len(polys) + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        v = np.concatenate([np.asarray(p, dtype=np.int64) for p in polys]) if polys else np.empty(0, np.int64)
        pm = cls(count=len(polys), positions=np.empty(0))
        pm._positions = None
        pm._h_off, pm._h_verts = off, v
        return pm

    @classmethod
    def from_csr(cls, offsets, verts) -> "PolygonMesh":
        pm = cls(count=len(offsets) - 1, positions=np.empty(0))
        pm._positions = None
        pm._h_off = np.asarray(offsets, dtype=np.int64)
        pm._h_verts = np.asarray(verts, dtype=np.int64)
        return pm


# ---------------------------------------------------------------- analytics
# The reference's polygon analytics (traversal.py:94-166), computed by the
# tm_polygon_stats / tm_polygon_areas kernels over the device CSR.
def _stats(pm: PolygonMesh, want_flags: bool = False, want_unique: bool = False, n_vertices: int = -1):
    import torch
    off, v = pm.device_csr()
    P = pm.count
    dev = off.device
    tip = rep = uniq = None
    if want_flags:
        tip = torch.empty(max(P, 1), dtype=torch.uint8, device=dev)
        rep = torch.empty(max(P, 1), dtype=torch.uint8, device=dev)
    if want_unique:  # distinct ids <= slots
        uniq = torch.empty(max(int(v.numel()), 1), dtype=torch.int32, device=dev)
    extra, count, edges = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_polygon_stats(ctx.ptr, _capi.ptr(off), _capi.ptr(v), P, n_vertices, _capi.ptr(tip),
                                      _capi.ptr(rep), _capi.ptr(uniq), ctypes.byref(extra), ctypes.byref(count),
                                      ctypes.byref(edges), _capi.stream_ptr(dev))
    ctx.check(rc)
    return {"tip": tip, "rep": rep, "extra": extra.value, "n_unique": count.value, "unique": uniq,
            "edges": edges.value}


def tip_flags(pm: PolygonMesh) -> np.ndarray:
    """Per polygon: any cyclic triple (a, b, a) (traversal.py:112-124)."""
    if pm.count == 0:
        return np.zeros(0, dtype=bool)
    return _stats(pm, want_flags=True)["tip"][: pm.count].cpu().numpy().astype(bool)


def repeated_vertex_flags(pm: PolygonMesh) -> np.ndarray:
    """Per polygon: any vertex more than once (traversal.py:127-137)."""
    if pm.count == 0:
        return np.zeros(0, dtype=bool)
    return _stats(pm, want_flags=True)["rep"][: pm.count].cpu().numpy().astype(bool)


def extra_vertex_visits(pm: PolygonMesh) -> int:
    """Sum over polygons of (length - distinct vertices) (traversal.py:140-147)."""
    return 0 if pm.count == 0 else int(_stats(pm)["extra"])


def unique_vertices(pm: PolygonMesh, n_vertices: int = -1) -> np.ndarray:
    """Sorted distinct vertex ids (traversal.py:150-153)."""
    if pm.count == 0:
        return np.zeros(0, dtype=np.int64)
    st = _stats(pm, want_unique=True, n_vertices=n_vertices)
    return st["unique"][: st["n_unique"]].cpu().numpy().astype(np.int64)


def unique_vertex_count(pm: PolygonMesh, n_vertices: int = -1) -> int:
    """len(unique_vertices(pm)) without the D2H of the ids (PhaseStats.final_vertices)."""
    return 0 if pm.count == 0 else int(_stats(pm, n_vertices=n_vertices)["n_unique"])


def boundary_edge_count(pm: PolygonMesh) -> int:
    """Distinct undirected boundary edges (traversal.py:156-166)."""
    return 0 if pm.count == 0 else int(_stats(pm)["edges"])


def enclosed_signed_areas(pm: PolygonMesh, vertices) -> np.ndarray:
    """Shoelace area per polygon walk (traversal.py:94-109), numpy's summation order."""
    import torch
    if pm.count == 0:
        return np.zeros(0, dtype=np.float64)
    off, v = pm.device_csr()
    dev = off.device
    xy = torch.from_numpy(np.ascontiguousarray(vertices, dtype=np.float64).ravel()).to(dev)
    area = torch.empty(pm.count, dtype=torch.float64, device=dev)
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_polygon_areas(ctx.ptr, _capi.ptr(off), _capi.ptr(v), pm.count, _capi.ptr(xy),
                                      _capi.ptr(area), _capi.stream_ptr(dev))
    ctx.check(rc)
    return area.cpu().numpy()


# ---------------------------------------------------------------- traversal
def build_polygon_mesh(tri: Triangulation, labels, backend: Backend = SEQUENTIAL) -> PolygonMesh:
    """One polygon per seed triangle, ascending seed order (traversal.py:303)."""
    import torch
    dm = labels.device_mesh(tri)
    T = dm.T
    dev = dm.hw.device
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    verts = torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
    n_polys, n_slots = ctypes.c_int64(), ctypes.c_int64()
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_traverse(ctx.ptr, _capi.ptr(dm.tri32), _capi.ptr(dm.hw), _capi.ptr(dm.seed), T,
                                 _capi.ptr(off), _capi.ptr(verts), T, 3 * T, ctypes.byref(n_polys),
                                 ctypes.byref(n_slots), _capi.stream_ptr(dev))
    ctx.check(rc, "traversal")
    P, F = n_polys.value, n_slots.value
    return PolygonMesh(count=P, offsets=off[: P + 1], verts=verts[:F])
