"""Region boundary walks on the GPU (drop-in for the reference traversal.py).

build_polygon_mesh (traversal.py:303-347) calls tm_traverse: start edges
(smallest frontier slot, else the reference BFS), walk lengths, exclusive scan
in ascending seed order, walk write.  The result is device CSR; the
reference's length-prefixed `mesh` / `positions` layout (traversal.py:30-45)
is materialised on first access and equals the reference SEQUENTIAL output
byte for byte.

The polygon analytics (tip_flags, repeated_vertex_flags, extra_vertex_visits,
unique_vertices, boundary_edge_count, enclosed_signed_areas) are untimed
statistics in the reference (pipeline.py:150-171) and are provided here as
numpy restatements over the host CSR.
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
def _flat(pm: PolygonMesh):
    off, v = pm.csr()
    lens = np.diff(off)
    pid = np.repeat(np.arange(pm.count, dtype=np.int64), lens)
    intra = np.arange(v.size, dtype=np.int64) - off[:-1][pid] if v.size else np.empty(0, np.int64)
    return v, pid, intra, lens, off[:-1]


def tip_flags(pm: PolygonMesh) -> np.ndarray:
    """Per polygon: any cyclic triple (a, b, a)."""
    v, pid, intra, lens, starts = _flat(pm)
    flags = np.zeros(pm.count, dtype=bool)
    if v.size:
        L = lens[pid]
        prv = starts[pid] + np.where(intra == 0, L - 1, intra - 1)
        nxt = starts[pid] + np.where(intra == L - 1, 0, intra + 1)
        flags[pid[v[prv] == v[nxt]]] = True
    return flags


def _dup_mask(v, pid):
    """Duplicate marks (all but the first occurrence of each (polygon, vertex))."""
    order = np.lexsort((v, pid))
    sp, sv = pid[order], v[order]
    dup = np.zeros(v.size, dtype=bool)
    dup[1:] = (sp[1:] == sp[:-1]) & (sv[1:] == sv[:-1])
    return dup, sp


def repeated_vertex_flags(pm: PolygonMesh) -> np.ndarray:
    v, pid, _, _, _ = _flat(pm)
    flags = np.zeros(pm.count, dtype=bool)
    if v.size:
        dup, sp = _dup_mask(v, pid)
        flags[sp[dup]] = True
    return flags


def extra_vertex_visits(pm: PolygonMesh) -> int:
    v, pid, _, _, _ = _flat(pm)
    if v.size == 0:
        return 0
    dup, _ = _dup_mask(v, pid)
    return int(dup.sum())


def unique_vertices(pm: PolygonMesh) -> np.ndarray:
    _, v = pm.csr()
    return np.unique(v)


def boundary_edge_count(pm: PolygonMesh) -> int:
    v, pid, intra, lens, starts = _flat(pm)
    if v.size == 0:
        return 0
    nxt = v[starts[pid] + np.where(intra == lens[pid] - 1, 0, intra + 1)]
    lo, hi = np.minimum(v, nxt), np.maximum(v, nxt)
    return int(np.unique(lo * (int(hi.max()) + 1) + hi).size)


def enclosed_signed_areas(pm: PolygonMesh, vertices) -> np.ndarray:
    v, pid, intra, lens, starts = _flat(pm)
    out = np.zeros(pm.count, dtype=np.float64)
    if v.size == 0:
        return out
    pts = np.asarray(vertices, dtype=np.float64).reshape(-1, 2)
    nv = v[starts[pid] + np.where(intra == lens[pid] - 1, 0, intra + 1)]
    cross = pts[v, 0] * pts[nv, 1] - pts[nv, 0] * pts[v, 1]
    np.add.at(out, pid, cross)
    return 0.5 * out


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
