"""CPU oracle for the mesh -> polygons path (TEST INFRASTRUCTURE ONLY).

ctypes front end of oracle.c, a C restatement of the reference `termesh`
algorithm (labeling.py, traversal.py, reparation.py, oracle.py:124-141).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package; the product path (paper_2204_05438_b200) never does.

Inputs are duck-typed reference triangulations: objects with `vertices`
(f64[2n]), `triangles` (i64[3T]), `neighbors` (i64[3T], -1 = border) and
optional `trivertex` (i64[n]).  Polygon meshes are CSR pairs
(offsets i64[P+1], verts i64[offsets[-1]]).
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .build import LIB, build

_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        lib.or_last_error.restype = ctypes.c_char_p
        lib.or_max_threads.restype = ctypes.c_int
        lib.or_compute_trivertex.argtypes = [_P, _I64, _I64, _P]
        lib.or_label.argtypes = [_P, _P, _P, _I64, ctypes.c_int, _P, _P, _P]
        lib.or_traverse.argtypes = [_P, _P, _I64, _P, _P, ctypes.c_int, _P, _P, _I64, _I64, _P]
        lib.or_repair.argtypes = [_P, _P, _P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _I64, _I64, _P, _P, _I64]
        lib.or_canonicalize.argtypes = [_P, _P, _I64, _P, _P]
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    """Raised with the oracle's message; `code` is 1 structural, 2 value, 3 capacity."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, _load().or_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().or_max_threads())


@dataclass
class Labels:
    max_edge: np.ndarray  # int8[T]
    frontier: np.ndarray  # bool[3T]
    seed: np.ndarray      # bool[T]


def _arrays(tri):
    xy = np.ascontiguousarray(tri.vertices, dtype=np.float64).ravel()
    tr = np.ascontiguousarray(tri.triangles, dtype=np.int64).ravel()
    nb = np.ascontiguousarray(tri.neighbors, dtype=np.int64).ravel()
    return xy, tr, nb


def compute_trivertex(triangles, n_vertices) -> np.ndarray:
    tr = np.ascontiguousarray(triangles, dtype=np.int64).ravel()
    out = np.empty(int(n_vertices), dtype=np.int64)
    _load().or_compute_trivertex(_ptr(tr), tr.size // 3, out.size, _ptr(out))
    return out


def label_all(tri, threads: int = 0) -> Labels:
    """labeling.py:118-145 (without validation)."""
    xy, tr, nb = _arrays(tri)
    T = tr.size // 3
    me = np.empty(T, dtype=np.int8)
    fr = np.empty(3 * T, dtype=np.bool_)
    sd = np.empty(T, dtype=np.bool_)
    _check(_load().or_label(_ptr(xy), _ptr(tr), _ptr(nb), T, threads, _ptr(me), _ptr(fr), _ptr(sd)))
    return Labels(me, fr, sd)


def build_polygon_mesh(tri, labels: Labels, threads: int = 0):
    """traversal.py:303-347 under SEQUENTIAL order -> CSR (offsets, verts)."""
    _, tr, nb = _arrays(tri)
    T = tr.size // 3
    fr = np.ascontiguousarray(labels.frontier, dtype=np.bool_)
    sd = np.ascontiguousarray(labels.seed, dtype=np.bool_)
    P = int(sd.sum())
    cap = int(fr.sum())
    off = np.zeros(P + 1, dtype=np.int64)
    verts = np.empty(max(cap, 1), dtype=np.int64)
    n = np.zeros(1, dtype=np.int64)
    _check(_load().or_traverse(_ptr(tr), _ptr(nb), T, _ptr(fr), _ptr(sd), threads,
                               _ptr(off), _ptr(verts), P, cap, _ptr(n)))
    return off, verts[: off[-1]].copy()


def repair_all(tri, labels: Labels, mesh, guard_extra: int = -1):
    """reparation.py:343-377 (round schedule).  Mutates labels.frontier.

    guard_extra >= 0 replaces the extra-visit count of the pinch guard
    (reparation.py:322) -- a seed-partitioned run uses the global one.
    Returns ((offsets, verts), stats dict rounds/splits/initial_tips/unrepaired/
    tip_extra), tip_extra = extra visits of the tip-phase output.
    """
    _, tr, nb = _arrays(tri)
    T = tr.size // 3
    n = np.asarray(tri.vertices).size // 2
    tv = getattr(tri, "trivertex", None)
    if tv is None:
        tv = compute_trivertex(tr, n)
    tv = np.ascontiguousarray(tv, dtype=np.int64)
    if labels.frontier.dtype != np.bool_ or not labels.frontier.flags.c_contiguous:
        raise TypeError("labels.frontier must be a contiguous bool array (mutated in place)")
    off_in, v_in = (np.ascontiguousarray(a, dtype=np.int64) for a in mesh)
    P = off_in.size - 1
    cap_p = T + 1
    cap_s = int(v_in.size) + 2 * T + 8
    off = np.zeros(cap_p + 1, dtype=np.int64)
    verts = np.empty(cap_s, dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    stats = np.zeros(5, dtype=np.int64)
    _check(_load().or_repair(_ptr(tr), _ptr(nb), _ptr(tv), T, n, _ptr(labels.frontier),
                             _ptr(off_in), _ptr(v_in), P, _ptr(off), _ptr(verts), cap_p, cap_s,
                             _ptr(cnt), _ptr(stats), int(guard_extra)))
    c = int(cnt[0])
    off = off[: c + 1].copy()
    s = dict(zip(("rounds", "splits", "initial_tips", "unrepaired", "tip_extra"), (int(x) for x in stats)))
    return (off, verts[: off[-1]].copy()), s


def canonicalize(mesh):
    """oracle.py:124-141: min rotation per polygon, then tuple-order sort."""
    off, v = (np.ascontiguousarray(a, dtype=np.int64) for a in mesh)
    P = off.size - 1
    o2 = np.empty_like(off)
    v2 = np.empty(max(v.size, 1), dtype=np.int64)
    _check(_load().or_canonicalize(_ptr(off), _ptr(v), P, _ptr(o2), _ptr(v2)))
    return o2, v2[: v.size]


def execute(tri, threads: int = 0):
    """label -> traverse -> repair (pipeline.py:124-172 minus validation/stats).

    Returns dict with labels (frontier post-repair), frontier_pre, mesh0, final, stats.
    """
    labels = label_all(tri, threads)
    frontier_pre = labels.frontier.copy()
    mesh0 = build_polygon_mesh(tri, labels, threads)
    final, stats = repair_all(tri, labels, mesh0)
    return {"labels": labels, "frontier_pre": frontier_pre, "mesh0": mesh0,
            "final": final, "stats": stats}


def polygons(mesh):
    """CSR -> list of python int lists."""
    off, v = mesh
    return [v[off[i]:off[i + 1]].tolist() for i in range(off.size - 1)]
