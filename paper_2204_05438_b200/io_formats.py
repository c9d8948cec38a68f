"""Input generation and output formats around the mesh -> polygons path.

These sit OUTSIDE the device hot path (the reference leaves them untimed,
pipeline.py:1-7): synthetic Delaunay inputs built with scipy's Qhull exactly
as the reference builds them (io_formats.py:351-388), the canonical polygon
form (oracle.py:124-141) and the byte-stable polymesh writer
(io_formats.py:251-262).
"""

import ctypes
import hashlib
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ParseError
from .mesh_core import Triangulation
from .traversal import PolygonMesh


def _reorient(pts, simplices, neighbors):
    """CW triangles get corners 1<->2 and neighbor slots 1<->2 swapped."""
    t3 = np.ascontiguousarray(simplices, dtype=np.int64)
    n3 = np.ascontiguousarray(neighbors, dtype=np.int64)
    a, b, c = pts[t3[:, 0]], pts[t3[:, 1]], pts[t3[:, 2]]
    area2 = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    cw = area2 < 0
    t3[cw] = t3[cw][:, [0, 2, 1]]
    n3[cw] = n3[cw][:, [0, 2, 1]]
    return t3, n3


def _lowest_incident(triangles, n):
    """Lowest incident triangle per vertex (input preparation on the host)."""
    out = np.full(n, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(out, triangles, np.repeat(np.arange(triangles.size // 3, dtype=np.int64), 3))
    out[out == np.iinfo(np.int64).max] = -1
    return out


def triangulate_points(pts) -> Triangulation:
    """scipy Delaunay + the reference's post-processing (io_formats.py:367-382)."""
    from scipy.spatial import Delaunay
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    d = Delaunay(pts)
    if d.coplanar.size:
        raise ValueError("a point was dropped by Qhull (coplanar)")
    t3, n3 = _reorient(pts, d.simplices, d.neighbors)
    tri = Triangulation(pts.ravel(), t3.ravel(), n3.ravel())
    tri.trivertex = _lowest_incident(tri.triangles, tri.n_vertices)
    return tri


def generate_random_delaunay(n: int, bbox=(0.0, 0.0, 10000.0, 10000.0), seed: int = 0) -> Triangulation:
    """Delaunay triangulation of n uniform points (same draw and Qhull call as
    the reference generator, so the arrays are identical)."""
    from scipy.spatial import QhullError
    if n < 3:
        raise ValueError("need at least 3 points to triangulate")
    x0, y0, x1, y1 = map(float, bbox)
    rng = np.random.default_rng(seed)
    last = None
    for _ in range(5):
        pts = rng.uniform((x0, y0), (x1, y1), (n, 2))
        try:
            return triangulate_points(pts)
        except QhullError as e:
            last = e
        except ValueError:
            continue
    raise ValueError(f"could not triangulate a degenerate point draw: {last}")


def generate_clustered_delaunay(n: int, clusters: int = 64, sigma: float = 0.002, seed: int = 0) -> Triangulation:
    """Gaussian clusters around uniform centres in the unit square."""
    rng = np.random.default_rng(seed)
    for _ in range(5):
        c = rng.uniform(0, 1, (clusters, 2))
        lab = rng.integers(0, clusters, n)
        pts = c[lab] + rng.normal(0, sigma, (n, 2))
        try:
            return triangulate_points(pts)
        except ValueError:
            continue
    raise ValueError("could not triangulate the clustered draw")


def generate_anisotropic_delaunay(n: int, seed: int = 0, ratio: float = 0.01) -> Triangulation:
    """N(0,1) x N(0,ratio) points: long hull slivers, deep repair."""
    rng = np.random.default_rng(seed)
    pts = np.stack([rng.normal(0, 1, n), rng.normal(0, ratio, n)], 1)
    return triangulate_points(pts)


def cached(name: str, make, cache_dir=None) -> Triangulation:
    """Load a generated triangulation from an .npz cache, or build and store it."""
    d = Path(cache_dir or os.environ.get("TERMESH_CACHE", "/tmp/termesh_cache"))
    d.mkdir(parents=True, exist_ok=True)
    f = d / f"{name}.npz"
    if f.exists():
        z = np.load(f)
        return Triangulation(z["vertices"], z["triangles"], z["neighbors"], z["trivertex"])
    tri = make()
    tmp = d / f"{name}.{os.getpid()}.tmp.npz"
    np.savez(tmp, vertices=tri.vertices, triangles=tri.triangles, neighbors=tri.neighbors,
             trivertex=tri.trivertex)
    os.replace(tmp, f)
    return tri


def array_hash(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# ---------------------------------------------------------------- canonical form
def canonicalize(pm: PolygonMesh, n_vertices: int = -1) -> PolygonMesh:
    """Each polygon rotated to its lexicographically smallest rotation,
    polygons sorted in tuple order (oracle.py:124-141) -- tm_canonicalize on
    the device (counting sort on the minimum vertex, lexicographic order inside
    each bucket).  The result is a device-backed PolygonMesh."""
    import torch
    from . import _capi
    off, v = pm.device_csr()
    P = pm.count
    dev = off.device
    off_out = torch.empty(P + 1, dtype=torch.int64, device=dev)
    v_out = torch.empty(max(int(v.numel()), 1), dtype=torch.int32, device=dev)
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_canonicalize(ctx.ptr, _capi.ptr(off), _capi.ptr(v), P, n_vertices, _capi.ptr(off_out),
                                     _capi.ptr(v_out), _capi.stream_ptr(dev))
    ctx.check(rc)
    return PolygonMesh(count=P, offsets=off_out, verts=v_out[: int(v.numel())])


def _fmt(x: float) -> str:
    """repr of a Python float (io_formats.py:44-46); the native writers use
    tm_format_double, which prints the same bytes."""
    return repr(float(x))


def format_double(x: float) -> str:
    """The native writers' float formatting (tm_format_double): Python repr."""
    from . import _capi
    buf = ctypes.create_string_buffer(64)
    n = _capi.lib().tm_format_double(float(x), buf, 64)
    if n < 0:
        raise ValueError("format buffer too small")
    return buf.value.decode()


def write_polymesh(mesh: PolygonMesh, vertices, path) -> None:
    """Canonical text form (io_formats.py:251-262): `<#v> <#polys>`, one
    `x y` line per vertex (repr floats), one `<len> v0 v1 ...` per polygon.
    Canonical order on the device (tm_canonicalize), text by the native
    multi-threaded writer (tm_write_polymesh) -- byte-identical output."""
    from . import _capi
    verts = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).ravel())
    n = verts.size // 2
    cm = canonicalize(mesh, n_vertices=n if n else -1)
    d_off, d_v = cm.device_csr()
    off = np.ascontiguousarray(d_off.cpu().numpy(), dtype=np.int64)
    v = np.ascontiguousarray(d_v.cpu().numpy(), dtype=np.int32)
    err = ctypes.create_string_buffer(512)
    rc = _capi.lib().tm_write_polymesh(str(path).encode(), verts.ctypes.data_as(ctypes.c_void_p), n,
                                       off.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p),
                                       cm.count, err, 512)
    if rc != 0:
        raise OSError(err.value.decode())


# ---------------------------------------------------------------- Triangle file sets
@dataclass
class TriangleFileSet:
    """Paths of one triangulation: .node, .ele, .neigh, optional .trivertex
    (io_formats.py:33-41)."""

    node: Path
    ele: Path
    neigh: Path
    trivertex: Path | None = None


_KIND = {"node": 0, "ele": 1, "neigh": 2, "trivertex": 3}


def _read_native(path, kind: str, n_expected: int = 0) -> np.ndarray:
    """tm_file_read: the reference's _data_lines + row readers (io_formats.py:48-158)
    in native code; parse failures raise ParseError(path, line, message) with
    the reference's messages."""
    from . import _capi
    L = _capi.lib()
    h = L.tm_file_read(str(path).encode(), _KIND[kind], int(n_expected))
    try:
        rows, cols, line = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        msg = ctypes.create_string_buffer(1024)
        if L.tm_file_status(h, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(line), msg, 1024):
            raise ParseError(path, int(line.value), msg.value.decode())
        out = np.empty(rows.value * cols.value, dtype=np.float64 if kind == "node" else np.int64)
        L.tm_file_copy(h, out.ctypes.data_as(ctypes.c_void_p))
    finally:
        L.tm_file_close(h)
    return out


def read_triangulation(files: TriangleFileSet) -> Triangulation:
    """Read and normalize a Triangle file set (io_formats.py:161-210): one-based
    sets shifted to zero-based (border -1 kept), range checks, clockwise
    triangles reoriented (vertex and neighbor slots 1, 2 swapped), trivertex
    computed (device) when no file gives it, and the result validated (device)."""
    from .errors import ValidationError
    from .mesh_core import compute_trivertex, signed_areas, validate
    coords = _read_native(files.node, "node")
    n = coords.size // 2
    tris = _read_native(files.ele, "ele").reshape(-1, 3)
    neigh = _read_native(files.neigh, "neigh").reshape(-1, 3)
    if neigh.shape[0] != tris.shape[0]:
        raise ParseError(files.neigh, 0, f"{neigh.shape[0]} neighbor rows for {tris.shape[0]} triangles")
    one_based = bool((tris == n).any())  # one-based sets reference vertex n
    if one_based:
        tris = tris - 1
        neigh = np.where(neigh >= 0, neigh - 1, neigh)
    if tris.size and ((tris < 0) | (tris >= n)).any():
        bad = int(np.argwhere((tris < 0) | (tris >= n))[0][0])
        raise ParseError(files.ele, 0, f"triangle row {bad} references a vertex outside [0, {n})")
    T = tris.shape[0]
    if neigh.size and ((neigh < -1) | (neigh >= T)).any():
        bad = int(np.argwhere((neigh < -1) | (neigh >= T))[0][0])
        raise ParseError(files.neigh, 0, f"neighbor row {bad} references a triangle outside [0, {T})")
    trivertex = None
    if files.trivertex is not None:
        trivertex = _read_native(files.trivertex, "trivertex", n)
        if one_based:
            trivertex = np.where(trivertex >= 0, trivertex - 1, trivertex)
    tri = Triangulation(coords, tris.ravel(), neigh.ravel(), trivertex)
    cw = signed_areas(tri) < 0
    if cw.any():
        t3 = tri.triangles.reshape(-1, 3)
        n3 = tri.neighbors.reshape(-1, 3)
        t3[cw] = t3[cw][:, [0, 2, 1]]
        n3[cw] = n3[cw][:, [0, 2, 1]]
    if tri.trivertex is None:
        tri.trivertex = compute_trivertex(tri)
    report = validate(tri)
    if not report.ok:
        raise ValidationError(f"{files.node}: triangulation is invalid: {report.summary()}", report)
    return tri


def write_triangulation(tri: Triangulation, basepath) -> TriangleFileSet:
    """.node/.ele/.neigh (+ .trivertex) next to basepath, zero-based, repr
    coordinates (io_formats.py:213-248), written by tm_write_triangle_file."""
    from . import _capi
    base = Path(basepath)
    paths = [base.with_suffix(x) for x in (".node", ".ele", ".neigh")]
    err = ctypes.create_string_buffer(512)
    xy = np.ascontiguousarray(tri.vertices, dtype=np.float64).ravel()
    t3 = np.ascontiguousarray(tri.triangles, dtype=np.int64).ravel()
    n3 = np.ascontiguousarray(tri.neighbors, dtype=np.int64).ravel()
    jobs = [(paths[0], 0, xy, None, tri.n_vertices), (paths[1], 1, None, t3, tri.n_triangles),
            (paths[2], 2, None, n3, tri.n_triangles)]
    tv_path = None
    if tri.trivertex is not None:
        tv_path = base.with_suffix(".trivertex")
        jobs.append((tv_path, 3, None, np.ascontiguousarray(tri.trivertex, dtype=np.int64), tri.n_vertices))
    for path, which, a, b, count in jobs:
        rc = _capi.lib().tm_write_triangle_file(str(path).encode(), which, _ptr_np(a), _ptr_np(b), int(count), err,
                                                512)
        if rc != 0:
            raise OSError(err.value.decode())
    return TriangleFileSet(paths[0], paths[1], paths[2], tv_path)


def _ptr_np(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def read_polymesh(path):
    """Parse a polymesh file into (flat vertex array, PolygonMesh)."""
    lines = [(i, ln.split("#", 1)[0].split()) for i, ln in enumerate(Path(path).read_text().splitlines(), 1)]
    lines = [(i, t) for i, t in lines if t]
    if not lines or len(lines[0][1]) != 2:
        raise ParseError(path, lines[0][0] if lines else 0, "header must be <#vertices> <#polygons>")
    n, count = int(lines[0][1][0]), int(lines[0][1][1])
    if len(lines) - 1 != n + count:
        raise ParseError(path, 0, f"header promises {n} vertex and {count} polygon rows, file has {len(lines) - 1}")
    verts = np.array([[float(t[0]), float(t[1])] for _, t in lines[1:1 + n]], dtype=np.float64).ravel()
    polys = []
    for lineno, t in lines[1 + n:]:
        ln = int(t[0])
        if len(t) != 1 + ln:
            raise ParseError(path, lineno, f"polygon row promises {ln} vertices, has {len(t) - 1}")
        polys.append([int(x) for x in t[1:]])
    return verts, PolygonMesh.from_polygons(polys)
