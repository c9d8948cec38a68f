"""Input generation and output formats around the mesh -> polygons path.

These sit OUTSIDE the device hot path (the reference leaves them untimed,
pipeline.py:1-7): synthetic Delaunay inputs built with scipy's Qhull exactly
as the reference builds them (io_formats.py:351-388), the canonical polygon
form (oracle.py:124-141) and the byte-stable polymesh writer
(io_formats.py:251-262).
"""

import hashlib
import os
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
def _min_rotation(p):
    p = list(p)
    m = min(p)
    best = None
    for i, x in enumerate(p):
        if x == m:
            r = p[i:] + p[:i]
            if best is None or r < best:
                best = r
    return tuple(best)


def canonicalize(pm: PolygonMesh) -> PolygonMesh:
    """Each polygon rotated to its lexicographically smallest rotation,
    polygons sorted in tuple order (oracle.py:124-141)."""
    off, v = pm.csr()
    lens = np.diff(off)
    polys = []
    for i in range(pm.count):
        s = v[off[i]:off[i + 1]]
        if lens[i] == 0:
            polys.append(())
            continue
        k = int(np.argmin(s))
        if np.count_nonzero(s == s[k]) == 1:
            polys.append(tuple(np.concatenate((s[k:], s[:k])).tolist()))
        else:
            polys.append(_min_rotation(s.tolist()))
    polys.sort()
    return PolygonMesh.from_polygons(polys)


def _fmt(x: float) -> str:
    return repr(float(x))


def write_polymesh(mesh: PolygonMesh, vertices, path) -> None:
    """Canonical text form (io_formats.py:251-262): `<#v> <#polys>`, one
    `x y` line per vertex (repr floats), one `<len> v0 v1 ...` per polygon."""
    verts = np.asarray(vertices, dtype=np.float64).ravel()
    cm = canonicalize(mesh)
    n = verts.size // 2
    with open(path, "w") as f:
        f.write(f"{n} {cm.count}\n")
        for i in range(n):
            f.write(f"{_fmt(verts[2 * i])} {_fmt(verts[2 * i + 1])}\n")
        for p in cm.polygons():
            f.write(f"{p.size} " + " ".join(str(int(x)) for x in p) + "\n")


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
