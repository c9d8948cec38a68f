"""Triangulation data model and half-edge index algebra (drop-in for the
reference's mesh_core.py).

Storage and conventions are the reference's (mesh_core.py:1-14, 47-93): flat
`vertices` f64[2n], `triangles` i64[3T] CCW, `neighbors` i64[3T] (BORDER=-1),
optional `trivertex` i64[n]; half-edge h = 3t + j is the edge opposite corner
j with origin corner (j+1)%3 and target (j+2)%3.

The scalar index helpers below are plain arithmetic on those arrays.  The
array-wide operations that sit on the mesh -> polygons path
(`compute_trivertex`, adjacency and the structural checks of `validate`) run
on the GPU through the C ABI; there is no host implementation of them.
"""

from dataclasses import dataclass

import numpy as np

from .errors import StructuralError

BORDER = -1


@dataclass
class ValidationReport:
    """Outcome of validate(); ok is true exactly when defects is empty.

    Each defect is a (kind, element index, message) triple with the kinds of
    the reference report (mesh_core.py:28-35): index_range, orientation,
    degenerate, duplicate, reciprocity, edge_count, trivertex.  The device
    check reports, per kind, the first offending element and the count.
    """

    ok: bool
    defects: list

    def summary(self, limit: int = 5) -> str:
        if self.ok:
            return "ok"
        head = "; ".join(f"{kind}[{idx}]: {msg}" for kind, idx, msg in self.defects[:limit])
        extra = len(self.defects) - limit
        return head + (f"; ... {extra} more" if extra > 0 else "")


@dataclass
class Triangulation:
    """Flat-array triangle mesh with neighbor adjacency (mesh_core.py:47-93)."""

    vertices: np.ndarray
    triangles: np.ndarray
    neighbors: np.ndarray
    trivertex: np.ndarray | None = None

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).ravel()
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int64).ravel()
        self.neighbors = np.ascontiguousarray(self.neighbors, dtype=np.int64).ravel()
        if self.trivertex is not None:
            self.trivertex = np.ascontiguousarray(self.trivertex, dtype=np.int64).ravel()
        if self.vertices.size % 2:
            raise ValueError("vertex array length must be a multiple of 2")
        if self.triangles.size % 3:
            raise ValueError("triangle array length must be a multiple of 3")
        if self.neighbors.size != self.triangles.size:
            raise ValueError("neighbor array must match the triangle array length")
        if self.trivertex is not None and self.trivertex.size != self.n_vertices:
            raise ValueError("trivertex array must hold one entry per vertex")

    @property
    def n_vertices(self) -> int:
        return self.vertices.size // 2

    @property
    def n_triangles(self) -> int:
        return self.triangles.size // 3

    @property
    def n_halfedges(self) -> int:
        return self.triangles.size

    def points(self) -> np.ndarray:
        return self.vertices.reshape(-1, 2)


def triangle_of(h: int) -> int:
    return h // 3


def local_edge(h: int) -> int:
    return h % 3


def next_halfedge(h: int) -> int:
    t, j = divmod(h, 3)
    return 3 * t + (j + 1) % 3


def prev_halfedge(h: int) -> int:
    t, j = divmod(h, 3)
    return 3 * t + (j + 2) % 3


def edge_endpoints(tri: Triangulation, h: int) -> tuple[int, int]:
    t, j = divmod(h, 3)
    return int(tri.triangles[3 * t + (j + 1) % 3]), int(tri.triangles[3 * t + (j + 2) % 3])


def origin(tri: Triangulation, h: int) -> int:
    return edge_endpoints(tri, h)[0]


def target(tri: Triangulation, h: int) -> int:
    return edge_endpoints(tri, h)[1]


def twin(tri: Triangulation, h: int) -> int:
    """Opposite half-edge across `neighbors[h]`, or BORDER (scalar helper)."""
    n = int(tri.neighbors[h])
    if n == BORDER:
        return BORDER
    o, g = edge_endpoints(tri, h)
    for k in range(3):
        if edge_endpoints(tri, 3 * n + k) == (g, o):
            return 3 * n + k
    raise StructuralError(f"triangle {n} is recorded as neighbor of half-edge {h} "
                          f"but shares no edge with endpoints ({o}, {g})")


def squared_length(tri: Triangulation, h: int) -> float:
    o, g = edge_endpoints(tri, h)
    dx = tri.vertices[2 * o] - tri.vertices[2 * g]
    dy = tri.vertices[2 * o + 1] - tri.vertices[2 * g + 1]
    return float(dx * dx + dy * dy)


def signed_areas(tri: Triangulation) -> np.ndarray:
    """Signed triangle areas (input preparation helper: CW reorientation)."""
    p = tri.points()
    t3 = tri.triangles.reshape(-1, 3)
    a, b, c = p[t3[:, 0]], p[t3[:, 1]], p[t3[:, 2]]
    return 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0]))


def compute_trivertex(tri: Triangulation) -> np.ndarray:
    """Lowest incident triangle per vertex, -1 if unreferenced (device atomicMin)."""
    from .device import DeviceMesh
    dm = DeviceMesh.upload(tri, check=False)
    return dm.trivertex_host()


def validate(tri: Triangulation) -> ValidationReport:
    """Structural check on the device: index ranges, orientation, degenerate
    triangles, edge sharing counts and endpoint reciprocity (from the twin
    build), agreement of `neighbors` with the twin build, and trivertex
    containment.  Returns the report instead of raising."""
    from .device import DeviceMesh
    from .errors import ValidationError
    try:
        dm = DeviceMesh.upload(tri, check=True)
        dm.check_neighbors(tri.neighbors)
        if tri.trivertex is not None:
            dm.check_trivertex(tri.trivertex)
    except ValidationError as e:
        return e.report if e.report is not None else ValidationReport(False, [("structural", -1, str(e))])
    return ValidationReport(True, [])
