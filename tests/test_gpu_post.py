"""Device kernels around the path (tm_post.cu): canonical form, polygon
analytics, trivertex validation -- against the reference's own results
(goldens produced by the Python reference) and numpy restatements of the
reference formulas (the checkers, traversal.py:94-166, oracle.py:124-141)."""
import numpy as np
import pytest

import oracle
from conftest import CASE_NAMES, load_case, load_hashes

pytestmark = pytest.mark.gpu


def tm():
    import paper_2204_05438_b200 as m
    return m


# ---------------------------------------------------------------- numpy checkers (reference formulas)
def _flat(off, v):
    lens = np.diff(off)
    pid = np.repeat(np.arange(lens.size, dtype=np.int64), lens)
    intra = np.arange(v.size, dtype=np.int64) - off[:-1][pid] if v.size else np.empty(0, np.int64)
    return pid, intra, lens, off[:-1]


def ref_tip_flags(off, v):  # traversal.py:112-124
    pid, intra, lens, starts = _flat(off, v)
    flags = np.zeros(lens.size, dtype=bool)
    if v.size:
        L = lens[pid]
        prv = np.where(intra == 0, L - 1, intra - 1)
        nxt = np.where(intra == L - 1, 0, intra + 1)
        base = starts[pid]
        flags[pid[v[base + prv] == v[base + nxt]]] = True
    return flags


def ref_repeated(off, v):  # traversal.py:127-137
    pid, _, lens, _ = _flat(off, v)
    flags = np.zeros(lens.size, dtype=bool)
    if v.size:
        width = int(v.max()) + 1
        keys = np.sort(pid * width + v)
        dup = keys[1:] == keys[:-1]
        flags[keys[1:][dup] // width] = True
    return flags


def ref_extra(off, v):  # traversal.py:140-147
    pid, _, _, _ = _flat(off, v)
    if v.size == 0:
        return 0
    width = int(v.max()) + 1
    return int(v.size - np.unique(pid * width + v).size)


def ref_edges(off, v):  # traversal.py:156-166
    pid, intra, lens, starts = _flat(off, v)
    if v.size == 0:
        return 0
    nxt = np.where(intra == lens[pid] - 1, 0, intra + 1)
    nv = v[starts[pid] + nxt]
    lo, hi = np.minimum(v, nv), np.maximum(v, nv)
    width = int(hi.max()) + 1
    return int(np.unique(lo * width + hi).size)


def ref_areas(off, v, xy):  # traversal.py:94-109
    pid, intra, lens, starts = _flat(off, v)
    pts = np.asarray(xy, dtype=np.float64).reshape(-1, 2)
    nxt = np.where(intra == lens[pid] - 1, 0, intra + 1)
    nv = v[starts[pid] + nxt]
    p, q = pts[v], pts[nv]
    cross = p[:, 0] * q[:, 1] - q[:, 0] * p[:, 1]
    return 0.5 * np.add.reduceat(cross, starts)


def ref_canon(polys):  # oracle.py:124-141
    out = []
    for p in polys:
        p = tuple(int(x) for x in p)
        m = min(p)
        out.append(min(p[i:] + p[:i] for i, x in enumerate(p) if x == m))
    return sorted(out)


def csr(polys):
    return tm().PolygonMesh.from_polygons([list(p) for p in polys])


# ---------------------------------------------------------------- canonical form
@pytest.mark.parametrize("name", CASE_NAMES)
def test_canonicalize_matches_reference_goldens(cuda, name):
    _, g = load_case(name)
    pm = tm().PolygonMesh.from_csr(g["final_off"], g["final_verts"])
    off, v = tm().canonicalize(pm).csr()
    assert np.array_equal(off, g["canon_off"]) and np.array_equal(v, g["canon_verts"])


@pytest.mark.parametrize("seed", range(6))
def test_canonicalize_random_polygons(cuda, seed):
    """Repeated minimum vertices, shared minima, duplicate polygons, shared
    prefixes of different lengths: tuple order throughout."""
    rng = np.random.default_rng(seed)
    polys = []
    for _ in range(400):
        L = int(rng.integers(1, 30))
        polys.append(rng.integers(0, 12 if seed % 2 else 400, L).tolist())
    polys += [[3, 1, 2], [1, 2, 3], [1, 2], [1, 2, 3, 4], [5, 1, 5, 1], [1, 5, 1, 5]]
    want = ref_canon(polys)
    off, v = tm().canonicalize(csr(polys)).csr()
    got = [tuple(v[off[i]:off[i + 1]].tolist()) for i in range(off.size - 1)]
    assert got == want
    o2, v2 = oracle.canonicalize(csr(polys).csr())
    assert np.array_equal(o2, off) and np.array_equal(v2, v)


def test_canonicalize_empty(cuda):
    off, v = tm().canonicalize(csr([])).csr()
    assert off.tolist() == [0] and v.size == 0


def test_canonicalize_u1m_hashes(cuda):
    from conftest import big_input
    import paper_2204_05438_b200.io_formats as io
    h = load_hashes().get("u1m_unit")
    if not h:
        pytest.skip("no u1m hashes")
    tri = big_input("u1m_unit")
    final, _ = tm().execute(tri)
    off, v = tm().canonicalize(final, n_vertices=tri.n_vertices).csr()
    assert io.array_hash(off) == h["canon_off"] and io.array_hash(v.astype(np.int64)) == h["canon_verts"]


# ---------------------------------------------------------------- analytics
@pytest.mark.parametrize("name", CASE_NAMES)
@pytest.mark.parametrize("which", ["mesh0", "final"])
def test_polygon_analytics_match_reference_formulas(cuda, name, which):
    tri, g = load_case(name)
    off, v = g[f"{which}_off"], g[f"{which}_verts"]
    pm = tm().PolygonMesh.from_csr(off, v)
    assert np.array_equal(tm().tip_flags(pm), ref_tip_flags(off, v))
    assert np.array_equal(tm().repeated_vertex_flags(pm), ref_repeated(off, v))
    assert tm().extra_vertex_visits(pm) == ref_extra(off, v)
    assert np.array_equal(tm().unique_vertices(pm), np.unique(v))
    assert tm().boundary_edge_count(pm) == ref_edges(off, v)
    got = tm().enclosed_signed_areas(pm, tri.vertices)
    want = ref_areas(off, v, tri.vertices)
    assert np.array_equal(got, want), np.max(np.abs(got - want))


def test_polygon_analytics_long_polygons(cuda):
    """Polygons over the short-path limit (64 slots) and over the pairwise
    block (128): the one-block stamp pass and the pairwise recursion."""
    rng = np.random.default_rng(5)
    polys = [rng.integers(0, 3000, L).tolist() for L in (65, 129, 300, 1000, 5000, 3, 7, 8, 9)]
    pm = csr(polys)
    off, v = pm.csr()
    xy = rng.normal(0, 1, (3000, 2))
    assert np.array_equal(tm().repeated_vertex_flags(pm), ref_repeated(off, v))
    assert tm().extra_vertex_visits(pm) == ref_extra(off, v)
    assert tm().boundary_edge_count(pm) == ref_edges(off, v)
    assert np.array_equal(tm().enclosed_signed_areas(pm, xy), ref_areas(off, v, xy))


# ---------------------------------------------------------------- trivertex rule
def test_trivertex_check(cuda):
    from paper_2204_05438_b200.errors import ValidationError
    tri, _ = load_case("u1k_unit")
    assert tm().validate(tri).ok
    for bad_v, val in ((5, -2), (7, tri.n_triangles), (9, -1)):
        t2 = tm().Triangulation(tri.vertices, tri.triangles, tri.neighbors, tri.trivertex.copy())
        t2.trivertex[bad_v] = val
        rep = tm().validate(t2)
        assert not rep.ok and rep.defects[0][0] == "trivertex" and rep.defects[0][1] == bad_v
    # a triangle that does not contain the vertex
    t2 = tm().Triangulation(tri.vertices, tri.triangles, tri.neighbors, tri.trivertex.copy())
    t3 = tri.triangles.reshape(-1, 3)
    v = 11
    t2.trivertex[v] = int(np.flatnonzero(~(t3 == v).any(axis=1))[0])
    rep = tm().validate(t2)
    assert not rep.ok and rep.defects[0][:2] == ("trivertex", v)
    with pytest.raises(ValidationError):
        tm().execute(t2)
