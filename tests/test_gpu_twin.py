"""Twin build (K0) robustness: displacement overflow grows the table and
reruns (no valid mesh is rejected), and vertex ids only enter through the
hashed keys -- a permuted numbering gives the permuted result."""
import ctypes

import numpy as np
import pytest

import oracle
from conftest import load_case

pytestmark = pytest.mark.gpu


def _whole_path(ctx, tri, dev):
    import torch
    from paper_2204_05438_b200 import _capi
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(np.ascontiguousarray(tri.vertices)).to(dev)
    tr = torch.from_numpy(np.ascontiguousarray(tri.triangles)).to(dev)
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    v = torch.empty(3 * T, dtype=torch.int32, device=dev)
    npol, nsl = ctypes.c_int64(), ctypes.c_int64()
    st = (ctypes.c_int64 * _capi.NUM_STATS)()
    ctx.check(_capi.lib().tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                              _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st,
                                              _capi.stream_ptr(dev)))
    P, F = npol.value, nsl.value
    return off[: P + 1].cpu().numpy(), v[:F].cpu().numpy().astype(np.int64)


def _host_path(ctx, tri):
    from paper_2204_05438_b200 import _capi
    n, T = tri.n_vertices, tri.n_triangles
    xy = np.ascontiguousarray(tri.vertices, dtype=np.float64)
    tr = np.ascontiguousarray(tri.triangles, dtype=np.int64)
    off = np.empty(T + 1, dtype=np.int64)
    v = np.empty(3 * T, dtype=np.int32)
    npol, nsl = ctypes.c_int64(), ctypes.c_int64()
    st = (ctypes.c_int64 * _capi.NUM_STATS)()
    ctx.check(_capi.lib().tm_mesh_to_polygons_host(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), T, 0, _capi.ptr(off),
                                                   _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl),
                                                   st))
    return off[: npol.value + 1].copy(), v[: nsl.value].astype(np.int64)


@pytest.mark.parametrize("shrink", ["4", "7"])
def test_table_overflow_grows_and_reruns(cuda, shrink, monkeypatch):
    """TERMESH_TABLE_SHRINK starts the context with a table 2^-s the size: the
    inserts overflow, the call reruns with twice the buckets until they fit, and
    the output is the reference's."""
    import paper_2204_05438_b200 as tm
    from paper_2204_05438_b200 import _capi
    monkeypatch.setenv("TERMESH_TABLE_SHRINK", shrink)
    tri = tm.generate_random_delaunay(20_000, seed=3)
    ref = oracle.execute(tri)
    for run in (_whole_path, _host_path):
        ctx = _capi.Context(cuda.index or 0)  # reads the hook at creation
        off, v = run(ctx, tri) if run is _host_path else run(ctx, tri, cuda)
        assert np.array_equal(off, ref["final"][0]) and np.array_equal(v, ref["final"][1]), run.__name__
        ctx.close()


@pytest.mark.parametrize("name", ["u1k_unit", "aniso2k_s1", "clust5k_s0", "sun"])
def test_permuted_vertex_ids(cuda, name):
    """Relabel the vertices with a random permutation: labels are unchanged and
    every output polygon is the permuted reference polygon (same raw order and
    rotation -- walks start from triangle slots, not vertex ids)."""
    import paper_2204_05438_b200 as tm
    tri, g = load_case(name)
    n = tri.n_vertices
    perm = np.random.default_rng(11).permutation(n).astype(np.int64)
    xy = tri.vertices.reshape(-1, 2)
    xy2 = np.empty_like(xy)
    xy2[perm] = xy
    t2 = tm.Triangulation(xy2.ravel().copy(), perm[tri.triangles], tri.neighbors.copy(), None)
    lab = tm.label_all(t2, check=True)
    assert np.array_equal(lab.max_edge, g["max_edge"]) and np.array_equal(lab.seed, g["seed"])
    final, _ = tm.execute(t2)
    off, v = final.csr()
    assert np.array_equal(off, g["final_off"]) and np.array_equal(v, perm[g["final_verts"]])



@pytest.mark.parametrize("name", ["u1k_unit", "aniso2k_s1", "clust5k_s0", "sun", "tie5", "single", "grid2x2", "u1k_box"])
def test_single_pass_labels(cuda, name, monkeypatch):
    """Single-pass labels (both half-edges of a far edge meet in pass A,
    table_meet; pass B scans the table for borders) -- the host-array entry's
    default, and every unchecked call with TERMESH_LABEL_ONE=1: the
    reference's final polygons through both entries."""
    from paper_2204_05438_b200 import _capi
    tri, g = load_case(name)
    ctx = _capi.Context(cuda.index or 0)  # default: single pass on the host entry only
    off, v = _host_path(ctx, tri)
    assert np.array_equal(off, g["final_off"]) and np.array_equal(v, g["final_verts"])
    ctx.close()
    monkeypatch.setenv("TERMESH_LABEL_ONE", "1")
    ctx = _capi.Context(cuda.index or 0)
    off, v = _whole_path(ctx, tri, cuda)
    assert np.array_equal(off, g["final_off"]) and np.array_equal(v, g["final_verts"])
    ctx.close()


def test_single_pass_labels_repeatable(cuda, monkeypatch):
    """The rendezvous races (two arrivals on one empty slot, pairs labelled from
    either side) on a 300k-point mesh, ten runs of each entry: every output
    equals the two-pass device path's."""
    import paper_2204_05438_b200 as tm
    from paper_2204_05438_b200 import _capi
    tri = tm.generate_random_delaunay(300_000, seed=5)
    monkeypatch.setenv("TERMESH_LABEL_ONE", "0")
    ctx = _capi.Context(cuda.index or 0)
    ref = _whole_path(ctx, tri, cuda)
    ctx.close()
    monkeypatch.setenv("TERMESH_LABEL_ONE", "1")
    ctx = _capi.Context(cuda.index or 0)
    for _ in range(10):
        for off, v in (_whole_path(ctx, tri, cuda), _host_path(ctx, tri)):
            assert np.array_equal(off, ref[0]) and np.array_equal(v, ref[1])
    ctx.close()
