"""GPU Delaunay input generation (tm_delaunay + the hull band through Qhull):
the same triangle set as scipy's Qhull on the reference generator's points,
and the mesh -> polygons output on it equals the output on Qhull's mesh in
canonical form (the triangle order differs; regions and polygons do not)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sorted_rows(t):
    t = np.sort(np.asarray(t, dtype=np.int64).reshape(-1, 3), axis=1)
    return t[np.lexsort(t.T[::-1])]


@pytest.mark.parametrize("n,seed", [(1000, 0), (10_000, 1), (200_000, 2), (1_000_000, 0)])
def test_same_triangles_as_qhull(cuda, n, seed):
    from scipy.spatial import Delaunay
    from paper_2204_05438_b200.delaunay import delaunay_gpu
    pts = np.random.default_rng(seed).uniform((0.0, 0.0), (1.0, 1.0), (n, 2))
    t, info = delaunay_gpu(pts)
    assert info["T"] == t.shape[0] == 2 * n - 2 - info["hull"]
    assert np.array_equal(_sorted_rows(t), _sorted_rows(Delaunay(pts).simplices))
    # CCW
    p = pts[t]
    area2 = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    assert (area2 > 0).all()


def test_pipeline_on_gpu_mesh_matches_qhull_mesh_canonically(cuda):
    import paper_2204_05438_b200 as tm
    from paper_2204_05438_b200.delaunay import generate_random_delaunay_gpu
    n = 100_000
    tq = tm.generate_random_delaunay(n, (0, 0, 1, 1), 0)
    tg, info = generate_random_delaunay_gpu(n, 0)
    assert np.array_equal(tg.vertices, tq.vertices)
    lab_q, lab_g = tm.label_all(tq, check=False), tm.label_all(tg, check=False)
    m_q, m_g = tm.build_polygon_mesh(tq, lab_q), tm.build_polygon_mesh(tg, lab_g)
    c_q, c_g = tm.canonicalize(m_q).csr(), tm.canonicalize(m_g).csr()
    assert np.array_equal(c_q[0], c_g[0]) and np.array_equal(c_q[1], c_g[1])  # regions: order-independent
    f_q, _ = tm.execute(tq)
    f_g, _ = tm.execute(tg)
    a, b = tm.canonicalize(f_q).csr(), tm.canonicalize(f_g).csr()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_rejects_points_off_the_grid(cuda):
    from paper_2204_05438_b200.delaunay import delaunay_gpu
    pts = np.random.default_rng(0).normal(0.5, 0.1, (100, 2))
    with pytest.raises(ValueError):
        delaunay_gpu(pts)
