"""Generate golden vectors from the Python reference (run in the build
container, where /root/reference exists; the outputs are committed).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Small cases (inputs + outputs) -> tests/golden/cases/<name>.npz
Large cases (hashes only; inputs are regenerated with scipy on the GPU box)
                                -> tests/golden/hashes.json

Outputs per case, all from the reference's SEQUENTIAL backend:
  max_edge int8[T], frontier_pre bool[3T], seed bool[T]          (label_all)
  mesh0 CSR (offsets, verts)                                      (build_polygon_mesh)
  final CSR, frontier_post, stats rounds/splits/initial_tips/unrepaired   (repair_all)
  canon CSR of the final mesh                                     (oracle.canonicalize)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import termesh as tm  # noqa: E402  (the reference)
from conftest import build_triangulation, make_grid, make_sun, make_tie_strip  # noqa: E402
from scipy.spatial import Delaunay  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = os.path.join(HERE, "cases")


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def csr_of(pm):
    lens = np.array([len(p) for p in pm.polygons()], dtype=np.int64)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    verts = np.concatenate([np.asarray(p, dtype=np.int64) for p in pm.polygons()]) if len(lens) else \
        np.empty(0, np.int64)
    return off, verts


def tri_from_points(pts):
    d = Delaunay(pts)
    assert not d.coplanar.size
    t3 = d.simplices.astype(np.int64)
    n3 = d.neighbors.astype(np.int64)
    tri = tm.Triangulation(pts.ravel(), t3.ravel(), n3.ravel())
    cw = tm.signed_areas(tri) < 0
    t3v = tri.triangles.reshape(-1, 3)
    n3v = tri.neighbors.reshape(-1, 3)
    t3v[cw] = t3v[cw][:, [0, 2, 1]]
    n3v[cw] = n3v[cw][:, [0, 2, 1]]
    tri.trivertex = tm.compute_trivertex(tri)
    assert tm.validate(tri).ok
    return tri


def run_reference(tri):
    labels = tm.label_all(tri, check=True)
    out = {"max_edge": labels.max_edge.copy(), "frontier_pre": labels.frontier.copy(), "seed": labels.seed.copy()}
    t0 = time.perf_counter()
    m0 = tm.build_polygon_mesh(tri, labels)
    out["mesh0_off"], out["mesh0_verts"] = csr_of(m0)
    out["mesh0_raw_mesh"], out["mesh0_raw_positions"] = m0.mesh.copy(), m0.positions.copy()
    info = {}
    fin = tm.repair_all(tri, labels, m0, stats_out=info)
    out["t_repair"] = time.perf_counter() - t0
    out["final_off"], out["final_verts"] = csr_of(fin)
    out["frontier_post"] = labels.frontier.copy()
    canon = tm.canonicalize(fin)
    out["canon_off"], out["canon_verts"] = csr_of(canon)
    out["stats"] = np.array([info["rounds"], info["splits"], info["initial_tips"], info["unrepaired"]], np.int64)
    return out


def small_cases():
    cases = {
        "single": build_triangulation([(0, 0), (3, 0), (0, 4)], [(0, 1, 2)]),
        "square": build_triangulation([(0, 0), (1, 0), (1, 1), (0, 1)], [(0, 1, 2), (0, 2, 3)]),
        "sun": make_sun(),
        "grid2x2": make_grid(2, 2),
        "grid6x5": make_grid(6, 5),
        "tie5": make_tie_strip(5),
        "u1k_unit": tm.generate_random_delaunay(1000, (0, 0, 1, 1), 0),
        "u1k_box": tm.generate_random_delaunay(1000, seed=0),
    }
    for s in (0, 4, 17):
        cases[f"u500_s{s}"] = tm.generate_random_delaunay(500, seed=s)
    for s in (0, 1, 2, 7, 11, 13, 17):
        rng = np.random.default_rng(s)
        n = 2000
        cases[f"aniso2k_s{s}"] = tri_from_points(np.stack([rng.normal(0, 1, n), rng.normal(0, 0.01, n)], 1))
    for s in (0, 3):
        rng = np.random.default_rng(s)
        n = 5000
        c = rng.uniform(0, 1, (16, 2))
        lab = rng.integers(0, 16, n)
        cases[f"clust5k_s{s}"] = tri_from_points(c[lab] + rng.normal(0, 0.002, (n, 2)))
    return cases


def write_small():
    os.makedirs(CASES, exist_ok=True)
    for name, tri in small_cases().items():
        out = run_reference(tri)
        out.pop("t_repair")
        np.savez_compressed(os.path.join(CASES, f"{name}.npz"), vertices=tri.vertices,
                            triangles=tri.triangles.astype(np.int32), neighbors=tri.neighbors.astype(np.int32),
                            trivertex=tri.trivertex.astype(np.int32), **out)
        print(name, "T", tri.n_triangles, "polys", out["mesh0_off"].size - 1, "->", out["final_off"].size - 1,
              "stats", out["stats"].tolist(), flush=True)


def clustered(n, clusters=64, sigma=0.002, seed=0):
    """Gaussian clusters around uniform centres in the unit square."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0, 1, (clusters, 2))
    lab = rng.integers(0, clusters, n)
    return tri_from_points(c[lab] + rng.normal(0, sigma, (n, 2)))


def big_case(name, tri):
    t0 = time.perf_counter()
    out = run_reference(tri)
    rec = {
        "n": tri.n_vertices, "T": tri.n_triangles,
        "input": {"vertices": h16(tri.vertices), "triangles": h16(tri.triangles),
                  "neighbors": h16(tri.neighbors), "trivertex": h16(tri.trivertex)},
        "max_edge": h16(out["max_edge"]), "frontier_pre": h16(out["frontier_pre"]), "seed": h16(out["seed"]),
        "mesh0_off": h16(out["mesh0_off"]), "mesh0_verts": h16(out["mesh0_verts"]),
        "mesh0_raw_mesh": h16(out["mesh0_raw_mesh"]), "mesh0_raw_positions": h16(out["mesh0_raw_positions"]),
        "final_off": h16(out["final_off"]), "final_verts": h16(out["final_verts"]),
        "frontier_post": h16(out["frontier_post"]),
        "canon_off": h16(out["canon_off"]), "canon_verts": h16(out["canon_verts"]),
        "polygons_after_traversal": int(out["mesh0_off"].size - 1),
        "final_polygons": int(out["final_off"].size - 1),
        "frontier_halfedges": int(out["frontier_pre"].sum()),
        "stats": out["stats"].tolist(),
        "reference_seconds": round(time.perf_counter() - t0, 2),
    }
    print(name, rec, flush=True)
    return rec


def write_big(which):
    path = os.path.join(HERE, "hashes.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    gens = {
        "u100k_unit": lambda: tm.generate_random_delaunay(100_000, (0, 0, 1, 1), 0),
        "u1m_unit": lambda: tm.generate_random_delaunay(1_000_000, (0, 0, 1, 1), 0),
        "u10m_unit": lambda: tm.generate_random_delaunay(10_000_000, (0, 0, 1, 1), 0),
        "c10m_clustered": lambda: clustered(10_000_000),
    }
    for name in which:
        data[name] = big_case(name, gens[name]())
        with open(path, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--big" in sys.argv:
        write_big([a for a in sys.argv[2:]] or ["u100k_unit", "u1m_unit"])
    else:
        write_small()
