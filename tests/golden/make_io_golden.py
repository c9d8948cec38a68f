"""Golden fixtures for the text formats, produced by the Python reference
(run in the build container, where /root/reference exists; outputs committed).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py

tests/golden/io/
  <case>.node/.ele/.neigh[/.trivertex]   Triangle file sets (reference
                                         write_triangulation, plus hand-made
                                         variants: one-based, comments,
                                         attributes/markers, clockwise rows)
  expected.npz                           read_triangulation arrays per set
  parse_errors.json                      malformed files -> ParseError text
  polymesh.json                          sha256 of write_polymesh output for
                                         golden final meshes
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import termesh as tm  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))
IO = os.path.join(HERE, "io")
CASES = os.path.join(HERE, "cases")


def case_tri(name):
    z = np.load(os.path.join(CASES, f"{name}.npz"))
    return tm.Triangulation(z["vertices"], z["triangles"].astype(np.int64), z["neighbors"].astype(np.int64),
                            z["trivertex"].astype(np.int64)), z


def main():
    os.makedirs(IO, exist_ok=True)
    expected = {}
    sets = {}
    # 1. reference writer output
    for name in ("sun", "u1k_unit", "aniso2k_s1", "clust5k_s0"):
        tri, _ = case_tri(name)
        fs = tm.write_triangulation(tri, os.path.join(IO, name))
        sets[name] = fs
    # 2. hand-made variants of the sun fixture
    tri, _ = case_tri("sun")
    n, T = tri.n_vertices, tri.n_triangles
    pts = tri.points()
    t3 = tri.triangles.reshape(-1, 3)
    n3 = tri.neighbors.reshape(-1, 3)

    def w(path, text):
        with open(path, "w") as f:
            f.write(text)

    # one-based, comments, blank lines, attributes and markers, CW rows (corners 1,2 swapped)
    base = os.path.join(IO, "sun_variant")
    node = f"# points\n{n} 2 1 1\n" + "".join(f"{i + 1} {float(pts[i, 0])!r} {float(pts[i, 1])!r} 0.5 1  # p{i}\n" for i in range(n))
    ele = f"{T} 3 0\n\n" + "".join(
        f"{i + 1} {t3[i, 0] + 1} {t3[i, 2] + 1} {t3[i, 1] + 1}\n" if i % 2 else
        f"{i + 1} {t3[i, 0] + 1} {t3[i, 1] + 1} {t3[i, 2] + 1}\n" for i in range(T))
    nb = f"{T} 3\n" + "".join(
        "{} {} {} {}\n".format(i + 1, *[(x + 1 if x >= 0 else -1) for x in (
            (n3[i, 0], n3[i, 2], n3[i, 1]) if i % 2 else (n3[i, 0], n3[i, 1], n3[i, 2]))]) for i in range(T))
    w(base + ".node", node)
    w(base + ".ele", ele)
    w(base + ".neigh", nb)
    sets["sun_variant"] = tm.TriangleFileSet(base + ".node", base + ".ele", base + ".neigh")
    for name, fs in sets.items():
        t = tm.read_triangulation(fs)
        expected[f"{name}_vertices"] = t.vertices
        expected[f"{name}_triangles"] = t.triangles
        expected[f"{name}_neighbors"] = t.neighbors
        expected[f"{name}_trivertex"] = t.trivertex
    np.savez_compressed(os.path.join(IO, "expected.npz"), **expected)
    with open(os.path.join(IO, "sets.json"), "w") as f:
        json.dump({k: {"node": os.path.basename(str(v.node)), "ele": os.path.basename(str(v.ele)),
                       "neigh": os.path.basename(str(v.neigh)),
                       "trivertex": os.path.basename(str(v.trivertex)) if v.trivertex else None}
                   for k, v in sets.items()}, f, indent=1, sort_keys=True)

    # 3. parse errors: (file kind, text) -> the reference's ParseError message
    bad = {
        "node_empty": ("node", "# nothing\n\n"),
        "node_header_short": ("node", "3\n"),
        "node_dim3": ("node", "3 3 0 0\n"),
        "node_bad_count": ("node", "x 2\n"),
        "node_markers": ("node", "1 2 0 2\n0 0.0 0.0 1\n"),
        "node_cols": ("node", "2 2 0 0\n0 0.0 0.0\n1 1.0\n"),
        "node_float": ("node", "1 2\n0 0.0 abc\n"),
        "node_too_many": ("node", "1 2\n0 0 0\n1 1 1\n"),
        "node_too_few": ("node", "3 2\n0 0 0\n1 1 1\n"),
        "node_underscore_ok": ("node", "1 2\n0 1_0.5 2e1_0\n"),
        "node_hex": ("node", "1 2\n0 0x10 1\n"),
        "ele_width": ("ele", "1 4\n0 1 2 3\n"),
        "ele_short_row": ("ele", "1 3\n0 1 2\n"),
        "ele_int": ("ele", "1 3\n0 1 2 3.0\n"),
        "ele_rows": ("ele", "2 3\n0 1 2 3\n"),
        "neigh_header": ("neigh", "5\n"),
        "trivertex_count": ("trivertex", "4\n0 1\n"),
        "trivertex_cols": ("trivertex", "2\n0 1 2\n1 1\n"),
    }
    errs = {}
    for key, (kind, text) in bad.items():
        path = os.path.join(IO, f"bad_{key}.{kind}")
        w(path, text)
        try:
            if kind == "node":
                r = tm.io_formats._read_node(path)
            elif kind == "ele":
                r = tm.io_formats._read_indexed_rows(path, "triangle", 4)
            elif kind == "neigh":
                r = tm.io_formats._read_indexed_rows(path, "neighbor", 4)
            else:
                r = tm.io_formats._read_trivertex(path, 2)
            errs[key] = {"kind": kind, "ok": True, "values": np.asarray(r).ravel().tolist()}
        except tm.ParseError as e:
            errs[key] = {"kind": kind, "ok": False, "line": e.line, "message": str(e).split(": ", 1)[1]}
    with open(os.path.join(IO, "parse_errors.json"), "w") as f:
        json.dump(errs, f, indent=1, sort_keys=True)

    # 4. polymesh bytes of golden final meshes
    out = {}
    for name in ("sun", "u1k_unit", "aniso2k_s1", "clust5k_s0", "grid6x5"):
        tri, z = case_tri(name)
        off, v = z["final_off"], z["final_verts"]
        pm = tm.PolygonMesh.from_polygons([v[off[i]:off[i + 1]].tolist() for i in range(off.size - 1)]) \
            if hasattr(tm.PolygonMesh, "from_polygons") else None
        if pm is None:
            from termesh.traversal import PolygonMesh
            pm = PolygonMesh.from_polygons([v[off[i]:off[i + 1]].tolist() for i in range(off.size - 1)])
        path = os.path.join("/tmp", f"{name}.polymesh")
        tm.write_polymesh(pm, tri.vertices, path)
        data = open(path, "rb").read()
        out[name] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data)}
        if name == "sun":
            with open(os.path.join(IO, "sun.polymesh"), "wb") as f:
                f.write(data)
    with open(os.path.join(IO, "polymesh.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("ok", len(sets), "sets", len(errs), "error cases", len(out), "polymesh files")


if __name__ == "__main__":
    main()
