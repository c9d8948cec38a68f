"""Text formats (tm_io.cu) against fixtures produced by the Python reference
(tests/golden/make_io_golden.py): Triangle file parsing incl. the reference's
ParseError messages, repr float formatting, byte-identical writers."""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, load_case

IO = os.path.join(GOLDEN, "io")


def io():
    from paper_2204_05438_b200 import io_formats
    return io_formats


def test_repr_formatting_matches_python():
    rng = np.random.default_rng(1)
    vals = list(rng.standard_normal(5000) * 10.0 ** rng.integers(-30, 30, 5000))
    vals += [struct.unpack("<d", rng.bytes(8))[0] for _ in range(20000)]
    vals += [1e16, 1e15, 1.5e15, 1234567890123456.0, 1e-4, 1e-5, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3,
             2.0 ** 53, -0.0, 0.0, float("inf"), -float("inf"), float("nan"), 100.0, 1e22, 1e23]
    bad = [x for x in vals if io().format_double(x) != repr(float(x))]
    assert not bad, bad[:5]


@pytest.mark.parametrize("key", sorted(json.load(open(os.path.join(IO, "parse_errors.json")))))
def test_parse_errors_match_reference(key):
    from paper_2204_05438_b200.errors import ParseError
    e = json.load(open(os.path.join(IO, "parse_errors.json")))[key]
    path = os.path.join(IO, f"bad_{key}.{e['kind']}")
    if e["ok"]:
        got = io()._read_native(path, e["kind"], 2)
        assert got.tolist() == e["values"]
        return
    with pytest.raises(ParseError) as ei:
        io()._read_native(path, e["kind"], 2)
    assert ei.value.line == e["line"]
    assert str(ei.value) == f"{path}:{e['line']}: {e['message']}"


@pytest.mark.parametrize("name", ["sun", "u1k_unit", "aniso2k_s1", "clust5k_s0"])
def test_triangle_writer_bytes_match_reference(name, tmp_path):
    tri, _ = load_case(name)
    fs = io().write_triangulation(tri, tmp_path / name)
    for suffix in (".node", ".ele", ".neigh", ".trivertex"):
        got = (tmp_path / (name + suffix)).read_bytes()
        want = open(os.path.join(IO, name + suffix), "rb").read()
        assert got == want, suffix
    assert fs.trivertex is not None


@pytest.mark.parametrize("name", ["sun", "u1k_unit", "sun_variant"])
def test_native_parse_of_reference_files(name):
    """The raw rows (before normalization) equal a direct reading of the files."""
    sets = json.load(open(os.path.join(IO, "sets.json")))[name]
    xy = io()._read_native(os.path.join(IO, sets["node"]), "node")
    rows = [ln.split("#")[0].split() for ln in open(os.path.join(IO, sets["node"])).read().splitlines()]
    rows = [r for r in rows if r][1:]
    assert np.array_equal(xy.reshape(-1, 2), np.array([[float(r[1]), float(r[2])] for r in rows]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sun", "u1k_unit", "aniso2k_s1", "clust5k_s0", "sun_variant"])
def test_read_triangulation_matches_reference(cuda, name):
    import paper_2204_05438_b200 as tm
    sets = json.load(open(os.path.join(IO, "sets.json")))[name]
    fs = tm.TriangleFileSet(*(os.path.join(IO, sets[k]) if sets[k] else None
                              for k in ("node", "ele", "neigh", "trivertex")))
    tri = tm.read_triangulation(fs)
    z = np.load(os.path.join(IO, "expected.npz"))
    for k in ("vertices", "triangles", "neighbors", "trivertex"):
        assert np.array_equal(getattr(tri, k), z[f"{name}_{k}"]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sun", "u1k_unit", "aniso2k_s1", "clust5k_s0", "grid6x5"])
def test_write_polymesh_bytes_match_reference(cuda, name, tmp_path):
    import paper_2204_05438_b200 as tm
    tri, g = load_case(name)
    pm = tm.PolygonMesh.from_csr(g["final_off"], g["final_verts"])
    out = tmp_path / f"{name}.polymesh"
    tm.write_polymesh(pm, tri.vertices, out)
    want = json.load(open(os.path.join(IO, "polymesh.json")))[name]
    data = out.read_bytes()
    assert len(data) == want["bytes"] and hashlib.sha256(data).hexdigest() == want["sha256"]
    if name == "sun":
        assert data == open(os.path.join(IO, "sun.polymesh"), "rb").read()


@pytest.mark.gpu
def test_pipeline_reads_triangle_files(cuda, tmp_path):
    """PipelineConfig(files=...) -> load_input -> execute (pipeline.py:107-111)."""
    import paper_2204_05438_b200 as tm
    tri, g = load_case("aniso2k_s1")
    fs = tm.write_triangulation(tri, tmp_path / "m")
    cfg = tm.PipelineConfig(files=fs)
    t2 = tm.load_input(cfg)
    final, stats = tm.execute(t2, cfg)
    off, v = final.csr()
    assert np.array_equal(off, g["final_off"]) and np.array_equal(v, g["final_verts"])
