"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every golden case through both device entry points (phase API and
the whole graph-captured path, unpartitioned and as 3 seed partitions), plus
a 100k uniform mesh when SAN_BIG=1; outputs checked against the reference
goldens so a sanitizer-visible hazard that changes results also fails here.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_05438_b200 as tm  # noqa: E402
from conftest import CASE_NAMES, load_case  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402
from paper_2204_05438_b200 import distributed as D  # noqa: E402


def whole_path(tri, dev, parts=1):
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).to(dev)
    tr = torch.from_numpy(tri.triangles).to(dev)
    outs, table, ranks = [], [], []
    for b, e in D.partition(T, parts):
        ctx = _capi.Context(0)
        off, v, p, f, st = D.run_partition(xy, tr, n, T, b, e, ctx=ctx)
        ranks.append([ctx, off, v, p, f])
        table.append([p, f, st["pinch_extra"], st["pinch_deferred"]])
    if D.needs_resume(table):
        tot = D.global_pinch_extra(table)
        for r, row in enumerate(table):
            if row[3]:
                ranks[r][3], ranks[r][4], _ = D.resume_partition(ranks[r][0], ranks[r][1], ranks[r][2], T, tot)
    base = 0
    for ctx, off, v, p, f in ranks:
        o = off[: p + 1].cpu().numpy() + base
        outs.append((o[:-1], v[:f].cpu().numpy()))
        base += f
    return np.concatenate([o for o, _ in outs] + [np.array([base])]), np.concatenate([v for _, v in outs])


def main():
    dev = torch.device("cuda", 0)
    bad = 0
    for name in CASE_NAMES:
        tri, g = load_case(name)
        fin, st = tm.execute(tri)
        off, v = fin.csr()
        ok = np.array_equal(off, g["final_off"]) and np.array_equal(v, g["final_verts"])
        for parts in (1, 3):
            o2, v2 = whole_path(tri, dev, parts)
            ok &= np.array_equal(o2, g["final_off"]) and np.array_equal(v2, g["final_verts"])
        print(name, "ok" if ok else "MISMATCH", flush=True)
        bad += not ok
    if os.environ.get("SAN_BIG"):
        tri = tm.generate_random_delaunay(100_000, (0, 0, 1, 1), 0)
        fin, st = tm.execute(tri)
        print("u100k", fin.count, st.reparation_rounds, flush=True)
    print("SANITIZE_RUN_DONE mismatches", bad, flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
