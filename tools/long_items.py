"""Longest pre-repair polygons of a workload (the repair lineage's size)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2204_05438_b200 as tm  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "u100m"
tri = bench.load_mesh(w, 0)
lab = tm.label_all(tri, check=False)
m0 = tm.build_polygon_mesh(tri, lab)
off, v = m0.csr()
L = np.diff(off)
rep = tm.repeated_vertex_flags(m0)
order = np.argsort(-L)[:12]
print(w, "polygons", L.size, "max", int(L.max()), ">8192:", int((L > 8192).sum()), ">21760:", int((L > 21760).sum()))
for i in order:
    print(" poly", int(i), "len", int(L[i]), "repeated", bool(rep[i]))
