"""GPU Delaunay (paper_2204_05438_b200.delaunay) timing and cross-check:
same triangle set as Qhull (n <= 10M) or as the tile-parallel Qhull
triangulation (tools/tiled_delaunay.py) at 100M.

    python tools/delaunay_check.py N [--against qhull|tiled]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_05438_b200.delaunay import delaunay_gpu  # noqa: E402


def rows(t):
    t = np.sort(np.asarray(t, dtype=np.int64).reshape(-1, 3), axis=1)
    return t[np.lexsort(t.T[::-1])]


def main():
    n = int(sys.argv[1])
    against = sys.argv[sys.argv.index("--against") + 1] if "--against" in sys.argv else "qhull"
    pts = np.random.default_rng(0).uniform((0.0, 0.0), (1.0, 1.0), (n, 2))
    delaunay_gpu(pts[:1000])  # warm-up (context, library)
    torch.cuda.synchronize()
    t0 = time.time()
    t, info = delaunay_gpu(pts)
    info["seconds"] = round(time.time() - t0, 2)
    t0 = time.time()
    if against == "qhull":
        from scipy.spatial import Delaunay
        ref = Delaunay(pts).simplices
    else:
        import tiled_delaunay
        ref, _ = tiled_delaunay.tiled_delaunay(pts)
    info["reference"] = against
    info["reference_seconds"] = round(time.time() - t0, 1)
    info["same_triangle_set"] = bool(np.array_equal(rows(t), rows(ref)))
    print(json.dumps(info), flush=True)


if __name__ == "__main__":
    main()
