"""Print tm_launch_count deltas per whole-path call (graph capture + replays)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_05438_b200 as tm  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402

tri = tm.generate_random_delaunay(100_000, (0, 0, 1, 1), 0)
dev = torch.device("cuda", 0)
n, T = tri.n_vertices, tri.n_triangles
xy = torch.from_numpy(tri.vertices).to(dev)
tr = torch.from_numpy(tri.triangles).to(dev)
off = torch.empty(T + 1, dtype=torch.int64, device=dev)
v = torch.empty(3 * T, dtype=torch.int32, device=dev)
ctx = _capi.context(dev)
L = _capi.lib()
npol, nsl = ctypes.c_int64(), ctypes.c_int64()
st = (ctypes.c_int64 * _capi.NUM_STATS)()
for k in range(6):
    a = L.tm_launch_count()
    ctx.check(L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off), _capi.ptr(v),
                                    T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st, _capi.stream_ptr(dev)))
    print("call", k, "launches", L.tm_launch_count() - a, flush=True)
