"""Print the repair-lineage trace of the longest item (debug timestamps)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402

tri = bench.load_mesh("u1m", 0)
n, T = tri.n_vertices, tri.n_triangles
xy = torch.from_numpy(tri.vertices).cuda()
tr = torch.from_numpy(tri.triangles).cuda()
off = torch.empty(T + 1, dtype=torch.int64, device="cuda")
v = torch.empty(3 * T, dtype=torch.int32, device="cuda")
ctx = _capi.context()
P, F = ctypes.c_int64(), ctypes.c_int64()
st = (ctypes.c_int64 * 8)()
for _ in range(3):
    rc = _capi.lib().tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                         _capi.ptr(v), T, 3 * T, ctypes.byref(P), ctypes.byref(F), st,
                                         _capi.stream_ptr())
    ctx.check(rc)
d = ctx.debug()
t0 = d[0]
print("item L", d[2], "tips", d[3], "precompute us", (d[1] - t0) / 1e3)
prev = d[1]
for r in range(1, 56):
    if d[4 + r] == 0:
        break
    print(f"round {r:3d} end {(d[4 + r] - t0) / 1e3:8.1f} us  (+{(d[4 + r] - prev) / 1e3:6.1f})")
    prev = d[4 + r]
