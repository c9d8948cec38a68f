"""Long-item kernel spills (items handed to the warp kernel) of one whole-path run."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "u100m"
tri = bench.load_mesh(w, 0)
dev = torch.device("cuda", 0)
n, T = tri.n_vertices, tri.n_triangles
xy = torch.from_numpy(tri.vertices).to(dev)
tr = torch.from_numpy(tri.triangles).to(dev)
off = torch.empty(T + 1, dtype=torch.int64, device=dev)
v = torch.empty(3 * T, dtype=torch.int32, device=dev)
ctx = _capi.context(dev)
npol, nsl = ctypes.c_int64(), ctypes.c_int64()
st = (ctypes.c_int64 * _capi.NUM_STATS)()
ctx.check(_capi.lib().tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                          _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st,
                                          _capi.stream_ptr(dev)))
d = ctx.debug()
last = d[74]
print(w, "spills shared", d[72], "pool", d[73], "last spilled: L", last >> 40, "pieces", (last >> 20) & 0xFFFFF,
      "depth", last & 0xFFFFF, "slowest item (0.1us, depth, qi)", d[60] >> 32, (d[60] >> 16) & 0xFFFF, d[60] & 0xFFFF)
