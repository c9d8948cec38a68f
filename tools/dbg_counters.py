"""Print the repair kernels' debug counters (Counters.dbg) after one whole-path run."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2204_05438_b200 import _capi
w = sys.argv[1] if len(sys.argv) > 1 else "u1m"
tri = bench.load_mesh(w, 0)
n, T = tri.n_vertices, tri.n_triangles
dev = torch.device("cuda", 0)
xy = torch.from_numpy(tri.vertices).to(dev); tr = torch.from_numpy(tri.triangles).to(dev)
off = torch.empty(T + 1, dtype=torch.int64, device=dev); v = torch.empty(3 * T, dtype=torch.int32, device=dev)
ctx = _capi.context(dev); L = _capi.lib()
npol, nsl = ctypes.c_int64(), ctypes.c_int64(); st = (ctypes.c_int64 * _capi.NUM_STATS)()
for k in range(3):
    ctx.check(L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off), _capi.ptr(v),
                                    T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st, _capi.stream_ptr(dev)))
torch.cuda.synchronize()
d = ctx.debug()
print("stats", list(st))
print("dbg", {i: int(x) for i, x in enumerate(d) if x})
