import ctypes, sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
from conftest import load_case
from paper_2204_05438_b200 import _capi
tri, g = load_case(sys.argv[1] if len(sys.argv) > 1 else 'clust5k_s0')
n, T = tri.n_vertices, tri.n_triangles
dev = torch.device('cuda', 0)
xy = torch.from_numpy(tri.vertices).to(dev); tr = torch.from_numpy(tri.triangles).to(dev)
off = torch.empty(T + 1, dtype=torch.int64, device=dev); v = torch.empty(3 * T, dtype=torch.int32, device=dev)
ctx = _capi.context(dev); L = _capi.lib()
npol, nsl = ctypes.c_int64(), ctypes.c_int64(); st = (ctypes.c_int64 * _capi.NUM_STATS)()
sp = _capi.stream_ptr(dev)
prev = None
for k in range(4):
    rc = L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off), _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st, sp)
    torch.cuda.synchronize()
    hw = torch.empty(3 * T, dtype=torch.int32, device=dev); L.tm_ctx_debug_copy(ctx.ptr, 2, _capi.ptr(hw), 12 * T)
    sd = torch.empty(T, dtype=torch.uint8, device=dev); L.tm_ctx_debug_copy(ctx.ptr, 4, _capi.ptr(sd), T)
    hw = hw.cpu().numpy(); sd = sd.cpu().numpy()
    ok = rc == 0 and np.array_equal(v[:nsl.value].cpu().numpy(), g['final_verts'])
    print('step', k, 'rc', rc, 'ok', ok, 'seeds', int(sd.sum()), flush=True)
    if prev is not None:
        d = np.nonzero(hw != prev[0])[0]
        print('  hw differ', len(d), d[:10].tolist(), hw[d[:10]].tolist(), prev[0][d[:10]].tolist())
        ds = np.nonzero(sd != prev[1])[0]
        print('  seed differ', ds[:10].tolist())
    prev = (hw, sd)
