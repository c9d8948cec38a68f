"""Repeat the device path on one workload and report the failing steps
(intermittent-failure hunt).  python tools/dbg_walk.py WORKLOAD STEPS"""
import ctypes, hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2204_05438_b200 import _capi
w = sys.argv[1] if len(sys.argv) > 1 else "u10m"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tri = bench.load_mesh(w, 0)
n, T = tri.n_vertices, tri.n_triangles
dev = torch.device("cuda", 0)
xy = torch.from_numpy(tri.vertices).to(dev); tr = torch.from_numpy(tri.triangles).to(dev)
off = torch.empty(T + 1, dtype=torch.int64, device=dev); v = torch.empty(3 * T, dtype=torch.int32, device=dev)
ctx = _capi.context(dev); L = _capi.lib()
npol, nsl = ctypes.c_int64(), ctypes.c_int64(); st = (ctypes.c_int64 * _capi.NUM_STATS)()
sp = _capi.stream_ptr(dev)
import json
GOLD = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                   "hashes.json")))
ref = None
ref_v = ref_off = ref_st = None
fails = 0
import numpy as np
for k in range(steps):
    rc = L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off), _capi.ptr(v), T,
                               3 * T, ctypes.byref(npol), ctypes.byref(nsl), st, sp)
    torch.cuda.synchronize()
    if rc:
        fails += 1
        try:
            ctx.check(rc)
        except Exception as e:  # noqa: BLE001
            print(f"step {k}: rc={rc} {e}", flush=True)
        continue
    bufs = {}
    for wh, (dt, cnt) in {0: (torch.int64, T + 1), 1: (torch.int32, 3 * T), 2: (torch.int32, 3 * T),
                          3: (torch.int32, 3 * T), 4: (torch.uint8, T)}.items():
        t_ = torch.empty(cnt, dtype=dt, device=dev)
        L.tm_ctx_debug_copy(ctx.ptr, wh, _capi.ptr(t_), t_.numel() * t_.element_size())
        bufs[wh] = t_.cpu().numpy()
    P0 = int(bufs[4].astype(bool).sum()); F0 = int(bufs[0][P0])
    bufs[0] = bufs[0][:P0 + 1]; bufs[1] = bufs[1][:F0]; bufs[3] = bufs[3][:F0]
    dbuf = {wh: hashlib.sha256(a.tobytes()).hexdigest()[:12] for wh, a in bufs.items()}
    if k == 0:
        ref_dbuf, ref_bufs = dbuf, bufs
    elif dbuf != ref_dbuf:
        print(f"step {k}: internal buffers differ {dbuf} vs {ref_dbuf}", flush=True)
        sd = np.nonzero(bufs[4] != ref_bufs[4])[0]
        for t in sd[:4].tolist():
            print(f"   seed diff tri {t} (block {t // 256}, lane {t % 256}): {bufs[4][t]} vs {ref_bufs[4][t]}; "
                  f"hw {bufs[2][3*t:3*t+3].tolist()} vs {ref_bufs[2][3*t:3*t+3].tolist()}", flush=True)
            for j in range(3):
                tw = ref_bufs[2][3 * t + j] >> 1
                if tw >= 0 and bufs[2][3 * t + j] != ref_bufs[2][3 * t + j]:
                    tt = tw // 3
                    print(f"     slot {j}: ref twin {tw} (tri {tt}, block {tt // 256}); partner word {bufs[2][tw]} vs {ref_bufs[2][tw]}",
                          flush=True)
        for wh in (0, 1, 3):
            a, b = bufs[wh], ref_bufs[wh]
            if len(a) == len(b):
                d = np.nonzero(a != b)[0]
                if len(d):
                    print(f"   buf {wh}: {len(d)} differ, first at {d[:6].tolist()}: {a[d[:6]].tolist()} vs {b[d[:6]].tolist()}", flush=True)
            else:
                print(f"   buf {wh}: length {len(a)} vs {len(b)}", flush=True)
    vv = v[:nsl.value].cpu().numpy(); oo = off[:npol.value + 1].cpu().numpy()
    gold = GOLD.get(w + "_unit")
    if gold:
        gv = hashlib.sha256(vv.astype(np.int64).tobytes()).hexdigest()[:16]
        print(f"step {k}: golden final_verts {'OK' if gv == gold['final_verts'] else 'MISMATCH'}", flush=True)
    h = hashlib.sha256(vv.tobytes()).hexdigest()[:16]
    if ref is None:
        ref, ref_v, ref_off, ref_st = h, vv, oo, list(st)
    elif h != ref:
        fails += 1
        print(f"step {k}: output hash {h} != {ref}; stats {list(st)} vs {ref_st}; P {len(oo)-1} vs {len(ref_off)-1}",
              flush=True)
        m = min(len(oo), len(ref_off))
        d = np.nonzero(oo[:m] != ref_off[:m])[0]
        i = int(d[0]) - 1 if len(d) else m - 2
        i = max(i, 0)
        print("  first offset diff at polygon", i, "len", oo[i + 1] - oo[i], "ref len", ref_off[i + 1] - ref_off[i],
              "verts", vv[oo[i]:oo[i + 1]][:40].tolist(), "ref", ref_v[ref_off[i]:ref_off[i + 1]][:40].tolist(),
              flush=True)
print(f"{w} env={[k for k in os.environ if k.startswith('TERMESH')]} steps={steps} fails={fails}", flush=True)
