"""Stream timeline of one whole-path step (TERMESH_STAMPS=1: globaltimer stamps
when the main / long-item streams reach each point), in microseconds from the
start of label pass A.  Best of 5 graph replays.

    TERMESH_STAMPS=1 python tools/trace_step.py [workload]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = {0: "main: label A start", 1: "main: labels done", 2: "main: chain count done", 3: "main: scans done",
         4: "main: chain emit done (fork)", 5: "main: ruler write done", 6: "main: classify done",
         16: "main: short items start (item list complete)", 7: "main: short items done",
         17: "main: short pinch done", 8: "main: joined the long items", 9: "main: pinch of handed-back items done",
         10: "main: stitch done", 11: "aux: start (after the fork)", 12: "aux: long runs written",
         13: "aux: long items classified", 14: "aux: long-item kernel done", 15: "aux: long pinch done"}


def main():
    import torch
    import bench
    from paper_2204_05438_b200 import _capi
    assert os.environ.get("TERMESH_STAMPS"), "set TERMESH_STAMPS=1"
    w = sys.argv[1] if len(sys.argv) > 1 else "u10m"
    tri = bench.load_mesh(w, 0)
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).cuda()
    tr = torch.from_numpy(tri.triangles).cuda()
    off = torch.empty(T + 1, dtype=torch.int64, device="cuda")
    v = torch.empty(3 * T, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ctx = _capi.context()
    P, F = ctypes.c_int64(), ctypes.c_int64()
    st = (ctypes.c_int64 * _capi.NUM_STATS)()
    best = None
    for _ in range(6):
        flush.zero_()
        ctx.check(_capi.lib().tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                                  _capi.ptr(v), T, 3 * T, ctypes.byref(P), ctypes.byref(F), st,
                                                  _capi.stream_ptr()))
        d = ctx.debug()
        t = {k: (d[100 + k] - d[100]) / 1e3 for k in NAMES if d[100 + k]}
        if best is None or t[10] < best[10]:
            best = t
    print(f"workload {w}: step {best[10]:.1f} us (stamp launches included)")
    for k, us in sorted(best.items(), key=lambda x: x[1]):
        print(f"  {us:8.1f} us  {NAMES[k]}")


if __name__ == "__main__":
    main()
