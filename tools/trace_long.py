"""Repair-lineage timeline of the long-item kernel (debug timestamps).

    python tools/trace_long.py            # slowest item + stale/reuse counts, then its rounds
"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


WORKLOAD = os.environ.get("TRACE_WORKLOAD", "u1m")


def run():
    import torch
    import bench
    from paper_2204_05438_b200 import _capi
    tri = bench.load_mesh(WORKLOAD, 0)
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).cuda()
    tr = torch.from_numpy(tri.triangles).cuda()
    off = torch.empty(T + 1, dtype=torch.int64, device="cuda")
    v = torch.empty(3 * T, dtype=torch.int32, device="cuda")
    ctx = _capi.context()
    P, F = ctypes.c_int64(), ctypes.c_int64()
    st = (ctypes.c_int64 * _capi.NUM_STATS)()
    for _ in range(3):
        rc = _capi.lib().tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                             _capi.ptr(v), T, 3 * T, ctypes.byref(P), ctypes.byref(F), st,
                                             _capi.stream_ptr())
        ctx.check(rc)
    return ctx.debug()


if __name__ == "__main__":
    if "--child" not in sys.argv:
        d = run()
        slow = d[60]
        qi, depth, dur = slow & 0xFFFF, (slow >> 16) & 0xFFFF, (slow >> 32) / 10.0
        print(f"slowest long item: qi={qi} depth={depth} {dur:.1f} us; split infos stale={d[61]} reused={d[62]} "
              f"re-walk fallbacks={d[63]}")
        print(f"pinch kernel: slowest item {d[48]} cycles, all items {d[49]} cycles")
        print(f"  pinch splits attempted {d[69]} ({d[68]} cyc), first-repeat scans {d[64]} cyc (max L {d[70]}), "
              f"trials wedge {d[66]} + inner {d[67]} ({d[65]} cyc), piece flags {d[71]} cyc")
        env = dict(os.environ, TERMESH_TRACE_QI=str(qi))
        subprocess.run([sys.executable, __file__, "--child"], env=env, check=True)
    else:
        d = run()
        t0 = d[0]
        print("item L", d[2], "tips", d[3], "precompute us", (d[1] - t0) / 1e3)
        print(f"splits {d[59]}: info {d[56] / max(d[59], 1):.0f} cyc, plan {d[57] / max(d[59], 1):.0f} cyc, "
              f"emit + first tip of pa {d[58] / max(d[59], 1):.0f} cyc per split")
        ns = max(d[59], 1)
        print(f"  plan: cut {d[52] / ns:.0f} cyc, rotations+alloc {d[53] / ns:.0f} cyc, "
              f"mean parent segments {d[55] / ns:.1f}")
        prev = d[1]
        for r in range(1, 48):
            if d[4 + r] == 0:
                break
            print(f"round {r:3d} end {(d[4 + r] - t0) / 1e3:8.1f} us  (+{(d[4 + r] - prev) / 1e3:6.1f})")
            prev = d[4 + r]
