"""Projected strong scaling of the seed-partitioned path on ONE GPU: each of
the G rank ranges runs as its own context (graph-captured), timed with CUDA
events after warm-up with the L2 flushed; the projected G-GPU step is the
slowest rank (the 32-byte NCCL count all-gather is not included).
--split: seed-partitioned labels too (tools/split_emulation.py): each rank's
label_range + resolve + traversal/repair kernels are measured, the
all-gathers (boundary entries, 14 B/triangle of labels) are modeled at
--nvlink-gbs per rank.

    python tools/partition_scaling.py [--workload u1m] [--steps 10]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402
from paper_2204_05438_b200 import distributed as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="u1m")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--gpus", default="1,2,4,8")
ap.add_argument("--split", action="store_true",
                help="seed-partitioned labels (tm_label_range + boundary exchange + label all-gather)")
ap.add_argument("--nvlink-gbs", type=float, default=700.0,
                help="modeled all-gather bandwidth per rank (GB/s received) for --split")
a = ap.parse_args()
tri = bench.load_mesh(a.workload, 0)
n, T = tri.n_vertices, tri.n_triangles
dev = torch.device("cuda", 0)
xy = torch.from_numpy(tri.vertices).to(dev)
tr = torch.from_numpy(tri.triangles).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
L = _capi.lib()
if a.split:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import split_emulation  # noqa: E402
    res = {}
    ctx = _capi.Context(0)
    for G in [int(x) for x in a.gpus.split(",")]:
        split_emulation.run(xy, tr, n, T, G, flush=flush, ctx=ctx)  # warm-up: scratch sizes for this G, graphs
        runs = [split_emulation.run(xy, tr, n, T, G, flush=flush, ctx=ctx)[2] for _ in range(max(1, a.steps // 3))]
        ranks = []
        for r in range(G):
            med = lambda k: sorted(x[r][k] for x in runs)[len(runs) // 2]  # noqa: E731
            nb_all = sum(runs[0][q]["boundary_entries"] for q in range(G))
            own = D.partition_chunks(T, G)[r]
            recv = 12 * (nb_all - runs[0][r]["boundary_entries"]) + 14 * (T - (own[1] - own[0])) + 8 * G
            xch = (recv / (a.nvlink_gbs * 1e9) * 1e3 + 5 * 0.01) if G > 1 else 0.0  # 5 collectives, ~10 us each
            ranks.append({"label_range_ms": round(med("label_range"), 4), "resolve_ms": round(med("resolve"), 4),
                          "polygons_ms": round(med("polygons"), 4), "exchange_ms_modeled": round(xch, 4),
                          "boundary_entries": runs[0][r]["boundary_entries"],
                          "step_ms": round(med("label_range") + med("resolve") + med("polygons") + xch, 4)})
        step = max(x["step_ms"] for x in ranks)
        res[G] = {"rank_ms": [x["step_ms"] for x in ranks], "ranks": ranks, "step_ms": round(step, 4),
                  "triangles_per_s": round(T / (step / 1e3), 1)}
    base = res[min(res)]["step_ms"]
    for G in res:
        res[G]["projected_speedup"] = round(base / res[G]["step_ms"], 3)
    print(json.dumps({"workload": a.workload, "T": T, "mode": "split labels", "nvlink_gbs_modeled": a.nvlink_gbs,
                      "projected": res}, indent=1))
    sys.exit(0)

res = {}
off = torch.empty(T + 1, dtype=torch.int64, device=dev)
v = torch.empty(3 * T, dtype=torch.int32, device=dev)
for G in [int(x) for x in a.gpus.split(",")]:
    per = []
    for b, e in D.partition(T, G):
        ctx = _capi.Context(0)  # one rank's context (its scratch is freed after the rank: 100M fits one at a time)
        ctx.check(L.tm_ctx_set_partition(ctx.ptr, b, e))
        npol, nsl = ctypes.c_int64(), ctypes.c_int64()
        st = (ctypes.c_int64 * _capi.NUM_STATS)()
        sp = _capi.stream_ptr(dev)

        def step():
            ctx.check(L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                            _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st, sp))
        for _ in range(3):
            step()
        ms = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        per.append(sorted(ms)[len(ms) // 2])
        ctx.close()
    res[G] = {"rank_ms": [round(x, 4) for x in per], "step_ms": round(max(per), 4),
              "triangles_per_s": round(T / (max(per) / 1e3), 1)}
base = res[min(res)]["step_ms"]
for G in res:
    res[G]["projected_speedup"] = round(base / res[G]["step_ms"], 3)
print(json.dumps({"workload": a.workload, "T": T, "projected": res}, indent=1))
