"""Projected strong scaling of the seed-partitioned path on ONE GPU: each of
the G rank ranges runs as its own context (graph-captured), timed with CUDA
events after warm-up with the L2 flushed; the projected G-GPU step is the
slowest rank (the 32-byte NCCL count all-gather is not included).
--split: seed-partitioned labels too (tools/split_emulation.py): each rank's
label_range + resolve + traversal/repair kernels are measured, the
all-gathers (boundary entries, 14 B/triangle of labels) are modeled at
--nvlink-gbs per rank.  --balance K: K iterations of measured-cost seed-range
rebalancing (distributed.balance_partition; label chunks stay equal), the
best iteration reported as "projected_balanced".

    python tools/partition_scaling.py [--workload u1m] [--steps 10] [--split [--balance 3] [--segments]]
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
ap.add_argument("--balance", type=int, default=0,
                help="--split: iterations of measured-cost seed-range rebalancing (distributed.balance_partition)")
ap.add_argument("--segments", action="store_true", help="--split: per-kernel device times of every rank")
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

    def measure(G, seeds):
        """(per-rank projection rows, seeds used) for the seed ranges `seeds`"""
        split_emulation.run(xy, tr, n, T, G, flush=flush, ctx=ctx, seeds=seeds)  # warm-up: scratch, graphs
        runs = []
        for k in range(max(1, a.steps // 3)):
            seeds_used, _, tt = split_emulation.run(xy, tr, n, T, G, flush=flush, ctx=ctx, seeds=seeds,
                                                    segments=a.segments and k == 0)
            runs.append(tt)
        ranks = []
        nb_all = sum(runs[0][q]["boundary_entries"] for q in range(G))
        for r in range(G):
            med = lambda k: sorted(x[r][k] for x in runs)[len(runs) // 2]  # noqa: E731
            own = D.partition_chunks(T, G)[r]
            recv = 12 * (nb_all - runs[0][r]["boundary_entries"]) + 14 * (T - (own[1] - own[0])) + 8 * G
            xch = (recv / (a.nvlink_gbs * 1e9) * 1e3 + 5 * 0.01) if G > 1 else 0.0  # 5 collectives, ~10 us each
            row = {"label_range_ms": round(med("label_range"), 4), "resolve_ms": round(med("resolve"), 4),
                   "seeds": list(seeds_used[r]), "polygons_ms": round(med("polygons"), 4),
                   "exchange_ms_modeled": round(xch, 4), "boundary_entries": runs[0][r]["boundary_entries"],
                   "step_ms": round(med("label_range") + med("resolve") + med("polygons") + xch, 4)}
            if "segments" in runs[0][r]:
                row["segments"] = runs[0][r]["segments"]
            ranks.append(row)
        step = max(x["step_ms"] for x in ranks)
        return {"rank_ms": [x["step_ms"] for x in ranks], "ranks": ranks, "step_ms": round(step, 4),
                "triangles_per_s": round(T / (step / 1e3), 1)}

    res, bal = {}, {}
    ctx = _capi.Context(0)
    for G in [int(x) for x in a.gpus.split(",")]:
        res[G] = measure(G, None)
        if a.balance and G > 1:
            # measured-cost rebalancing of the seed ranges (the label chunks stay equal):
            # each iteration re-cuts the ranges at equal quantiles of the last measured polygon-phase cost
            seeds = [tuple(x["seeds"]) for x in res[G]["ranks"]]
            hist = []
            best = res[G]
            for it in range(a.balance):
                seeds = D.balance_partition(seeds, [x["polygons_ms"] for x in (hist[-1] if hist else res[G])["ranks"]])
                m = measure(G, seeds)
                hist.append(m)
                if m["step_ms"] < best["step_ms"]:
                    best = m
            bal[G] = dict(best, iterations=[h["step_ms"] for h in hist])
    base = res[min(res)]["step_ms"]
    for G in res:
        res[G]["projected_speedup"] = round(base / res[G]["step_ms"], 3)
    for G in bal:
        bal[G]["projected_speedup"] = round(base / bal[G]["step_ms"], 3)
    out = {"workload": a.workload, "T": T, "mode": "split labels", "nvlink_gbs_modeled": a.nvlink_gbs,
           "projected": res}
    if bal:
        out["projected_balanced"] = bal
    print(json.dumps(out, indent=1))
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
