"""Parity at the 100M-point config (BASELINE.json configs[3]), where the Python
reference cannot run (hours of repair, > 60 GB): the GPU path against the CPU
oracle (oracle/, the reference algorithm in C) on the same triangulation.

  1. labels (max_edge, seed, frontier) of the whole mesh: bit-exact;
  2. the traversal output (raw CSR, reference SEQUENTIAL order): bit-exact;
  3. repair: the seeds of S sampled 1/64 slices, GPU seed-partitioned path
     (tm_ctx_set_partition + tm_resume_pinch under the GLOBAL pinch guard) vs
     the oracle restricted to the same seeds with the same global guard:
     raw CSR bit-exact (distinct polygons repair independently);
  4. the whole-path final CSR hash over 3 graph replays (determinism) and its
     size laws: P' = P + splits, F' = F + 2 splits.

    python tools/check_100m.py [--workload u100m] [--slices 0,21,42,63]
"""
import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2204_05438_b200 as tm  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402
from paper_2204_05438_b200 import distributed as D  # noqa: E402


def h16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="u100m")
    ap.add_argument("--slices", default="0,21,42,63")
    ap.add_argument("--nslices", type=int, default=64)
    a = ap.parse_args()
    out = {"workload": a.workload}
    t0 = time.time()
    tri = bench.load_mesh(a.workload, 0)
    n, T = tri.n_vertices, tri.n_triangles
    out.update(n=n, T=T, load_s=round(time.time() - t0, 1))
    dev = torch.device("cuda", 0)

    # 1 + 2: labels and traversal, whole mesh
    lab = tm.label_all(tri, check=False)
    ol = oracle.label_all(tri)
    out["labels_equal"] = {k: bool(np.array_equal(getattr(lab, k), getattr(ol, k)))
                           for k in ("max_edge", "seed", "frontier")}
    m0 = tm.build_polygon_mesh(tri, lab)
    go, gv = m0.csr()
    oo, ov = oracle.build_polygon_mesh(tri, ol)
    out["traversal_equal"] = bool(np.array_equal(go, oo) and np.array_equal(gv, ov))
    out["polygons_after_traversal"] = int(go.size - 1)
    P0, F0 = int(go.size - 1), int(go[-1])
    del go, gv, oo, ov
    print({k: out[k] for k in ("labels_equal", "traversal_equal")}, flush=True)
    # whole-mesh repair (phase API) for the global guard and the stats
    info = {}
    fin = tm.repair_all(tri, lab, m0, stats_out=info)
    fo, fv = fin.csr()
    out["stats"] = {k: info[k] for k in ("rounds", "splits", "initial_tips", "unrepaired", "pinch_extra")}
    out["size_laws"] = bool(fo.size - 1 == P0 + info["splits"] and int(fo[-1]) == F0 + 2 * info["splits"])
    out["final_phase_api"] = {"off": h16(fo), "verts": h16(fv)}
    extra = info["pinch_extra"]
    del lab, m0, fin, fo, fv, ol
    torch.cuda.empty_cache()

    # 4: whole path (graph) replays
    xy = torch.from_numpy(tri.vertices).to(dev)
    tr = torch.from_numpy(tri.triangles).to(dev)
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    v = torch.empty(3 * T, dtype=torch.int32, device=dev)
    ctx = _capi.context(dev)
    L = _capi.lib()
    hashes = []
    for _ in range(3):
        npol, nsl = ctypes.c_int64(), ctypes.c_int64()
        st = (ctypes.c_int64 * _capi.NUM_STATS)()
        ctx.check(L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                        _capi.ptr(v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), st,
                                        _capi.stream_ptr(dev)))
        P, F = npol.value, nsl.value
        hashes.append((h16(off[: P + 1].cpu().numpy()), h16(v[:F].cpu().numpy().astype(np.int64))))
    out["whole_path_hashes"] = hashes[0]
    out["whole_path_deterministic"] = len(set(hashes)) == 1
    out["whole_path_equals_phase_api"] = hashes[0] == (out["final_phase_api"]["off"], out["final_phase_api"]["verts"])
    print({k: out[k] for k in ("stats", "size_laws", "whole_path_deterministic", "whole_path_equals_phase_api")},
          flush=True)

    # 3: sampled seed slices, GPU partition (global guard) vs oracle slice
    res = []
    S = a.nslices
    olab = oracle.label_all(tri)
    for k in [int(x) for x in a.slices.split(",")]:
        b, e = k * T // S, (k + 1) * T // S
        t1 = time.time()
        _, _, p, f, st = D.run_partition(xy, tr, n, T, b, e, ctx=ctx, off=off, verts=v)
        if st["pinch_deferred"]:
            p, f, st = D.resume_partition(ctx, off, v, T, extra)
        g_off, g_v = off[: p + 1].cpu().numpy(), v[:f].cpu().numpy().astype(np.int64)
        sd = olab.seed.copy()
        sd[:b] = False
        sd[e:] = False
        sub = oracle.Labels(olab.max_edge, olab.frontier.copy(), sd)
        om0 = oracle.build_polygon_mesh(tri, sub)
        (r_off, r_v), rst = oracle.repair_all(tri, sub, om0, guard_extra=extra)
        res.append({"slice": k, "range": [b, e], "polygons": int(p), "equal": bool(
            np.array_equal(g_off, r_off) and np.array_equal(g_v, r_v)), "oracle_stats": rst,
            "seconds": round(time.time() - t1, 1)})
        print(res[-1], flush=True)
    out["slices"] = res
    out["all_equal"] = bool(all(out["labels_equal"].values()) and out["traversal_equal"] and out["size_laws"] and
                            out["whole_path_deterministic"] and out["whole_path_equals_phase_api"] and
                            all(r["equal"] for r in res))
    out["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
