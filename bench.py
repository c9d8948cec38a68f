"""Benchmark: mesh -> polygons throughput (input triangles/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload u10m]

A step is one pass of the whole hot path -- twin build + labels (K0-K2),
traversal (K3), repair + stitch (K4) -- over one synthetic Delaunay
triangulation.  Default workload: BASELINE.json configs[2], 10M uniform points
in the unit square (scipy Qhull, seed 0; T = 19,999,954 triangles), the config
SURVEY.md 8(d) quotes the roofline on (at 1M the vertex array fits in L2).
--workload u1m | c10m | ... selects another config.  --gpus N without a
torchrun environment re-launches this script under torch.distributed.run with
N ranks (127.0.0.1); under torchrun, WORLD_SIZE wins.

GPU arm (default):
  value  device-resident: inputs (xy f64, triangles i64) already in HBM, CUDA
         events on the launching stream around each step, L2 flushed (256 MiB
         write) between steps outside the events; max over ranks.
  e2e    the one-call C ABI (tm_mesh_to_polygons_host) from pinned host arrays
         in the reference dtypes: H2D of the inputs, the path, D2H of the final
         CSR, all inside the timed region (host wall clock per call).
  roofline  the dominant kernel (largest device-time share) over its
         algorithmic bytes, peak = measured HBM
         copy bandwidth from MEASURED_PEAKS.json.
  cpu_baseline  the CPU oracle port (oracle/, the reference algorithm in C,
         OpenMP label+traversal, sequential repair as the reference's "mixed"
         mode) on the same mesh, rank 0 at N=1 only.
Multi-GPU (torchrun): the mesh is replicated on every rank and
the seeds are partitioned (rank r owns triangles [rT/G, (r+1)T/G)); each step
ends with the exchange -- NCCL all-gather of the per-rank (polygons, slots)
counts and the shift of the local CSR to its global base.  Strong scaling:
value = T / (slowest rank's step time); barrier + max-over-ranks timing.

Parity: the final CSR of the last timed step (gathered to rank 0 when N > 1)
is hashed and compared with the reference's own output for this workload
(tests/golden/hashes.json, produced by the Python reference); the line's
"parity" object says whether it matched.

Reference arm (--impl reference): the reference algorithm's CPU port (oracle/)
on the box's host cores over the same workload, rank 0 only.  Each step is a
bounded sample: labels of the whole mesh (OpenMP), then traversal + repair of
the seeds of one 1/S slice of the triangles (slices rotate across steps);
value = T / (t_label + S * t_slice), i.e. the whole mesh's throughput
extrapolated from the sampled slice.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "u1m": dict(n=1_000_000, gen="uniform", desc="1M uniform random points in the unit square, scipy Delaunay (seed 0)"),
    "u10m": dict(n=10_000_000, gen="uniform", desc="10M uniform random points in the unit square, scipy Delaunay (seed 0)"),
    "u100k": dict(n=100_000, gen="uniform", desc="100k uniform random points in the unit square, scipy Delaunay (seed 0)"),
    "c1m": dict(n=1_000_000, gen="clustered",
                desc="1M points in 64 Gaussian clusters (sigma 0.002) in the unit square, scipy Delaunay (seed 0)"),
    "c10m": dict(n=10_000_000, gen="clustered",
                 desc="10M points in 64 Gaussian clusters (sigma 0.002) in the unit square, scipy Delaunay (seed 0)"),
    # BASELINE.json configs[3]: one Qhull call would take ~1 h and ~150 GB on the
    # host, so the same points go through the tile-parallel exact Delaunay
    # (tools/tiled_delaunay.py: the identical triangle set as Qhull, checked at
    # 300k / 1M / 10M; tile-major triangle order)
    "u100m": dict(n=100_000_000, gen="tiled",
                  desc="100M uniform random points in the unit square, exact Delaunay (tile-parallel Qhull, seed 0)"),
}
METRIC = "triangles/sec end-to-end mesh->polygons"
UNIT = "triangles/s"


def load_mesh(workload, seed):
    from paper_2204_05438_b200 import io_formats as io
    w = WORKLOADS[workload]
    if w["gen"] == "clustered":
        return io.cached(f"{workload}_s{seed}_clustered", lambda: io.generate_clustered_delaunay(w["n"], seed=seed))
    if w["gen"] == "tiled":
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import tiled_delaunay
        return io.cached(f"{workload}_s{seed}_tiled", lambda: tiled_delaunay.triangulation(w["n"], seed)[0])
    return io.cached(f"{workload}_s{seed}_unit", lambda: io.generate_random_delaunay(w["n"], (0.0, 0.0, 1.0, 1.0), seed))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_bytes(n, T, F, P, Fp, Pp):
    """Compulsory bytes per segment: every
    array touched once in its device dtype.  R = rulers = seeds + F/8."""
    R = P + F // 8
    return {
        # pass A: tri i64 in, xy gathers, tri32 + max_edge out, 1.5 ascending keys (8 B) into the twin table
        "label_a_tri_pass": 24 * T + 16 * n + 12 * T + 1 * T + 12 * T,
        # pass B: tri32 + max_edge in, 1.5 key probes, packed half-edge words + seeds out
        "label_b_edges": 12 * T + 1 * T + 12 * T + 12 * T + 1 * T,
        "select_seeds": 1 * T + 4 * P,
        "trav_start": 4 * P + 12 * P + 4 * P,
        "trav_rulers": 12 * T + 12 * T + 8 * R,                                 # hw scan + rotations, rnext/rdist
        "trav_chain": 4 * P + 8 * R + 16 * P,
        "trav_scan": 32 * P,
        "trav_write": 4 * P + 8 * R + 24 * R + 12 * T + 4 * F + 4 * F,
        "repair_classify": 8 * P + 4 * F + 4 * P,
        "repair_tips": 0,
        "repair_pinch": 0,
        "repair_stitch": 8 * P + 4 * F + 8 * Pp + 4 * Fp + 48 * P,
    }


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2204_05438_b200 as tm
    from paper_2204_05438_b200 import _capi

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2204_05438_b200 import distributed as D
    tri = load_mesh(args.workload, 0)  # one mesh, replicated on every rank
    n, T = tri.n_vertices, tri.n_triangles
    t_begin, t_end = D.partition(T, world)[rank]  # this rank's seed range
    xy = torch.from_numpy(tri.vertices).to(dev)
    tr = torch.from_numpy(tri.triangles).to(dev)
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    verts = torch.empty(3 * T, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = _capi.context(dev)
    L = _capi.lib()
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    npol, nsl = ctypes.c_int64(), ctypes.c_int64()
    stats = (ctypes.c_int64 * _capi.NUM_STATS)()

    ctx.check(L.tm_ctx_set_partition(ctx.ptr, t_begin, t_end))

    shard = [None]
    comm = D.Comm() if world > 1 else None  # the library's NCCL communicator (tm_comm_*, C ABI)

    split = args.split_labels and world > 1
    if split:  # seed-partitioned labels: chunk ranges, labels exchanged (distributed.split_labels)
        t_begin, t_end = D.partition_chunks(T, world)[rank]
        ctx.check(L.tm_ctx_set_partition(ctx.ptr, t_begin, t_end))

    def step():
        if split:
            D.split_labels(ctx, xy, tr, n, T, comm, rank, world)
            ctx.check(L.tm_polygons_from_labels(ctx.ptr, n, T, _capi.ptr(off), _capi.ptr(verts), T, 3 * T,
                                                ctypes.byref(npol), ctypes.byref(nsl), stats, sp))
        else:
            rc = L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, 0, _capi.ptr(off),
                                       _capi.ptr(verts), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), stats, sp)
            ctx.check(rc)
        if world > 1:  # the exchange step: all-gather counts (NCCL), shift to the global slot base
            shard[0] = D.stitch(off, verts, npol.value, nsl.value, pinch=(stats[8], stats[10]),
                                resume=D.device_resume(ctx, off, verts, T, stats), comm=comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = L.tm_launch_count()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = L.tm_launch_count() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = T / (ms_per_step / 1e3)  # the one mesh's triangles over the slowest rank's time
    P_out, F_out = npol.value, nsl.value
    repair_stats = dict(zip(_capi.STAT_NAMES, list(stats)))
    parity = check_parity(args.workload, off, verts, P_out, F_out, shard[0], world, rank)

    # per-kernel device time (separate profiled pass; not part of `value`)
    ctx.set_profiling(True)
    ctx.segments(reset=True)
    prof_steps = max(3, min(args.steps, 10))
    for _ in range(prof_steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    segs = ctx.segments(reset=True)
    ctx.set_profiling(False)

    # traversal-phase counts for the byte model (this rank's seed range)
    lab = tm.label_all(tri, check=False)
    m0 = tm.build_polygon_mesh(tri, lab)
    P0, F0 = m0.count, int(m0.csr()[0][-1])
    abytes = algorithmic_bytes(n, T, F0, P0, F_out, P_out)
    peak, peak_src = measured_peak()
    kernels = {}
    for name, (ms, cnt) in segs.items():
        if cnt == 0:
            continue
        per = ms / cnt
        b = abytes.get(name, 0)
        kernels[name] = {"ms": round(per, 4), "share": None, "alg_bytes": b,
                         "gbs": round(b / (per / 1e3) / 1e9, 1) if b and per > 0 else None}
    tot = sum(k["ms"] for k in kernels.values()) or 1.0
    for k in kernels.values():
        k["share"] = round(k["ms"] / tot, 4)
    dom = max(kernels, key=lambda k: kernels[k]["ms"]) if kernels else None
    hbm_kernels = [k for k in kernels if kernels[k]["alg_bytes"]]
    dom_hbm = max(hbm_kernels, key=lambda k: kernels[k]["ms"]) if hbm_kernels else None
    d = kernels.get(dom_hbm, {})
    achieved = d.get("gbs") or 0.0
    # DRAM bytes per launch of the roofline kernel from the committed ncu --set full capture
    # (tools/ncu_summary.py -> profiles/ncu_traffic.json), same workload, or null
    traffic, traffic_src = None, None
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[args.workload][dom_hbm]
        traffic, traffic_src = t["dram_bytes"], f"profiles/{t['source']} (ncu, {t['kernel']})"
    except Exception:
        pass
    dram_gbs = round(traffic / (d["ms"] / 1e3) / 1e9, 1) if traffic and d.get("ms") else None
    roofline = {"bound": "hbm", "kernel": dom_hbm, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if peak else None, "traffic": traffic,
                "algorithmic_bytes": d.get("alg_bytes"), "traffic_source": traffic_src,
                # the DRAM bytes the kernel actually moves (random sectors of the gathers) over its time
                "dram_achieved": dram_gbs, "dram_frac": round(dram_gbs / peak, 4) if dram_gbs and peak else None,
                "peak_source": peak_src, "dominant_by_time": dom,
                "note": "dominant HBM kernel; repair_tips is latency-bound (no byte roofline)"}

    # e2e: one C-ABI call from pinned host buffers (reference dtypes)
    h_xy = torch.from_numpy(tri.vertices).pin_memory()
    h_tr = torch.from_numpy(tri.triangles).pin_memory()
    h_off = torch.empty(T + 1, dtype=torch.int64).pin_memory()
    h_v = torch.empty(3 * T, dtype=torch.int32).pin_memory()

    def e2e_step():
        if split:  # host arrays in, the split path, the rank's CSR out
            xy.copy_(h_xy, non_blocking=True)
            tr.copy_(h_tr, non_blocking=True)
            step()
            P, F = shard[0].n_polys, int(shard[0].verts.numel())
            h_off[: P + 1].copy_(shard[0].offsets, non_blocking=True)
            h_v[:F].copy_(shard[0].verts, non_blocking=True)
            torch.cuda.synchronize()
            return
        rc = L.tm_mesh_to_polygons_host(ctx.ptr, _capi.ptr(h_xy), n, _capi.ptr(h_tr), T, 0, _capi.ptr(h_off),
                                        _capi.ptr(h_v), T, 3 * T, ctypes.byref(npol), ctypes.byref(nsl), stats)
        ctx.check(rc)
        if world > 1:
            D.stitch(h_off, h_v, npol.value, nsl.value, pinch=(stats[8], stats[10]),
                     resume=D.device_resume(ctx, h_off, h_v, T, stats), comm=comm)

    for _ in range(args.warmup):
        e2e_step()
    if world > 1:
        dist.barrier()
    e2e_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    e2e_tot = torch.tensor([sum(e2e_s)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_tot.item()) / args.steps * 1e3
    e2e = {"value": round(T / (e2e_ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(e2e_ms, 3),
           "h2d_bytes_per_step": 16 * n + 24 * T, "d2h_bytes_per_step": 8 * (npol.value + 1) + 4 * nsl.value,
           "api": "tm_mesh_to_polygons_host (C ABI, pinned host buffers)"}
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32/f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"], "n_vertices": n,
                   "triangles": T, "seed_range_rank0": [t_begin, t_end], "polygons_rank0": P_out,
                   "polygon_slots_rank0": F_out, "l2": "flushed (256 MiB write) between steps",
                   "parallelism": f"replicated mesh, seeds partitioned x{world}, NCCL all-gather of counts "
                                  f"(tm_comm_allgather)" + (", labels partitioned" if split else "")},
        "e2e": e2e, "roofline": roofline, "kernels": kernels, "repair_stats": repair_stats,
        "gpu_launches": int(launches), "clocks": clk.summary(), "parity": parity,
        "step_ms": {"min": round(min(step_ms), 4), "median": round(statistics.median(step_ms), 4),
                    "max": round(max(step_ms), 4)},
    }
    return out, tri


# reference outputs of the bench workloads (tests/golden/hashes.json, made by the Python reference)
GOLDEN_KEY = {"u100k": "u100k_unit", "u1m": "u1m_unit", "u10m": "u10m_unit", "c10m": "c10m_clustered"}


def _h16(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def check_parity(workload, off, verts, P, F, shard, world, rank):
    """Hash the timed path's final CSR (int64 offsets / int64 vertices, the
    reference dtypes) and compare with the reference's hashes for this input.
    With N > 1 the rank CSRs are gathered to rank 0 first (outside the timing)."""
    from paper_2204_05438_b200 import distributed as D
    if world > 1:
        g = D.gather_csr(shard, 0)
        if rank != 0:
            return None
        o, v = g
    else:
        o = off[: P + 1].cpu().numpy()
        v = verts[:F].cpu().numpy()
    got = {"final_off": _h16(o.astype(np.int64)), "final_verts": _h16(v.astype(np.int64)),
           "final_polygons": int(o.size - 1)}
    ref = {}
    try:
        ref = json.load(open(os.path.join(ROOT, "tests", "golden", "hashes.json"))).get(GOLDEN_KEY.get(workload), {})
    except Exception:
        pass
    if not ref:
        return {**got, "reference": None, "match": None}
    match = all(got[k] == ref.get(k) for k in got)
    return {**got, "reference": f"tests/golden/hashes.json[{GOLDEN_KEY[workload]}]", "match": bool(match)}


def reference_sample(tri, k, slices):
    """One bounded sample of the reference algorithm (CPU port, oracle/): labels
    of the whole mesh, then traversal + repair of the seeds in slice k of S
    equal triangle ranges.  Returns (t_label, t_slice) in seconds."""
    import oracle
    T = tri.n_triangles
    b, e = k * T // slices, (k + 1) * T // slices
    th = host_threads()
    t0 = time.perf_counter()
    lab = oracle.label_all(tri, th)
    t1 = time.perf_counter()
    sd = lab.seed.copy()
    sd[:b] = False
    sd[e:] = False
    sub = oracle.Labels(lab.max_edge, lab.frontier, sd)
    m0 = oracle.build_polygon_mesh(tri, sub, th)
    oracle.repair_all(tri, sub, m0)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def host_threads():
    """Every host thread (torchrun sets OMP_NUM_THREADS=1 per rank; the reference
    arm runs on rank 0 alone and uses the whole host)."""
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def reference_slices(T):
    """Slices per sample so that one step is a few seconds of 16-core CPU work
    (the 10M mesh takes ~1 min per full pass: 16 slices)."""
    return max(1, min(64, -(-T // 1_250_000)))


def cpu_baseline(tri, budget_s=15.0):
    S = reference_slices(tri.n_triangles)
    reference_sample(tri, 0, S)  # warm (page-in)
    runs = []
    t_start = time.perf_counter()
    k = 0
    while not runs or (time.perf_counter() - t_start < budget_s and len(runs) < 8):
        runs.append(reference_sample(tri, k % S, S))
        k += 1
    est = [tl + S * ts for tl, ts in runs]
    s = statistics.mean(est)
    return {"value": round(tri.n_triangles / s, 1), "unit": UNIT, "cores": host_threads(), "kind": "port",
            "sample": f"{len(runs)} sample(s) of the workload mesh (T={tri.n_triangles}): labels of the whole mesh "
                      f"(OpenMP) + traversal and sequential repair of one 1/{S} seed slice each (the reference "
                      f"'mixed' mode); full-mesh time extrapolated as t_label + {S} * t_slice = {s:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    tri = load_mesh(args.workload, 0)
    T = tri.n_triangles
    S = reference_slices(T)
    for k in range(args.warmup):
        reference_sample(tri, k % S, S)
    est = []
    for k in range(args.steps):
        tl, ts = reference_sample(tri, (args.warmup + k) % S, S)
        est.append(tl + S * ts)
    s = statistics.mean(est)
    v = round(T / s, 1)
    sample = (f"per step: labels of the whole mesh (OpenMP) + traversal and sequential repair of the seeds of one "
              f"1/{S} triangle slice (slices rotate); full-mesh time t_label + {S} * t_slice")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(s * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"], "triangles": T,
                       "n_vertices": tri.n_vertices},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def launch_command(argv, nproc, port):
    """torch.distributed.run command that re-launches this script with nproc ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def probe_launch(rank, world):
    """--probe-launch: every rank joins a gloo group and rank 0 reports who joined
    (the CPU test of the self-launch)."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([rank], dtype=torch.int64)
    allr = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, t)
    if rank == 0:
        print(json.dumps({"probe": True, "world": world, "ranks": [int(x.item()) for x in allr]}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="u10m")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-labels", action="store_true",
                    help="N > 1: each rank labels its own triangle chunk (distributed.split_labels)")
    ap.add_argument("--probe-launch", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver may also launch us that way)
        r = subprocess.run(launch_command(sys.argv[1:], args.gpus, _free_port()))
        sys.exit(r.returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.probe_launch:
        probe_launch(rank, world)
        return
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out, tri = run_gpu(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(tri)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
