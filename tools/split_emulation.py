"""Seed-partitioned labels on G logical ranks of ONE GPU (the single-GPU stand-in
for distributed.split_labels).  One context is reused rank after rank (a
100M-point rank needs ~62 GB of scratch); the all-gathers of the boundary
entries and of the label chunks are device copies through whole-mesh arrays,
timed separately from the ranks' kernels (the projection models them as
NVLink transfers).  Returns the ranks' CSR outputs (local offsets, after the
global pinch guard's resume) and each rank's device time per phase.

Used by tests/test_distributed.py (parity) and tools/partition_scaling.py
(--split, projected scaling)."""
import ctypes

import torch

from paper_2204_05438_b200 import _capi
from paper_2204_05438_b200 import distributed as D


def _timed(fn, flush=None):
    if flush is not None:
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


def run(xy, tr, n, T, G, flush=None, ctx=None, seeds=None, segments=False):
    """seeds: the ranks' seed ranges for traversal + repair (default: the label
    chunks; D.balance_partition gives cost-balanced ones -- the label chunks stay
    equal so the all-gathers have one size per rank).  segments: also collect
    each rank's per-kernel device times (a separate profiled run)."""
    dev = xy.device
    L = _capi.lib()
    sp = _capi.stream_ptr(dev)
    parts = D.partition_chunks(T, G)
    seeds = seeds or parts
    own = ctx is None
    ctx = ctx or _capi.Context(dev.index or 0)
    hw = torch.empty(3 * T, dtype=torch.int32, device=dev)  # the label all-gather's result
    sd = torch.empty(T, dtype=torch.uint8, device=dev)
    me = torch.empty(T, dtype=torch.int8, device=dev)
    t = {r: {} for r in range(G)}
    entries = []
    # phase 1: every rank labels its chunk, lists its boundary entries
    for r, (b, e) in enumerate(parts):
        cap = 3 * (e - b) + 1
        keys = torch.empty(cap, dtype=torch.int64, device=dev)
        vals = torch.empty(cap, dtype=torch.int32, device=dev)
        nb = ctypes.c_int64()
        _, t[r]["label_range"] = _timed(lambda: ctx.check(L.tm_label_range(
            ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tr), 64, T, b, e, _capi.ptr(keys), _capi.ptr(vals), cap,
            ctypes.byref(nb), sp)), flush)
        t[r]["boundary_entries"] = nb.value
        entries.append((keys[: nb.value].clone(), vals[: nb.value].clone()))
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 0, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), b, e, sp))
    k_all = torch.cat([k for k, _ in entries])  # all-gather of the boundary entries
    v_all = torch.cat([v for _, v in entries])
    offs = [0]
    for k, _ in entries:
        offs.append(offs[-1] + k.numel())
    # phase 2: every rank pairs its cross-chunk half-edges
    for r, (b, e) in enumerate(parts):
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), b, e, sp))
        _, t[r]["resolve"] = _timed(lambda: ctx.check(L.tm_label_resolve(
            ctx.ptr, _capi.ptr(k_all), _capi.ptr(v_all), k_all.numel(), offs[r], offs[r + 1] - offs[r], sp)), flush)
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 0, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), b, e, sp))
    # phase 3: traversal + repair of each rank's seeds from the whole labels
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    v = torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
    extras = []
    for r, (b, e) in enumerate(seeds):
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), 0, T, sp))
        D.polygons_from_labels(ctx, n, T, b, e, off, v)  # graph capture / warm-up outside the timing
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), 0, T, sp))
        res, t[r]["polygons"] = _timed(lambda: D.polygons_from_labels(ctx, n, T, b, e, off, v), flush)
        extras.append(res[4]["pinch_extra"])
        if segments:
            ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), 0, T, sp))
            ctx.set_profiling(True)
            ctx.segments(reset=True)
            if flush is not None:
                flush.zero_()
            D.polygons_from_labels(ctx, n, T, b, e, off, v)
            torch.cuda.synchronize()
            t[r]["segments"] = {k: round(ms, 4) for k, (ms, c) in ctx.segments(reset=True).items() if c}
            ctx.set_profiling(False)
    total = sum(extras)
    out = []
    for r, (b, e) in enumerate(seeds):  # the outputs, with the global pinch guard's resume
        ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), 0, T, sp))
        o, vv, p, f, st = D.polygons_from_labels(ctx, n, T, b, e, off, v)
        if st["pinch_deferred"]:
            p, f, st = D.resume_partition(ctx, off, v, T, total)
        out.append((off[: p + 1].clone(), v[:f].clone(), p, f, st))
    if own:
        ctx.close()
    return seeds, out, t
