"""Multi-GPU mesh -> polygons: replicated mesh, seed-partitioned.

Every rank holds the whole (read-only) half-edge mesh on its own GPU and
labels all of it -- a boundary walk may leave the rank's triangle range, and
K0-K2 are streaming passes.  Rank r then traverses and repairs only the
polygons whose seed triangle lies in its range

    [r * T // G, (r + 1) * T // G)          (partition(T, G)[r])

(tm_ctx_set_partition: seed selection, the sampled ruler walks, repair and
the stitch are all restricted to that range).  Distinct polygons have
disjoint interiors, so the ranks' frontier promotions never interact
 and no label exchange is needed afterwards.

The exchange step is an all-gather of each rank's (polygon count, slot count,
pinch extra visits, deferred items) -- 32 bytes per rank, NCCL over NVLink on
GPUs, gloo in the CPU tests.  The pinch pass's round guard is global
(reparation.py:322); a rank that parked items at its local guard finishes them
under the global one (tm_resume_pinch) and the counts go round once more.
Its exclusive prefix gives every rank its global polygon / slot base; shifting
the local CSR offsets by the slot base (tm_shift_offsets) stitches the global
CSR, whose rank-ordered concatenation is exactly the single-GPU output
(ascending seed order = the reference's raw order).  The CSR
can stay sharded (ShardedCSR) or be gathered to one rank (gather_csr).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np


def partition(T: int, world: int) -> list[tuple[int, int]]:
    """Consecutive seed-triangle ranges, one per rank, covering [0, T)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    return [(r * T // world, (r + 1) * T // world) for r in range(world)]


def balance_partition(bounds, rank_cost, damping: float = 1.0) -> list[tuple[int, int]]:
    """Cost-balanced consecutive seed ranges for the next call on the same mesh.

    bounds: the ranges just used (consecutive, covering [0, T)); rank_cost: the
    cost each rank measured for its range (device ms of its traversal + repair).
    Each range's cost is taken as spread evenly over its triangles; the new
    boundaries cut the resulting piecewise-linear cumulative cost into G equal
    parts (damping < 1 moves each boundary only part of the way).  Repeated
    calls converge onto the measured cost profile -- e.g. the rank holding the
    hull-sliver repair lineage (one dependent chain) ends up with a narrow
    range.  Any consecutive ranges give the single-GPU output (the
    rank-ordered concatenation is the ascending seed order), so balancing
    never changes the result, only who does which seeds."""
    G = len(bounds)
    if G != len(rank_cost) or G == 0:
        raise ValueError("one cost per range")
    T = bounds[-1][1]
    edges = np.array([b for b, _ in bounds] + [T], dtype=np.float64)
    cost = np.maximum(np.asarray(rank_cost, dtype=np.float64), 0.0)
    if G == 1 or T == 0 or cost.sum() <= 0:
        return [tuple(map(int, x)) for x in bounds]
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    targets = cum[-1] * np.arange(1, G) / G
    cuts = np.interp(targets, cum, edges)  # inverse of the piecewise-linear cumulative cost
    cuts = edges[1:-1] + damping * (cuts - edges[1:-1])
    c = np.round(cuts).astype(np.int64)
    c = np.clip(c, 0, T)
    c = np.maximum.accumulate(c)  # monotone
    out = [0] + c.tolist() + [T]
    return [(int(out[r]), int(out[r + 1])) for r in range(G)]


def exclusive_bases(counts) -> tuple[np.ndarray, np.ndarray]:
    """counts[r] = (polygons, slots) of rank r -> (polygon base, slot base) per rank."""
    c = np.asarray(counts, dtype=np.int64).reshape(-1, 2)
    pb = np.concatenate([[0], np.cumsum(c[:, 0])[:-1]]).astype(np.int64)
    sb = np.concatenate([[0], np.cumsum(c[:, 1])[:-1]]).astype(np.int64)
    return pb, sb


class Comm:
    """The library's own NCCL communicator for this rank (tm_comm_init, C ABI):
    rank 0's unique id goes round once through torch.distributed, then every
    exchange of the path is a tm_comm_allgather on the device stream."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        from . import _capi
        L = _capi.lib()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = ctypes.create_string_buffer(L.tm_comm_id_bytes())
        if self.rank == 0 and L.tm_comm_unique_id(uid) != 0:
            raise _capi.TermeshError(L.tm_comm_last_error().decode())
        obj = [uid.raw]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.device = torch.cuda.current_device()
        p = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(obj[0], len(obj[0]))
        if L.tm_comm_init(ctypes.byref(p), self.rank, self.world, idbuf, self.device) != 0:
            raise _capi.TermeshError(L.tm_comm_last_error().decode())
        self.ptr = p

    def allgather(self, send, recv):
        """recv (device, world x send.nbytes) <- every rank's send (device)."""
        from . import _capi
        L = _capi.lib()
        rc = L.tm_comm_allgather(self.ptr, _capi.ptr(send), _capi.ptr(recv), send.numel() * send.element_size(),
                                 _capi.stream_ptr(send.device))
        if rc != 0:
            raise _capi.TermeshError(L.tm_comm_last_error().decode())

    def close(self):
        if self.ptr:
            from . import _capi
            _capi.lib().tm_comm_destroy(self.ptr)
            self.ptr = None


def exchange_counts(n_polys: int, n_slots: int, device, group=None, pinch=(0, 0), comm: Comm | None = None) -> np.ndarray:
    """All-gather (polygons, slots, pinch extra visits, pinch-deferred items) of
    every rank: int64[world, 4] on every rank (32 bytes per rank) -- through the
    library's NCCL communicator when one is given, else torch.distributed
    (gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    if comm is not None:
        dev = torch.device("cuda", comm.device)
        mine = torch.tensor([n_polys, n_slots, int(pinch[0]), int(pinch[1])], dtype=torch.int64, device=dev)
        allc = torch.empty(comm.world * 4, dtype=torch.int64, device=dev)
        comm.allgather(mine, allc)
        return allc.view(comm.world, 4).cpu().numpy()
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        device = torch.device("cuda", torch.cuda.current_device())
    mine = torch.tensor([n_polys, n_slots, int(pinch[0]), int(pinch[1])], dtype=torch.int64, device=device)
    allc = torch.empty(world * 4, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allc, mine, group=group)
    return allc.view(world, 4).cpu().numpy()


def global_pinch_extra(table) -> int:
    """The pinch guard's extra-visit count of the whole mesh (reparation.py:322:
    extra_vertex_visits of the tip-phase output): the sum of every rank's share.
    table rows: (polygons, slots, extra, deferred)."""
    return int(np.asarray(table, dtype=np.int64).reshape(-1, 4)[:, 2].sum())


def needs_resume(table) -> bool:
    """Some rank parked items at its local pinch guard (TM_STAT_PINCH_DEFERRED):
    those ranks resume under the global guard and the counts are exchanged again."""
    return bool((np.asarray(table, dtype=np.int64).reshape(-1, 4)[:, 3] > 0).any())


@dataclass
class ShardedCSR:
    """This rank's slice of the global polygon CSR.  offsets are GLOBAL slot
    offsets (already shifted): polygon poly_base + i of the global mesh is
    verts[offsets[i] - offsets[0] : offsets[i + 1] - offsets[0]]."""
    offsets: object     # int64[P_r + 1] (device tensor)
    verts: object       # int32[F_r] (device tensor)
    poly_base: int
    slot_base: int
    counts: np.ndarray  # int64[world, 2]

    @property
    def n_polys(self) -> int:
        return int(self.offsets.numel() - 1)


def stitch(local_off, local_verts, n_polys: int, n_slots: int, group=None, shift=None, pinch=(0, 0),
           resume=None, comm: Comm | None = None) -> ShardedCSR:
    """Exchange counts and place this rank's CSR at its global base.

    pinch = this rank's (TM_STAT_PINCH_EXTRA, TM_STAT_PINCH_DEFERRED).  The pinch
    guard is global (reparation.py:322), so a rank that parked items at its local
    guard must finish them under the global one before its counts are final:
    `resume(extra_total) -> (n_polys, n_slots)` does that (tm_resume_pinch on the
    device) and a second all-gather publishes the final counts.  Without deferred
    items anywhere (the usual case) the first exchange is the only one.
    `shift` adds the slot base to the offsets in place (default: the C ABI kernel
    on a CUDA tensor, a plain add on CPU tensors).  comm: the library's NCCL
    communicator (Comm) for the exchange, else torch.distributed."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = local_off.device if local_off.is_cuda else "cpu"
    table = exchange_counts(n_polys, n_slots, dev, group, pinch, comm)
    if needs_resume(table):
        if int(pinch[1]) > 0:
            if resume is None:
                from .errors import StructuralError
                raise StructuralError("items parked at the local pinch guard and no resume step given",
                                      phase="reparation")
            n_polys, n_slots = resume(global_pinch_extra(table))
        table = exchange_counts(n_polys, n_slots, dev, group, (int(pinch[0]), 0), comm)
    counts = table[:, :2]
    pb, sb = exclusive_bases(counts)
    off = local_off[: n_polys + 1]
    if shift is None:
        shift = _shift_device if off.is_cuda else _shift_host
    shift(off, n_polys, int(sb[rank]))
    return ShardedCSR(off, local_verts[:n_slots], int(pb[rank]), int(sb[rank]), counts)


def device_resume(ctx, off, verts, T: int, stats=None):
    """resume callable for stitch(): tm_resume_pinch on `ctx`'s last whole-path
    call (device output buffers off / verts), stats updated in place."""
    from . import _capi

    def run(extra_total: int):
        npol, nsl = ctypes.c_int64(), ctypes.c_int64()
        st = stats if stats is not None else (ctypes.c_int64 * _capi.NUM_STATS)()
        rc = _capi.lib().tm_resume_pinch(ctx.ptr, int(extra_total), _capi.ptr(off), _capi.ptr(verts), T, 3 * T,
                                         ctypes.byref(npol), ctypes.byref(nsl), st,
                                         _capi.stream_ptr(off.device) if off.is_cuda else None)
        ctx.check(rc, "reparation")
        return npol.value, nsl.value
    return run


def _shift_host(off, n_polys, delta):
    off += delta


def _shift_device(off, n_polys, delta):
    from . import _capi
    rc = _capi.lib().tm_shift_offsets(_capi.ptr(off), n_polys, delta, _capi.stream_ptr(off.device))
    if rc != 0:
        raise _capi.TermeshError(f"tm_shift_offsets failed with status {rc}")


def gather_csr(shard: ShardedCSR, dst: int = 0, group=None):
    """Global CSR (numpy offsets int64[P+1], verts int32[F]) on rank `dst`,
    None elsewhere.  Padded all-gather, so it works on NCCL and gloo alike."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    counts = shard.counts
    maxp, maxf = int(counts[:, 0].max()), int(counts[:, 1].max())
    dev = shard.offsets.device
    po = torch.zeros(maxp + 1, dtype=torch.int64, device=dev)
    pv = torch.zeros(max(maxf, 1), dtype=torch.int32, device=dev)
    po[: shard.n_polys + 1] = shard.offsets
    pv[: shard.verts.numel()] = shard.verts
    go = [torch.empty_like(po) for _ in range(world)]
    gv = [torch.empty_like(pv) for _ in range(world)]
    dist.all_gather(go, po, group=group)
    dist.all_gather(gv, pv, group=group)
    if rank != dst:
        return None
    offs, verts = [], []
    for r in range(world):
        p, f = int(counts[r, 0]), int(counts[r, 1])
        offs.append(go[r][:p].cpu().numpy())
        verts.append(gv[r][:f].cpu().numpy())
    total = int(counts[:, 1].sum())
    return (np.concatenate(offs + [np.array([total], dtype=np.int64)]).astype(np.int64),
            np.concatenate(verts).astype(np.int32) if verts else np.zeros(0, np.int32))


def run_partition(xy, tri, n: int, T: int, t_begin: int, t_end: int, ctx=None, off=None, verts=None):
    """Device path of one rank: the whole pipeline restricted to the seeds in
    [t_begin, t_end).  xy float64 / tri int64 device tensors.  Returns
    (offsets, verts, n_polys, n_slots, stats) with LOCAL offsets (from 0)."""
    import torch
    from . import _capi
    dev = xy.device
    ctx = ctx or _capi.context(dev)
    off = off if off is not None else torch.empty(T + 1, dtype=torch.int64, device=dev)
    verts = verts if verts is not None else torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
    L = _capi.lib()
    ctx.check(L.tm_ctx_set_partition(ctx.ptr, t_begin, t_end))
    npol, nsl = ctypes.c_int64(), ctypes.c_int64()
    stats = (ctypes.c_int64 * _capi.NUM_STATS)()
    try:
        rc = L.tm_mesh_to_polygons(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tri), 64 if tri.dtype == torch.int64 else 32,
                                   T, 0, _capi.ptr(off), _capi.ptr(verts), T, 3 * T, ctypes.byref(npol),
                                   ctypes.byref(nsl), stats, _capi.stream_ptr(dev))
        ctx.check(rc, "traversal")
    finally:
        L.tm_ctx_set_partition(ctx.ptr, 0, -1)
    return off, verts, npol.value, nsl.value, dict(zip(_capi.STAT_NAMES, list(stats)))


def resume_partition(ctx, off, verts, T: int, extra_total: int):
    """Second phase of a partition run whose stats report pinch_deferred > 0:
    tm_resume_pinch under the global guard.  Returns (n_polys, n_slots, stats)."""
    from . import _capi
    stats = (ctypes.c_int64 * _capi.NUM_STATS)()
    p, f = device_resume(ctx, off, verts, T, stats)(extra_total)
    return p, f, dict(zip(_capi.STAT_NAMES, list(stats)))


def partition_chunks(T: int, world: int) -> list[tuple[int, int]]:
    """Equal chunks of ceil(T / world) triangles (the last one shorter): the
    split-label mode's ranges, so the label all-gathers have one size per rank."""
    C = -(-T // world) if world else 0
    return [(min(r * C, T), min((r + 1) * C, T)) for r in range(world)]


def split_labels(ctx, xy, tri, n: int, T: int, comm: Comm, rank: int, world: int):
    """SURVEY.md 8(e) "each GPU labels its own edge range": this rank labels its
    chunk with a range-local twin table (tm_label_range), the ranks all-gather
    their boundary entries (half-edges whose partner may lie in another chunk),
    tm_label_resolve pairs this chunk's cross-chunk half-edges, and an in-place
    all-gather of the packed half-edge words, seeds and longest edges (14 B per
    triangle) gives every rank the labels of the whole mesh in its context."""
    import torch
    from . import _capi
    L = _capi.lib()
    dev = xy.device
    sp = _capi.stream_ptr(dev)
    C = -(-T // world)
    b, e = partition_chunks(T, world)[rank]
    cap = 3 * (e - b) + 1
    keys = torch.empty(cap, dtype=torch.int64, device=dev)
    vals = torch.empty(cap, dtype=torch.int32, device=dev)
    nb = ctypes.c_int64()
    ctx.check(L.tm_label_range(ctx.ptr, _capi.ptr(xy), n, _capi.ptr(tri), 64 if tri.dtype == torch.int64 else 32, T,
                               b, e, _capi.ptr(keys), _capi.ptr(vals), cap, ctypes.byref(nb), sp), "label")
    cnt = torch.tensor([nb.value], dtype=torch.int64, device=dev)
    cnts = torch.empty(world, dtype=torch.int64, device=dev)
    comm.allgather(cnt, cnts)
    counts = cnts.cpu().tolist()
    maxc = max(1, max(counts))
    kp = torch.full((maxc,), -1, dtype=torch.int64, device=dev)  # padding key ~0
    vp = torch.full((maxc,), -1, dtype=torch.int32, device=dev)
    kp[: nb.value] = keys[: nb.value]
    vp[: nb.value] = vals[: nb.value]
    k_all = torch.empty(world * maxc, dtype=torch.int64, device=dev)
    v_all = torch.empty(world * maxc, dtype=torch.int32, device=dev)
    comm.allgather(kp, k_all)
    comm.allgather(vp, v_all)
    ctx.check(L.tm_label_resolve(ctx.ptr, _capi.ptr(k_all), _capi.ptr(v_all), world * maxc, rank * maxc, nb.value,
                                 sp), "label")
    hw = torch.empty(3 * world * C, dtype=torch.int32, device=dev)
    sd = torch.empty(world * C, dtype=torch.uint8, device=dev)
    me = torch.empty(world * C, dtype=torch.int8, device=dev)
    ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 0, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), b, e, sp))
    comm.allgather(hw[3 * rank * C: 3 * (rank + 1) * C], hw)  # in place: rank r's chunk at r * C
    comm.allgather(sd[rank * C: (rank + 1) * C], sd)
    comm.allgather(me[rank * C: (rank + 1) * C], me)
    ctx.check(L.tm_ctx_copy_labels(ctx.ptr, 1, _capi.ptr(hw), _capi.ptr(sd), _capi.ptr(me), 0, T, sp))
    return b, e


def polygons_from_labels(ctx, n: int, T: int, t_begin: int, t_end: int, off=None, verts=None):
    """Traversal, repair and stitch of the seeds in [t_begin, t_end) from the
    labels already in the context (tm_polygons_from_labels).  Returns
    (offsets, verts, n_polys, n_slots, stats) with LOCAL offsets."""
    import torch
    from . import _capi
    dev = torch.device("cuda", ctx.device_index)
    off = off if off is not None else torch.empty(T + 1, dtype=torch.int64, device=dev)
    verts = verts if verts is not None else torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
    L = _capi.lib()
    ctx.check(L.tm_ctx_set_partition(ctx.ptr, t_begin, t_end))
    npol, nsl = ctypes.c_int64(), ctypes.c_int64()
    stats = (ctypes.c_int64 * _capi.NUM_STATS)()
    try:
        ctx.check(L.tm_polygons_from_labels(ctx.ptr, n, T, _capi.ptr(off), _capi.ptr(verts), T, 3 * T,
                                            ctypes.byref(npol), ctypes.byref(nsl), stats, _capi.stream_ptr(dev)),
                  "traversal")
    finally:
        L.tm_ctx_set_partition(ctx.ptr, 0, -1)
    return off, verts, npol.value, nsl.value, dict(zip(_capi.STAT_NAMES, list(stats)))


def execute_distributed(tri, group=None, gather: bool = True, comm: Comm | None = None, split_labels_mode=False,
                        seed_ranges=None):
    """Drop-in multi-GPU execute: every rank passes the same Triangulation; the
    global final CSR comes back on rank 0 (gather=True) or as shards.
    seed_ranges: consecutive per-rank seed ranges covering [0, T) (e.g. from
    balance_partition after a previous call on the same mesh); default equal."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n, T = tri.n_vertices, tri.n_triangles
    dev = torch.device("cuda", torch.cuda.current_device())
    xy = torch.from_numpy(np.ascontiguousarray(tri.vertices)).to(dev)
    tr = torch.from_numpy(np.ascontiguousarray(tri.triangles)).to(dev)
    from . import _capi
    ctx = _capi.context(dev)
    if comm is None and (split_labels_mode or dist.get_backend(group) == "nccl"):
        comm = Comm(group)  # the library's own communicator for the exchange
    if seed_ranges is not None and (len(seed_ranges) != world or seed_ranges[0][0] != 0 or seed_ranges[-1][1] != T
                                    or any(seed_ranges[r][1] != seed_ranges[r + 1][0] for r in range(world - 1))):
        raise ValueError("seed_ranges must be consecutive ranges covering [0, T), one per rank")
    if split_labels_mode:
        b, e = split_labels(ctx, xy, tr, n, T, comm, rank, world)
        if seed_ranges is not None:
            b, e = seed_ranges[rank]
        off, verts, p, f, stats = polygons_from_labels(ctx, n, T, b, e)
    else:
        b, e = partition(T, world)[rank] if seed_ranges is None else seed_ranges[rank]
        off, verts, p, f, stats = run_partition(xy, tr, n, T, b, e, ctx=ctx)
    shard = stitch(off, verts, p, f, group, pinch=(stats["pinch_extra"], stats["pinch_deferred"]),
                   resume=device_resume(ctx, off, verts, T), comm=comm)
    if not gather:
        return shard, stats
    return gather_csr(shard, 0, group), stats
