"""Multi-GPU path: replicated mesh, seed-partitioned ranks,
one all-gather of per-rank counts to stitch the global CSR.

CPU (gloo, world_size 2 and 3): the product's partition / exchange / stitch /
gather code (paper_2204_05438_b200.distributed) with each rank's local result
produced by the CPU oracle restricted to the rank's seed range -- the
concatenation must equal the reference's single-process output byte for byte.
GPU: the same partitions run through the C ABI (tm_ctx_set_partition) as
logical ranks on one device (the G-way partitioned path on one
GPU), stitched with the same bases."""
import os

import numpy as np
import pytest

import oracle
from conftest import load_case
from paper_2204_05438_b200 import distributed as D

CASES = ("aniso2k_s1", "clust5k_s0", "sun", "u1k_unit")


def _store_path():
    """A fresh file for a file:// rendezvous (no TCP port to race for)."""
    import tempfile
    fd, path = tempfile.mkstemp(prefix="termesh_pg_")
    os.close(fd)
    os.unlink(path)
    return path


def oracle_partition(tri, b, e, guard_extra=-1):
    """The reference algorithm on the polygons whose seed lies in [b, e), pinch
    guard from `guard_extra` (the global extra visits) or, with -1, from this
    range alone.  Returns (offsets, verts, tip-phase extra visits)."""
    lab = oracle.label_all(tri)
    off, v = oracle.build_polygon_mesh(tri, lab)
    seeds = np.flatnonzero(lab.seed)
    i0, i1 = np.searchsorted(seeds, b), np.searchsorted(seeds, e)
    sub = (off[i0:i1 + 1] - off[i0], v[off[i0]:off[i1]])
    (fo, fv), st = oracle.repair_all(tri, lab, sub, guard_extra)
    return fo, fv, st["tip_extra"]


def test_partition_covers_range():
    for T in (0, 1, 7, 1000, 1999963):
        for G in (1, 2, 3, 8):
            parts = D.partition(T, G)
            assert parts[0][0] == 0 and parts[-1][1] == T
            assert all(parts[k][1] == parts[k + 1][0] for k in range(G - 1))
            assert max(e - b for b, e in parts) - min(e - b for b, e in parts) <= 1


def test_exclusive_bases():
    pb, sb = D.exclusive_bases([[3, 10], [0, 0], [2, 7]])
    assert pb.tolist() == [0, 3, 3] and sb.tolist() == [0, 10, 10]


def _worker(rank, world, store, names, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{store}", rank=rank, world_size=world)
    try:
        for name in names:
            tri, g = load_case(name)
            b, e = D.partition(tri.n_triangles, world)[rank]
            fo, fv, extra = oracle_partition(tri, b, e)
            p, f = fo.size - 1, int(fo[-1])
            bufs = {"off": torch.from_numpy(np.zeros(tri.n_triangles + 1, np.int64)),
                    "v": torch.from_numpy(np.zeros(3 * tri.n_triangles + 1, np.int32))}
            bufs["off"][: p + 1] = torch.from_numpy(fo)
            bufs["v"][:f] = torch.from_numpy(fv.astype(np.int32))

            def resume(extra_total, tri=tri, b=b, e=e, bufs=bufs):
                # second phase under the GLOBAL pinch guard (reparation.py:322)
                ro, rv, _ = oracle_partition(tri, b, e, extra_total)
                bufs["off"][: ro.size] = torch.from_numpy(ro)
                bufs["v"][: rv.size] = torch.from_numpy(rv.astype(np.int32))
                return ro.size - 1, int(ro[-1])

            # every rank reports a deferred item, so the two-exchange protocol runs
            shard = D.stitch(bufs["off"], bufs["v"], p, f, pinch=(extra, 1), resume=resume)
            assert shard.counts.shape == (world, 2)
            out = D.gather_csr(shard, 0)
            if rank == 0:
                ok = np.array_equal(out[0], g["final_off"]) and np.array_equal(out[1], g["final_verts"])
                q.put((name, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_stitch_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _store_path(), CASES, q), nprocs=world, join=True,
                       start_method="spawn")
    res = [q.get() for _ in CASES]
    assert all(ok for _, ok in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("cap", [None, "1"])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", CASES)
def test_partitioned_device_path(cuda, name, world, cap, monkeypatch):
    """Logical ranks on one GPU (one context each), the two-phase pinch guard:
    ranks that parked items at their local guard resume under the global one.
    cap = "1" (TERMESH_PINCH_GUARD_CAP) forces the local guard down to one round,
    so every pinch-prone item takes the park -> resume path."""
    import torch
    from paper_2204_05438_b200 import _capi
    if cap:
        monkeypatch.setenv("TERMESH_PINCH_GUARD_CAP", cap)
    tri, g = load_case(name)
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).to(cuda)
    tr = torch.from_numpy(tri.triangles).to(cuda)
    ranks, table = [], []
    for b, e in D.partition(T, world):
        ctx = _capi.Context(cuda.index or 0)
        off, v, p, f, st = D.run_partition(xy, tr, n, T, b, e, ctx=ctx)
        ranks.append([ctx, off, v, p, f])
        table.append([p, f, st["pinch_extra"], st["pinch_deferred"]])
    total = D.global_pinch_extra(table)
    if D.needs_resume(table):
        for r, row in enumerate(table):
            if row[3] > 0:
                ctx, off, v = ranks[r][:3]
                ranks[r][3], ranks[r][4], _ = D.resume_partition(ctx, off, v, T, total)
    if cap and name.startswith("aniso"):
        assert D.needs_resume(table)  # the hook really exercised the resume path
    pb, sb = D.exclusive_bases([[p, f] for _, _, _, p, f in ranks])
    for (_, off, _, p, _), base in zip(ranks, sb):
        D._shift_device(off, p, int(base))
    torch.cuda.synchronize()
    got_off = np.concatenate([off[:p].cpu().numpy() for _, off, _, p, _ in ranks] + [np.array([int(sb[-1]) + ranks[-1][4]])])
    got_v = np.concatenate([v[:f].cpu().numpy() for _, _, v, _, f in ranks])
    assert np.array_equal(got_off, g["final_off"]) and np.array_equal(got_v, g["final_verts"])


@pytest.mark.gpu
def test_library_nccl_comm_single_rank(cuda):
    """The C-ABI communicator (tm_comm_*: NCCL bound at run time) on a
    one-rank group: the counts exchange and the stitch go through it."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{_store_path()}", rank=0, world_size=1)
    try:
        comm = D.Comm()
        send = torch.arange(8, dtype=torch.int64, device=cuda)
        recv = torch.empty(8, dtype=torch.int64, device=cuda)
        comm.allgather(send, recv)
        torch.cuda.synchronize()
        assert torch.equal(send, recv)
        table = D.exchange_counts(5, 17, cuda, pinch=(3, 0), comm=comm)
        assert table.tolist() == [[5, 17, 3, 0]]
        tri, g = load_case("aniso2k_s1")
        xy = torch.from_numpy(tri.vertices).to(cuda)
        tr = torch.from_numpy(tri.triangles).to(cuda)
        off, v, p, f, st = D.run_partition(xy, tr, tri.n_vertices, tri.n_triangles, 0, tri.n_triangles)
        shard = D.stitch(off, v, p, f, pinch=(st["pinch_extra"], st["pinch_deferred"]), comm=comm)
        assert np.array_equal(shard.offsets.cpu().numpy(), g["final_off"])
        assert np.array_equal(shard.verts.cpu().numpy(), g["final_verts"])
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", CASES + ("aniso2k_s2", "clust5k_s3", "grid6x5", "tie5"))
def test_split_labels_logical_ranks(cuda, name, world):
    """Seed-partitioned LABELS (tm_label_range + boundary exchange +
    tm_label_resolve + label all-gather) on logical ranks of one GPU: every
    rank's labels equal the single-GPU ones and the stitched output equals the
    reference golden."""
    import sys
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import split_emulation
    tri, g = load_case(name)
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).to(cuda)
    tr = torch.from_numpy(tri.triangles).to(cuda)
    parts, out, _ = split_emulation.run(xy, tr, n, T, world)
    offs, verts, base = [], [], 0
    for off, v, p, f, st in out:
        offs.append(off[:p].cpu().numpy() + base)
        verts.append(v[:f].cpu().numpy())
        base += f
    got_off = np.concatenate(offs + [np.array([base])])
    got_v = np.concatenate(verts)
    assert np.array_equal(got_off, g["final_off"]) and np.array_equal(got_v, g["final_verts"])


@pytest.mark.gpu
def test_split_labels_single_rank_nccl(cuda):
    """The real split-label path (distributed.split_labels over the library's
    NCCL communicator) on a one-rank group."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{_store_path()}", rank=0, world_size=1)
    try:
        for name in ("aniso2k_s1", "u1k_unit"):
            tri, g = load_case(name)
            csr, stats = D.execute_distributed(tri, split_labels_mode=True)
            assert np.array_equal(csr[0], g["final_off"]) and np.array_equal(csr[1], g["final_verts"])
    finally:
        dist.destroy_process_group()


def test_balance_partition_properties():
    """Measured-cost rebalancing: consecutive ranges covering [0, T), and on a
    cost profile with one expensive point (a repair lineage) the iteration
    converges to ranges of near-equal cost."""
    T, G = 1_000_000, 8
    dens = np.ones(T)
    dens[T - 1000:T - 990] += 2e5 / 10  # a concentrated chain near the end (hull band last)
    cum = np.concatenate([[0.0], np.cumsum(dens)])

    def cost(bounds):
        return [cum[e] - cum[b] for b, e in bounds]

    bounds = D.partition(T, G)
    first = max(cost(bounds))
    for _ in range(6):
        bounds = D.balance_partition(bounds, cost(bounds))
        assert bounds[0][0] == 0 and bounds[-1][1] == T
        assert all(b <= e for b, e in bounds) and all(bounds[r][1] == bounds[r + 1][0] for r in range(G - 1))
    c = cost(bounds)
    floor = max(2e5, cum[-1] / G)  # the chain cannot be split
    assert max(c) <= 1.05 * floor < 0.7 * first
    assert D.balance_partition([(0, 10)], [3.0]) == [(0, 10)]
    assert D.balance_partition([(0, 5), (5, 10)], [0.0, 0.0]) == [(0, 5), (5, 10)]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [3, 8])
@pytest.mark.parametrize("name", CASES)
def test_split_labels_rebalanced_seed_ranges(cuda, name, world):
    """Seed ranges that differ from the label chunks (measured-cost
    rebalancing, here from a skewed synthetic cost) give the same stitched
    output: only the seed ranges decide who repairs what."""
    import sys
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import split_emulation
    tri, g = load_case(name)
    n, T = tri.n_vertices, tri.n_triangles
    xy = torch.from_numpy(tri.vertices).to(cuda)
    tr = torch.from_numpy(tri.triangles).to(cuda)
    seeds = D.balance_partition(D.partition_chunks(T, world), [1.0 + 5.0 * (r == world - 1) for r in range(world)])
    assert seeds != D.partition_chunks(T, world)
    _, out, _ = split_emulation.run(xy, tr, n, T, world, seeds=seeds, segments=True)
    offs, verts, base = [], [], 0
    for off, v, p, f, st in out:
        offs.append(off[:p].cpu().numpy() + base)
        verts.append(v[:f].cpu().numpy())
        base += f
    got_off = np.concatenate(offs + [np.array([base])])
    got_v = np.concatenate(verts)
    assert np.array_equal(got_off, g["final_off"]) and np.array_equal(got_v, g["final_verts"])
