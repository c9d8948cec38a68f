"""Barrier-edge tip removal and pinch splitting on the GPU (drop-in for the
reference reparation.py).

repair_all (reparation.py:343-377) calls tm_repair: one device work item per
non-simple polygon replays the reference's rounds on its own pieces (tip
splits as arc copies, pinch trials as re-walks), then a scan-and-stitch
kernel writes the final CSR in the reference's raw order.  labels.frontier is
mutated exactly as the reference mutates it.
"""

import ctypes

from . import _capi
from .backend import SEQUENTIAL, Backend
from .mesh_core import Triangulation
from .traversal import PolygonMesh


def repair_all(tri: Triangulation, labels, mesh: PolygonMesh, backend: Backend = SEQUENTIAL,
               stats_out: dict | None = None) -> PolygonMesh:
    """Split every non-simple polygon until none has a tip, then resolve
    pinches.  stats_out receives rounds, splits, initial_tips, unrepaired
    (reparation.py:372-376) plus nonsimple / tip_splits / pinch_splits /
    work_items."""
    import torch
    # trivertex on the device is the caller's tri.trivertex when it was set at
    # label time, else the lowest incident triangle (compute_trivertex's rule)
    dm = labels.device_mesh(tri)
    T = dm.T
    dev = dm.hw.device
    off_in, v_in = mesh.device_csr()
    P = off_in.numel() - 1
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    verts = torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
    n_polys, n_slots = ctypes.c_int64(), ctypes.c_int64()
    stats = (ctypes.c_int64 * _capi.NUM_STATS)()
    ctx = _capi.context(dev)
    rc = _capi.lib().tm_repair(ctx.ptr, _capi.ptr(dm.tri32), _capi.ptr(dm.hw), _capi.ptr(dm.tv), T,
                               _capi.ptr(off_in), _capi.ptr(v_in), P, _capi.ptr(off), _capi.ptr(verts), T, 3 * T,
                               ctypes.byref(n_polys), ctypes.byref(n_slots), stats, _capi.stream_ptr(dev))
    ctx.check(rc, "reparation")
    labels._refresh_frontier_from_device()
    if stats_out is not None:
        for k, name in enumerate(_capi.STAT_NAMES):
            stats_out[name] = int(stats[k])
        stats_out["tip_extra"] = stats_out["pinch_extra"]  # extra visits of the tip-phase output
    Pn, Fn = n_polys.value, n_slots.value
    return PolygonMesh(count=Pn, offsets=off[: Pn + 1], verts=verts[:Fn])
