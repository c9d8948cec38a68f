"""Device-resident mesh state (torch tensors as plain device buffers).

DeviceMesh owns, for one Triangulation on one GPU:
    xy        float64[n, 2]      vertex coordinates
    tri_in    int64[3T]          the reference's corner array as uploaded
    tri32     int32[3T]          corners (written by the label pass)
    hw        int32[3T]          packed half-edge words (twin << 1) | frontier
    max_edge  int8[T]            labeling.label_max
    seed      uint8[T]           labeling.label_seeds
    tv        int32[n]           trivertex (lowest incident triangle, or the
                                 caller's own trivertex when given)
Every array-wide computation goes through the C ABI (_capi).
"""

import numpy as np

from . import _capi
from .errors import ValidationError
from .mesh_core import Triangulation, ValidationReport


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _capi.TermeshError("termesh-b200 requires a CUDA device (sm_100a); no CPU fallback exists")
    return torch


def to_device(a, dtype=None, pin=True):
    """numpy -> cuda tensor (via pinned staging for large arrays)."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    if pin and t.numel() * t.element_size() >= (1 << 20):
        t = t.pin_memory()
    return t.to("cuda", non_blocking=True)


class DeviceMesh:
    def __init__(self):
        self.n = self.T = 0

    # ------------------------------------------------------------ creation
    @classmethod
    def upload(cls, tri: Triangulation, check: bool = False, use_trivertex: bool = True) -> "DeviceMesh":
        torch = _torch()
        dm = cls()
        dm.n, dm.T = tri.n_vertices, tri.n_triangles
        dm.xy = to_device(tri.vertices).view(-1, 2)
        dm.tri_in = to_device(tri.triangles)
        dm.label(check=check)
        if use_trivertex and tri.trivertex is not None:
            tv = to_device(tri.trivertex)
            if check:
                dm.check_trivertex(tri.trivertex)
            dm.tv = tv.to(torch.int32)
        return dm

    @classmethod
    def from_device(cls, xy, tri, check: bool = False) -> "DeviceMesh":
        """Wrap device tensors (xy float64[n,2] or [2n], tri int32/int64[3T] or [T,3])."""
        dm = cls()
        dm.xy = xy.reshape(-1, 2)
        dm.tri_in = tri.reshape(-1)
        dm.n, dm.T = dm.xy.shape[0], dm.tri_in.numel() // 3
        dm.label(check=check)
        return dm

    def label(self, check: bool = False):
        """K0+K1+K2 (tm_label): twins, trivertex, max_edge, frontier, seed."""
        torch = _torch()
        T, n = self.T, self.n
        dev = self.xy.device
        bits = 64 if self.tri_in.dtype == torch.int64 else 32
        if bits == 32 and self.tri_in.dtype != torch.int32:
            self.tri_in = self.tri_in.to(torch.int32)
        self.tri32 = self.tri_in if bits == 32 else torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
        self.hw = torch.empty(max(3 * T, 1), dtype=torch.int32, device=dev)
        self.max_edge = torch.empty(max(T, 1), dtype=torch.int8, device=dev)
        self.seed = torch.empty(max(T, 1), dtype=torch.uint8, device=dev)
        self.tv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        ctx = _capi.context(dev)
        rc = _capi.lib().tm_label(ctx.ptr, _capi.ptr(self.xy), n, _capi.ptr(self.tri_in), bits, T, int(check),
                                  _capi.ptr(self.tri32), _capi.ptr(self.hw), _capi.ptr(self.max_edge),
                                  _capi.ptr(self.seed), _capi.ptr(self.tv), _capi.stream_ptr(dev))
        ctx.check(rc, "label")
        return self

    # ------------------------------------------------------------ checks
    def check_neighbors(self, neighbors):
        torch = _torch()
        nb = to_device(np.asarray(neighbors, dtype=np.int64))
        ctx = _capi.context(self.xy.device)
        rc = _capi.lib().tm_check_neighbors(ctx.ptr, _capi.ptr(self.hw), _capi.ptr(nb), 64, self.T,
                                            _capi.stream_ptr(self.xy.device))
        ctx.check(rc, "validate")
        del torch

    def check_trivertex(self, trivertex):
        """mesh_core.validate's trivertex rule (mesh_core.py:268-283): each entry
        is -1 for an unreferenced vertex or a triangle containing the vertex
        (tm_check_trivertex)."""
        tv = to_device(np.asarray(trivertex, dtype=np.int64))
        bits = 64 if self.tri_in.dtype == _torch().int64 else 32
        ctx = _capi.context(self.xy.device)
        rc = _capi.lib().tm_check_trivertex(ctx.ptr, _capi.ptr(self.tri_in), bits, self.T, _capi.ptr(tv), self.n,
                                            _capi.stream_ptr(self.xy.device))
        try:
            ctx.check(rc, "validate")
        except ValidationError as e:
            rep = e.report if e.report is not None else ValidationReport(False, [])
            raise ValidationError("refusing to run on an invalid triangulation: " + rep.summary(), rep) from None

    # ------------------------------------------------------------ host views
    def trivertex_host(self) -> np.ndarray:
        return self.tv[: self.n].to("cpu").numpy().astype(np.int64)

    def unpack(self):
        """(twin int32[3T], frontier bool[3T]) on the device."""
        torch = _torch()
        H = 3 * self.T
        twin = torch.empty(max(H, 1), dtype=torch.int32, device=self.hw.device)
        fr = torch.empty(max(H, 1), dtype=torch.uint8, device=self.hw.device)
        ctx = _capi.context(self.hw.device)
        rc = _capi.lib().tm_unpack_halfedges(ctx.ptr, _capi.ptr(self.hw), self.T, _capi.ptr(twin), _capi.ptr(fr),
                                             _capi.stream_ptr(self.hw.device))
        ctx.check(rc)
        return twin[:H], fr[:H]

    def pack_frontier(self, frontier):
        torch = _torch()
        fr = frontier if hasattr(frontier, "data_ptr") else to_device(np.asarray(frontier, dtype=np.uint8))
        fr = fr.to(torch.uint8).contiguous()
        ctx = _capi.context(self.hw.device)
        rc = _capi.lib().tm_pack_frontier(ctx.ptr, _capi.ptr(self.hw), _capi.ptr(fr), self.T,
                                          _capi.stream_ptr(self.hw.device))
        ctx.check(rc)

    def frontier_host(self) -> np.ndarray:
        _, fr = self.unpack()
        return fr.to("cpu").numpy().astype(bool)

    def twin_host(self) -> np.ndarray:
        tw, _ = self.unpack()
        return tw.to("cpu").numpy()
