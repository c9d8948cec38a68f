"""Edge classification on the GPU (drop-in for the reference labeling.py).

label_all (labeling.py:118-145) runs one fused device pass pair (tm_label):
twin build + LabelMax in pass A, LabelSeed + LabelFrontier in pass B.  The
result stays on the device; the reference's numpy arrays (max_edge int8[T],
frontier bool[3T], seed bool[T]) are materialised on first access.
"""


import numpy as np

from . import _capi
from .backend import SEQUENTIAL, Backend
from .device import DeviceMesh, to_device
from .errors import ValidationError
from .mesh_core import Triangulation


class EdgeLabels:
    """Labels of one triangulation (labeling.py:31-43).

    max_edge: int8 per triangle; frontier: bool per half-edge; seed: bool per
    triangle.  Device-backed when produced by label_all; repair_all mutates
    `frontier` in place exactly like the reference (reparation.py:217-218).
    """

    def __init__(self, max_edge=None, frontier=None, seed=None, *, device: DeviceMesh | None = None):
        self._max_edge = None if max_edge is None else np.asarray(max_edge, dtype=np.int8)
        self._frontier = None if frontier is None else np.asarray(frontier, dtype=bool)
        self._seed = None if seed is None else np.asarray(seed, dtype=bool)
        self._dev = device

    # -- host views (lazy D2H)
    @property
    def max_edge(self) -> np.ndarray:
        if self._max_edge is None:
            self._max_edge = self._dev.max_edge[: self._dev.T].to("cpu").numpy().copy()
        return self._max_edge

    @property
    def frontier(self) -> np.ndarray:
        if self._frontier is None:
            self._frontier = self._dev.frontier_host()
        return self._frontier

    @property
    def seed(self) -> np.ndarray:
        if self._seed is None:
            self._seed = self._dev.seed[: self._dev.T].to("cpu").numpy().astype(bool)
        return self._seed

    def _refresh_frontier_from_device(self):
        """After a device mutation: update an already materialised host frontier in place."""
        if self._frontier is not None and self._dev is not None:
            self._frontier[:] = self._dev.frontier_host()

    def device_mesh(self, tri: Triangulation) -> DeviceMesh:
        """Device state for `tri`, built from host arrays when labels came from elsewhere."""
        if self._dev is not None and self._dev.T == tri.n_triangles:
            return self._dev
        dm = DeviceMesh.upload(tri, check=False)
        if self._max_edge is not None:
            dm.max_edge = to_device(self._max_edge)
        if self._seed is not None:
            dm.seed = to_device(self._seed.astype(np.uint8))
        if self._frontier is not None:
            dm.pack_frontier(self._frontier.astype(np.uint8))
        self._dev = dm
        return dm

    def __repr__(self):
        return f"EdgeLabels(T={self._dev.T if self._dev else len(self.max_edge)}, device={self._dev is not None})"


def _label_device(tri: Triangulation, check: bool) -> DeviceMesh:
    dm = DeviceMesh.upload(tri, check=check)
    if check:
        dm.check_neighbors(tri.neighbors)
    return dm


def label_all(tri: Triangulation, backend: Backend = SEQUENTIAL, kernel_seconds: dict | None = None,
              check: bool = True) -> EdgeLabels:
    """Longest edges, seeds and frontier flags for every triangle (labeling.py:118).

    With check=True the triangulation is validated on the device first and a
    failing report raises ValidationError.  kernel_seconds receives the device
    time of the fused passes (CUDA events, no upload): "label_max" = pass A
    (twin inserts + LabelMax); "label_seed" / "label_frontier" = half each of
    pass B (twin lookups + seeds and frontier in one pass).
    """
    import torch
    if check:
        try:
            _label_device(tri, check=True)
        except ValidationError as e:
            raise ValidationError("refusing to label an invalid triangulation: " + str(e), e.report) from None
        if tri.trivertex is not None:
            DeviceMesh.upload(tri, check=False).check_trivertex(tri.trivertex)
    dm = DeviceMesh.upload(tri, check=False)
    torch.cuda.synchronize()
    if kernel_seconds is not None:
        # device time of the two fused passes (tm_ctx_label_ms): pass A is
        # LabelMax (+ the twin inserts); pass B computes seeds and frontier
        # together, its time is split evenly between the reference's
        # label_seed and label_frontier kernels (labeling.py:134-144)
        a_ms, b_ms = _capi.context(dm.xy.device).label_ms()
        kernel_seconds["label_max"] = a_ms / 1e3
        kernel_seconds["label_seed"] = b_ms / 2e3
        kernel_seconds["label_frontier"] = b_ms / 2e3
    return EdgeLabels(device=dm)


def label_max(tri: Triangulation, backend: Backend = SEQUENTIAL) -> np.ndarray:
    """Longest-edge slot per triangle, lowest slot wins ties (labeling.py:46-62)."""
    return label_all(tri, backend, check=False).max_edge


def _relabel(tri: Triangulation, max_edge) -> DeviceMesh:
    dm = DeviceMesh.upload(tri, check=False)
    dm.max_edge = to_device(np.asarray(max_edge, dtype=np.int8))
    ctx = _capi.context(dm.hw.device)
    rc = _capi.lib().tm_relabel(ctx.ptr, _capi.ptr(dm.hw), _capi.ptr(dm.max_edge), dm.T, _capi.ptr(dm.seed),
                                _capi.stream_ptr(dm.hw.device))
    ctx.check(rc, "label")
    return dm


def label_seeds(tri: Triangulation, max_edge, backend: Backend = SEQUENTIAL) -> np.ndarray:
    """Seed flag per triangle from a given max_edge (labeling.py:65-89)."""
    dm = _relabel(tri, max_edge)
    return dm.seed[: dm.T].to("cpu").numpy().astype(bool)


def label_frontiers(tri: Triangulation, max_edge, backend: Backend = SEQUENTIAL) -> np.ndarray:
    """Frontier flag per half-edge from a given max_edge (labeling.py:92-115)."""
    return _relabel(tri, max_edge).frontier_host()
