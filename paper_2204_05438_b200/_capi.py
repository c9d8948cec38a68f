"""ctypes binding of libtermesh_b200.so (include/termesh_b200.h).

The product path has exactly one implementation: the sm_100a kernels behind
this C ABI.  If the library is missing or no CUDA device is visible, every
entry point raises -- there is no CPU fallback.
"""

import atexit
import ctypes
import os
import threading

from .errors import CapacityError, StructuralError, TermeshError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# TERMESH_LIB_VARIANT: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("TERMESH_LIB_VARIANT") or os.path.join(_HERE, "libtermesh_b200.so")

TM_OK, TM_ERR_STRUCTURAL, TM_ERR_VALIDATION, TM_ERR_CAPACITY, TM_ERR_CUDA, TM_ERR_ARGUMENT = range(6)
NUM_KINDS = 16
NUM_STATS = 11
KIND_NAMES = ("index_range", "orientation", "degenerate", "duplicate", "reciprocity", "edge_count",
              "trivertex", "neighbors", "walk", "no_frontier", "no_converge", "split_law", "pool",
              "barrier", "no_internal", "structural")
STAT_NAMES = ("rounds", "splits", "initial_tips", "unrepaired", "nonsimple", "tip_splits",
              "pinch_splits", "work_items", "pinch_extra", "pinch_truncated", "pinch_deferred")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_PI64 = ctypes.POINTER(ctypes.c_int64)

_lib = None
_lock = threading.RLock()
_ctxs = {}
_all_ctxs = []  # every Context ever created (destroyed at exit)


class ExtensionMissing(TermeshError, ImportError):
    """libtermesh_b200.so is not built (run `python -m paper_2204_05438_b200.build`)."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(f"{LIB_PATH} not built; run `python -m paper_2204_05438_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.tm_version.restype = _I
        L.tm_ctx_create.argtypes = [ctypes.POINTER(_P)]
        L.tm_ctx_destroy.argtypes = [_P]
        L.tm_ctx_destroy.restype = None
        L.tm_ctx_last_error.argtypes = [_P]
        L.tm_ctx_last_error.restype = ctypes.c_char_p
        L.tm_ctx_defects.argtypes = [_P, _PI64, _PI64]
        L.tm_ctx_phase_ms.argtypes = [_P, ctypes.POINTER(ctypes.c_double)]
        L.tm_ctx_label_ms.argtypes = [_P, ctypes.POINTER(ctypes.c_double)]
        L.tm_ctx_set_profiling.argtypes = [_P, _I]
        L.tm_ctx_segment_ms.argtypes = [_P, ctypes.POINTER(ctypes.c_double), _PI64, _I, _I]
        L.tm_segment_name.argtypes = [_I]
        L.tm_segment_name.restype = ctypes.c_char_p
        L.tm_launch_count.restype = ctypes.c_int64
        L.tm_ctx_debug.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64), _I]
        L.tm_ctx_debug_copy.argtypes = [_P, _I, _P, ctypes.c_size_t]
        L.tm_ctx_set_partition.argtypes = [_P, _I64, _I64]
        L.tm_shift_offsets.argtypes = [_P, _I64, _I64, _P]
        L.tm_label.argtypes = [_P, _P, _I64, _P, _I, _I64, _I, _P, _P, _P, _P, _P, _P]
        L.tm_relabel.argtypes = [_P, _P, _P, _I64, _P, _P]
        L.tm_check_neighbors.argtypes = [_P, _P, _P, _I, _I64, _P]
        L.tm_unpack_halfedges.argtypes = [_P, _P, _I64, _P, _P, _P]
        L.tm_pack_frontier.argtypes = [_P, _P, _P, _I64, _P]
        L.tm_traverse.argtypes = [_P, _P, _P, _P, _I64, _P, _P, _I64, _I64, _PI64, _PI64, _P]
        L.tm_repair.argtypes = [_P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _I64, _PI64, _PI64, _PI64, _P]
        L.tm_mesh_to_polygons.argtypes = [_P, _P, _I64, _P, _I, _I64, _I, _P, _P, _I64, _I64, _PI64, _PI64,
                                          _PI64, _P]
        L.tm_mesh_to_polygons_host.argtypes = [_P, _P, _I64, _P, _I64, _I, _P, _P, _I64, _I64, _PI64, _PI64,
                                               _PI64]
        L.tm_resume_pinch.argtypes = [_P, _I64, _P, _P, _I64, _I64, _PI64, _PI64, _PI64, _P]
        L.tm_check_trivertex.argtypes = [_P, _P, _I, _I64, _P, _I64, _P]
        L.tm_polygon_stats.argtypes = [_P, _P, _P, _I64, _I64, _P, _P, _P, _PI64, _PI64, _PI64, _P]
        L.tm_polygon_areas.argtypes = [_P, _P, _P, _I64, _P, _P, _P]
        L.tm_canonicalize.argtypes = [_P, _P, _P, _I64, _I64, _P, _P, _P]
        L.tm_delaunay.argtypes = [_P, _P, _I64, _P, _P, _I64, _PI64, _P, _PI64, _PI64, _P]
        L.tm_label_range.argtypes = [_P, _P, _I64, _P, _I, _I64, _I64, _I64, _P, _P, _I64, _PI64, _P]
        L.tm_ctx_label_buffers.argtypes = [_P] + [ctypes.POINTER(_P)] * 4
        L.tm_ctx_copy_labels.argtypes = [_P, _I, _P, _P, _P, _I64, _I64, _P]
        L.tm_ctx_copy_labels.restype = _I
        L.tm_label_resolve.argtypes = [_P, _P, _P, _I64, _I64, _I64, _P]
        L.tm_polygons_from_labels.argtypes = [_P, _I64, _I64, _P, _P, _I64, _I64, _PI64, _PI64, _PI64, _P]
        for name in ("tm_label_range", "tm_ctx_label_buffers", "tm_label_resolve", "tm_polygons_from_labels"):
            getattr(L, name).restype = _I
        L.tm_delaunay.restype = _I
        # multi-GPU exchange (tm_comm.cu; NCCL bound at run time)
        L.tm_comm_id_bytes.restype = _I
        L.tm_comm_unique_id.argtypes = [_P]
        L.tm_comm_unique_id.restype = _I
        L.tm_comm_init.argtypes = [ctypes.POINTER(_P), _I, _I, _P, _I]
        L.tm_comm_init.restype = _I
        L.tm_comm_allgather.argtypes = [_P, _P, _P, ctypes.c_size_t, _P]
        L.tm_comm_allgather.restype = _I
        L.tm_comm_destroy.argtypes = [_P]
        L.tm_comm_destroy.restype = None
        L.tm_comm_last_error.restype = ctypes.c_char_p
        # host-side text I/O (tm_io.cu; no GPU needed)
        L.tm_format_double.argtypes = [ctypes.c_double, ctypes.c_char_p, ctypes.c_size_t]
        L.tm_format_double.restype = _I
        L.tm_file_read.argtypes = [ctypes.c_char_p, _I, _I64]
        L.tm_file_read.restype = _P
        L.tm_file_status.argtypes = [_P, _PI64, _PI64, _PI64, ctypes.c_char_p, ctypes.c_size_t]
        L.tm_file_status.restype = _I
        L.tm_file_copy.argtypes = [_P, _P]
        L.tm_file_copy.restype = _I
        L.tm_file_close.argtypes = [_P]
        L.tm_file_close.restype = None
        L.tm_write_polymesh.argtypes = [ctypes.c_char_p, _P, _I64, _P, _P, _I64, ctypes.c_char_p, ctypes.c_size_t]
        L.tm_write_polymesh.restype = _I
        L.tm_write_triangle_file.argtypes = [ctypes.c_char_p, _I, _P, _P, _I64, ctypes.c_char_p, ctypes.c_size_t]
        L.tm_write_triangle_file.restype = _I
        for name in ("tm_ctx_create", "tm_ctx_defects", "tm_ctx_phase_ms", "tm_ctx_label_ms", "tm_ctx_set_profiling", "tm_ctx_debug",
                     "tm_ctx_debug_copy",
                     "tm_ctx_set_partition", "tm_shift_offsets", "tm_ctx_segment_ms", "tm_label", "tm_relabel",
                     "tm_check_neighbors",
                     "tm_unpack_halfedges", "tm_pack_frontier", "tm_traverse", "tm_repair",
                     "tm_mesh_to_polygons", "tm_mesh_to_polygons_host", "tm_resume_pinch", "tm_check_trivertex",
                     "tm_polygon_stats", "tm_polygon_areas", "tm_canonicalize"):
            getattr(L, name).restype = _I
        _lib = L
    return _lib


def exported_symbols():
    """Names declared in include/termesh_b200.h (checked by the CPU tests)."""
    return ("tm_version", "tm_ctx_create", "tm_ctx_destroy", "tm_ctx_last_error", "tm_ctx_defects",
            "tm_ctx_phase_ms", "tm_ctx_label_ms", "tm_ctx_set_profiling", "tm_ctx_segment_ms", "tm_segment_name", "tm_launch_count",
            "tm_ctx_debug", "tm_ctx_debug_copy", "tm_ctx_set_partition", "tm_shift_offsets",
            "tm_label", "tm_relabel", "tm_check_neighbors", "tm_unpack_halfedges",
            "tm_pack_frontier",
            "tm_traverse", "tm_repair", "tm_mesh_to_polygons_host", "tm_mesh_to_polygons", "tm_resume_pinch",
            "tm_check_trivertex", "tm_polygon_stats", "tm_polygon_areas", "tm_canonicalize",
            "tm_delaunay", "tm_label_range", "tm_ctx_label_buffers", "tm_ctx_copy_labels", "tm_label_resolve",
            "tm_polygons_from_labels", "tm_comm_id_bytes", "tm_comm_unique_id", "tm_comm_init", "tm_comm_allgather", "tm_comm_destroy",
            "tm_comm_last_error", "tm_format_double", "tm_file_read", "tm_file_status", "tm_file_copy", "tm_file_close",
            "tm_write_polymesh", "tm_write_triangle_file")


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise TermeshError("termesh-b200 requires a CUDA device (sm_100a); no CPU fallback exists")
    return torch


class Context:
    """One tm_ctx per CUDA device (owns the library's scratch buffers)."""

    def __init__(self, device_index: int):
        self.device_index = device_index
        p = _P()
        rc = lib().tm_ctx_create(ctypes.byref(p))
        if rc != TM_OK:
            raise TermeshError(f"tm_ctx_create failed with status {rc}")
        self.ptr = p
        _all_ctxs.append(self)

    def close(self):
        """Free this context's device scratch (also done for every context at exit)."""
        if self.ptr:
            lib().tm_ctx_destroy(self.ptr)
            self.ptr = None

    def defects(self):
        counts = (ctypes.c_int64 * NUM_KINDS)()
        first = (ctypes.c_int64 * NUM_KINDS)()
        lib().tm_ctx_defects(self.ptr, counts, first)
        return [(KIND_NAMES[k], int(first[k]), int(counts[k])) for k in range(NUM_KINDS) if counts[k]]

    def phase_ms(self):
        ms = (ctypes.c_double * 3)()
        lib().tm_ctx_phase_ms(self.ptr, ms)
        return list(ms)

    def label_ms(self):
        """[pass A ms, pass B ms] of the last tm_label call (device time)."""
        ms = (ctypes.c_double * 2)()
        lib().tm_ctx_label_ms(self.ptr, ms)
        return list(ms)

    def set_profiling(self, on: bool):
        lib().tm_ctx_set_profiling(self.ptr, int(on))

    def segments(self, reset: bool = True) -> dict:
        """{segment name: (total device ms, launches)} since the last reset."""
        ms = (ctypes.c_double * 32)()
        cnt = (ctypes.c_int64 * 32)()
        n = lib().tm_ctx_segment_ms(self.ptr, ms, cnt, 32, int(reset))
        return {lib().tm_segment_name(k).decode(): (ms[k], int(cnt[k])) for k in range(n)}

    def debug(self):
        out = (ctypes.c_uint64 * 128)()
        lib().tm_ctx_debug(self.ptr, out, 128)
        return list(out)

    def last_error(self) -> str:
        return lib().tm_ctx_last_error(self.ptr).decode()

    def check(self, rc: int, phase: str | None = None):
        if rc == TM_OK:
            return
        msg = self.last_error()
        if rc == TM_ERR_VALIDATION:
            from .mesh_core import ValidationReport
            defects = [(kind, idx, f"{count} defect(s), first at element {idx}")
                       for kind, idx, count in self.defects() if KIND_NAMES.index(kind) <= 7]
            raise ValidationError("refusing to run on an invalid triangulation: " + msg,
                                  ValidationReport(False, defects))
        if rc == TM_ERR_STRUCTURAL:
            # the library tags its messages "[phase] ..."; keep the tag as e.phase
            # (the reference's _phase guarantees e.phase, pipeline.py:114-121)
            if msg.startswith("[") and "] " in msg:
                tag, rest = msg[1:].split("] ", 1)
                raise StructuralError(rest, phase=tag)
            raise StructuralError(msg, phase=phase)
        if rc == TM_ERR_CAPACITY:
            raise CapacityError(msg)
        if rc == TM_ERR_ARGUMENT:
            raise ValueError(msg)
        raise TermeshError(f"CUDA failure: {msg}")


def _destroy_contexts():
    """Free every context's device scratch at interpreter exit (clean
    compute-sanitizer leak reports; the CUDA context is still alive here)."""
    if _lib is None:
        return
    for c in _all_ctxs:
        try:
            c.close()
        except Exception:
            pass
    _all_ctxs.clear()
    _ctxs.clear()


atexit.register(_destroy_contexts)


def context(device=None) -> Context:
    torch = _require_cuda()
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    c = _ctxs.get(idx)
    if c is None:
        with _lock:
            c = _ctxs.get(idx)
            if c is None:
                with torch.cuda.device(idx):
                    c = Context(idx)
                _ctxs[idx] = c
    return c


def stream_ptr(device=None):
    torch = _require_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    """Device/host pointer of a torch tensor or numpy array as c_void_p (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)
