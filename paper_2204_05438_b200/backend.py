"""Backend selector kept for signature compatibility with the reference
(backend.py:20-45).  The reference maps phase kernels onto a thread pool; here
every phase runs as CUDA grids on the current device, so the backend argument
of label_all / build_polygon_mesh / repair_all is accepted and only recorded
in PhaseStats.  "gpu" is accepted as a kind; "sequential" and "parallel" are
aliases of it for drop-in callers.
"""

from dataclasses import dataclass


@dataclass(frozen=True)
class Backend:
    kind: str = "gpu"
    workers: int = 1

    def __post_init__(self):
        if self.kind not in ("sequential", "parallel", "gpu"):
            raise ValueError(f"unknown backend kind {self.kind!r}")
        if self.workers < 1:
            raise ValueError("worker count must be positive")

    @property
    def is_parallel(self) -> bool:
        return self.kind != "sequential"

    def __str__(self):
        return "gpu"


GPU = Backend("gpu")
SEQUENTIAL = GPU


def parallel(workers: int) -> Backend:
    return Backend("parallel", workers)
