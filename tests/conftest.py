"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""
import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
CASE_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "cases", "*.npz")))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running (large meshes)")


def load_case(name):
    """Golden case -> (Triangulation in reference dtypes, dict of reference outputs)."""
    from paper_2204_05438_b200 import Triangulation
    z = np.load(os.path.join(GOLDEN, "cases", f"{name}.npz"))
    tri = Triangulation(z["vertices"], z["triangles"].astype(np.int64), z["neighbors"].astype(np.int64),
                        z["trivertex"].astype(np.int64))
    return tri, {k: z[k] for k in z.files}


def load_hashes():
    p = os.path.join(GOLDEN, "hashes.json")
    return json.load(open(p)) if os.path.exists(p) else {}


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


_BIG = {}


def big_input(name):
    """Regenerate a large golden input with scipy (cached per process and on disk)."""
    if name in _BIG:
        return _BIG[name]
    from paper_2204_05438_b200 import io_formats as io
    n = {"u100k_unit": 100_000, "u1m_unit": 1_000_000, "u10m_unit": 10_000_000}[name]
    tri = io.cached(name, lambda: io.generate_random_delaunay(n, (0, 0, 1, 1), 0))
    _BIG[name] = tri
    return tri
