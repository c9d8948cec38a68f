"""Step-by-step GPU debug run with a watchdog traceback (development tool)."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
faulthandler.dump_traceback_later(int(os.environ.get("WATCHDOG", "90")), exit=True)

t0 = time.time()


def log(*a):
    print(f"[{time.time() - t0:7.2f}s]", *a, flush=True)


import numpy as np  # noqa: E402
import torch  # noqa: E402

log("torch", torch.__version__, torch.cuda.is_available())
torch.zeros(1, device="cuda")
log("cuda init ok")
import paper_2204_05438_b200 as tm  # noqa: E402
from conftest import load_case  # noqa: E402

for name in sys.argv[1:] or ["sun", "u1k_unit", "aniso2k_s1"]:
    tri, g = load_case(name)
    log(name, "T", tri.n_triangles)
    lab = tm.label_all(tri, check=False)
    torch.cuda.synchronize()
    log(" label ok", np.array_equal(lab.max_edge, g["max_edge"]), np.array_equal(lab.frontier, g["frontier_pre"]),
        np.array_equal(lab.seed, g["seed"]))
    m0 = tm.build_polygon_mesh(tri, lab)
    torch.cuda.synchronize()
    off, v = m0.csr()
    log(" traverse ok", np.array_equal(off, g["mesh0_off"]), np.array_equal(v, g["mesh0_verts"]))
    info = {}
    fin = tm.repair_all(tri, lab, m0, stats_out=info)
    torch.cuda.synchronize()
    off, v = fin.csr()
    log(" repair ok", info, np.array_equal(off, g["final_off"]), np.array_equal(v, g["final_verts"]),
        g["stats"].tolist())
log("done")
