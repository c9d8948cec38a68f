"""Determinism check per phase: labels (hw words, seeds) over repeated
label_all calls, then traversal over repeated build_polygon_mesh calls on one
fixed labelling.  python tools/dbg_phases.py WORKLOAD N"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2204_05438_b200 as tm
w = sys.argv[1] if len(sys.argv) > 1 else "u10m"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
tri = bench.load_mesh(w, 0)
H = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
ref = None
bad = 0
keep = None
for k in range(N):
    lab = tm.label_all(tri, check=False)
    dm = lab._dev
    hw = dm.hw[: 3 * dm.T].cpu().numpy()
    h = (H(hw), H(dm.seed[: dm.T].cpu().numpy()), H(dm.max_edge[: dm.T].cpu().numpy()))
    if ref is None:
        ref, ref_hw, keep = h, hw, lab
    elif h != ref:
        bad += 1
        d = np.nonzero(hw != ref_hw)[0]
        print(f"labels run {k}: {h} vs {ref}; {len(d)} hw words differ, first {d[:8].tolist()} "
              f"{hw[d[:4]].tolist()} vs {ref_hw[d[:4]].tolist()}", flush=True)
print(f"labels: {bad}/{N} differ", flush=True)
ref = None
bad = 0
for k in range(N):
    m0 = tm.build_polygon_mesh(tri, keep)
    off, v = m0.csr()
    h = (H(off), H(v))
    if ref is None:
        ref = h
    elif h != ref:
        bad += 1
        print(f"traversal run {k}: {h} vs {ref}", flush=True)
print(f"traversal: {bad}/{N} differ", flush=True)
