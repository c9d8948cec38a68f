"""Label-pass device times (tm_ctx_label_ms, best of 7) of the library named by
TERMESH_LIB_VARIANT (A/B timing builds; their labels may be wrong)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_05438_b200 as tm  # noqa: E402
from paper_2204_05438_b200 import _capi  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "u10m"
tri = bench.load_mesh(w, 0)
ctx = _capi.context()
res = []
for _ in range(7):
    tm.label_all(tri, check=False)
    res.append(ctx.label_ms())
a = min(r[0] for r in res)
b = min(r[1] for r in res)
print(json.dumps({"lib": os.path.basename(os.environ.get("TERMESH_LIB_VARIANT", "default")), "workload": w,
                  "pass_a_ms": round(a, 4), "pass_b_ms": round(b, 4)}))
