"""One bench.py JSON line (stdin) -> one text line: tag, workload, ms/step, e2e ms, parity, segments."""
import json
import sys

d = json.loads(sys.stdin.readline())
seg = " ".join(f"{k}={v['ms']:.3f}" for k, v in d.get("kernels", {}).items())
print(sys.argv[1] if len(sys.argv) > 1 else "-", d["config"]["workload"], d["ms_per_step"], d["e2e"]["ms_per_step"],
      (d.get("parity") or {}).get("match"), seg)
