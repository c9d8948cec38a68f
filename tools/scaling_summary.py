"""Print a partition_scaling.py JSON (per G: step, speed-up, per-rank phases; balanced iterations)."""
import json
import sys

d = json.load(open(sys.argv[1]))
for key in ("projected", "projected_balanced"):
    if key not in d:
        continue
    print(key)
    for g, v in d[key].items():
        print(f"  G={g} step {v['step_ms']} ms  x{v['projected_speedup']}", "iters", v.get("iterations", ""))
        for r in v.get("ranks", []):
            segs = r.get("segments", {})
            top = sorted(segs.items(), key=lambda kv: -kv[1])[:4]
            print(f"    seeds {r.get('seeds')} label {r['label_range_ms']} poly {r['polygons_ms']} xch "
                  f"{r['exchange_ms_modeled']} step {r['step_ms']}  top: {top}")
