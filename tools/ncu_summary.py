"""Summarise ncu --set full reports into profiles/: per-kernel CSV (time,
DRAM bytes, L2 hit rate, occupancy, divergence) and ncu_traffic.json, from
which bench.py fills roofline.traffic (DRAM bytes per launch of the roofline
kernel, measured by ncu; cold-cache and serialised, like every ncu number).

    python tools/ncu_summary.py OUT_DIR WORKLOAD REPORT.ncu-rep [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
           "smsp__sass_inst_executed_op_global_atom.sum", "launch__registers_per_thread"]
SEGMENT = {"k_tri_pass": "label_a_tri_pass", "k_pair_pass": "label_b_edges", "k_ruler_walk": "trav_rulers",
           "k_repair_tips_seg": "repair_tips", "k_stitch_plain": "repair_stitch"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.split("::")[-1].split("<")[0]


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[i]
                if m.startswith("dram__bytes"):
                    x *= SCALE.get(u, 1)
                if m == "gpu__time_duration.sum":
                    x *= SCALE.get(u, 1e-9) * 1e3  # -> ms
                d[m] = x
        res.append(d)
    return res


def main():
    out_dir, workload, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    rows = [d for rep in reps for d in read(rep)]
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, f"ncu_summary_{workload}.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "ms", "dram_read_MB", "dram_write_MB", "L2_hit_%", "L1_hit_%", "warps_active_%",
                    "threads_per_inst", "dram_throughput_%", "mem_compute_throughput_%", "global_atomics",
                    "registers"])
        for d in rows:
            w.writerow([d["kernel"], round(d.get("gpu__time_duration.sum", 0), 4),
                        round(d.get("dram__bytes_read.sum", 0) / 1e6, 2),
                        round(d.get("dram__bytes_write.sum", 0) / 1e6, 2),
                        round(d.get("lts__t_sector_hit_rate.pct", 0), 1),
                        round(d.get("l1tex__t_sector_hit_rate.pct", 0), 1),
                        round(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0), 1),
                        round(d.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0), 2),
                        round(d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0), 1),
                        round(d.get("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 0), 1),
                        int(d.get("smsp__sass_inst_executed_op_global_atom.sum", 0)),
                        int(d.get("launch__registers_per_thread", 0))])
    tj = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for d in rows:
        seg = SEGMENT.get(d["kernel"])
        if seg and "dram__bytes_read.sum" in d:
            traffic.setdefault(workload, {})[seg] = {
                "kernel": d["kernel"], "dram_bytes": int(d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0)),
                "ncu_ms": round(d.get("gpu__time_duration.sum", 0), 4), "source": os.path.basename(out_dir)}
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)
    print(open(os.path.join(out_dir, f"ncu_summary_{workload}.csv")).read())


if __name__ == "__main__":
    main()
