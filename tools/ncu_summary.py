"""Summarise ncu --set full reports into profiles/: a per-kernel CSV (time,
DRAM bytes and % of peak, L2/L1 hit rates, warps active, threads per
instruction (divergence), global atomic/reduction sectors, long-scoreboard
stalls, registers) and ncu_traffic.json, from which bench.py fills
roofline.traffic (DRAM bytes per launch of the roofline kernel, measured by
ncu; cold-cache and serialised, like every ncu number).

Every metric below must be present in the report: a missing name is an
error (no silent zero columns).  Capture with
    ncu --set full --metrics l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum,\
l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum ...

    python tools/ncu_summary.py OUT_DIR WORKLOAD REPORT.ncu-rep|RAW.csv [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

# (column, metric, scale kind)
COLUMNS = [
    ("ms", "gpu__time_duration.sum", "time"),
    ("dram_read_MB", "dram__bytes_read.sum", "bytes"),
    ("dram_write_MB", "dram__bytes_write.sum", "bytes"),
    ("dram_throughput_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("sm_throughput_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("mem_throughput_%", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("L2_hit_%", "lts__t_sector_hit_rate.pct", None),
    ("L1_hit_%", "l1tex__t_sector_hit_rate.pct", None),
    ("warps_active_%", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("threads_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio", None),
    ("global_atom_sectors", "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum", None),
    ("global_red_sectors", "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum", None),
    ("long_scoreboard_warps_per_issue", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     None),
    ("registers", "launch__registers_per_thread", None),
]
SEGMENT = {"k_tri_pass": "label_a_tri_pass", "k_pair_pass": "label_b_edges", "k_ruler_walk": "trav_rulers",
           "k_ruler_write": "trav_write", "k_chain_count": "trav_chain", "k_repair_tips_seg": "repair_tips",
           "k_repair_tips": "repair_tips_short", "k_stitch_plain": "repair_stitch", "k_stitch": "repair_stitch"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1, "nsecond": 1e-9}


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.split("::")[-1].split("<")[0]


def raw_rows(src):
    if src.endswith(".csv"):
        text = open(src).read()
    else:
        text = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True,
                              check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    missing = [m for _, m, _ in COLUMNS if m not in hdr]
    if missing:
        raise SystemExit(f"{src}: metrics not in the report: {missing}")
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for col, m, kind in COLUMNS:
            i = hdr.index(m)
            v = r[i].replace(",", "")
            if v in ("", "n/a"):
                raise SystemExit(f"{src}: {m} has no value for {d['kernel']}")
            x = float(v)
            if kind == "bytes":
                x *= SCALE[units[i]] if units[i] in SCALE else 1
            if kind == "time":
                x *= SCALE.get(units[i], 1e-9) * 1e3  # -> ms
            d[m] = x
        out.append(d)
    return out


def main():
    out_dir, workload, srcs = sys.argv[1], sys.argv[2], sys.argv[3:]
    rows = [d for s in srcs for d in raw_rows(s)]
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"ncu_summary_{workload}.csv")
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + [c for c, _, _ in COLUMNS])
        for d in rows:
            vals = []
            for col, m, kind in COLUMNS:
                x = d[m]
                if kind == "bytes":
                    x /= 1e6
                vals.append(round(x, 4) if isinstance(x, float) else x)
            w.writerow([d["kernel"]] + vals)
    tj = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for d in rows:
        seg = SEGMENT.get(d["kernel"])
        prev = traffic.get(workload, {}).get(seg, {})
        if seg and not (prev.get("source") == os.path.basename(out_dir.rstrip("/")) and
                        prev.get("ncu_ms", 0) > d["gpu__time_duration.sum"]):  # keep a kernel's longest launch
            traffic.setdefault(workload, {})[seg] = {
                "kernel": d["kernel"], "dram_bytes": int(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]),
                "ncu_ms": round(d["gpu__time_duration.sum"], 4), "source": os.path.basename(out_dir.rstrip("/"))}
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)
    print(open(path).read())


if __name__ == "__main__":
    main()
