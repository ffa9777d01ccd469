"""Summarise an `ncu --set full` capture of the TF-update kernels (raw page as CSV).

Writes a markdown summary (duration, DRAM bytes, throughput, occupancy, issue activity,
top stall reasons per launch) to stdout and, with --traffic FILE, the per-launch DRAM
bytes (read + write) per kernel as JSON -- the `roofline.traffic` that bench.py reports.

usage: ncu -i gpurun_out/prof.ncu-rep --page raw --csv > raw.csv
       python profiles/summarize_full.py raw.csv --traffic profiles/ncu_dram_per_launch.json
"""
import csv
import json
import re
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}


def short(name):
    m = re.search(r"(weights_reduce_tma|bin_reduce_tma|agg_reduce|agg_build|bin_boundary|\w+_kernel)", name)
    return m.group(1) if m else name[:40]


def main(path, traffic_out=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    traffic = {}
    print(f"# ncu --set full summary ({path})\n")
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        k = short(r[col["Kernel Name"]])
        print(f"## {k}\n")
        print("| metric | value | unit |")
        print("|---|---|---|")
        for m, label in METRICS:
            if m in col:
                print(f"| {label} | {r[col[m]]} | {units[col[m]]} |")
        stalls = [(h, r[i]) for h, i in col.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0))
                         for h, v in stalls), key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        print("\nTop stall reasons (pc sampling): " +
              ", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in stalls[:6]) + "\n")
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[m]]) * SCALE.get(units[col[m]], 1)
        traffic[k] = b
    if traffic_out:
        with open(traffic_out, "w") as f:
            json.dump({k: int(v) for k, v in traffic.items()}, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    out = None
    if "--traffic" in sys.argv:
        out = sys.argv[sys.argv.index("--traffic") + 1]
    main(sys.argv[1], out)
