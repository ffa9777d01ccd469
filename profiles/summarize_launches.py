"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`) of bench.py.

Prints, per kernel (short name), the launch count and mean / total device time, and the
share of each dvl::* update kernel in the TF-update step (maxv/prologue, pass 1, pass 2,
epilogue), from the mean of each update kernel's last STEADY launches: the steady state of
bench.py's repeated edits of one member (the first edits of each member build the edit cache
and run longer).  ncu serialises launches and runs them cold-cache, so compare shares with
the live CUDA-event numbers of bench.py, not absolute times.

usage: python profiles/summarize_launches.py gpurun_out/launches_r01.csv > profiles/r01_launches.md
"""
import collections
import csv
import re
import sys

# the kernels of one TF-update step (acc_init runs once per context / pixel count)
STEADY = 8
UPDATE = ("tf_prologue_kernel", "maxv_exact_kernel", "weights_reduce_tma", "agg_reduce",
          "bin_boundary", "epilogue_kernel", "weights_scan_kernel", "bin_reduce_kernel")


def short(name):
    m = re.search(r"dvl::(\w+)", name) or re.search(r"\b(agg_reduce|agg_build|bin_boundary|weights_reduce_tma|bin_reduce_tma)\b", name)
    if m:
        return m.group(1)
    m = re.match(r"(?:void )?([\w:]+)", name)
    return (m.group(1) if m else name)[:60]


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    launches = [(short(r[ki]), float(r[vi]), r[gi], r[bi]) for r in rows[h + 1:]
                if len(r) == len(hdr) and r[mi] == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for name, ns, g, b in launches:
        a = agg.setdefault(name, [0, 0.0, g, b])
        a[0] += 1
        a[1] += ns
    print(f"# ncu launch list: {path}\n")
    print(f"{len(launches)} launches (gpu__time_duration.sum, --clock-control none)\n")
    print("| kernel | grid | block | launches | mean us | total us |")
    print("|---|---|---|---|---|---|")
    for name, (c, tot, g, b) in agg.items():
        print(f"| {name} | {g} | {b} | {c} | {tot / c / 1e3:.2f} | {tot / 1e3:.1f} |")
    per = collections.OrderedDict()
    for name, ns, _, _ in launches:
        if name in UPDATE:
            per.setdefault(name, []).append(ns)
    upd = {k: sum(v[-STEADY:]) / len(v[-STEADY:]) for k, v in per.items()}
    step = sum(upd.values())
    print(f"\n## TF-update step (mean of the last {STEADY} launches of each update kernel)\n")
    print("| kernel | mean us | share of step |")
    print("|---|---|---|")
    for name, ns in upd.items():
        print(f"| {name} | {ns / 1e3:.2f} | {ns / step:.3f} |")
    print(f"| **sum** | {step / 1e3:.2f} | 1.000 |")


if __name__ == "__main__":
    main(sys.argv[1])
