"""Per-kernel table from an ncu --csv metrics log (time, DRAM read / write, GB/s).

usage: python tools/ncu_csv.py gpurun_out/x.csv
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("<")[0].split("(")[0].replace("void ", "").replace("dvl::", "")
            key = (d["ID"], k)
            data.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return data


if __name__ == "__main__":
    data = load(sys.argv[1])
    print("| kernel | us | DRAM read MB | DRAM write MB | GB/s |\n|---|---|---|---|---|")
    for (i, k), v in data.items():
        t = v.get("gpu__time_duration.sum", 0) / 1e3
        rd = v.get("dram__bytes_read.sum", 0) / 1e6
        wr = v.get("dram__bytes_write.sum", 0) / 1e6
        print(f"| {k} | {t:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) / max(t, 1e-9) / 1e3 * 1e3 / 1e3:.0f} |")
