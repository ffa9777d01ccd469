"""Static SASS instruction counts of the hot kernels of the built library (sm_100a):
UBLKCP = cp.async.bulk (1D TMA), SYNCS = mbarrier operations, REDUX = warp reductions
(redux.sync), MATCH = match.any, ATOMS / ATOMG / RED = shared / global atomics and
reductions.  One instantiation per kernel family (the ones the C2 / C3 / C5 edits run).

usage: python tools/sass_counts.py > profiles/r02f_sass_counts.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2306_11612_b200", "libdvl.so")
KERNELS = [   # (label, regex on the demangled name)
    ("tf_prologue_kernel", r"dvl::tf_prologue_kernel"),
    ("weights_reduce_tma<4, 4, smem table, M == 4, edit cache>", r"weights_reduce_tma<4, 4, true, true, 1>"),
    ("weights_reduce_tma<4, 16, L1 table, M == 16, edit cache>", r"weights_reduce_tma<4, 16, false, true, 1>"),
    ("agg_reduce<4, 24, inline>", r"agg_reduce<4, 24, false, false>"),
    ("agg_reduce<8, 16, listed>", r"agg_reduce<8, 16, true, false>"),
    ("agg_jobs<4, 24, 32 jobs / warp>", r"agg_jobs<4, 24, 1>"),
    ("bin_boundary<8>", r"bin_boundary<8>"),
    ("epilogue_kernel", r"dvl::epilogue_kernel"),
    ("encode_bucket_kernel<u64>", r"encode_bucket_kernel<unsigned long long, true>"),
    ("bucket_scatter_kernel<u64>", r"bucket_scatter_kernel<unsigned long long, true>"),
    ("bucket_rank_kernel<u32>", r"bucket_rank_kernel<unsigned int>"),
    ("gather_validate8_kernel<u32>", r"gather_validate8_kernel<unsigned int>"),
    ("onesweep_kernel<u32>", r"onesweep_kernel<unsigned int, false>"),
]
COLS = ["UBLKCP", "SYNCS", "REDUX", "MATCH", "ATOMS", "ATOMG", "RED", "SHFL", "LDG", "STG", "LDS", "STS", "BAR"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur].append(m.group(1))
    names = {}
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
    for mangled, d in zip(funcs, dem):
        names[mangled] = d
    print("# SASS instruction counts of the hot kernels (`python tools/sass_counts.py`, sm_100a)\n")
    print(__doc__.split("\n\n")[0].replace("\n", " ") + "\n")
    print("| kernel | " + " | ".join(COLS) + " | total |")
    print("|---" * (len(COLS) + 2) + "|")
    for label, rx in KERNELS:
        hit = [k for k, d in names.items() if re.search(re.escape(rx) if "<" in rx else rx, d)]
        if not hit:
            print(f"| `{label}` | " + " | ".join("-" for _ in COLS) + " | not found |")
            continue
        ops = funcs[hit[0]]
        c = collections.Counter("RED" if o in ("RED", "REDG") else o for o in ops)
        print(f"| `{label}` | " + " | ".join(str(c.get(k, 0)) for k in COLS) + f" | {len(ops)} |")


if __name__ == "__main__":
    sys.exit(main())
