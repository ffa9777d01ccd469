"""Probe: live timeline of one TF-update step (built with --define=DVL_PROF, run with
DVL_DBG=4): first-block start / last-block end (globaltimer) of pass 1, agg_reduce and
bin_boundary, relative to pass 1's first block, median over steps.  Dev tool, not a bench.

usage: DVL_DBG=4 python tools/timeline.py [config] [W]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402

SLOTS = 8 + 2048 + 4096
BASE = SLOTS - 32
NAMES = [("pass1 entry", 0), ("pass1 after wait", 10), ("pass1 stream end", 11), ("pass1 end", 1),
         ("agg entry", 2), ("agg after wait", 4), ("bnd entry", 6), ("bnd after wait", 8),
         ("bnd end", 7)]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    cfg = synth.make_config(name)
    lib = dvl.load()
    ctx = dvl.Context(device=0)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    M = cfg["M"]
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    out = torch.empty((M, W, 8), dtype=torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    buf = (ctypes.c_ulonglong * SLOTS)()
    rows = []
    st = torch.cuda.ExternalStream(ctx.stream)
    for it in range(24):
        flush.zero_()
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.update_tf(0, synth.tf_edit(1, 1 + it, 256, member=0))
        ctx.get_polylines(W, out=out)
        e1.record(st)
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        v = np.array(list(buf[BASE:BASE + 16]), dtype=np.uint64)
        if it < 4:
            continue
        t = {}
        for nm, k in NAMES:
            x = int(v[k])
            if k % 2 == 0:
                x = (~np.uint64(x)) & np.uint64(0xFFFFFFFFFFFFFFFF) if x else 0
            t[nm] = int(x)
        t0 = t["pass1 entry"]
        rows.append([(t[nm] - t0) / 1e3 if t[nm] else float("nan") for nm, _ in NAMES] +
                    [e0.elapsed_time(e1) * 1e3])
    med = np.nanmedian(np.array(rows), axis=0)
    for (nm, _), x in zip(NAMES, med):
        print(f"  {nm:18s} {x:8.1f} us")
    print(f"  {'step (events)':18s} {med[-1]:8.1f} us")


if __name__ == "__main__":
    main()
