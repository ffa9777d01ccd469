"""Probe: per-warp phase times of agg_reduce in the live pipeline (build with
--define=DVL_PROF, run with DVL_DBG=4): after the grid wait -> loads done -> uniform part
done -> end, for the first 2048 warps.  Dev tool, not a bench.

usage: DVL_DBG=4 python tools/aggprobe.py [config] [W]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402


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
    buf = (ctypes.c_ulonglong * (8 + 2048 + 4096))()
    bt = (ctypes.c_ulonglong * (4096 * 6))()
    for it in range(12):
        flush.zero_()
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        lib.dvl_debug_bt(bt)
        ctx.update_tf(0, synth.tf_edit(1, 1 + it, 256, member=0))
        ctx.get_polylines(W, out=out)
        if os.environ.get("AGG_TWICE") == "1":   # the reduction again, its code now warm
            torch.cuda.synchronize()
            lib.dvl_debug_stats(buf)
            lib.dvl_debug_bt(bt)
            if os.environ.get("AGG_FLUSH") == "1":
                flush.zero_()
            ctx.get_polylines(W, out=out)
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        lib.dvl_debug_bt(bt)
    v = np.array(list(buf), dtype=np.uint64)
    a = v[8:8 + 2048]
    ts = v[8 + 2048:].astype(np.int64).reshape(-1, 2)
    ok = ts[:, 0] > 0
    a, ts = a[ok], ts[ok]
    loads = (a >> np.uint64(40)).astype(np.int64) / 1e3
    uni = ((a >> np.uint64(16)) & np.uint64((1 << 24) - 1)).astype(np.int64) / 1e3
    nb = (a & np.uint64(0xffff)).astype(np.int64)
    t0 = ts[:, 0].min()
    start = (ts[:, 0] - t0) / 1e3
    end = (ts[:, 1] - t0) / 1e3
    dur = (ts[:, 1] - ts[:, 0]) / 1e3
    print("warps %d (of the first 2048), with boundary tiles %d" % (len(a), int((nb > 0).sum())))
    print("  boundary tiles per warp (histogram):", dict(zip(*np.unique(nb, return_counts=True))))
    for nm, x in (("start after first", start), ("loads", loads), ("uniform done", uni),
                  ("total", dur), ("end after first start", end)):
        print("  %-22s p10 %.2f p50 %.2f p90 %.2f max %.2f us" % ((nm,) + tuple(np.percentile(x, [10, 50, 90, 100]))))
    b = nb > 0
    if b.any():
        print("  boundary part (end - uniform done) for warps with boundary tiles: p50 %.2f p90 %.2f max %.2f us" % tuple(
            np.percentile((dur - uni)[b], [50, 90, 100])))
    phases(bt)


def phases(bt):
    b = np.array(list(bt), dtype=np.int64).reshape(-1, 6)
    stride = int(os.environ.get("BT_STRIDE", "0"))   # bin_boundary: a warp's second tile is e + stride
    if stride:
        for nm, sl in (("first tiles", b[:min(stride, 4096)]), ("second tiles", b[stride:4096])):
            s = sl[(sl > 0).all(axis=1)]
            if len(s):
                d = np.diff(s, axis=1) / 1e3
                print("  bin_boundary %s (%d): stage %.2f | weights %.2f | bins %.2f | fold %.2f | mid+flush %.2f us (p50)" % (
                    (nm, len(s)) + tuple(np.median(d, axis=0))))
        return
    b = b[(b > 0).all(axis=1)]
    if len(b):
        d = np.diff(b, axis=1) / 1e3
        print("  first boundary tile of a warp (%d): stage %.2f | weights %.2f | bins %.2f | fold %.2f | mid+flush %.2f us (p50)" % (
            (len(b),) + tuple(np.median(d, axis=0))))


if __name__ == "__main__":
    main()
