"""Probe: live timeline of one TF-update step (built with --define=DVL_PROF, run with
DVL_DBG=4): first-block start / last-block end (globaltimer) of pass 1 and agg_reduce (with
its boundary tiles), relative to pass 1's first block, median over steps.  Dev tool, not a bench.

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
         ("agg entry", 2), ("agg after wait", 4), ("agg end", 3),
         ("bin_boundary entry", 6), ("bin_boundary after wait", 8), ("bin_boundary end", 7),
         ("agg_jobs entry", 12), ("agg_jobs after wait", 14), ("agg_jobs end", 13)]
NAMES2 = [("prologue start", 0), ("prologue end", 1), ("epilogue entry", 2),
          ("epilogue after wait", 4), ("epilogue after wait (last)", 5),
          ("epilogue loads done (last)", 7), ("epilogue vertex done (last)", 6), ("epilogue end", 3)]
ALL = NAMES2[:2] + NAMES + NAMES2[2:]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    cfg = synth.make_config(name)
    lib = dvl.load()
    if os.environ.get("TL_NORED") == "1":   # timing experiment: pass 2 without its atomics
        lib.dvl_debug_nored(1)
    ctx = dvl.Context(device=0, pass2=os.environ.get("TL_PASS2") or None)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    M = cfg["M"]
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    out = torch.empty((M, W, 8), dtype=torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    buf = (ctypes.c_ulonglong * SLOTS)()
    buf2 = (ctypes.c_ulonglong * (8 + 1 + 64 * 4))()
    if os.environ.get("TL_LOOP") == "1":   # back-to-back steps as in bench.py: per-step gaps
        tfs = [synth.tf_edit(1, 1 + it, 256, member=0) for it in range(48)]
        for it in range(8):
            ctx.update_tf(0, tfs[it])
            ctx.get_polylines(W, out=out)
        torch.cuda.synchronize()
        lib.dvl_debug_tl2(buf2)
        for it in range(40):
            ctx.update_tf(0, tfs[8 + it])
            ctx.get_polylines(W, out=out)
        torch.cuda.synchronize()
        lib.dvl_debug_tl2(buf2)
        st = np.array(list(buf2[9:9 + 160]), dtype=np.int64).reshape(40, 4)
        per = np.diff(st[:, 0]) / 1e3
        gap = (st[1:, 0] - st[:-1, 3]) / 1e3
        pro = (st[:, 1] - st[:, 0]) / 1e3
        body = (st[:, 2] - st[:, 1]) / 1e3
        epi = (st[:, 3] - st[:, 2]) / 1e3
        print("  per-step medians (us): period %.1f | prologue %.1f | prologue end -> epilogue after wait %.1f"
              " | epilogue %.1f | epilogue end -> next prologue start %.1f" % (
                  np.median(per), np.median(pro), np.median(body), np.median(epi), np.median(gap)))
        return
    rows = []
    st = torch.cuda.ExternalStream(ctx.stream)
    do_flush = os.environ.get("TL_FLUSH", "1") == "1"
    for it in range(24):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        lib.dvl_debug_tl2(buf2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.update_tf(0, synth.tf_edit(1, 1 + it, 256, member=0))
        ctx.get_polylines(W, out=out)
        e1.record(st)
        torch.cuda.synchronize()
        lib.dvl_debug_stats(buf)
        lib.dvl_debug_tl2(buf2)
        v = np.array(list(buf[BASE:BASE + 16]), dtype=np.uint64)
        v2 = np.array(list(buf2), dtype=np.uint64)
        if it < 4:
            continue
        t = {}
        for nm, k in NAMES:
            x = int(v[k])
            if k % 2 == 0:
                x = (~np.uint64(x)) & np.uint64(0xFFFFFFFFFFFFFFFF) if x else 0
            t[nm] = int(x)
        for nm, k in NAMES2:
            x = int(v2[k])
            if k % 2 == 0 and k != 6:   # (slot 6: a plain max stamp)
                x = (~np.uint64(x)) & np.uint64(0xFFFFFFFFFFFFFFFF) if x else 0
            t[nm] = int(x)
        t0 = t["pass1 entry"]
        rows.append([(t[nm] - t0) / 1e3 if t[nm] else float("nan") for nm, _ in ALL] +
                    [e0.elapsed_time(e1) * 1e3])
    med = np.nanmedian(np.array(rows), axis=0)
    for (nm, _), x in zip(ALL, med):
        print(f"  {nm:18s} {x:8.1f} us")
    print(f"  {'step (events)':18s} {med[-1]:8.1f} us")


if __name__ == "__main__":
    main()
