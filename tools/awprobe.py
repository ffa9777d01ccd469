"""Probe: every agg_reduce warp's (after the grid wait, loads done, end) globaltimer stamps
in one live edit step (build with --define=DVL_PROF, run with DVL_DBG=4): how the kernel's
time splits into waves, load latency and per-warp work.  Dev tool, not a bench.

usage: DVL_DBG=4 python tools/awprobe.py [config]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2306_11612_b200 as dvl  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    dev = torch.device("cuda", 0)
    c = bench.device_workload(cfg, dev, 2306)
    M, W = c["M"], c["W"]
    lib = dvl.load()
    if os.environ.get("TL_NORED") == "1":   # timing experiment: pass 2 without its atomics
        lib.dvl_debug_nored(1)
    ctx = dvl.Context(device=0)
    ctx.build(c["lower"], c["level"], c["scal"])
    base, seq = bench.tf_sequence(cfg, 12, 256, M)
    for m in range(M):
        if c["domain"] is not None:
            ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
        ctx.update_tf(m, base[m])
    out = torch.empty(M * W * 8, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    buf = (ctypes.c_ulonglong * (32768 * 6))()
    res = []
    for e in range(12):
        flush.fill_(e)
        torch.cuda.synchronize()
        lib.dvl_debug_aw(buf)
        ctx.update_tf(0, seq[e])
        ctx.get_polylines(W, out=out)
        torch.cuda.synchronize()
        lib.dvl_debug_aw(buf)
        if e >= 4:
            res.append(np.array(list(buf), dtype=np.int64).reshape(-1, 6))
    a = res[-1]
    b = a[(a > 0).all(axis=1)]   # the warps that went past the job-level pixel test
    if len(b):
        d = np.diff(b[:, [0, 1, 3, 4, 5, 2]], axis=1) / 1e3
        print(f"{cfg}: {len(b)} straddling warps, p50 (us): loads {np.median(d[:, 0]):.2f} | pixel test "
              f"{np.median(d[:, 1]):.2f} | lazy records {np.median(d[:, 2]):.2f} | single-pixel groups "
              f"{np.median(d[:, 3]):.2f} | boundary tiles / list {np.median(d[:, 4]):.2f}")
    u = a[(a[:, :4] > 0).all(axis=1) & (a[:, 4] == 0)]   # jobs inside one pixel (lazy test)
    if len(u):
        d = np.diff(u[:, [0, 1, 3, 2]], axis=1) / 1e3
        print(f"{cfg}: {len(u)} single-pixel jobs (lazy test), p50 (us): loads {np.median(d[:, 0]):.2f} | "
              f"pixel test {np.median(d[:, 1]):.2f} | fold + exit {np.median(d[:, 2]):.2f}; p90 fold + exit "
              f"{np.percentile(d[:, 2], 90):.2f}")
    a = a[(a[:, :3] > 0).all(axis=1)][:, :3]
    t0 = a[:, 0].min()
    st = (a[:, 0] - t0) / 1e3
    ld = (a[:, 1] - a[:, 0]) / 1e3
    tot = (a[:, 2] - a[:, 0]) / 1e3
    en = (a[:, 2] - t0) / 1e3
    print(f"{cfg}: {len(a)} warps; kernel span (first after-wait -> last end) {en.max():.1f} us")
    for nm, x in (("start", st), ("loads", ld), ("warp total", tot), ("end", en)):
        print("  %-10s p10 %6.2f p50 %6.2f p90 %6.2f max %6.2f us" % ((nm,) + tuple(np.percentile(x, [10, 50, 90, 100]))))
    h, edges = np.histogram(st, bins=20)
    print("  starts histogram:", " ".join(f"{edges[i]:.0f}:{h[i]}" for i in range(len(h))))
    # warps of the first and the later waves
    early = st < 1.0
    print("  warps starting within 1 us of the first: %d, their total p50 %.2f p90 %.2f" % (
        early.sum(), np.median(tot[early]), np.percentile(tot[early], 90)))
    late = ~early
    if late.any():
        print("  later warps: total p50 %.2f p90 %.2f, loads p50 %.2f" % (
            np.median(tot[late]), np.percentile(tot[late], 90), np.median(ld[late])))


if __name__ == "__main__":
    main()
