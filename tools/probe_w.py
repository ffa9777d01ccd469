"""Probe: TF-update kernel times on one workload as the pixel count W varies (W = 2 has
almost no pixel boundaries, so pass 2 is all uniform warp tiles).  Dev tool, not a bench.

usage: python tools/probe_w.py [config] [W ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    Ws = [int(w) for w in sys.argv[2:]] or [2, 64, 1024, 8192, 65536]
    cfg = synth.make_config(name)
    dvl.load()
    ctx = dvl.Context(device=0, timing=True)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    if cfg["domain"] is not None:
        for m in range(cfg["M"]):
            ctx.set_domain(m, float(cfg["domain"][m, 0]), float(cfg["domain"][m, 1]))
    M = cfg["M"]
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    out = torch.empty((M, max(Ws), 8), dtype=torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    mode = os.environ.get("PROBE_FLUSH", "write")
    twice = os.environ.get("PROBE_TWICE", "0") == "1"
    for W in Ws:
        acc = {}
        for it in range(8):
            flush.zero_()
            if mode == "write+read":
                clean.sum()
            ctx.update_tf(0, synth.tf_edit(1, 1 + it, 256, member=0))
            ctx.get_polylines(W, out=out)
            if twice:
                torch.cuda.synchronize()
                t0 = ctx.timings()
                ctx.get_polylines(W, out=out)
            torch.cuda.synchronize()
            t = ctx.timings()
            if int(os.environ.get("DVL_DBG", "0")) & 4:
                import ctypes
                buf = (ctypes.c_ulonglong * (8 + 2048 + 4096))()
                dvl.load().dvl_debug_stats(buf)
                v = list(buf)
                if it == 7 and any(v[8:8 + 2048]):
                    cta = np.array(v[8:8 + 2048], dtype=np.uint64)
                    ts = np.array(v[8 + 2048:], dtype=np.int64).reshape(-1, 2)
                    cyc = (cta & np.uint64((1 << 40) - 1)).astype(np.int64)
                    sm = (cta >> np.uint64(40)).astype(np.int64)
                    G = int((cyc > 0).sum())
                    cyc, sm = cyc[:G], sm[:G]
                    print("  CTA kcycles: min %.0f p50 %.0f p90 %.0f max %.0f" % tuple(
                        np.percentile(cyc, [0, 50, 90, 100]) / 1e3))
                    order = np.argsort(-cyc)[:12]
                    print("  slowest CTAs (chunk, sm, kc):", [(int(i), int(sm[i]), int(cyc[i] // 1000)) for i in order])
                    per_sm = np.zeros(sm.max() + 1)
                    np.maximum.at(per_sm, sm, cyc)
                    print("  by SM: slowest-CTA kc per SM, p10/p50/p90:", np.percentile(per_sm, [10, 50, 90]) // 1000,
                          " chunk-index corr %.2f" % np.corrcoef(np.arange(G), cyc)[0, 1])
                    ts = ts[:G]
                    t0 = ts[:, 0].min()
                    st, en = (ts[:, 0] - t0) / 1e3, (ts[:, 1] - t0) / 1e3
                    for lo_, hi_ in ((0, 148), (148, 296), (296, 444)):
                        print("  blocks %d-%d: start us p50 %.1f max %.1f | end us p50 %.1f max %.1f" % (
                            lo_, hi_, np.median(st[lo_:hi_]), st[lo_:hi_].max(), np.median(en[lo_:hi_]), en[lo_:hi_].max()))
                    h = np.histogram(cyc / 1e3, bins=8)
                    print("  hist:", list(h[0]), [int(x) for x in h[1]])
                bd = v[8 + 2048 + 4096 - 8:]
                if it >= 3 and bd[5]:
                    ne = bd[5]
                    print("  boundary per entry (kcycles): to-entry %.1f stage %.1f weights %.1f bins %.1f fold+mid %.1f flush %.1f | per warp total %.1f | entries %d" % (
                        bd[0] / ne / 1e3, bd[1] / ne / 1e3, bd[2] / ne / 1e3, bd[3] / ne / 1e3, bd[4] / ne / 1e3, bd[6] / ne / 1e3, bd[7] / (2 * 148 * 8) / 1e3, ne))
                if it >= 3:
                    nw = max(v[5], 1)
                    print("  agg_reduce per warp (kcycles): wait %.1f loads %.1f scan+thr %.1f reduce+atomics %.1f (unused %.2f)"
                          " | max warp %.1f | warps %d tiles %d" % (v[0] / nw / 1e3, v[1] / nw / 1e3,
                          v[2] / nw / 1e3, v[3] / nw / 1e3, v[4] / nw / 1e3, v[6] / 1e3, nw, v[7] // 8))
            if it >= 3:
                for k, v in t.items():
                    if isinstance(v, float):
                        acc.setdefault(k, []).append(v)
        print(W, {k: round(float(np.median(v)) * 1e3, 2) for k, v in acc.items()}, flush=True)


if __name__ == "__main__":
    main()
