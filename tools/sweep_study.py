"""The P / eps sweep and the cells-per-bin distribution (the paper's Fig. 3 and
Fig. 4), through the library on the GPU: for every (scale, P, eps) the
device time of one TF edit (update + polylines, CUDA events, L2 flushed before each) and the
quartiles of the number of cells per pixel bin of member 0 -- how strongly the importance
warps the x axis.  P = 0 gives every cell the same weight (the bins hold equal cell counts);
larger P concentrates the plot width on the varying, coarse cells.

usage: python tools/sweep_study.py [config] > profiles/sweep_study.md
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
    cfg = synth.make_config(name)
    M, W = cfg["M"], cfg["W"]
    dvl.load()
    ctx = dvl.Context(device=0)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    if cfg["domain"] is not None:
        for m in range(M):
            ctx.set_domain(m, float(cfg["domain"][m, 0]), float(cfg["domain"][m, 1]))
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    st = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = torch.empty((M, W, 8), dtype=torch.float32, device="cuda")
    n = len(cfg["level"])
    print(f"# P / eps sweep, {name} (n = {n}, M = {M}, W = {W})\n")
    print("| scale | P | eps | edit us (median of 10) | cells per bin: min | p25 | median | p75 | max |")
    print("|---|---|---|---|---|---|---|---|---|")
    for scale in ("width", "volume"):
        ctx.set_level_scale(scale)
        for P in (0.0, 0.5, 1.0, 2.0, 5.0):
            for eps in (0.0, 0.025, 0.1, 0.25):
                try:
                    ctx.set_params(P, eps, "conservative")
                except dvl.DvlError as ex:   # e.g. ceil(3 Lmax P) > 100
                    print(f"| {scale} | {P} | {eps} | {ex} | | | | | |")
                    continue
                times = []
                for k in range(12):
                    flush.zero_()
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    ctx.update_tf(0, synth.tf_edit(1, 1 + k, 256, member=0))
                    ctx.get_polylines(W, out=out)
                    b.record(st)
                    torch.cuda.synchronize()
                    times.append(a.elapsed_time(b) * 1e3)
                counts = ctx.get_polylines(W)["count"][0].astype(np.int64)
                q = np.percentile(counts, [0, 25, 50, 75, 100])
                print(f"| {scale} | {P} | {eps} | {np.median(times[2:]):.1f} | " +
                      " | ".join(f"{int(x)}" for x in q) + " |")
    ctx.close()


if __name__ == "__main__":
    main()
