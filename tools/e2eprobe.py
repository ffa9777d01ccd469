"""Probe: where the end-to-end time of one TF edit goes on the host (update_tf call,
get_polylines call incl. D2H + sync), against the device time of the same step.
Dev tool, not a bench.

usage: python tools/e2eprobe.py [config] [W]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    cfg = synth.make_config(name)
    dvl.load()
    ctx = dvl.Context(device=0)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    M = cfg["M"]
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    pin = torch.empty(M * W * 32, dtype=torch.uint8, pin_memory=True)
    res = pin.numpy().view(dvl.VERTEX_DTYPE).reshape(M, W)
    dev = torch.empty((M, W, 8), dtype=torch.float32, device="cuda")
    tfs = [synth.tf_edit(1, 1 + k, 256, member=0) for k in range(40)]
    st = torch.cuda.ExternalStream(ctx.stream)
    rows = []
    for k in range(40):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        ctx.update_tf(0, tfs[k])
        t1 = time.perf_counter()
        ctx.get_polylines(W, out=res)
        t2 = time.perf_counter()
        e1.record(st)
        torch.cuda.synchronize()
        rows.append((t1 - t0, t2 - t1, t2 - t0, e0.elapsed_time(e1) / 1e3))
    r = np.median(np.array(rows[5:]), axis=0) * 1e6
    print("host out: update_tf call %.1f us | get_polylines(host) call %.1f us | total %.1f us | device events %.1f us" % tuple(r))
    rows = []
    for k in range(40):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.update_tf(0, tfs[k])
        t1 = time.perf_counter()
        ctx.get_polylines(W, out=dev)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rows.append((t1 - t0, t2 - t1, t3 - t0))
    r = np.median(np.array(rows[5:]), axis=0) * 1e6
    print("device out: update_tf call %.1f us | get_polylines(dev) call %.1f us | total incl. sync %.1f us" % tuple(r))


if __name__ == "__main__":
    main()
