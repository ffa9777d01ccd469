"""Step time of repeated edits of member 0 under each pass-2 launch mode (stream = the
persistent default, inline / list = one warp per job), L2 flushed before every step.

usage: python tools/pass2_probe.py [config] [steps] [W] [modes, comma-separated: auto,inline,list,jobs]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_11612_b200 as dvl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
M, W = c["M"], c["W"]
if len(sys.argv) > 3:
    W = int(sys.argv[3])
modes = [None if m == "auto" else m for m in (sys.argv[4] if len(sys.argv) > 4 else "auto,inline,list,jobs").split(",")]
n = int(c["level"].shape[0])
base, seq = bench.tf_sequence(cfg, steps + 5, 256, M)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = torch.empty(M * W * 8, dtype=torch.int32, device=dev)
ref = None
for mode in modes:
    stream = torch.cuda.Stream()
    ctx = dvl.Context(device=0, stream=stream, timing=True, pass2=mode)
    ctx.build(c["lower"], c["level"], c["scal"])
    for m in range(M):
        if c["domain"] is not None:
            ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
        ctx.update_tf(m, base[m])
    for e in range(5):
        ctx.update_tf(0, seq[e])
        ctx.get_polylines(W, out=out)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xff)
        evs[k][0].record(stream)
        ctx.update_tf(0, seq[5 + k])
        ctx.get_polylines(W, out=out)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in evs]
    ctx.set_timing(True)
    kern = {}
    for k in range(10):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xff)
        ctx.update_tf(0, seq[5 + k])
        ctx.get_polylines(W, out=out)
        tk = ctx.timings()
        for key in ("weights_scan_ms", "bin_reduce_ms", "bin_boundary_ms", "epilogue_ms", "maxv_ms"):
            kern.setdefault(key, []).append(tk[key] * 1e3)
    res = ctx.get_polylines(W)
    if ref is None:
        ref = res
    same = (res.view("u1") == ref.view("u1")).all()
    print(f"{cfg} W={W} pass2={mode or 'auto'}: step median {statistics.median(t):.1f} us "
          f"({n / statistics.median(t) / 1e3:.1f} Gcells/s) | " +
          " ".join(f"{k[:-3]} {statistics.median(v):.1f}" for k, v in kern.items()) +
          f" | same bits as the first mode: {bool(same)}", flush=True)
    ctx.close()
