"""Median step time (L2 flushed, device events) of repeated edits of member 0 for a config,
with the library at the given path (A/B comparisons of two builds).

usage: python tools/step_probe.py [config] [lib path] [steps]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_11612_b200 import dvl  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
path = sys.argv[2] if len(sys.argv) > 2 else dvl.LIB_PATH
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
mode = sys.argv[4] if len(sys.argv) > 4 else "write"   # L2 flush: write, or write then read
dvl.load(path)
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
M, W = c["M"], c["W"]
n = int(c["level"].shape[0])
base, seq = bench.tf_sequence(cfg, steps + 5, 256, M)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev).view(torch.int64)
out = torch.empty(M * W * 8, dtype=torch.int32, device=dev)
stream = torch.cuda.Stream()
ctx = dvl.Context(device=0, stream=stream)
ctx.build(c["lower"], c["level"], c["scal"])
for m in range(M):
    if c["domain"] is not None:
        ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
    ctx.update_tf(m, base[m])
for e in range(5):
    ctx.update_tf(0, seq[e])
    ctx.get_polylines(W, out=out)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for k in range(steps):
    with torch.cuda.stream(stream):
        flush.fill_(k & 0xff)
        if mode == "write+read":
            flush2.sum()   # clean lines: the dirty flush lines are written back before the step
    evs[k][0].record(stream)
    ctx.update_tf(0, seq[5 + k])
    ctx.get_polylines(W, out=out)
    evs[k][1].record(stream)
torch.cuda.synchronize()
t = [a.elapsed_time(b) * 1e3 for a, b in evs]
print(f"{cfg} {os.path.basename(path)} flush={mode}: median {statistics.median(t):.1f} us, "
      f"{n / statistics.median(t) / 1e3:.1f} Gcells/s", flush=True)
