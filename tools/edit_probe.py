"""Runs a config's repeated TF edits of member 0 (the bench's step) for ncu captures: build
from HBM-generated inputs, every member's TF installed, then `edits` edits + get_polylines.

usage: python tools/edit_probe.py [config] [edits]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_11612_b200 as dvl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
edits = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
M, W = c["M"], c["W"]
ctx = dvl.Context(device=0)
ctx.build(c["lower"], c["level"], c["scal"])
base, seq = bench.tf_sequence(cfg, edits, 256, M)
for m in range(M):
    if c["domain"] is not None:
        ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
    ctx.update_tf(m, base[m])
out = torch.empty(M * W * 8, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for e in range(edits):
    flush.fill_(e & 0xff)
    ctx.update_tf(0, seq[e])
    ctx.get_polylines(W, out=out)
torch.cuda.synchronize()
print("edit_probe", cfg, "n", int(c["level"].shape[0]), "edits", edits)
