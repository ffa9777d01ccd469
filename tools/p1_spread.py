"""Probe (DVL_PROF build, DVL_DBG=4): per-chunk (= per pass-1 CTA) entry, end of streaming
and end times of pass 1 in one edit, relative to the first CTA's entry: how much of the pass
is ramp, spread and look-back tail.

usage: DVL_DBG=4 python tools/p1_spread.py [config]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2306_11612_b200 as dvl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
M, W = c["M"], c["W"]
lib = dvl.load()
ctx = dvl.Context(device=0)
ctx.build(c["lower"], c["level"], c["scal"])
base, seq = bench.tf_sequence(cfg, 24, 256, M)
for m in range(M):
    if c["domain"] is not None:
        ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
    ctx.update_tf(m, base[m])
out = torch.empty(M * W * 8, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
buf = (ctypes.c_ulonglong * 1024)()
rows = []
for it in range(24):
    flush.fill_(it & 0xff)
    torch.cuda.synchronize()
    ctx.update_tf(0, seq[it])
    ctx.get_polylines(W, out=out)
    torch.cuda.synchronize()
    lib.dvl_debug_p1(buf)
    a = np.array(list(buf), dtype=np.int64)[:3 * 341].reshape(-1, 3)
    a = a[a[:, 0] > 0]
    if it >= 4:
        t0 = a[:, 0].min()
        rows.append(((a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3))
ent = np.median([np.percentile(r[0], [0, 50, 100]) for r in rows], axis=0)
se = np.median([np.percentile(r[1], [0, 10, 50, 90, 100]) for r in rows], axis=0)
en = np.median([np.percentile(r[2], [0, 50, 100]) for r in rows], axis=0)
print(f"{cfg}: chunks {len(rows[0][0])}")
print("  entry        min/med/max (us):", np.round(ent, 2))
print("  stream end   min/p10/med/p90/max:", np.round(se, 2))
print("  look-back end min/med/max:", np.round(en, 2))
