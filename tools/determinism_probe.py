"""Race check at size (in place of compute-sanitizer, which this GPU pool refuses): two
contexts on the same data run the same sequence of TF edits (the bench's edit-cache steps,
L2 flushed in between, so the look-backs, the self-resetting counters and the boundary /
job lists are exercised in their production launch configuration) and every edit's
vertices must be bit-identical between the two contexts and across the pass-2 forms.

usage: python tools/determinism_probe.py [config] [edits] [pass-2 forms, comma-separated]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2306_11612_b200 as dvl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
edits = int(sys.argv[2]) if len(sys.argv) > 2 else 40
forms = [None if f == "auto" else f for f in (sys.argv[3] if len(sys.argv) > 3 else "auto,auto").split(",")]
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
M, W = c["M"], c["W"]
base, seq = bench.tf_sequence(cfg, edits, 256, M)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ctxs = []
for f in forms:
    ctx = dvl.Context(device=0, pass2=f)
    ctx.build(c["lower"], c["level"], c["scal"])
    for m in range(M):
        if c["domain"] is not None:
            ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
        ctx.update_tf(m, base[m])
    ctxs.append(ctx)
outs = [torch.empty(M * W * 8, dtype=torch.int32, device=dev) for _ in forms]
bad = 0
for e in range(edits):
    res = []
    for ctx, out in zip(ctxs, outs):
        flush.fill_(e & 0xff)
        ctx.update_tf(0 if e % 5 else (e // 5) % M, seq[e])
        ctx.get_polylines(W, out=out)
        torch.cuda.synchronize()
        res.append(out.cpu().numpy().copy())
    for r in res[1:]:
        if not np.array_equal(r, res[0]):
            bad += 1
print(f"{cfg}: {edits} edits x {len(forms)} contexts ({','.join(f or 'auto' for f in forms)}): "
      f"{'all bit-identical' if bad == 0 else f'{bad} edits differ'}", flush=True)
for ctx in ctxs:
    ctx.close()
sys.exit(1 if bad else 0)
