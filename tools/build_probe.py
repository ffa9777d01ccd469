"""Times the build (B0-B3) of a config with device-resident inputs through the C ABI and
prints the library's per-phase event times (used with ncu for the build kernels).

usage: python tools/build_probe.py [config] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11612_b200 as dvl  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sort = sys.argv[3] if len(sys.argv) > 3 else "auto"
dev = torch.device("cuda", 0)
c = bench.device_workload(cfg, dev, 2306)
torch.cuda.synchronize()
ctx = dvl.Context(device=0, timing=True, sort=sort)
for r in range(reps):
    ctx.build(c["lower"], c["level"], c["scal"])
    t = ctx.timings()
    print(cfg, sort, {k: round(v, 4) for k, v in t.items() if k in ("ingest_ms", "encode_ms", "sort_ms", "gather_ms")},
          "passes", t["sort_passes"], flush=True)
