"""Debug probe: G contexts in a LocalGroup build one dataset; prints per-rank sortedness."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
from oracle import oracle as o  # noqa: E402
from tests.test_gpu_parity import octree  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sort = sys.argv[2] if len(sys.argv) > 2 else "auto"
alloc = (sys.argv[3] if len(sys.argv) > 3 else "torch") == "torch"
lower, level = octree(64, 3, 22)
n = len(level)
scal = np.random.default_rng(0).standard_normal((4, n)).astype(np.float32)
parts = [np.arange(r, n, G) for r in range(G)]
grp = dvl.LocalGroup(G)
ctxs = [dvl.Context(device=0, sort=sort, torch_allocator=alloc) for _ in range(G)]
for r, c in enumerate(ctxs):
    c.set_local_comm(grp, r)
errs = [None] * G


def run(r):
    try:
        ctxs[r].build(lower[parts[r]], level[parts[r]], np.ascontiguousarray(scal[:, parts[r]]))
    except Exception as e:  # noqa: BLE001
        errs[r] = e


ts = [threading.Thread(target=run, args=(r,)) for r in range(G)]
[t.start() for t in ts]
[t.join() for t in ts]
print("errors", errs)
B = o.build(lower, level, scal)
for r, c in enumerate(ctxs):
    codes, ids = c.get_sorted()
    d = np.diff(codes.astype(np.int64))
    bad = np.nonzero(d <= 0)[0]
    print(f"rank {r}: n={len(codes)} shard={c.shard()} unsorted_at={bad[:5]} first={codes[:3]} last={codes[-3:]}")
allc = np.concatenate([c.get_sorted()[0] for c in ctxs])
print("union == oracle:", np.array_equal(allc, B.codes), "sorted union:", np.array_equal(np.sort(allc), B.codes))
for c in ctxs:
    c.close()
print("done")
