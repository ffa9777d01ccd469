"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): C1-sized builds and TF edits through the C ABI on every kernel family --
encode + onesweep sort (u32 and u64 keys), gather/validate, the TMA pass 1 in full and
edit-cache modes, pass 2 inline and listed (bin_boundary), the epilogue, the generic
kernels, the exact-maxV pass, q export, locate, W changes, and the single-rank sharded
export/merge path.  Each result is checked against the oracle so a run is also a parity run.

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402
from oracle import oracle as o  # noqa: E402
from tests.test_gpu_parity import check_update, octree, scalars, sparse_cells, tfs_for  # noqa: E402


def one(lower, level, scal, W_list, generic=False, pass2=None, mode="conservative", edits=3):
    M = scal.shape[0]
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0, generic=generic, pass2=pass2)
    ctx.build(lower, level, scal)
    ctx.set_params(1.0, 0.025, mode)
    tfs = tfs_for(M, 256, 5)
    for m in range(M):
        ctx.update_tf(m, tfs[m])
    for e in range(edits):
        tfs[0] = synth.tf_edit(9, e)
        ctx.update_tf(0, tfs[0])
        for W in W_list:
            out = ctx.get_polylines(W)
            U = o.update(B, tfs, W, mode=mode)
            check_update(U, B, tfs, dict(out=out, info=ctx.info(), Q=ctx.get_prefix(),
                                         ranges=ctx.get_bin_ranges(W)), W)
    ctx.locate(np.array([[0, 0, 0], [5, 7, 9], [1, 1, 1]], np.uint32))
    ctx.close()


def main():
    lower, level = octree(32, 3, 1)
    scal = scalars(len(level), 4, 2)
    one(lower, level, scal, [1024, 300, 700])
    one(lower, level, scal, [64], pass2="list")
    one(lower, level, scal, [64], pass2="inline", mode="exact")
    one(lower, level, scal, [512], generic=True, edits=2)
    l8, v8 = octree(32, 2, 3)
    one(l8, v8, scalars(len(v8), 8, 4), [4096, 100], edits=2)
    one(l8, v8, scalars(len(v8), 16, 5), [1000], edits=2)
    lu, vu = sparse_cells(4096, 30000, 6, Lmax=4)   # u64 keys
    one(lu, vu, scalars(len(vu), 3, 7), [1024], edits=2)
    print("sanitize_run: all parity checks passed")


if __name__ == "__main__":
    main()
