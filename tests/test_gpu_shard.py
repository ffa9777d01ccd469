"""Sharded TF update through the C ABI on one GPU: G contexts in one process, each holding a
contiguous piece of the global curve order (given to it in shuffled order), with the two
exchanges (gather of the shard totals, MIN/MAX/SUM merge of the accumulator planes) done by
torch ops in place of the collectives.  The merged polylines must equal the unsharded
context and the oracle: bit for bit on bin ranges, counts, min/max; means within 1e-5.
(NCCL cannot put two ranks on one GPU; the collectives themselves are covered by the gloo
test and by bench.py under torchrun.)"""
import numpy as np
import pytest

from oracle import oracle as o
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dvl():
    import paper_2306_11612_b200 as m
    m.load()
    return m


def octree(E, Lmax, seed, p=0.45):
    rng = np.random.default_rng(seed)
    lower, level = synth.uniform_cells(E >> Lmax)
    lower = (lower << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(level), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < p)
        lower, level = synth.refine(lower, level, mask)
    return lower, level


def run_sharded(dvl, lower, level, scal, tfs, W, G, generic, B):
    import torch
    from paper_2306_11612_b200 import shard
    rng = np.random.default_rng(G)
    cuts = np.linspace(0, B.n, G + 1).astype(int)
    perm = B.perm.astype(np.int64)
    ctxs = []
    for g in range(G):
        ids = perm[cuts[g]:cuts[g + 1]].copy()
        rng.shuffle(ids)
        c = dvl.Context(device=0, generic=generic)
        c.set_global_bits(B.b)
        c.build(lower[ids], level[ids], scal[:, ids])
        c.set_shard(int(cuts[g]), B.n, B.Lmax, B.vmin, B.vmax)
        for m in range(B.M):
            c.update_tf(m, tfs[m])
        ctxs.append(c)
    totals = torch.zeros(G, dtype=torch.int64, device="cuda")
    for g, c in enumerate(ctxs):
        c.shard_total(totals[g:g + 1])
    torch.cuda.synchronize()
    exports = []
    for g, c in enumerate(ctxs):
        buf = torch.empty(c.shard_export_words(W), dtype=torch.int64, device="cuda")
        c.shard_reduce(W, totals, g, buf)
        exports.append(buf)
    torch.cuda.synchronize()
    planes = [shard.split_planes(e, W, B.M) for e in exports]
    mn = torch.stack([p[0] for p in planes]).max(0).values
    mx = torch.stack([p[1] for p in planes]).max(0).values
    sm = torch.stack([p[2] for p in planes]).sum(0)
    merged = torch.cat([mn, mx, sm])
    out = ctxs[-1].shard_finish(W, merged)
    ranges = ctxs[-1].get_bin_ranges(W)
    for c in ctxs:
        c.close()
    return out, ranges, int(totals.sum().item())


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("W", [3, 256, 4096])
def test_sharded_equals_unsharded(dvl, G, generic, W):
    lower, level = octree(64, 3, 10 + G)
    rng = np.random.default_rng(G)
    scal = rng.standard_normal((4, len(level))).astype(np.float32)
    tfs = np.stack([synth.random_tf(50 + m, 256, member=m) for m in range(4)])
    B = o.build(lower, level, scal)
    U = o.update(B, tfs, W)
    out, (lo, hi), qtot = run_sharded(dvl, lower, level, scal, tfs, W, G, generic, B)
    assert qtot == U.Qtot
    assert np.array_equal(lo, U.lo) and np.array_equal(hi, U.hi)
    ref = U.vertices
    assert np.array_equal(out["count"], ref["count"])
    assert np.array_equal(out["t_min"], ref["t_min"])
    assert np.array_equal(out["t_max"], ref["t_max"])
    rel = np.abs(out["t_mean"].astype(np.float64) - ref["t_mean"]) / np.maximum(ref["t_mean"], 1e-30)
    assert rel.max() <= 1e-5
    full = dvl.Context(device=0, generic=generic)
    full.build(lower, level, scal)
    for m in range(4):
        full.update_tf(m, tfs[m])
    one = full.get_polylines(W)
    full.close()
    for k in ("count", "t_min", "t_max"):
        assert np.array_equal(one[k], out[k])


@pytest.mark.parametrize("generic", [False, True])
def test_native_comm_single_rank(dvl, generic):
    """The library's own NCCL path (dvl_set_comm + dvl_get_polylines of a sharded context,
    both exchanges inside the call) with one rank: every output equals the unsharded
    context bit for bit, over several edits (one rank is all NCCL allows on one GPU; the
    multi-rank exchanges are the same collectives as the torch path above)."""
    from paper_2306_11612_b200 import dvl as D
    lower, level = octree(32, 3, 81)
    M = 4
    scal = np.random.default_rng(82).standard_normal((M, len(level))).astype(np.float32)
    B = o.build(lower, level, scal)
    tfs = np.stack([synth.random_tf(83 + m, 256, member=m) for m in range(M)])
    plain = dvl.Context(device=0, generic=generic)
    plain.build(lower, level, scal)
    sh = dvl.Context(device=0, generic=generic)
    sh.build(lower, level, scal)
    sh.set_shard(0, B.n, B.Lmax, B.vmin, B.vmax)
    sh.set_comm(1, 0, D.nccl_unique_id())
    W = 512
    for e in range(3):
        for c in (plain, sh):
            for m in range(M):
                c.update_tf(m, tfs[m] if e == 0 else synth.tf_edit(4, e, 256, member=m))
        a, b = plain.get_polylines(W), sh.get_polylines(W)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), e
        la, ha = plain.get_bin_ranges(W)
        lb, hb = sh.get_bin_ranges(W)
        assert np.array_equal(la, lb) and np.array_equal(ha, hb)
    plain.close()
    sh.close()
