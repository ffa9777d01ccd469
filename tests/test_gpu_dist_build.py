"""Distributed build + sharded TF update through the C ABI on one GPU: G ranks as G threads
(paper_2306_11612_b200.dist_build.ThreadCollectives), each with its own dvl context and a
round-robin slice of the input order.  After the sample sort each context must hold one
contiguous piece of the global curve order (the union equals a one-context build: codes,
levels, scalars), and the sharded polylines must equal the one-context polylines (bit for
bit on counts, min/max and bin ranges) and the oracle.  (NCCL cannot put two ranks on one
GPU; the same function runs over torch.distributed in bench.py under torchrun.)
"""
import threading

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


def run_threads(fns):
    errs = [None] * len(fns)

    def wrap(i):
        try:
            fns[i]()
        except BaseException as e:   # noqa: BLE001
            errs[i] = e

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e


@pytest.mark.parametrize("G", [2, 3])
def test_distributed_build_and_sharded_update(dvl, G):
    import torch
    from paper_2306_11612_b200 import dist_build as db, shard
    lower, level = octree(64, 3, 20 + G)
    M = 4
    rng = np.random.default_rng(G)
    scal = rng.standard_normal((M, len(level))).astype(np.float32)
    tfs = np.stack([synth.random_tf(70 + m, 256, member=m) for m in range(M)])
    W = 300
    ctxs = [dvl.Context(device=0) for _ in range(G)]
    colls = db.ThreadCollectives.group(G)
    infos = [None] * G

    def rank_fn(r):
        def f():
            idx = np.arange(r, len(level), G)
            lo = torch.from_numpy(lower[idx].astype(np.int32)).cuda()
            lv = torch.from_numpy(level[idx]).cuda()
            sc = torch.from_numpy(np.ascontiguousarray(scal[:, idx])).cuda()
            infos[r] = db.distributed_build(ctxs[r], lo, lv, sc, colls[r], samples=128)
        return f

    run_threads([rank_fn(r) for r in range(G)])
    B = o.build(lower, level, scal)
    codes = np.concatenate([c.get_sorted()[0] for c in ctxs])
    assert np.array_equal(codes, B.codes)
    data = [c.get_sorted_data() for c in ctxs]
    assert np.array_equal(np.concatenate([d[0] for d in data]), B.level_s)
    assert np.array_equal(np.concatenate([d[1] for d in data], axis=1), B.scal_s)
    assert [i["offset"] for i in infos] == list(np.cumsum([0] + [i["n_local"] for i in infos])[:-1])
    assert all(min(i["sent"]) > 0 for i in infos)
    # sharded update with the two exchanges done by torch ops (as in test_gpu_shard)
    for c in ctxs:
        for m in range(M):
            c.update_tf(m, tfs[m])
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
    planes = [shard.split_planes(e, W, M) for e in exports]
    merged = torch.cat([torch.stack([p[0] for p in planes]).max(0).values,
                        torch.stack([p[1] for p in planes]).max(0).values,
                        torch.stack([p[2] for p in planes]).sum(0)])
    out = ctxs[0].shard_finish(W, merged)
    U = o.update(B, tfs, W)
    assert int(totals.sum().item()) == U.Qtot
    ref = U.vertices
    for k in ("count", "t_min", "t_max"):
        assert np.array_equal(out[k], ref[k])
    rel = np.abs(out["t_mean"].astype(np.float64) - ref["t_mean"]) / np.maximum(ref["t_mean"], 1e-30)
    assert rel.max() <= 1e-5
    one = dvl.Context(device=0)
    one.build(lower, level, scal)
    for m in range(M):
        one.update_tf(m, tfs[m])
    single = one.get_polylines(W)
    for k in ("count", "t_min", "t_max"):
        assert np.array_equal(single[k], out[k])
    for c in ctxs + [one]:
        c.close()
