"""The sharded TF-update decomposition on CPU with world_size 2 over gloo.

Each rank takes one contiguous piece of the global curve order and computes, with the
oracle's definitions, its fixed-point weights, its total, and (after the product's
`shard.gather_totals` all_gather and `shard.scan_offset` rule) the global pixel ranges of
its cells and its per-pixel MIN / MAX / SUM planes; the product's `shard.merge_planes`
all_reduces them.  The merged planes must equal the unsharded oracle: bit for bit on cell
ranges, counts, min/max; the means to double rounding.  This pins the decomposition math
that the GPU path (dvl_shard_reduce / dvl_shard_finish) implements, without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dataset(seed):
    import synth
    rng = np.random.default_rng(seed)
    E, Lmax = 32, 3
    lower, level = synth.uniform_cells(E >> Lmax)
    lower = (lower << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(level), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < 0.5)
        lower, level = synth.refine(lower, level, mask)
    M = 3
    scal = rng.standard_normal((M, len(level))).astype(np.float32)
    tfs = np.stack([synth.random_tf(seed + m, 64, member=m) for m in range(M)])
    return lower, level, scal, tfs


def _shard_planes(B, tfs, a, b, W, offset, Qtot, s, maxV):
    """Planes of cells [a, b) of the curve order: lo/hi (global cell ids), tmin/tmax bits,
    double sums of t -- the definitions O13/O14 applied to a contiguous piece."""
    from oracle import oracle as o
    M, N = B.M, tfs.shape[1]
    lo_, _, inv = o.domains(B)
    alpha = np.ascontiguousarray(tfs[:, :, 3])
    n = b - a
    lv = np.ascontiguousarray(B.level_s[a:b])
    sc = np.ascontiguousarray(B.scal_s[:, a:b])
    q = np.empty(n, np.uint64)
    o.lib().or_weights(n, M, N, o._p(lv), o._p(sc), o._p(alpha), o._p(lo_), o._p(inv), maxV, 1.0,
                       0.025, s, None, o._p(q))
    Q = (np.cumsum(q.astype(object)) + offset).astype(np.uint64) if n else q
    b1, b2 = o.bins_ext(Q, offset, Qtot, W)
    big = np.iinfo(np.int64).max
    mn = np.full(W + M * W, big, np.int64)
    mx = np.zeros(W + M * W, np.int64)
    sm = np.zeros(M * W, np.float64)
    for h in range(n):
        t = [o.normalize(float(sc[m, h]), float(lo_[m]), float(inv[m])) for m in range(M)]
        for x in range(b1[h], b2[h] + 1):
            g = a + h
            mn[x] = min(mn[x], g)
            mx[x] = max(mx[x], g)
            for m in range(M):
                bits = int(np.float32(t[m]).view(np.uint32))
                mn[W + m * W + x] = min(mn[W + m * W + x], bits)
                mx[W + m * W + x] = max(mx[W + m * W + x], bits)
                sm[m * W + x] += t[m]
    return int(q.sum(dtype=np.uint64)) if n else 0, mn, mx, sm


def _worker(rank, world, port, seed, W, results):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as o
    from paper_2306_11612_b200 import shard
    lower, level, scal, tfs = _dataset(seed)
    B = o.build(lower, level, scal)
    lo_, _, inv = o.domains(B)
    maxV = o.maxv(B, tfs, lo_, inv)
    s = o.shift(B.n, B.Lmax, 1.0)
    cuts = np.linspace(0, B.n, world + 1).astype(int)
    a, b = int(cuts[rank]), int(cuts[rank + 1])
    # 1. weight totals -> scan offset and Qtot
    local_total = _shard_planes(B, tfs, a, b, W, 0, 1, s, maxV)[0]
    totals = shard.gather_totals(torch.tensor([local_total], dtype=torch.int64))
    offset, Qtot = shard.scan_offset(totals.tolist(), rank)
    # 2. planes of this shard's cells with the global offset, merged over the ranks
    _, mn, mx, sm = _shard_planes(B, tfs, a, b, W, offset, Qtot, s, maxV)
    tmn, tmx, tsm = torch.from_numpy(mn), torch.from_numpy(mx), torch.from_numpy(sm)
    shard.merge_planes(tmn, tmx, tsm)
    if rank == 0:
        results.put((offset, Qtot, tmn.numpy(), tmx.numpy(), tsm.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed,W", [(3, 64), (4, 7), (5, 1000)])
def test_sharded_update_matches_unsharded(seed, W):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as o
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, W, q)) for r in range(2)]
    for p in procs:
        p.start()
    offset, Qtot, mn, mx, sm = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lower, level, scal, tfs = _dataset(seed)
    B = o.build(lower, level, scal)
    U = o.update(B, tfs, W)
    M = B.M
    assert offset == 0 and Qtot == U.Qtot
    assert np.array_equal(mn[:W].astype(np.uint64), U.lo)
    assert np.array_equal(mx[:W].astype(np.uint64), U.hi)
    cnt = (mx[:W] - mn[:W] + 1).astype(np.uint32)
    for m in range(M):
        v = U.vertices[m]
        assert np.array_equal(cnt, v["count"])
        assert np.array_equal(mn[W + m * W: W + (m + 1) * W].astype(np.uint32).view(np.float32), v["t_min"])
        assert np.array_equal(mx[W + m * W: W + (m + 1) * W].astype(np.uint32).view(np.float32), v["t_max"])
        mean = (sm[m * W:(m + 1) * W] / cnt).astype(np.float32)
        assert np.allclose(mean, v["t_mean"], rtol=1e-6, atol=0)


def test_scan_offset_rule():
    from paper_2306_11612_b200 import shard
    assert shard.scan_offset([5, 7, 11], 0) == (0, 23)
    assert shard.scan_offset([5, 7, 11], 2) == (12, 23)
    (a, b), (c, d), (e, f) = shard.export_layout(4, 3)
    assert (a, b, c, d, e, f) == (0, 16, 16, 32, 32, 68)
