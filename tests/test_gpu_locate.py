"""GPU parity of point location (dvl_locate; brushing / linking) against the
oracle's containment test: points inside cells, in gaps and outside the grid, for u32 and
u64 keys, host and device buffers; and the brush of a pixel range selects exactly the cells
of its bin ranges."""
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


def octree(E, Lmax, seed, p=0.45, keep=1.0):
    rng = np.random.default_rng(seed)
    lower, level = synth.uniform_cells(E >> Lmax)
    lower = (lower << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(level), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < p)
        lower, level = synth.refine(lower, level, mask)
    k = rng.random(len(level)) < keep
    return lower[k], level[k]


def points(E, n, seed, lower=None, level=None):
    rng = np.random.default_rng(seed)
    pts = [rng.integers(0, E, size=(n, 3))]
    if lower is not None:   # cell corners
        idx = rng.integers(0, len(level), size=n // 4)
        w = (1 << level[idx].astype(np.int64))[:, None]
        pts += [lower[idx].astype(np.int64), lower[idx].astype(np.int64) + w - 1]
    pts.append(np.array([[E, 0, 0], [0, E + 5, 0], [2 ** 21 - 1] * 3]))
    return np.concatenate(pts).astype(np.uint32)


@pytest.mark.parametrize("E,Lmax,seed,keep", [(32, 3, 1, 1.0), (64, 4, 2, 0.7), (16, 2, 3, 0.5)])
def test_locate_matches_oracle(dvl, E, Lmax, seed, keep):
    import torch
    lower, level = octree(E, Lmax, seed, keep=keep)
    scal = np.random.default_rng(seed).standard_normal((2, len(level))).astype(np.float32)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0)
    ctx.build(lower, level, scal)
    pts = points(E, 600, seed + 10, lower, level)
    ref = o.locate(lower, level, B, pts)
    assert np.array_equal(ctx.locate(pts), ref)
    dev = ctx.locate(torch.from_numpy(pts.astype(np.int32)).cuda())
    assert np.array_equal(dev.cpu().numpy(), ref)
    ctx.close()


def test_locate_u64_keys(dvl):
    rng = np.random.default_rng(5)
    E, n = 2 ** 14, 3000                        # 3b = 42 > 32: u64 keys
    blocks = E >> 3
    ids = rng.choice(blocks ** 3, size=n, replace=False)
    lower = np.stack([ids % blocks, (ids // blocks) % blocks, ids // blocks ** 2], 1).astype(np.uint32) * 8
    level = rng.integers(0, 4, size=n).astype(np.uint8)
    scal = rng.standard_normal((1, n)).astype(np.float32)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0)
    ctx.build(lower, level, scal)
    assert ctx.info()["key_bytes"] == 8
    w = (1 << level.astype(np.int64))[:, None]
    pts = np.concatenate([lower.astype(np.int64), lower.astype(np.int64) + w - 1,
                          rng.integers(0, E, size=(500, 3))]).astype(np.uint32)
    assert np.array_equal(ctx.locate(pts), o.locate(lower, level, B, pts))
    ctx.close()


def test_brush_selects_the_bin_cells(dvl):
    lower, level = octree(32, 3, 7)
    scal = np.random.default_rng(7).standard_normal((4, len(level))).astype(np.float32)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0)
    ctx.build(lower, level, scal)
    W = 64
    ctx.get_polylines(W)
    lo, hi = ctx.get_bin_ranges(W)
    br = ctx.brush(W, 10, 20)
    first, last = br["first"], br["last"]
    assert (first, last) == (int(lo[10]), int(hi[20]))
    # the ROI as Hilbert codes: the first and last brushed cells' codes
    assert (br["code_first"], br["code_last"]) == (int(B.codes[first]), int(B.codes[last]))
    # the brushed cells' centroids locate inside the range, the others outside
    half = ((1 << level.astype(np.int64)) >> 1)[:, None]
    cent = (lower.astype(np.int64) + half).astype(np.uint32)
    k = ctx.locate(cent)
    rank = np.empty(B.n, np.int64)
    rank[B.perm.astype(np.int64)] = np.arange(B.n)
    assert np.array_equal(k, rank)
    inside = (k >= first) & (k <= last)
    assert inside.sum() == last - first + 1
    ctx.close()


@pytest.mark.parametrize("seed", [3, 4])
def test_roi_contains_matches_oracle(dvl, seed):
    """dvl_roi_contains (a sample point is in the ROI iff the cell containing it
    has a code in the ROI's code range) against the oracle's containment test + its codes."""
    lower, level = octree(32, 3, seed)
    scal = np.random.default_rng(seed).standard_normal((3, len(level))).astype(np.float32)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0)
    ctx.build(lower, level, scal)
    W = 100
    ctx.get_polylines(W)
    br = ctx.brush(W, 30, 55)
    U = o.update(B, np.stack([o.identity_tf(256)] * 3), W)
    assert (br["first"], br["last"]) == (int(U.lo[30]), int(U.hi[55]))
    rng = np.random.default_rng(seed + 10)
    pts = rng.integers(0, 33, size=(20000, 3)).astype(np.uint32)   # includes points outside
    got = ctx.roi_contains(pts, br["code_first"], br["code_last"])
    idx = o.locate(lower, level, B, pts)
    ref = np.where(idx >= 0, (B.codes[np.maximum(idx, 0)] >= br["code_first"]) &
                   (B.codes[np.maximum(idx, 0)] <= br["code_last"]), False).astype(np.int64)
    assert np.array_equal(got, ref)
    assert 0 < got.sum() < len(pts)
    ctx.close()
