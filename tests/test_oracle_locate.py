"""Pins of the oracle's point location (brushing / linking) against facts other
than its own containment test: on a uniform L = 0 grid every cell is one point, so a point's
cell is the rank of its Hilbert code among all codes (an independent sort); every cell
contains its own lower corner, its far corner and its centroid; points in gaps or outside
the grid hit no cell."""
import numpy as np

from oracle import oracle as o
import synth


def test_uniform_grid_is_the_code_rank():
    lower, level = synth.uniform_cells(8)          # 8^3 cells, L = 0
    B = o.build(lower, level, np.zeros((1, len(level)), np.float32))
    rng = np.random.default_rng(1)
    pts = rng.integers(0, 8, size=(300, 3))
    got = o.locate(lower, level, B, pts)
    codes = o.hilbert_encode(pts.astype(np.uint32), B.b)
    assert np.array_equal(got, np.searchsorted(B.codes, codes))


def test_corners_centroids_gaps_and_outside():
    rng = np.random.default_rng(2)
    lower, level = synth.uniform_cells(4)
    lower = (lower << np.uint32(2)).astype(np.uint32)
    level = np.full(len(level), 2, np.uint8)
    lower, level = synth.refine(lower, level, rng.random(len(level)) < 0.5)
    keep = rng.random(len(level)) < 0.8             # holes in the grid
    lower, level = lower[keep], level[keep]
    B = o.build(lower, level, np.zeros((1, len(level)), np.float32))
    rank = np.empty(B.n, np.int64)
    rank[B.perm.astype(np.int64)] = np.arange(B.n)
    w = (1 << level.astype(np.int64))[:, None]
    lo = lower.astype(np.int64)
    for pts in (lo, lo + w - 1, lo + (w >> 1)):
        assert np.array_equal(o.locate(lower, level, B, pts), rank)
    # every point of the grid not covered by a kept cell hits nothing
    E = 16
    cover = np.zeros((E, E, E), bool)
    for (x, y, z), s in zip(lo, w[:, 0]):
        cover[x:x + s, y:y + s, z:z + s] = True
    gaps = np.argwhere(~cover)
    if len(gaps):
        assert (o.locate(lower, level, B, gaps[:200]) == -1).all()
    assert (o.locate(lower, level, B, [[E, 0, 0], [0, 0, 1 << 20]]) == -1).all()
