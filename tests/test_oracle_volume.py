"""Pins of the volume-scaled importance (the cell volume 2^3L instead of the
width 2^L in Eq. 3): on L = 0 data both choices are the same weights; for two cells of equal
variation the weight ratio is the size ratio, 2^L by width and 2^3L = 8^L by volume (exact
in fixed point: powers of two)."""
import numpy as np

from oracle import oracle as o
import synth


def test_level0_volume_equals_width():
    lower, level = synth.uniform_cells(6)
    scal = np.random.default_rng(3).standard_normal((3, len(level))).astype(np.float32)
    B = o.build(lower, level, scal)
    tfs = np.stack([synth.random_tf(5 + m, 256, member=m) for m in range(3)])
    a = o.update(B, tfs, 64)
    b = o.update(B, tfs, 64, scale="volume")
    assert np.array_equal(a.q, b.q) and a.s == b.s


def test_size_ratio_width_vs_volume():
    # a level-1 cell (a 2^3 cube) and a level-0 cell beside it, one member: V = 0 -> r = eps
    lower = np.array([[0, 0, 0], [2, 0, 0]], np.uint32)
    level = np.array([1, 0], np.uint8)
    scal = np.array([[0.5, 0.5]], np.float32)
    B = o.build(lower, level, scal)
    tfs = synth.random_tf(1, 256)[None]
    big = int(np.nonzero(B.level_s == 1)[0][0])
    small = 1 - big
    w = o.update(B, tfs, 4, eps=0.25)
    v = o.update(B, tfs, 4, eps=0.25, scale="volume")
    assert w.q[big] == 2 * w.q[small]
    assert v.q[big] == 8 * v.q[small]
    assert w.s == 61 - 1 - 1 and v.s == 61 - 1 - 3     # O11 with ceil(c Lmax P)
