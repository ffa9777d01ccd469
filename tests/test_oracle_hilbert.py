"""Pins of the oracle's Hilbert curve (reading A1/O3).

What pins it: bijection and face adjacency by exhaustive curve walks on 2^3..32^3 grids
(north_star: "brute-force curve walks on 2^3-8^3 grids; curve adjacency"), sampled
adjacency at b = 10, 20, 21, origin = 0, dyadic-block contiguity (the
property the AMR order relies on), and the Skilling-variant vectors of reading A1.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as o


def all_points(b):
    r = np.arange(1 << b, dtype=np.uint32)
    x, y, z = np.meshgrid(r, r, r, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], 1)


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_bijection_exhaustive(b):
    pts = all_points(b)
    h = o.hilbert_encode(pts, b)
    assert np.array_equal(np.sort(h), np.arange(8 ** b, dtype=np.uint64))
    back = o.hilbert_decode(h, b)
    assert np.array_equal(back, pts)


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_face_adjacency_exhaustive(b):
    pts = all_points(b).astype(np.int64)
    h = o.hilbert_encode(pts, b)
    walk = pts[np.argsort(h)]
    d = np.abs(np.diff(walk, axis=0)).sum(axis=1)
    assert np.all(d == 1), "consecutive curve points must be face neighbours"


@pytest.mark.parametrize("b", [10, 20, 21])
def test_adjacency_and_roundtrip_sampled(b):
    rng = np.random.default_rng(b)
    h = rng.integers(0, 8 ** b - 1, size=100_000, dtype=np.uint64)
    p0 = o.hilbert_decode(h, b).astype(np.int64)
    p1 = o.hilbert_decode(h + np.uint64(1), b).astype(np.int64)
    assert np.all(np.abs(p1 - p0).sum(axis=1) == 1)
    assert np.all(p0 < (1 << b))
    assert np.array_equal(o.hilbert_encode(p0, b), h)


@pytest.mark.parametrize("b", list(range(1, 22)))
def test_origin_and_end(b):
    assert o.hilbert_encode([[0, 0, 0]], b)[0] == 0
    # reading A1 (Skilling variant): the curve ends at (2^b - 1, 0, 0)
    assert np.array_equal(o.hilbert_decode([8 ** b - 1], b)[0], [(1 << b) - 1, 0, 0])


@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_dyadic_block_contiguity(b):
    """Every aligned 2^L cube maps to one aligned code range [s, s + 8^L)."""
    pts = all_points(b)
    h = o.hilbert_encode(pts, b).reshape(1 << b, 1 << b, 1 << b)
    for L in range(0, b + 1):
        w = 1 << L
        for x0, y0, z0 in itertools.product(range(0, 1 << b, w), repeat=3):
            blk = np.sort(h[x0:x0 + w, y0:y0 + w, z0:z0 + w].ravel())
            s = int(blk[0])
            assert s % (8 ** L) == 0
            assert np.array_equal(blk, np.arange(s, s + 8 ** L, dtype=np.uint64))


def test_skilling_variant_vectors():
    """Reading A1: Skilling (2004) AxestoTranspose + x-major interleave.  The b=1 walk is
    h bits = (x, x^y, x^y^z); the other vectors are SURVEY.md 8(c)'s cross-check values."""
    walk = [tuple(int(v) for v in p) for p in o.hilbert_decode(np.arange(8), 1)]
    assert walk == [(0, 0, 0), (0, 0, 1), (0, 1, 1), (0, 1, 0), (1, 1, 0), (1, 1, 1),
                    (1, 0, 1), (1, 0, 0)]
    for x, y, z in itertools.product(range(2), repeat=3):
        assert o.hilbert_encode([[x, y, z]], 1)[0] == (x << 2) | ((x ^ y) << 1) | (x ^ y ^ z)
    assert o.hilbert_encode([[1, 1, 1]], 2)[0] == 5
    assert o.hilbert_encode([[3, 5, 7]], 3)[0] == 177
    assert o.hilbert_encode([[1000, 2000, 3000]], 12)[0] == 16259960082
    assert o.hilbert_encode([[2 ** 20 - 1, 0, 0]], 20)[0] == 2 ** 60 - 1
    assert o.hilbert_encode([[2 ** 21 - 1] * 3], 21)[0] == 6588122883467697005
    b2 = [tuple(int(v) for v in p) for p in o.hilbert_decode(np.arange(4), 2)]
    assert b2 == [(0, 0, 0), (0, 1, 0), (1, 1, 0), (1, 0, 0)]


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5, 6])
def test_first_step_axis_cycles(b):
    """Reading A1 fact: the first step is along z, y, x for b = 1, 2, 0 (mod 3)."""
    p1 = o.hilbert_decode([1], b)[0]
    axis = int(np.nonzero(p1)[0][0])
    assert axis == {1: 2, 2: 1, 0: 0}[b % 3]
