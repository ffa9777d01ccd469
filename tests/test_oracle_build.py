"""Pins of the oracle's build stage (O1-O5).

What pins it: SPEC's worked build examples, the 57-cell
AMR example (re-derived here from the curve walk), the theorem that
dyadic blocks are disjoint contiguous code ranges (so the sort order is independent of
the representative point and consecutive cells share a face under complete coverage),
brute-force pairwise box overlap for the overlap detector, and the validation rules.
"""
import numpy as np
import pytest

from oracle import oracle as o

from synth import refine


def random_octree(E, Lmax, rng, p_refine=0.4):
    """Complete, non-overlapping AMR coverage of an E^3 grid (octree refinement)."""
    G = E >> Lmax
    r = np.arange(G, dtype=np.uint32)
    z, y, x = np.meshgrid(r, r, r, indexing="ij")
    lower = (np.stack([x.ravel(), y.ravel(), z.ravel()], 1) << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(lower), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < p_refine)
        lower, level = refine(lower, level, mask)
    return lower, level


def boxes_overlap(la, La, lb, Lb):
    wa, wb = 1 << int(La), 1 << int(Lb)
    return all(int(la[k]) < int(lb[k]) + wb and int(lb[k]) < int(la[k]) + wa for k in range(3))


def test_unit_block_codes_0_to_7():
    """8 level-0 cells forming a 2^3 block -> codes exactly 0..7 in order."""
    lower = np.array([[x, y, z] for z in range(2) for y in range(2) for x in range(2)], np.uint32)
    B = o.build(lower, np.zeros(8, np.uint8), np.zeros((1, 8), np.float32))
    assert B.b == 1 and B.E == 2
    assert np.array_equal(B.codes, np.arange(8, dtype=np.uint64))


def test_single_cell():
    """one cell; its centroid code."""
    B = o.build([[0, 0, 0]], [0], [[1.0]])
    assert B.n == 1 and B.codes[0] == 0 and B.perm[0] == 0
    B = o.build([[0, 0, 0]], [1], [[1.0]])          # centroid (1,1,1) on a 2^3 grid
    assert B.b == 1 and B.codes[0] == o.hilbert_encode([[1, 1, 1]], 1)[0]


def test_shuffled_input_identical():
    """shuffled input produces an identical dataset."""
    rng = np.random.default_rng(1)
    lower, level = random_octree(16, 2, rng)
    n = len(level)
    scal = rng.standard_normal((3, n)).astype(np.float32)
    B0 = o.build(lower, level, scal)
    p = rng.permutation(n)
    B1 = o.build(lower[p], level[p], scal[:, p])
    assert np.array_equal(B0.codes, B1.codes)
    assert np.array_equal(B0.level_s, B1.level_s)
    assert np.array_equal(B0.scal_s, B1.scal_s)
    assert np.array_equal(p[B1.perm.astype(np.int64)], B0.perm.astype(np.int64))


def test_structured_field_reorders_by_decode():
    """dims (4,4,4), field = x -> reordered values equal x(decode3d(h, 2))."""
    r = np.arange(4, dtype=np.uint32)
    z, y, x = np.meshgrid(r, r, r, indexing="ij")
    lower = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    B = o.build(lower, np.zeros(64, np.uint8), x.ravel()[None].astype(np.float32))
    assert B.b == 2
    assert np.array_equal(B.codes, np.arange(64, dtype=np.uint64))
    assert np.array_equal(B.scal_s[0], o.hilbert_decode(np.arange(64), 2)[:, 0].astype(np.float32))


def test_amr_57_cells():
    """4^3 grid, one L=1 cell at the origin + 56 L=0 cells.  The coarse
    cell's centroid (1,1,1) has code 5 and its block is [0, 8); the fine cells take
    codes 8..63 in curve order."""
    lower = [[0, 0, 0]]
    level = [1]
    for z in range(4):
        for y in range(4):
            for x in range(4):
                if x < 2 and y < 2 and z < 2:
                    continue
                lower.append([x, y, z])
                level.append(0)
    B = o.build(lower, level, np.zeros((1, 57), np.float32))
    assert B.codes[0] == 5 and B.perm[0] == 0 and B.level_s[0] == 1
    assert np.array_equal(B.codes[1:], np.arange(8, 64, dtype=np.uint64))
    walk = o.hilbert_decode(np.arange(8, 11), 2)
    assert [tuple(int(v) for v in p) for p in walk] == [(0, 0, 2), (0, 0, 3), (1, 0, 3)]
    got = np.asarray(lower)[B.perm[1:4].astype(np.int64)]
    assert np.array_equal(got, walk)


@pytest.mark.parametrize("seed", range(8))
def test_order_independent_of_representative_and_face_adjacent(seed):
    """Dyadic blocks are disjoint contiguous code ranges, so sorting by the centroid
    code, the lower-corner code, or the max-corner code gives the same order; with
    complete coverage consecutive cells share a face (positive-area contact)."""
    rng = np.random.default_rng(100 + seed)
    E, Lmax = 16, 3
    lower, level = random_octree(E, Lmax, rng)
    p = rng.permutation(len(level))
    lower, level = lower[p], level[p]
    B = o.build(lower, level, np.zeros((1, len(level)), np.float32))
    w = (1 << level.astype(np.int64))
    for off in (np.zeros_like(lower), (w - 1)[:, None] * np.ones((1, 3), np.int64)):
        codes = o.hilbert_encode((lower.astype(np.int64) + off).astype(np.uint32), B.b)
        assert np.array_equal(np.argsort(codes, kind="stable"), B.perm.astype(np.int64))
    lo = lower[B.perm.astype(np.int64)].astype(np.int64)
    ww = w[B.perm.astype(np.int64)]
    hi = lo + ww[:, None]
    for k in range(len(lo) - 1):
        a0, a1, b0, b1 = lo[k], hi[k], lo[k + 1], hi[k + 1]
        touch = [(a1[d] == b0[d] or b1[d] == a0[d]) for d in range(3)]
        over = [min(a1[d], b1[d]) - max(a0[d], b0[d]) > 0 for d in range(3)]
        assert sum(touch) == 1 and sum(over) == 2, (k, a0, a1, b0, b1)


@pytest.mark.parametrize("seed", range(20))
def test_overlap_detector_matches_pairwise(seed):
    """O4: the consecutive dyadic-range check equals a pairwise box-overlap brute force."""
    rng = np.random.default_rng(seed)
    lower, level = random_octree(8, 2, rng, 0.5)
    lower, level = list(lower), list(level)
    if seed % 2 == 0:   # inject an overlapping cell
        L = int(rng.integers(0, 3))
        c = (rng.integers(0, 8 >> L, size=3) << L).astype(np.uint32)
        lower.append(c)
        level.append(L)
    lower = np.array(lower, np.uint32)
    level = np.array(level, np.uint8)
    brute = any(boxes_overlap(lower[i], level[i], lower[j], level[j])
                for i in range(len(level)) for j in range(i))
    if brute:
        with pytest.raises(o.OracleError) as e:
            o.build(lower, level, np.zeros((1, len(level)), np.float32))
        assert e.value.status == "OVERLAP"
    else:
        o.build(lower, level, np.zeros((1, len(level)), np.float32))


def test_validation_rules():
    with pytest.raises(o.OracleError) as e:
        o.build(np.zeros((0, 3)), np.zeros(0), np.zeros((1, 0)))
    assert e.value.status == "INVAL"
    with pytest.raises(o.OracleError) as e:                  # lower not a multiple of 2^L
        o.build([[1, 0, 0]], [1], [[0.0]])
    assert e.value.status == "INVAL"
    with pytest.raises(o.OracleError) as e:                  # L > 20
        o.build([[0, 0, 0]], [21], [[0.0]])
    assert e.value.status == "INVAL"
    with pytest.raises(o.OracleError) as e:                  # E > 2^21
        o.build([[2 ** 21, 0, 0]], [0], [[0.0]])
    assert e.value.status == "RANGE"
    B = o.build([[2 ** 21 - 1, 0, 0]], [0], [[0.0]])         # E = 2^21 is allowed
    assert B.b == 21
    with pytest.raises(o.OracleError) as e:                  # duplicate cell
        o.build([[0, 0, 0], [0, 0, 0]], [0, 0], [[0.0, 1.0]])
    assert e.value.status == "OVERLAP"


@pytest.mark.parametrize("E,b", [(1, 1), (2, 1), (3, 2), (64, 6), (65, 7), (512, 9), (2048, 11)])
def test_bits_from_extent(E, b):
    """O1: b = max(1, ceil(log2 E)) with E = max(lower + 2^L)."""
    B = o.build([[E - 1, 0, 0]], [0], [[0.0]])
    assert B.E == E and B.b == b


def test_member_ranges_ignore_nonfinite():
    vals = np.array([[np.nan, 2.0, -1.0, np.inf], [np.nan] * 4], np.float32)
    lower = [[x, 0, 0] for x in range(4)]
    B = o.build(lower, [0] * 4, vals)
    assert B.vmin[0] == -1.0 and B.vmax[0] == 2.0
    assert B.vmin[1] == 0.0 and B.vmax[1] == 0.0
