"""Pins of the oracle's TF-update stage (O6-O15; Eq. 1-4).

What pins it: SPEC's worked examples for sample / importance /
x-pairs / rasterisation (S:187-189, S:196-198, S:205-207, S:270-272, S:279-281,
S:288-289); closed forms (level scaling exactly 2^L, P=0 uniform, M=1 -> eps);
the Weissenboeck reduction (L=0, exact maxV, identity alpha gives Eq. 2);
exact big-int / rational brute force of the scan, the bins and the per-bin reduction
(tests/bruteforce.py); the invariants "weights sum to the plot width", no empty bins,
n <= sum(count) <= n+W-1; R2 >= exact max(V_h); and the hand-worked 8-cell ensemble.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

from oracle import oracle as o
from tests import bruteforce as bf

f32 = np.float32


# ------------------------------------------------------------------ TF lookup (O7, O8)
def test_sample_examples():
    A = np.array([0.0, 1.0], f32)
    assert o.sample(A, 0.0) == 0.0 and o.sample(A, 1.0) == 1.0
    assert o.sample(A, 0.5) == 0.5
    rng = np.random.default_rng(0)
    C = np.full(17, 0.37, f32)
    assert all(o.sample(C, float(t)) == f32(0.37) for t in rng.random(100))


@pytest.mark.parametrize("N", [2, 3, 5, 17, 129, 257])
def test_sample_exact_at_knots_and_linear_between(N):
    rng = np.random.default_rng(N)
    A = rng.random(N).astype(f32)
    for k in range(N):     # N-1 = 2^j: t = k/(N-1) and t*(N-1) are exact in fp32
        assert o.sample(A, float(f32(k) / f32(N - 1))) == A[k]
    for t in rng.random(200).astype(f32):
        ref = np.interp(float(t) * (N - 1), np.arange(N), A.astype(np.float64))
        assert abs(o.sample(A, float(t)) - ref) <= 4e-7 * max(1.0, abs(ref))


def test_normalize_special_values():
    inv = o.domain_inv(-1.0, 3.0)
    assert inv == 0.25
    assert o.normalize(-1.0, -1.0, inv) == 0.0 and o.normalize(3.0, -1.0, inv) == 1.0
    assert o.normalize(1.0, -1.0, inv) == 0.5
    assert o.normalize(float("nan"), -1.0, inv) == 0.0
    assert o.normalize(float("inf"), -1.0, inv) == 1.0
    assert o.normalize(float("-inf"), -1.0, inv) == 0.0
    assert o.normalize(-5.0, -1.0, inv) == 0.0 and o.normalize(9.0, -1.0, inv) == 1.0
    assert o.domain_inv(2.0, 2.0) == 0.0 and o.normalize(7.0, 2.0, 0.0) == 0.0


def test_index_range_examples():
    """full range -> (0, N-1); constant field -> i == j; middle half, N=101
    -> (25, 75)."""
    inv = o.domain_inv(0.0, 1.0)
    assert o.index_range(0.0, 1.0, 0.0, inv, 256) == (0, 255)
    i, j = o.index_range(0.5, 0.5, 0.0, inv, 256)
    assert i == j or j == i + 1 and (0.5 * 255) % 1 != 0
    inv0 = o.domain_inv(0.3, 0.3)
    assert o.index_range(0.3, 0.3, 0.3, inv0, 64) == (0, 0)
    assert o.index_range(0.25, 0.75, 0.0, inv, 101) == (25, 75)


# ------------------------------------------------------------- importance (Eq. 1-3)
def test_importance_examples():
    eps = 0.025
    assert o.importance(0.0, 0.0, 0, 1.0, eps) == f32(eps)        # S:270 (M=1 -> V=0)
    assert o.importance(0.7, 0.7, 2, 1.0, eps) == 4.0
    for V, L in [(0.1, 0), (0.9, 3), (0.0, 5)]:
        assert o.importance(V, 0.9, L, 0.0, eps) == 1.0            # S:272 (P=0)


@pytest.mark.parametrize("L", range(0, 21))
def test_level_scaling_exact(L):
    """S:325 / Eq. 3: at P=1 a level-L cell weighs exactly 2^L times a level-0 cell."""
    for V in (0.0, 0.013, 0.5, 0.731, 1.0):
        f0 = o.importance(V, 1.0, 0, 1.0, 0.025)
        fL = o.importance(V, 1.0, L, 1.0, 0.025)
        assert Fraction(fL) == Fraction(f0) * 2 ** L


def test_integer_powers_left_to_right():
    rng = np.random.default_rng(3)
    for g in rng.random(50).astype(f32) * f32(8):
        acc = g
        for P in range(2, 9):
            acc = f32(acc * g)
            assert o.powP(float(g), float(P)) == acc


def test_detpow_accuracy():
    """The detpow recipe is deterministic by construction; its accuracy is checked against
    libm pow (bit pattern: parity unpinned)."""
    rng = np.random.default_rng(4)
    for g in np.concatenate([rng.random(200) * 64, [1e-3, 0.025, 1.0, 2.0, 1024.0]]).astype(f32):
        for P in (0.5, 1.5, 2.7, 4.9, 0.1):
            ref = float(g) ** P
            assert abs(o.detpow(float(g), P) - ref) <= 2e-5 * ref + 1e-30
    assert o.detpow(0.0, 0.5) == 0.0


def np_identity_weights(tvals, maxV, eps, P):
    """Eq. 2 written directly in fp32 numpy: f = max(V/maxV, eps)^P."""
    V = tvals.max(axis=0) - tvals.min(axis=0)
    r = (V / f32(maxV)).astype(f32) if maxV > 0 else np.zeros_like(V)
    r = np.minimum(np.maximum(r, f32(eps)), f32(1))
    if P == 0:
        return np.ones_like(r)
    f = r.copy()
    for _ in range(int(P) - 1):
        f = (f * r).astype(f32)
    return f


@pytest.mark.parametrize("P", [0, 1, 2])
def test_weissenboeck_reduction(P):
    """Uniform volume, L=0 everywhere, exact maxV, identity alpha, shared domain: the AMR
    importance (Eq. 3) reduces to Weissenboeck's DVL importance (Eq. 2), bit for bit."""
    rng = np.random.default_rng(7)
    E, M = 8, 3
    r = np.arange(E, dtype=np.uint32)
    z, y, x = np.meshgrid(r, r, r, indexing="ij")
    lower = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    n = len(lower)
    scal = rng.random((M, n)).astype(f32)
    B = o.build(lower, np.zeros(n, np.uint8), scal)
    tf = np.zeros((M, 2, 4), f32)
    tf[:, 1, 3] = 1.0       # alpha(t) = t
    U = o.update(B, tf, 16, P=float(P), eps=0.025, mode="exact", domain=[[0.0, 1.0]])
    # identity alpha and domain [0,1] with scal in [0,1): I(m,h) = v exactly
    V = B.scal_s.max(axis=0) - B.scal_s.min(axis=0)
    assert U.maxV == V.max()
    ref = np_identity_weights(B.scal_s, U.maxV, 0.025, P)
    assert np.array_equal(U.f, ref)


# ------------------------------------------------------------------------ maxV (O9)
def _built_random(seed, M=3, n=500):
    rng = np.random.default_rng(seed)
    lower = np.stack([np.arange(n), np.zeros(n), np.zeros(n)], 1).astype(np.uint32)
    scal = (rng.random((M, n)) * rng.uniform(0.5, 3, size=(M, 1))).astype(f32)
    return o.build(lower, np.zeros(n, np.uint8), scal), rng


def test_maxv_examples():
    """S:205-207.  S:205 (M=1 -> 0) is SPEC's per-entry formula (R1); the R2 bound of one
    member is that member's alpha range over [i, j] (>= the exact 0), and both give the
    same importance f = eps * 2^L because V_h = 0 (reading A8/A11)."""
    B, _ = _built_random(1, M=1)
    tf = np.random.default_rng(2).random((1, 64, 4)).astype(f32)
    lo, _, inv = o.domains(B)
    assert o.maxv(B, tf, lo, inv, "per_entry") == 0.0
    assert o.maxv(B, tf, lo, inv, "exact") == 0.0
    a = tf[0, :, 3]
    assert o.maxv(B, tf, lo, inv, "conservative") == a.max() - a.min()
    for mode in ("per_entry", "conservative"):
        U = o.update(B, tf, 16, mode=mode)
        assert np.all(U.f == f32(0.025))
    B, _ = _built_random(2, M=2)
    lo, _, inv = o.domains(B)
    tf = np.zeros((2, 8, 4), f32)
    tf[0, :, 3] = 1.0
    assert o.maxv(B, tf, lo, inv, "conservative") == 1.0
    assert o.maxv(B, tf, lo, inv, "per_entry") == 1.0
    same = np.repeat(np.random.default_rng(3).random((1, 32, 4)).astype(f32), 2, axis=0)
    assert o.maxv(B, same, lo, inv, "per_entry") == 0.0
    a = same[0, :, 3]
    assert o.maxv(B, same, lo, inv, "conservative") == a.max() - a.min()


@pytest.mark.parametrize("seed", range(30))
def test_r2_bounds_exact(seed):
    """Reading A8: R2 is a conservative bound of the exact max(V_h)."""
    B, rng = _built_random(10 + seed, M=int(2 + seed % 4))
    N = int(rng.integers(2, 300))
    tf = rng.random((B.M, N, 4)).astype(f32)
    if seed % 3 == 0:
        tf[:] = tf[0]
    dom = None if seed % 2 else [[float(B.vmin.min()), float(B.vmax.max())]]
    lo, _, inv = o.domains(B, dom)
    ex = o.maxv(B, tf, lo, inv, "exact")
    r2 = o.maxv(B, tf, lo, inv, "conservative")
    assert r2 >= ex - np.spacing(f32(ex))
    # exact = a direct numpy evaluation of Eq. 1 over all cells
    t = np.stack([np.clip((B.scal_s[m] - lo[m]) * inv[m], 0, 1) for m in range(B.M)])
    al = np.stack([np.interp(t[m].astype(np.float64) * (N - 1), np.arange(N), tf[m, :, 3])
                   for m in range(B.M)])
    assert abs(ex - (al.max(0) - al.min(0)).max()) <= 1e-4   # fp32 vs fp64 lookup


# ------------------------------------------------------------------- scan (O11, O12)
@pytest.mark.parametrize("n,Lmax,P,s", [(1, 0, 1.0, 61), (8, 0, 1.0, 58), (9, 4, 1.0, 53),
                                        (2 ** 30, 4, 1.0, 27), (1000, 10, 0.1, 49),
                                        (5, 3, 0.0, 58)])
def test_shift(n, Lmax, P, s):
    """O11: s = 61 - ceil(log2 n) - ceil(Lmax * P) (ceil of the fp32 P in double)."""
    assert o.shift(n, Lmax, P) == s


def _lines_fixture(seed, n, M, Lmax, N=64):
    rng = np.random.default_rng(seed)
    lower = np.zeros((n, 3), np.uint32)
    level = rng.integers(0, Lmax + 1, size=n).astype(np.uint8)
    x = 0
    for h in range(n):           # cells along the x axis, no overlap
        w = 1 << int(level[h])
        x = (x + w - 1) // w * w
        lower[h, 0] = x
        x += w
    scal = rng.random((M, n)).astype(f32)
    B = o.build(lower, level, scal)
    tf = rng.random((M, N, 4)).astype(f32)
    return B, tf, rng


@pytest.mark.parametrize("seed", range(6))
def test_scan_exact_prefix(seed):
    """Eq. 4 in u64 fixed point: Q equals the big-int prefix of q; Qtot < 2^62; when the
    dynamic-range condition of reading A12 holds, Q * 2^-s is the exact rational prefix
    sum of the fp32 importances."""
    B, tf, _ = _lines_fixture(seed, 300, 3, 3)
    U = o.update(B, tf, 64, P=1.0, eps=0.025)
    acc, ex = 0, Fraction(0)
    for h in range(B.n):
        acc += int(U.q[h])
        ex += Fraction(float(U.f[h]))
        assert int(U.Q[h]) == acc
        assert Fraction(acc, 2 ** U.s) == ex
        assert int(U.q[h]) == math.floor(Fraction(float(U.f[h])) * 2 ** U.s)
    assert U.Qtot == acc < 2 ** 62


# ------------------------------------------------------------------------- bins (O13)
def _spans(U):
    return list(zip(U.b1.tolist(), U.b2.tolist()))


def _bins_from_q(q, W):
    q = np.asarray(q, np.uint64)
    Q = np.cumsum(q).astype(np.uint64)
    b1 = np.empty(len(q), np.int32)
    b2 = np.empty(len(q), np.int32)
    o.lib().or_bins(len(q), o._p(Q), W, o._p(b1), o._p(b2))
    return list(zip(b1.tolist(), b2.tolist()))


def test_spec_x_pair_examples():
    """S:279-280 (x pairs) and S:288-289 (rasterisation)."""
    assert _bins_from_q([1, 1, 1, 1], 8) == [(0, 1), (2, 3), (4, 5), (6, 7)]
    assert _bins_from_q([1, 3], 8) == [(0, 1), (2, 7)]
    assert _bins_from_q([5, 5], 2) == [(0, 0), (1, 1)]
    assert _bins_from_q([7], 3) == [(0, 2)]


@pytest.mark.parametrize("seed", range(300))
def test_bins_equal_rational_overlap(seed):
    """O13 equals exact rational half-open overlap binning (incl. zero-width cells)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 30))
    W = int(rng.integers(2, 40))
    q = rng.integers(0, 6, size=n)
    if rng.random() < 0.5:
        q = q * int(rng.integers(1, 2 ** 40))
    if q.sum() == 0:
        q[rng.integers(0, n)] = 1
    assert _bins_from_q(q, W) == bf.bins_rational([int(v) for v in q], W)


@pytest.mark.parametrize("seed", range(10))
def test_bin_invariants(seed):
    B, tf, rng = _lines_fixture(seed, 400, 2, 4)
    W = int(rng.integers(2, 700))
    U = o.update(B, tf, W, P=float(rng.choice([0.0, 1.0, 2.0])), eps=0.025)
    sp = _spans(U)
    cnt = U.vertices["count"][0].astype(np.int64)
    assert np.all(cnt >= 1)                                   # A18: no empty bins
    assert B.n <= cnt.sum() <= B.n + W - 1
    assert int(U.Q[-1]) == U.Qtot                             # last xf2 == W exactly
    for x in range(W):                                        # contiguous membership
        cells = [h for h, (a, b) in enumerate(sp) if a <= x <= b]
        assert cells == list(range(int(U.lo[x]), int(U.hi[x]) + 1))
    assert all(sp[h + 1][0] >= sp[h][0] and sp[h + 1][0] <= sp[h][1] + 1 for h in range(B.n - 1))


def test_uniform_importance_spans_differ_by_at_most_one():
    """P = 0 -> all cells equally wide -> spans differ by <= 1 pixel."""
    B, tf, _ = _lines_fixture(5, 37, 2, 3)
    U = o.update(B, tf, 1000, P=0.0)
    widths = [b - a + 1 for a, b in _spans(U)]
    assert max(widths) - min(widths) <= 1


@pytest.mark.parametrize("seed", range(20))
def test_doubling_weight_never_shrinks_span(seed):
    """S:322."""
    rng = np.random.default_rng(seed)
    q = rng.integers(1, 50, size=12)
    W = int(rng.integers(2, 100))
    base = _bins_from_q(q, W)
    k = int(rng.integers(0, 12))
    q2 = q.copy()
    q2[k] *= 2
    a, b = _bins_from_q(q2, W)[k]
    assert b - a >= base[k][1] - base[k][0]


# ----------------------------------------------------------------- reduce (O14, O15)
@pytest.mark.parametrize("seed", range(12))
def test_reduce_matches_rational_bruteforce(seed):
    B, tf, rng = _lines_fixture(100 + seed, int(rng_n := 5 + seed * 3), 2, 3)
    W = int(np.random.default_rng(seed).integers(2, 50))
    U = o.update(B, tf, W, P=1.0, eps=0.025)
    lo, _, inv = o.domains(B)
    t_cols = [[o.normalize(float(v), float(lo[m]), float(inv[m])) for v in B.scal_s[m]]
              for m in range(B.M)]
    spans = bf.bins_rational([int(v) for v in U.q], W)
    assert spans == _spans(U)
    ref = bf.reduce_rational(t_cols, spans, W)
    for m in range(B.M):
        for x in range(W):
            c, mn, mx, mean = ref[m][x]
            v = U.vertices[m, x]
            assert v["count"] == c and v["t_min"] == f32(mn) and v["t_max"] == f32(mx)
            assert abs(Fraction(float(v["t_mean"])) - mean) <= Fraction(float(np.spacing(f32(mean))))
            A = tf[m, :, 3]
            assert v["y"] == f32(o.sample(A, float(v["t_mean"])))
            assert v["r"] == f32(o.sample(tf[m, :, 0], float(v["t_mean"])))
            assert v["g"] == f32(o.sample(tf[m, :, 1], float(v["t_mean"])))
            assert v["b"] == f32(o.sample(tf[m, :, 2], float(v["t_mean"])))
    assert rng_n == B.n


def test_identity_alpha_gives_mean_and_identical_members():
    """S:298 (identity alpha -> y = mean) and S:315 (identical members -> identical
    series)."""
    B, _, _ = _lines_fixture(9, 200, 1, 2)
    scal = np.repeat(B.scal_s, 3, axis=0)
    lower = np.zeros((B.n, 3), np.uint32)
    Bp = o.build(*_restore(B), scal[:, np.argsort(B.perm)])
    tf = np.zeros((3, 2, 4), f32)
    tf[:, 1, :] = 1.0
    U = o.update(Bp, tf, 37)
    v = U.vertices
    assert np.array_equal(v[0], v[1]) and np.array_equal(v[1], v[2])
    ok = v["t_mean"][0] < 1.0
    assert np.array_equal(v["y"][0][ok], v["t_mean"][0][ok])
    del lower


def _restore(B):
    """Recover input-order (lower, level) of a _lines_fixture build."""
    inv = np.argsort(B.perm)
    lvl = B.level_s[inv]
    x = 0
    lower = np.zeros((B.n, 3), np.uint32)
    for h in range(B.n):
        w = 1 << int(lvl[h])
        x = (x + w - 1) // w * w
        lower[h, 0] = x
        x += w
    return lower, lvl


def test_qtot_zero_is_degenerate():
    """total = 0 -> degenerate (only possible with eps = 0)."""
    B, _, _ = _lines_fixture(1, 10, 1, 0)
    tf = np.zeros((1, 4, 4), f32)
    with pytest.raises(o.OracleError) as e:
        o.update(B, tf, 8, eps=0.0)
    assert e.value.status == "DEGENERATE"


# ----------------------------------------------------- hand-worked 8-cell ensemble (A3)
def _eight_cells():
    lower = np.array([[i & 1, (i >> 1) & 1, (i >> 2) & 1] for i in range(8)], np.uint32)
    sorted_m1 = np.array([0.25, 0.25, 0.75, 0.25, 0.5, 0.25, 0.25, 0.25], f32)
    ids_sorted = [0, 4, 6, 2, 3, 7, 5, 1]
    m1 = np.empty(8, f32)
    m1[ids_sorted] = sorted_m1
    scal = np.stack([np.full(8, 0.25, f32), m1])
    B = o.build(lower, np.zeros(8, np.uint8), scal)
    assert B.perm.tolist() == ids_sorted
    assert o.hilbert_encode(lower, 1).tolist() == [0, 7, 3, 4, 1, 6, 2, 5]
    tf = np.zeros((2, 2, 4), f32)
    tf[:, 1, 3] = 1.0
    return B, tf


def test_eight_cell_ensemble_r2():
    """Worked by hand: R2 gives maxV = 1, s = 58, q = [e', e',
    2^57, e', 2^56, e', e', e'] with e' = 0.025f * 2^58 = 7205759511166976."""
    B, tf = _eight_cells()
    U = o.update(B, tf, 4, P=1.0, eps=0.025, domain=[[0.0, 1.0]])
    e = 7205759511166976
    assert U.maxV == 1.0 and U.s == 58
    assert U.q.tolist() == [e, e, 2 ** 57, e, 2 ** 56, e, e, e]
    assert U.Q.tolist() == [7205759511166976, 14411519022333952, 158526707098189824,
                            165732466609356800, 237790060647284736, 244995820158451712,
                            252201579669618688, 259407339180785664]
    assert U.b1.tolist() == [0, 0, 0, 2, 2, 3, 3, 3]
    assert U.b2.tolist() == [0, 0, 2, 2, 3, 3, 3, 3]
    v = U.vertices[1]
    assert v["count"].tolist() == [3, 1, 3, 4]
    assert v["t_min"].tolist() == [0.25, 0.75, 0.25, 0.25]
    assert v["t_max"].tolist() == [0.75, 0.75, 0.75, 0.5]
    assert v["t_mean"].tolist() == [f32(1.25 / 3), 0.75, 0.5, 0.3125]
    assert np.all(U.vertices[0]["t_mean"] == 0.25)
    assert U.vertices["count"][0].sum() == 11


def test_eight_cell_ensemble_exact_and_r1():
    B, tf = _eight_cells()
    U = o.update(B, tf, 4, P=1.0, eps=0.025, domain=[[0.0, 1.0]], mode="exact")
    assert U.maxV == 0.5 and U.q[2] == 2 ** 58 and U.q[4] == 2 ** 57
    assert U.Qtot == 475580121294569472
    assert U.b1.tolist() == [0, 0, 0, 2, 2, 3, 3, 3]
    U = o.update(B, tf, 4, P=1.0, eps=0.025, domain=[[0.0, 1.0]], mode="per_entry")
    assert U.maxV == 0.0
    assert U.b1.tolist() == [0, 0, 1, 1, 2, 2, 3, 3] and U.b1.tolist() == U.b2.tolist()
    assert U.vertices[1]["t_mean"].tolist() == [0.25, 0.5, 0.375, 0.25]


# ------------------------------------- maxV restricted to the data's TF index range [i, j]
def _index_range_fixture():
    """P:272-278 ("ranges [i_m, j_m] of the transfer-function indices ... iterate only over
    the transfer function values present in the data").  Two members on a shared domain
    [0, 8] with N = 9 entries (inv = 1/8 exactly, so t (N-1) = v): member 0 holds values in
    [2, 3] -> [i_0, j_0] = [2, 3]; member 1 in [4, 5] -> [4, 5]; so [i, j] = [2, 5].  The
    alpha extremes of both tables (1.0 and 0.0) lie outside [2, 5]."""
    n = 8
    lower = np.stack([np.arange(n), np.zeros(n), np.zeros(n)], 1).astype(np.uint32)
    m0 = np.array([2.0, 3.0, 2.5, 2.0, 3.0, 2.25, 2.75, 2.0], f32)
    m1 = np.array([4.0, 5.0, 4.5, 5.0, 4.0, 4.25, 4.75, 4.0], f32)
    B = o.build(lower, np.zeros(n, np.uint8), np.stack([m0, m1]))
    tf = np.zeros((2, 9, 4), f32)
    tf[0, :, 3] = [1.0, 0.9, 0.30, 0.50, 0.40, 0.60, 0.0, 0.1, 1.0]
    tf[1, :, 3] = [0.0, 0.05, 0.20, 0.35, 0.70, 0.45, 1.0, 0.8, 0.0]
    tf[:, :, 0], tf[:, :, 1], tf[:, :, 2] = 0.1, 0.2, 0.3
    return B, tf


def test_maxv_uses_only_the_data_index_range():
    """Hand-computed over a in [2, 5]: R2 = max{.30,.50,.40,.60,.20,.35,.70,.45}
    - min{...} = 0.70 - 0.20; R1 = max_a |alpha_0[a] - alpha_1[a]| = |0.40 - 0.70| (a = 4).
    Over the whole tables both would be 1.0 (a = 0 and the 0/1 entries), and with member
    0's range alone ([2, 3]) R2 would be 0.50 - 0.20 -- so a dropped [i, j] restriction or a
    wrong min/max over the members fails here."""
    B, tf = _index_range_fixture()
    lo, _, inv = o.domains(B, [[0.0, 8.0]])
    assert inv[0] == f32(0.125)
    assert o.index_range(float(B.vmin[0]), float(B.vmax[0]), 0.0, float(inv[0]), 9) == (2, 3)
    assert o.index_range(float(B.vmin[1]), float(B.vmax[1]), 0.0, float(inv[1]), 9) == (4, 5)
    r2 = o.maxv(B, tf, lo, inv, "conservative")
    r1 = o.maxv(B, tf, lo, inv, "per_entry")
    assert r2 == f32(f32(0.70) - f32(0.20))
    assert r1 == f32(f32(0.70) - f32(0.40))
    ex = o.maxv(B, tf, lo, inv, "exact")
    assert r2 >= ex
    # the importance follows (Eq. 3, P = 1, L = 0): the cell with member 0 at 2.0 (alpha
    # 0.30) and member 1 at 4.0 (alpha 0.70) has V = 0.70 - 0.30 and f = V / R2
    U = o.update(B, tf, 8, P=1.0, eps=0.025, domain=[[0.0, 8.0]])
    k = int(np.nonzero(B.perm == 0)[0][0])
    V = f32(f32(0.70) - f32(0.30))
    assert U.maxV == r2 and U.f[k] == f32(V / r2)


def test_index_range_floor_and_ceil_between_knots():
    """i = floor of the lower data position, j = ceil of the upper one;
    positions between knots widen the range outward; j is capped at N - 1."""
    inv = o.domain_inv(0.0, 8.0)
    assert o.index_range(2.5, 3.5, 0.0, inv, 9) == (2, 4)
    assert o.index_range(2.0, 3.0, 0.0, inv, 9) == (2, 3)
    assert o.index_range(-1.0, 9.0, 0.0, inv, 9) == (0, 8)
    assert o.index_range(7.9, 8.0, 0.0, inv, 9) == (7, 8)


def test_maxv_restricted_range_r2_bounds_exact_random():
    """R2 over [i, j] is still an upper bound of the exact max(V_h) (reading A8) when the
    domains are wider than the data, so [i, j] is a strict sub-range of [0, N-1]."""
    for seed in range(20):
        rng = np.random.default_rng(700 + seed)
        M, n, N = int(rng.integers(2, 5)), 300, int(rng.integers(5, 200))
        lower = np.stack([np.arange(n), np.zeros(n), np.zeros(n)], 1).astype(np.uint32)
        a, w = rng.uniform(1, 3, (M, 1)), rng.uniform(0.5, 2, (M, 1))
        scal = (a + w * rng.random((M, n))).astype(f32)
        B = o.build(lower, np.zeros(n, np.uint8), scal)
        lo, _, inv = o.domains(B, [[0.0, 6.0]])
        tf = rng.random((M, N, 4)).astype(f32)
        ex = o.maxv(B, tf, lo, inv, "exact")
        r2 = o.maxv(B, tf, lo, inv, "conservative")
        full = tf[:, :, 3].max() - tf[:, :, 3].min()
        assert ex <= r2 <= full


def test_reduce_rgb_channels_constant_tf():
    """P:250-256 (RGBa per bin after the division): with constant colour channels r = 0.1,
    g = 0.2, b = 0.3 every vertex carries exactly those values (O8 is exact for constant
    tables), so a channel-order mistake in the reduction's epilogue fails here."""
    B, tf = _index_range_fixture()
    U = o.update(B, tf, 5, P=1.0, eps=0.025, domain=[[0.0, 8.0]])
    for m in range(2):
        assert np.all(U.vertices[m]["r"] == f32(0.1))
        assert np.all(U.vertices[m]["g"] == f32(0.2))
        assert np.all(U.vertices[m]["b"] == f32(0.3))
    # distinct ramps per channel: r = t, g = 1 - t, b = t/2 (exact at every t on N = 2
    # tables with these knots up to one fp32 rounding); y uses alpha
    tf2 = np.zeros((2, 2, 4), f32)
    tf2[:, :, 0] = [0.0, 1.0]
    tf2[:, :, 1] = [1.0, 0.0]
    tf2[:, :, 2] = [0.0, 0.5]
    tf2[:, :, 3] = [0.0, 1.0]
    U = o.update(B, tf2, 5, P=1.0, eps=0.025, domain=[[0.0, 8.0]])
    for m in range(2):
        v = U.vertices[m]
        mu = v["t_mean"].astype(np.float64)
        assert np.all(v["r"] == v["t_mean"]) and np.all(v["y"] == v["t_mean"])
        assert np.allclose(v["g"], 1.0 - mu, atol=1e-7) and np.allclose(v["b"], mu / 2, atol=1e-7)
