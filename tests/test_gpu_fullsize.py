"""GPU parity at BASELINE.json's full sizes in the launch configuration bench.py times (C3:
103 M cells x 8 fields, W = 4096; C4: 134 M cells x 16 members; C5: 1.03 B cells x 4
members, 36-bit keys), on outputs the oracle computes one by one and on properties that hold
at any size (the whole-dataset oracle does not finish in seconds there; the element-wise
comparison at size is tests/test_gpu_scale.py on the same recipes):

* the order: codes strictly increasing, ids a permutation, 4096 sampled positions whose code
  is the oracle's centroid code of the input cell there, and whose level / scalars are that
  cell's (B1-B3);
* maxV (oracle R2 from the data ranges and the TFs) and the shift s, bit for bit (U0);
* 4096 sampled cells' q = Q(k) - Q(k-1) equal the oracle's per-cell Eq. 1 / Eq. 3 / fixed
  point (U1, U2);
* the bin ranges: contiguous, every pixel non-empty, and at 16 sampled pixel boundaries the
  oracle's O13 on the neighbouring cells' Q puts lo / hi exactly there (U3); counts = hi -
  lo + 1 for every pixel;
* at 4 sampled pixels, per member, min / max of t bit for bit and the mean within 1e-5 of the
  float64 mean over the pixel's cells (U4, U5), with t by the oracle's O7 (vectorised, pinned
  to the oracle's own function on a subset).
Run after two edits of member 0 (the second in edit-cache mode, as bench.py times)."""
import ctypes

import numpy as np
import pytest

from oracle import oracle as o

pytestmark = pytest.mark.gpu

f32 = np.float32


@pytest.fixture(scope="module")
def dvl():
    import paper_2306_11612_b200 as m
    m.load()
    return m


def t_of(v, lo, inv):
    """O7 vectorised: t = clamp((v - lo) inv, 0, 1) in fp32, NaN -> 0."""
    x = (v.astype(f32) - f32(lo)).astype(f32) * f32(inv)
    x = x.astype(f32)
    return np.where(x > 0, np.where(x < 1, x, f32(1)), f32(0)).astype(f32)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_sampled(dvl, name):
    import torch
    import bench
    dev = torch.device("cuda", 0)
    c = bench.device_workload(name, dev, 2306)
    M, W = c["M"], c["W"]
    n = int(c["level"].shape[0])
    base, edits = bench.tf_sequence(name, 2, 256, M)
    tfs = np.stack(base)
    ctx = dvl.Context(device=0)
    ctx.build(c["lower"], c["level"], c["scal"])
    if c["domain"] is not None:
        lo = c["domain"][:, 0].astype(f32)
        hi = c["domain"][:, 1].astype(f32)
        for m in range(M):
            ctx.set_domain(m, float(lo[m]), float(hi[m]))
    for m in range(M):
        ctx.update_tf(m, tfs[m])
    for e in range(2):
        tfs[0] = edits[e]
        ctx.update_tf(0, tfs[0])
    out = ctx.get_polylines(W)
    info = ctx.info()
    rng = np.random.default_rng(7)
    # ---- finite data ranges of the input (the default domains), from the input itself
    scal = c["scal"]
    fin = torch.isfinite(scal)
    vmin = torch.where(fin, scal, float("inf")).min(dim=1).values.cpu().numpy().astype(f32)
    vmax = torch.where(fin, scal, float("-inf")).max(dim=1).values.cpu().numpy().astype(f32)
    if c["domain"] is None:
        lo, hi = vmin.copy(), vmax.copy()
    inv = np.array([o.domain_inv(float(a), float(b)) for a, b in zip(lo, hi)], f32)
    # ---- B1-B3: order, sampled codes, sampled gathered data
    codes, ids = ctx.get_sorted(device=True)
    assert bool((codes[1:] > codes[:-1]).all())
    assert bool((torch.sort(ids).values == torch.arange(n, device=dev)).all())
    ks = np.sort(rng.choice(n, 4096, replace=False))
    kt = torch.from_numpy(ks).to(dev)
    cell = ids[kt].cpu().numpy()
    lower = c["lower"][ids[kt]].cpu().numpy().astype(np.uint32)
    level = c["level"][ids[kt]].cpu().numpy().astype(np.uint32)
    half = ((np.uint32(1) << level) >> np.uint32(1))[:, None]
    assert np.array_equal(o.hilbert_encode(lower + half, int(info["bits"])), codes[kt].cpu().numpy().astype(np.uint64))
    lv_s, sc_s = ctx.get_sorted_data(device=True)
    assert np.array_equal(lv_s[kt].cpu().numpy(), level.astype(np.uint8))
    vals = scal[:, ids[kt]].cpu().numpy()          # M x 4096, input values of the sampled cells
    assert np.array_equal(sc_s[:, kt].cpu().numpy().view(np.uint32), vals.view(np.uint32))
    del codes, sc_s
    # ---- U0: maxV (R2 from the data ranges) and s
    alpha = np.ascontiguousarray(tfs[:, :, 3])
    mv = float(o.lib().or_maxv_approx(0, M, 256, o._p(alpha), o._p(vmin), o._p(vmax), o._p(lo), o._p(inv)))
    assert f32(info["maxV"]) == f32(mv)
    Lmax = int(c["level"].max().item())
    s = o.shift(n, Lmax, 1.0)
    assert info["shift"] == s
    # ---- U1, U2: sampled q from the oracle, one cell at a time
    Q = ctx.get_prefix()
    assert int(Q[-1]) == info["Qtot"]
    for j, k in enumerate(ks):
        one = np.ascontiguousarray(vals[:, j].reshape(M, 1))
        V = float(o.lib().or_variation(0, 1, M, 256, o._p(one), o._p(alpha), o._p(lo), o._p(inv)))
        f = o.importance(V, mv, int(level[j]), 1.0, 0.025)
        q = int(Q[k]) - (int(Q[k - 1]) if k else 0)
        assert q == o.fixed(f, s), (k, q, o.fixed(f, s))
    # ---- U3: bin ranges
    blo, bhi = ctx.get_bin_ranges(W)
    assert blo[0] == 0 and bhi[W - 1] == n - 1 and np.all(bhi >= blo)
    assert np.all((blo[1:] == bhi[:-1]) | (blo[1:] == bhi[:-1] + 1))
    assert np.array_equal(out["count"][0].astype(np.int64), (bhi - blo + 1).astype(np.int64))
    Qtot = int(Q[-1])
    checked = 0
    for x in np.sort(rng.choice(np.arange(1, W - 1), 16, replace=False)):
        a, b = int(blo[x]), int(bhi[x])
        if a < 1 or b + 1 >= n:
            continue
        # O13 on the cells around the pixel's ends: lo is the first cell reaching x (the one
        # before it ends below x), hi the last cell starting at or before x
        b1a, b2a = o.bins_ext(np.array([Q[a - 1], Q[a]], np.uint64), int(Q[a - 2]) if a >= 2 else 0, Qtot, W)
        b1b, b2b = o.bins_ext(np.array([Q[b], Q[b + 1]], np.uint64), int(Q[b - 1]), Qtot, W)
        assert b2a[0] < x <= b2a[1] and b1b[0] <= x < b1b[1], (x, b1a, b2a, b1b, b2b)
        checked += 1
    assert checked >= 8
    # ---- U4, U5: sampled pixels, per member (t by O7, pinned to the oracle's function)
    for m in range(M):   # pin the vectorised O7 to the oracle's own function
        tt = t_of(vals[m, :64], lo[m], inv[m])
        assert np.array_equal(tt, np.array([o.normalize(float(v), float(lo[m]), float(inv[m])) for v in vals[m, :64]], f32))
    for x in rng.choice(W, 4, replace=False):
        a, b = int(blo[x]), int(bhi[x])
        cells = ids[a:b + 1]
        for m in range(M):
            t = t_of(scal[m, cells].cpu().numpy(), lo[m], inv[m])
            v = out[m, x]
            assert v["t_min"] == t.min() and v["t_max"] == t.max()
            mean = t.astype(np.float64).mean()
            assert abs(float(v["t_mean"]) - mean) <= 1e-5 * max(abs(mean), 1e-30)
            assert v["y"] == f32(o.sample(tfs[m, :, 3], float(v["t_mean"])))
    ctx.close()
