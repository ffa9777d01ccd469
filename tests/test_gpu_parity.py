"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bit-exact on every integer / index output (codes, permutation, levels, scalars in
curve order, maxV, shift, Q, bin ranges, counts) and on min/max; means within 1e-5
relative (north_star); y/rgb equal the oracle's TF sample at the GPU's mean, bit for bit,
and are within the propagated tolerance of the oracle's y."""
import numpy as np
import pytest

from oracle import oracle as o
import synth

pytestmark = pytest.mark.gpu

f32 = np.float32


@pytest.fixture(scope="module")
def dvl():
    import paper_2306_11612_b200 as m
    m.load()
    return m


def make_ctx(dvl, generic=False):
    """generic: a bool, or a path name of PATHS ("jobs": the TMA path with pass 2 in its
    many-jobs form, agg_jobs + the job list, forced at any size)."""
    if isinstance(generic, str):
        return dvl.Context(device=0, generic=generic == "generic",
                           pass2="jobs" if generic == "jobs" else None)
    return dvl.Context(device=0, generic=generic)


PATHS = ["tma", "generic", "jobs"]


# ------------------------------------------------------------------------ fixtures
def octree(E, Lmax, seed, p=0.45):
    rng = np.random.default_rng(seed)
    G = E >> Lmax
    lower, level = synth.uniform_cells(G)
    lower = (lower << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(level), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < p)
        lower, level = synth.refine(lower, level, mask)
    perm = rng.permutation(len(level))
    return lower[perm], level[perm]


def sparse_cells(E, n, seed, Lmax=3):
    """n non-overlapping cells scattered in a large grid (u64 keys when 3b > 32)."""
    rng = np.random.default_rng(seed)
    blocks = E >> Lmax
    ids = rng.choice(blocks ** 3, size=n, replace=False)
    bx, by, bz = ids % blocks, (ids // blocks) % blocks, ids // blocks ** 2
    level = rng.integers(0, Lmax + 1, size=n).astype(np.uint8)
    w = 1 << Lmax
    lower = np.stack([bx, by, bz], 1).astype(np.uint32) * np.uint32(w)
    # place the level-L cell at an aligned spot inside its block
    off = (rng.integers(0, w, size=(n, 3)) >> level[:, None].astype(np.int64)) << level[:, None].astype(np.int64)
    lower = lower + off.astype(np.uint32)
    return lower, level


def scalars(n, M, seed, nan_frac=0.0):
    rng = np.random.default_rng(seed)
    s = (rng.standard_normal((M, n)) * rng.uniform(0.5, 3, (M, 1)) + rng.uniform(-2, 2, (M, 1))).astype(f32)
    if nan_frac:
        s[rng.random(s.shape) < nan_frac] = np.nan
    return s


def tfs_for(M, N, seed, same=False):
    tfs = np.stack([synth.random_tf(seed + (0 if same else m), N, member=m) for m in range(M)])
    return tfs


def run_gpu(dvl, lower, level, scal, tfs, W, P=1.0, eps=0.025, mode="conservative", domain=None,
            generic=False, scale="width"):
    ctx = make_ctx(dvl, generic)
    ctx.build(lower, level, scal)
    ctx.set_params(P, eps, mode)
    if scale != "width":
        ctx.set_level_scale(scale)
    N = tfs.shape[1]
    if N != 256:
        ctx.reset_tfs(N)
    M = scal.shape[0]
    if domain is not None:
        d = np.asarray(domain, f32).reshape(-1, 2)
        d = np.repeat(d, M, axis=0) if d.shape[0] == 1 else d
        for m in range(M):
            ctx.set_domain(m, float(d[m, 0]), float(d[m, 1]))
    for m in range(M):
        ctx.update_tf(m, tfs[m])
    out = ctx.get_polylines(W)
    res = dict(out=out, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(W),
               sorted=ctx.get_sorted(), data=ctx.get_sorted_data())
    ctx.close()
    return res


def check_update(U, B, tfs, g, W):
    info = g["info"]
    assert np.float32(info["maxV"]) == np.float32(U.maxV), (info["maxV"], U.maxV)
    assert info["shift"] == U.s
    assert info["Qtot"] == U.Qtot
    assert np.array_equal(g["Q"], U.Q)
    lo, hi = g["ranges"]
    assert np.array_equal(lo, U.lo) and np.array_equal(hi, U.hi)
    out, ref = g["out"], U.vertices
    assert np.array_equal(out["count"], ref["count"])
    assert np.array_equal(out["t_min"], ref["t_min"])
    assert np.array_equal(out["t_max"], ref["t_max"])
    rel = np.abs(out["t_mean"].astype(np.float64) - ref["t_mean"]) / np.maximum(np.abs(ref["t_mean"]), 1e-30)
    bad = rel > 1e-5
    assert not bad.any(), (rel.max(), np.argwhere(bad)[:5])
    # y/rgb: the TF applied to the GPU mean, bit for bit (independent oracle sampler)
    M = out.shape[0]
    for m in range(M):
        for x in range(0, W, max(1, W // 64)):
            mu = float(out["t_mean"][m, x])
            assert out["y"][m, x] == f32(o.sample(tfs[m, :, 3], mu))
            assert out["r"][m, x] == f32(o.sample(tfs[m, :, 0], mu))
            assert out["b"][m, x] == f32(o.sample(tfs[m, :, 2], mu))


def check_build(B, g):
    codes, ids = g["sorted"]
    assert np.array_equal(codes, B.codes)
    assert np.array_equal(ids, B.perm)
    lv, sc = g["data"]
    assert np.array_equal(lv, B.level_s)
    assert np.array_equal(sc.view(np.uint32), B.scal_s.view(np.uint32))
    info = g["info"]
    assert info["bits"] == B.b and info["extent"] == B.E and info["Lmax"] == B.Lmax


def parity(dvl, lower, level, scal, tfs, W, generic=False, **kw):
    B = o.build(lower, level, scal)
    U = o.update(B, tfs, W, **kw)
    g = run_gpu(dvl, lower, level, scal, tfs, W, generic=generic, **kw)
    check_build(B, g)
    check_update(U, B, tfs, g, W)
    return B, U, g


# --------------------------------------------------------------------------- tests
@pytest.mark.parametrize("path", PATHS)
def test_c1_uniform_64(dvl, path):
    c = synth.make_config("C1")
    tfs = np.stack([synth.tf_edit(1, 0, member=m) for m in range(c["M"])])
    parity(dvl, c["lower"], c["level"], c["scal"], tfs, c["W"], domain=c["domain"],
           generic=path)


@pytest.mark.parametrize("seed,E,Lmax,M,W", [(1, 32, 3, 4, 1024), (2, 64, 4, 1, 37), (3, 16, 2, 5, 3),
                                             (4, 64, 2, 8, 4096), (5, 32, 5, 16, 1000),
                                             (6, 16, 1, 17, 65536), (7, 32, 3, 33, 2),
                                             (8, 16, 2, 64, 300), (9, 64, 3, 2, 64),
                                             (10, 64, 4, 12, 2048)])
@pytest.mark.parametrize("path", PATHS)
def test_amr_octrees(dvl, seed, E, Lmax, M, W, path):
    lower, level = octree(E, Lmax, seed)
    scal = scalars(len(level), M, seed)
    tfs = tfs_for(M, 256, 100 + seed)
    parity(dvl, lower, level, scal, tfs, W, generic=path)


@pytest.mark.parametrize("P", [0.0, 1.0, 2.0, 3.0, 0.5, 2.5])
@pytest.mark.parametrize("eps", [0.0, 0.025, 0.25])
@pytest.mark.parametrize("path", PATHS)
def test_params(dvl, P, eps, path):
    lower, level = octree(32, 3, 11)
    scal = scalars(len(level), 4, 12)
    tfs = tfs_for(4, 64, 13)
    parity(dvl, lower, level, scal, tfs, 512, P=P, eps=eps, generic=path)


@pytest.mark.parametrize("P", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("path", PATHS)
def test_volume_scaled_importance(dvl, P, path):
    """f = (V/maxV 2^3L)^P, the cell-volume variant of Eq. 3."""
    lower, level = octree(32, 3, 90)
    scal = scalars(len(level), 4, 91)
    parity(dvl, lower, level, scal, tfs_for(4, 256, 92), 700, generic=path, P=P,
           scale="volume")


@pytest.mark.parametrize("mode", ["conservative", "per_entry", "exact"])
@pytest.mark.parametrize("same", [False, True])
def test_maxv_modes(dvl, mode, same):
    lower, level = octree(32, 2, 21)
    scal = scalars(len(level), 3, 22)
    tfs = tfs_for(3, 128, 23, same=same)
    parity(dvl, lower, level, scal, tfs, 700, mode=mode, domain=[[-3.0, 3.0]])


@pytest.mark.parametrize("n", [1, 2, 7, 255, 2047, 2049, 4095, 4097, 20000, 300001])
@pytest.mark.parametrize("path", PATHS)
def test_sizes_and_ragged_tails(dvl, n, path):
    lower, level = sparse_cells(256 if n < 100000 else 1024, n, n)
    scal = scalars(n, 3, n + 1)
    tfs = tfs_for(3, 256, n + 2)
    for W in ((5,) if n == 1 else (1024, 3, 65536)):
        parity(dvl, lower, level, scal, tfs, W, generic=path)


@pytest.mark.parametrize("E,seed", [(4096, 1), (2 ** 21, 2)])
def test_u64_keys(dvl, E, seed):
    lower, level = sparse_cells(E, 30000, seed, Lmax=4)
    scal = scalars(len(level), 4, seed)
    tfs = tfs_for(4, 256, seed)
    B, _, g = parity(dvl, lower, level, scal, tfs, 1024)
    assert g["info"]["key_bytes"] == 8


def test_tf_sizes(dvl):
    lower, level = octree(16, 2, 31)
    scal = scalars(len(level), 2, 32)
    for N in (2, 3, 4096):
        parity(dvl, lower, level, scal, tfs_for(2, N, 33), 256)


def test_nan_and_inf_scalars(dvl):
    lower, level = octree(16, 2, 41)
    scal = scalars(len(level), 3, 42, nan_frac=0.05)
    scal[1, :7] = np.inf
    scal[2, 3:9] = -np.inf
    parity(dvl, lower, level, scal, tfs_for(3, 256, 43), 128)


def test_repeated_edits_and_determinism(dvl):
    """C2-style repeated TF edits on one member; two runs give identical bits."""
    lower, level = octree(32, 3, 51)
    scal = scalars(len(level), 4, 52)
    B = o.build(lower, level, scal)
    ctx = make_ctx(dvl)
    ctx.build(lower, level, scal)
    tfs = tfs_for(4, 256, 53)
    for m in range(4):
        ctx.update_tf(m, tfs[m])
    for e in range(4):
        tfs[0] = synth.tf_edit(2, e)
        ctx.update_tf(0, tfs[0])
        a = ctx.get_polylines(1024)
        b = ctx.get_polylines(1024)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
        U = o.update(B, tfs, 1024)
        g = dict(out=a, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(1024))
        check_update(U, B, tfs, g, 1024)
    # changing W reruns only the reduction
    for W in (2, 4096, 333):
        a = ctx.get_polylines(W)
        U = o.update(B, tfs, W)
        g = dict(out=a, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(W))
        check_update(U, B, tfs, g, W)
    ctx.close()


@pytest.mark.parametrize("pass2", [None, "jobs"])
@pytest.mark.parametrize("M", [3, 4, 5, 8, 16])
def test_edit_cache_sequences(dvl, M, pass2):
    """The edit cache (repeated edits of one member read that member and the cached alpha
    range of the others): edit sequences that switch members, change a domain, reset the
    TFs and change P / eps in between, each checked against the oracle, and against a
    context with the cache disabled and the default pass 2 (bit for bit)."""
    lower, level = octree(32, 3, 60 + M)
    scal = scalars(len(level), M, 61 + M, nan_frac=0.01)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0, pass2=pass2)
    ctx.build(lower, level, scal)
    ref_ctx = dvl.Context(device=0, edit_cache=False)
    ref_ctx.build(lower, level, scal)
    tfs = tfs_for(M, 256, 62)
    for c in (ctx, ref_ctx):
        for m in range(M):
            c.update_tf(m, tfs[m])
    domain = [[float(np.nanmin(scal[m])), float(np.nanmax(scal[m]))] for m in range(M)]
    W = 700
    steps = [("edit", 0), ("edit", 0), ("edit", 0), ("edit", M - 1), ("edit", M - 1), ("edit", 0),
             ("domain", 1), ("edit", 0), ("edit", 0), ("params", 2.0), ("edit", 0), ("reset", None),
             ("edit", 1), ("edit", 1), ("params", 1.0), ("edit", 1)]
    P = 1.0
    for k, (op, arg) in enumerate(steps):
        for c in (ctx, ref_ctx):
            if op == "edit":
                tfs[arg] = synth.tf_edit(3, k, 256, member=arg)
                c.update_tf(arg, tfs[arg])
            elif op == "domain":
                lo, hi = domain[arg][0] + 0.25, domain[arg][1] - 0.25
                c.set_domain(arg, lo, hi)
            elif op == "params":
                P = arg
                c.set_params(P, 0.025, "conservative")
            elif op == "reset":
                c.reset_tfs(256)
        if op == "domain":
            domain[arg] = [domain[arg][0] + 0.25, domain[arg][1] - 0.25]
        if op == "reset":
            tfs = np.stack([o.identity_tf(256)] * M)
        a = ctx.get_polylines(W)
        b = ref_ctx.get_polylines(W)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (k, op)
        U = o.update(B, tfs, W, P=P, domain=np.array(domain, f32))
        g = dict(out=a, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(W))
        check_update(U, B, tfs, g, W)
    ctx.close()
    ref_ctx.close()


def test_errors(dvl):
    ctx = make_ctx(dvl)
    with pytest.raises(dvl.DvlError) as e:
        ctx.update_tf(0, synth.identity_tf())
    assert e.value.status == "DVL_E_STATE"
    with pytest.raises(dvl.DvlError) as e:
        ctx.build([[0, 0, 0], [0, 0, 0]], [0, 0], [[1.0, 2.0]])
    assert e.value.status == "DVL_E_OVERLAP"
    with pytest.raises(dvl.DvlError) as e:
        ctx.build([[0, 0, 0], [1, 1, 1]], [1, 0], [[1.0, 2.0]])
    assert e.value.status == "DVL_E_OVERLAP"
    with pytest.raises(dvl.DvlError) as e:
        ctx.build([[1, 0, 0]], [1], [[1.0]])
    assert e.value.status == "DVL_E_INVAL"
    with pytest.raises(dvl.DvlError) as e:
        ctx.build([[2 ** 21, 0, 0]], [0], [[1.0]])
    assert e.value.status == "DVL_E_RANGE"
    ctx.build([[0, 0, 0], [1, 0, 0]], [0, 0], [[1.0, 2.0]])
    with pytest.raises(dvl.DvlError) as e:
        ctx.get_polylines(1)
    assert e.value.status == "DVL_E_INVAL"
    with pytest.raises(dvl.DvlError) as e:
        ctx.update_tf(0, np.full((8, 4), 1.5, f32))
    assert e.value.status == "DVL_E_INVAL"
    with pytest.raises(dvl.DvlError) as e:
        ctx.set_params(17.0, 0.025)
    assert e.value.status == "DVL_E_INVAL"
    # eps = 0 and a constant TF: every weight is 0 -> degenerate
    ctx.set_params(1.0, 0.0)
    ctx.update_tf(0, np.zeros((256, 4), f32))
    with pytest.raises(dvl.DvlError) as e:
        ctx.get_polylines(16)
    assert e.value.status == "DVL_E_DEGENERATE"
    ctx.set_params(1.0, 0.025)
    ctx.get_polylines(16)
    ctx.close()


def test_device_buffers(dvl):
    """Inputs and outputs as device (torch) tensors give the same result as host arrays."""
    import torch
    lower, level = octree(32, 3, 61)
    scal = scalars(len(level), 4, 62)
    tfs = tfs_for(4, 256, 63)
    B = o.build(lower, level, scal)
    U = o.update(B, tfs, 1024)
    ctx = make_ctx(dvl)
    ctx.build(torch.from_numpy(lower.astype(np.int32)).cuda(), torch.from_numpy(level).cuda(),
              torch.from_numpy(scal).cuda())
    for m in range(4):
        ctx.update_tf(m, tfs[m])
    out = torch.empty(4 * 1024 * 8, dtype=torch.int32, device="cuda")
    ctx.get_polylines(1024, out=out)
    # no explicit synchronize: the binding orders the caller's current stream after the
    # context stream, so reading 'out' on the current stream sees the epilogue's writes
    got = out.cpu().numpy().view(dvl.VERTEX_DTYPE).reshape(4, 1024)
    assert np.array_equal(got["count"], U.vertices["count"])
    assert np.array_equal(got["t_min"], U.vertices["t_min"])
    ctx.close()


@pytest.mark.parametrize("name", ["C2"])
@pytest.mark.parametrize("path", PATHS)
def test_full_size_config(dvl, name, path):
    """BASELINE configs[1] at full size (~10.9 M cells) in the launch configuration the
    bench times: complete comparison (the oracle finishes it in seconds)."""
    c = synth.make_config(name)
    tfs = np.stack([synth.tf_edit(2, 0, member=m) for m in range(c["M"])])
    parity(dvl, c["lower"], c["level"], c["scal"], tfs, c["W"], domain=c["domain"],
           generic=path)





@pytest.mark.parametrize("path", PATHS)
def test_negative_zero_and_domain_edges(dvl, path):
    """v = -0.0 with a domain starting at +0.0 gives (-0 - 0) * inv = -0, which the O7
    clamp maps to +0; values at, below and above the domain bounds clamp to 0 and 1."""
    lower, level = octree(16, 2, 71)
    n = len(level)
    scal = np.abs(scalars(n, 3, 72)).astype(f32)
    scal[0, ::3] = -0.0
    scal[1, ::5] = 0.0
    scal[2, ::7] = 2.0
    scal[2, 1::7] = -1.0
    dom = np.array([[0.0, 2.0], [0.0, 1.5], [0.0, 2.0]], f32)
    parity(dvl, lower, level, scal, tfs_for(3, 256, 73), 64, domain=dom, generic=path)


@pytest.mark.parametrize("path", PATHS)
def test_width_shrinks_then_grows(dvl, path):
    """W = 1024, 512, 700, 2048, 3 on one context, with and without TF edits in between:
    the two alternating lo / hi copies must not carry first / last cells of an earlier,
    wider call into a later one."""
    lower, level = octree(32, 3, 81)
    scal = scalars(len(level), 4, 82)
    B = o.build(lower, level, scal)
    ctx = make_ctx(dvl, path)
    ctx.build(lower, level, scal)
    tfs = tfs_for(4, 256, 83)
    for m in range(4):
        ctx.update_tf(m, tfs[m])
    for k, W in enumerate((1024, 512, 700, 2048, 3, 1500, 1499, 4096)):
        if k % 2:
            tfs[0] = synth.tf_edit(4, k)
            ctx.update_tf(0, tfs[0])
        a = ctx.get_polylines(W)
        U = o.update(B, tfs, W)
        g = dict(out=a, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(W))
        check_update(U, B, tfs, g, W)
    ctx.close()


@pytest.mark.parametrize("mode", ["conservative", "per_entry"])
@pytest.mark.parametrize("path", PATHS)
def test_maxv_data_index_range(dvl, mode, path):
    """the max(V_h) approximation only visits the TF entries [i, j] that the data
    reach.  Domains twice as wide as the data put [i, j] strictly inside [0, N-1], and the
    TFs' alpha extremes outside it: the device's maxV must equal the oracle's and differ
    from the whole-table value."""
    lower, level = octree(32, 2, 24)
    n = len(level)
    rng = np.random.default_rng(25)
    M, N = 3, 64
    scal = np.stack([(2.0 + m * 0.5 + rng.random(n)).astype(f32) for m in range(M)])
    # member ranges [2,3], [2.5,3.5], [3,4] on the domain [0, 8] -> [i, j] ~ [15, 32] of 63
    tfs = tfs_for(M, N, 26)
    tfs[:, :8, 3] = 0.0
    tfs[:, -8:, 3] = 1.0
    tfs[:, 8:-8, 3] = np.clip(tfs[:, 8:-8, 3], 0.1, 0.9)
    B, U, g = parity(dvl, lower, level, scal, tfs, 700, mode=mode, domain=[[0.0, 8.0]],
                     generic=path)
    lo, _, inv = o.domains(B, [[0.0, 8.0]])
    ij = [o.index_range(float(B.vmin[m]), float(B.vmax[m]), float(lo[m]), float(inv[m]), N) for m in range(M)]
    assert min(i for i, _ in ij) > 8 and max(j for _, j in ij) < N - 9
    full = float(tfs[:, :, 3].max() - tfs[:, :, 3].min()) if mode == "conservative" else \
        float((tfs[:, :, 3].max(0) - tfs[:, :, 3].min(0)).max())
    assert g["info"]["maxV"] == U.maxV and U.maxV < full


def test_binding_validates_device_arguments(dvl):
    """The binding rejects device tensors of the wrong dtype / size instead of letting the
    C library misread them."""
    import torch
    lower, level = octree(16, 2, 62)
    scal = scalars(len(level), 2, 63)
    ctx = make_ctx(dvl)
    with pytest.raises(ValueError):
        ctx.build(torch.from_numpy(lower.astype(np.int64)).cuda(), torch.from_numpy(level).cuda(),
                  torch.from_numpy(scal).cuda())
    with pytest.raises(ValueError):
        ctx.build(torch.from_numpy(lower.astype(np.int32)).cuda(), torch.from_numpy(level).cuda(),
                  torch.from_numpy(scal.astype(np.float64)).cuda())
    ctx.build(torch.from_numpy(lower.astype(np.int32)).cuda(), torch.from_numpy(level).cuda(),
              torch.from_numpy(scal).cuda())
    with pytest.raises(ValueError):
        ctx.get_polylines(64, out=torch.empty(2 * 64 * 8 - 1, dtype=torch.int32, device="cuda"))
    ctx.close()


@pytest.mark.parametrize("sort", ["auto", "lsd"])
@pytest.mark.parametrize("E,Lmax,n", [(2, 1, None), (8, 2, None), (64, 3, None), (512, 4, None),
                                      (4096, 4, 50000)])
def test_sort_paths(dvl, sort, E, Lmax, n):
    """The bucket sort (3b <= 36) and the onesweep LSD sort give the oracle's order bit for
    bit, from one-bucket grids (b = 1, 3) to 2^24 buckets (b = 12, u64 keys)."""
    if n is None:
        lower, level = octree(E, Lmax, E + Lmax)
    else:
        lower, level = sparse_cells(E, n, 5, Lmax=Lmax)
    scal = scalars(len(level), 3, 9)
    B = o.build(lower, level, scal)
    ctx = dvl.Context(device=0, sort=sort)
    ctx.build(lower, level, scal)
    check_build(B, dict(sorted=ctx.get_sorted(), data=ctx.get_sorted_data(), info=ctx.info()))
    ctx.close()


@pytest.mark.parametrize("sort", ["auto", "lsd"])
def test_duplicate_and_overlap_detection_both_sorts(dvl, sort):
    """Duplicates inside one bucket (bitmap and comparison ranks) and nested cells are
    rejected with DVL_E_OVERLAP by either sort."""
    lower, level = octree(64, 3, 12)
    for dup in (0, 5):
        lo2 = np.concatenate([lower, lower[dup:dup + 1]])
        lv2 = np.concatenate([level, level[dup:dup + 1]])
        ctx = dvl.Context(device=0, sort=sort)
        with pytest.raises(dvl.DvlError) as e:
            ctx.build(lo2, lv2, scalars(len(lv2), 2, 1))
        assert e.value.status == "DVL_E_OVERLAP"
        ctx.close()
    # a level-0 cell inside a coarser one
    big = np.nonzero(level > 0)[0][0]
    lo3 = np.concatenate([lower, lower[big:big + 1]])
    lv3 = np.concatenate([level, np.zeros(1, np.uint8)])
    ctx = dvl.Context(device=0, sort=sort)
    with pytest.raises(dvl.DvlError) as e:
        ctx.build(lo3, lv3, scalars(len(lv3), 2, 1))
    assert e.value.status == "DVL_E_OVERLAP"
    ctx.close()


@pytest.mark.parametrize("pass2,extra", [("inline", 0), ("list", 1), ("jobs", 2)])
def test_launch_count_per_edit(dvl, pass2, extra):
    """dvl_get_timings counts every kernel of an edit (bench.py's gpu_launches): prologue,
    pass 1, pass 2 (agg_reduce; + bin_boundary when listed; + agg_jobs in the jobs form, whose
    boundary tiles are listed here: W > pass-1 tiles), epilogue."""
    lower, level = octree(32, 3, 91)
    scal = scalars(len(level), 4, 92)
    tfs = tfs_for(4, 256, 93)
    ctx = dvl.Context(device=0, pass2=pass2)
    ctx.build(lower, level, scal)
    for m in range(4):
        ctx.update_tf(m, tfs[m])
    ctx.get_polylines(300)
    ctx.timings()                      # resets the counter
    ctx.update_tf(0, synth.tf_edit(9, 1, 256, member=0))
    ctx.get_polylines(300)
    assert ctx.timings()["launches"] == 4 + extra
    ctx.close()
