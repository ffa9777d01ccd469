"""The distributed build and the sharded TF update through the C ABI on one GPU: G contexts in
an in-process group (dvl.LocalGroup, driven by G host threads: the library's stand-in for an
NCCL communicator, same code above the transport), each given a slice of the input order --
round robin, or uneven with an empty rank.  dvl_build runs the whole Hilbert-key sample
sort in the library (SURVEY 8(e) "Build"); afterwards each context must hold one contiguous
piece of the global curve order whose union equals the oracle's one-process build (codes,
input ids, levels, scalars), and get_polylines -- the sharded edit with both exchanges in
the library -- must equal the oracle and a one-context run, over a run of edits of one
member (edit-cache mode).
"""
import threading

import numpy as np
import pytest

from oracle import oracle as o
import synth

from tests.test_gpu_parity import check_update, octree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dvl():
    import paper_2306_11612_b200 as m
    m.load()
    return m


def run_threads(fns):
    errs = [None] * len(fns)
    outs = [None] * len(fns)

    def wrap(i):
        try:
            outs[i] = fns[i]()
        except BaseException as e:   # noqa: BLE001
            errs[i] = e

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    return outs, errs


def slices(n, G, kind, rng):
    if kind == "round_robin":
        return [np.arange(r, n, G) for r in range(G)]
    perm = rng.permutation(n)
    cuts = [0, 0] + sorted(rng.choice(np.arange(1, n), G - 2, replace=False).tolist()) + [n]
    if G == 2:
        cuts = [0, 0, n]
    return [np.sort(perm[cuts[r]:cuts[r + 1]]) for r in range(G)]   # rank 0 holds nothing


def build_group(dvl, G, lower, level, scal, parts, **kw):
    grp = dvl.LocalGroup(G)
    ctxs = [dvl.Context(device=0, **kw) for _ in range(G)]
    for r, c in enumerate(ctxs):
        c.set_local_comm(grp, r)
    _, errs = run_threads([lambda r=r: ctxs[r].build(lower[parts[r]], level[parts[r]],
                                                      np.ascontiguousarray(scal[:, parts[r]]))
                           for r in range(G)])
    return ctxs, errs


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("kind,pass2", [("round_robin", None), ("uneven", None), ("round_robin", "jobs")])
def test_library_distributed_build_and_sharded_edits(dvl, G, kind, pass2):
    lower, level = octree(64, 3, 20 + G)
    n, M, W = len(level), 4, 300
    rng = np.random.default_rng(G)
    scal = rng.standard_normal((M, n)).astype(np.float32)
    parts = slices(n, G, kind, rng)
    ctxs, errs = build_group(dvl, G, lower, level, scal, parts, pass2=pass2)
    for e in errs:
        if e is not None:
            raise e
    B = o.build(lower, level, scal)
    order = np.concatenate(parts)            # global input id -> input index
    srt = [c.get_sorted() for c in ctxs]
    assert np.array_equal(np.concatenate([s[0] for s in srt]), B.codes)
    assert np.array_equal(order[np.concatenate([s[1] for s in srt]).astype(np.int64)], B.perm.astype(np.int64))
    data = [c.get_sorted_data() for c in ctxs]
    assert np.array_equal(np.concatenate([d[0] for d in data]), B.level_s)
    assert np.array_equal(np.concatenate([d[1] for d in data], axis=1).view(np.uint32), B.scal_s.view(np.uint32))
    shards = [c.shard() for c in ctxs]
    sizes = [len(s[0]) for s in srt]
    assert [s["cell_offset"] for s in shards] == np.cumsum([0] + sizes)[:-1].tolist()
    assert all(s["n_global"] == n and s["lmax_global"] == B.Lmax for s in shards)
    assert min(sizes) > 0
    # sharded edits: every rank's get_polylines runs both exchanges in the library
    tfs = np.stack([synth.random_tf(70 + m, 256, member=m) for m in range(M)])
    one = dvl.Context(device=0)
    one.build(lower, level, scal)
    for m in range(M):
        one.update_tf(m, tfs[m])
        for c in ctxs:
            c.update_tf(m, tfs[m])
    for e in range(3):
        if e:
            tfs[0] = synth.tf_edit(5, e)
            one.update_tf(0, tfs[0])
            for c in ctxs:
                c.update_tf(0, tfs[0])
        outs, errs = run_threads([lambda c=c: c.get_polylines(W) for c in ctxs])
        for err in errs:
            if err is not None:
                raise err
        U = o.update(B, tfs, W)
        single = one.get_polylines(W)
        for out in outs:
            assert np.array_equal(out.view(np.uint8), outs[0].view(np.uint8))
            for k in ("count", "t_min", "t_max"):
                assert np.array_equal(out[k], U.vertices[k]) and np.array_equal(out[k], single[k])
            rel = np.abs(out["t_mean"].astype(np.float64) - U.vertices["t_mean"]) / np.maximum(U.vertices["t_mean"], 1e-30)
            assert rel.max() <= 1e-5
        # brushing on a sharded dataset (collective): every rank gets the ROI's codes
        brs, errs = run_threads([lambda c=c: c.brush(W, 40, 90) for c in ctxs])
        for err in errs:
            if err is not None:
                raise err
        for br in brs:
            assert (br["first"], br["last"]) == (int(U.lo[40]), int(U.hi[90]))
            assert (br["code_first"], br["code_last"]) == (int(B.codes[br["first"]]), int(B.codes[br["last"]]))
        # each shard's prefix of its own cells (shard-relative) plus the earlier shards' total
        # is the global Q (Eq. 4)
        for c, sh in zip(ctxs, shards):
            off = sh["cell_offset"]
            q = c.get_prefix().astype(object) + (int(U.Q[off - 1]) if off else 0)
            assert np.array_equal(q.astype(np.uint64), U.Q[off:off + len(q)])
    for c in ctxs + [one]:
        c.close()


@pytest.mark.parametrize("G", [2, 3])
def test_overlap_across_ranks_fails_everywhere(dvl, G):
    """A duplicate cell held by two different ranks: every rank returns DVL_E_OVERLAP."""
    lower, level = octree(32, 2, 7)
    n = len(level)
    scal = np.random.default_rng(1).standard_normal((2, n)).astype(np.float32)
    parts = [np.arange(r, n, G) for r in range(G)]
    parts[1] = np.concatenate([parts[1], parts[0][:1]])     # rank 1 repeats a cell of rank 0
    ctxs, errs = build_group(dvl, G, lower, level, scal, parts)
    assert all(e is not None and getattr(e, "status", "") == "DVL_E_OVERLAP" for e in errs), errs
    for c in ctxs:
        c.close()


def test_u64_keys_and_lsd_combine(dvl):
    """3b > 36 (E = 2^13): the received runs are combined by the onesweep LSD sort."""
    from tests.test_gpu_parity import sparse_cells
    lower, level = sparse_cells(1 << 13, 20000, 3, Lmax=4)
    n = len(level)
    scal = np.random.default_rng(2).standard_normal((3, n)).astype(np.float32)
    G = 3
    parts = [np.arange(r, n, G) for r in range(G)]
    ctxs, errs = build_group(dvl, G, lower, level, scal, parts)
    for e in errs:
        if e is not None:
            raise e
    B = o.build(lower, level, scal)
    assert B.b == 13
    assert np.array_equal(np.concatenate([c.get_sorted()[0] for c in ctxs]), B.codes)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("M,generic", [(17, False), (3, True)])
def test_distributed_generic_path_and_width_changes(dvl, M, generic):
    """M > 16 (the portable update kernels) and the forced generic path in a distributed
    build; sharded edits at several W on one group (W shrinks and grows)."""
    lower, level = octree(32, 3, 40 + M)
    n = len(level)
    scal = np.random.default_rng(M).standard_normal((M, n)).astype(np.float32)
    G = 3
    parts = [np.arange(r, n, G) for r in range(G)]
    ctxs, errs = build_group(dvl, G, lower, level, scal, parts, generic=generic)
    for e in errs:
        if e is not None:
            raise e
    B = o.build(lower, level, scal)
    assert np.array_equal(np.concatenate([c.get_sorted()[0] for c in ctxs]), B.codes)
    tfs = np.stack([synth.random_tf(90 + m, 256, member=m) for m in range(M)])
    for m in range(M):
        for c in ctxs:
            c.update_tf(m, tfs[m])
    for W in (700, 256, 1024, 5):
        outs, errs = run_threads([lambda c=c: c.get_polylines(W) for c in ctxs])
        for err in errs:
            if err is not None:
                raise err
        U = o.update(B, tfs, W)
        for out in outs:
            for k in ("count", "t_min", "t_max"):
                assert np.array_equal(out[k], U.vertices[k]), (W, k)
    for c in ctxs:
        c.close()


def test_distributed_exact_maxv(dvl):
    """DVL_MAXV_EXACT on shards: max(V_h) over every shard's cells (an all_reduce MAX inside
    the library; TF installs are then collective), equal to the one-context result."""
    lower, level = octree(32, 3, 77)
    n, M, W, G = len(level), 3, 400, 2
    scal = np.random.default_rng(77).standard_normal((M, n)).astype(np.float32)
    parts = [np.arange(r, n, G) for r in range(G)]
    ctxs, errs = build_group(dvl, G, lower, level, scal, parts)
    for e in errs:
        if e is not None:
            raise e
    B = o.build(lower, level, scal)
    tfs = np.stack([synth.random_tf(300 + m, 256, member=m) for m in range(M)])
    _, errs = run_threads([lambda c=c: c.set_params(1.0, 0.025, "exact") for c in ctxs])
    assert all(e is None for e in errs), errs
    for m in range(M):
        _, errs = run_threads([lambda c=c, m=m: c.update_tf(m, tfs[m]) for c in ctxs])
        assert all(e is None for e in errs), errs
    outs, errs = run_threads([lambda c=c: c.get_polylines(W) for c in ctxs])
    assert all(e is None for e in errs), errs
    U = o.update(B, tfs, W, mode="exact")
    for c in ctxs:
        assert np.float32(c.info()["maxV"]) == np.float32(U.maxV)
    for out in outs:
        for k in ("count", "t_min", "t_max"):
            assert np.array_equal(out[k], U.vertices[k])
    for c in ctxs:
        c.close()
