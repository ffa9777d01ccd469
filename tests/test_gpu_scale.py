"""GPU parity at size, in the launch configurations bench.py times.

Every test compares the CUDA path (through the C ABI) with the CPU oracle element by element
on the same seeded inputs: codes, permutation, maxV, s, Q, bin ranges, counts and min/max
bit-exact, means within 1e-5 relative.

* C2 at full size (10.9 M cells, BASELINE configs[1]) with a run of consecutive edits of
  member 0 -- the edit-cache pass 1 (13 B/cell) whose stage ring wraps many times per CTA,
  exactly the step bench.py times -- in both pass-2 launch modes.
* The C3 recipe (5 levels, 8 fields, per-field domains, W = 4096) on a 1024^3 grid: pass 2
  forced inline and listed (bin_boundary), at M = 8.
* The C4 recipe (uniform, 16 members) on 256^3 = 16.8 M cells: the MR = 16 TMA kernels
  (8 consumer warps, one CTA per SM) with edit-cache edits, both pass-2 modes.
* The C5 recipe (4096^3 logical grid, b = 12: 36-bit u64 keys, 5 sort passes, 5 levels,
  rho = 0.32) on a slab of its coarse blocks, ~16 M cells.
"""
import numpy as np
import pytest

from oracle import oracle as o
import synth

from tests.test_gpu_parity import check_build, check_update

pytestmark = pytest.mark.gpu

_DATA = {}


@pytest.fixture(scope="module")
def dvl():
    import paper_2306_11612_b200 as m
    m.load()
    return m


def dataset(key, make):
    if key not in _DATA:
        c = make()
        _DATA[key] = (c, o.build(c["lower"], c["level"], c["scal"]))
    return _DATA[key]


def run_sequence(dvl, c, B, edits, modes, config_index):
    """Build one context per pass-2 mode, install every member's TF, then edit member 0
    `edits` times; after every edit each context is compared with the oracle."""
    M, W = c["M"], c["W"]
    tfs = np.stack([synth.tf_edit(config_index, 0, member=m) for m in range(M)])
    ctxs = []
    for mode in modes:
        ctx = dvl.Context(device=0, pass2=mode)
        ctx.build(c["lower"], c["level"], c["scal"])
        for m in range(M):
            if c["domain"] is not None:
                ctx.set_domain(m, float(c["domain"][m, 0]), float(c["domain"][m, 1]))
            ctx.update_tf(m, tfs[m])
        ctxs.append(ctx)
    g0 = dict(sorted=ctxs[0].get_sorted(), data=ctxs[0].get_sorted_data(), info=ctxs[0].info())
    check_build(B, g0)
    for e in range(edits + 1):
        if e:
            tfs[0] = synth.tf_edit(config_index, 100 + e, member=0)
            for ctx in ctxs:
                ctx.update_tf(0, tfs[0])
        U = o.update(B, tfs, W, domain=c["domain"])
        for ctx in ctxs:
            out = ctx.get_polylines(W)
            g = dict(out=out, info=ctx.info(), Q=ctx.get_prefix(), ranges=ctx.get_bin_ranges(W))
            check_update(U, B, tfs, g, W)
    for ctx in ctxs:
        ctx.close()


def test_c2_full_size_edit_cache_sequence(dvl):
    c, B = dataset("C2", lambda: synth.make_config("C2"))
    assert B.n > 10_000_000
    run_sequence(dvl, c, B, edits=5, modes=[None, "list", "jobs"], config_index=1)


def test_c3_recipe_pass2_inline_listed_and_jobs(dvl):
    c, B = dataset("C3s", lambda: synth.make_config("C3", scale_E=1024))
    assert B.n > 12_000_000 and c["M"] == 8
    run_sequence(dvl, c, B, edits=2, modes=["inline", "list", "jobs"], config_index=2)


def test_c4_recipe_sixteen_members(dvl):
    c, B = dataset("C4s", lambda: synth.make_config("C4", scale_E=256))
    assert B.n == 256 ** 3 and c["M"] == 16
    run_sequence(dvl, c, B, edits=2, modes=["inline", "list", "jobs"], config_index=3)


def test_c5_recipe_u64_keys(dvl):
    c, B = dataset("C5s", lambda: synth.make_config("C5", box=(256, 128, 8)))
    assert B.n > 15_000_000 and B.b == 12 and B.Lmax == 4
    run_sequence(dvl, c, B, edits=2, modes=[None, "jobs"], config_index=4)
    ctx = dvl.Context(device=0)
    ctx.build(c["lower"], c["level"], c["scal"])
    assert ctx.info()["key_bytes"] == 8
    ctx.close()
