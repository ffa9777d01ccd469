"""The distributed build's sample sort (paper_2306_11612_b200.dist_build) on CPU: world size 2
and 3 over gloo, every rank holding a round-robin slice of the input order (so the exchange
really moves cells), with a stand-in context whose local build is the oracle's definition
(O2-O4: centroid codes with the global b, stable sort by code).  The union of the ranks'
final sorted runs, in rank order, must equal the oracle's one-process build of all cells;
offsets, n and member ranges must be the global ones.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dataset(seed, E=32, Lmax=3, M=3):
    import synth
    rng = np.random.default_rng(seed)
    lower, level = synth.uniform_cells(E >> Lmax)
    lower = (lower << np.uint32(Lmax)).astype(np.uint32)
    level = np.full(len(level), Lmax, np.uint8)
    for L in range(Lmax, 0, -1):
        mask = (level == L) & (rng.random(len(level)) < 0.5)
        lower, level = synth.refine(lower, level, mask)
    scal = rng.standard_normal((M, len(level))).astype(np.float32)
    scal[0, :5] = np.nan
    return lower, level, scal


class OracleCtx:
    """The context calls distributed_build makes, with the oracle's build definition."""

    def __init__(self):
        self.bits = None

    def set_global_bits(self, b):
        self.bits = b

    def build(self, lower, level, scal):
        from oracle import oracle as o
        lower = lower.numpy().astype(np.uint32).reshape(-1, 3)
        level = level.numpy().astype(np.uint8)
        half = ((np.uint32(1) << level.astype(np.uint32)) >> np.uint32(1))[:, None]
        codes = o.hilbert_encode(lower + half, self.bits).astype(np.uint64)
        perm = np.argsort(codes, kind="stable")
        self.codes, self.perm = codes[perm], perm
        self.level_s, self.scal_s = level[perm], scal.numpy()[:, perm]
        self.n = len(level)

    def get_sorted(self, device=False):
        return (torch.from_numpy(self.codes.astype(np.int64)),
                torch.from_numpy(self.perm.astype(np.int64)))

    def get_sorted_data(self, device=False):
        return torch.from_numpy(self.level_s), torch.from_numpy(self.scal_s)

    def set_shard(self, offset, n_global, lmax, vmin, vmax):
        self.shard = (offset, n_global, lmax, np.asarray(vmin), np.asarray(vmax))


def _worker(rank, world, port, seed, results):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_11612_b200 import dist_build as db
    lower, level, scal = _dataset(seed)
    idx = np.arange(rank, len(level), world)          # round-robin slice of the input order
    ctx = OracleCtx()
    info = db.distributed_build(ctx, torch.from_numpy(lower[idx].astype(np.int32)),
                                torch.from_numpy(level[idx]), torch.from_numpy(scal[:, idx]),
                                db.TorchCollectives(), samples=64)
    results.put((rank, ctx.codes, ctx.level_s, ctx.scal_s, ctx.shard, info))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 7), (3, 8)])
def test_distributed_build_matches_one_process(world, seed):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as o
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lower, level, scal = _dataset(seed)
    B = o.build(lower, level, scal)
    codes = np.concatenate([r[1] for r in res])
    assert np.array_equal(codes, B.codes)
    assert np.array_equal(np.concatenate([r[2] for r in res]), B.level_s)
    assert np.array_equal(np.concatenate([r[3] for r in res], axis=1), B.scal_s, equal_nan=True)
    off = 0
    for r in res:
        offset, n_global, lmax, vmin, vmax = r[4]
        assert offset == off and n_global == B.n and lmax == B.Lmax
        assert np.array_equal(vmin, B.vmin) and np.array_equal(vmax, B.vmax)
        assert r[5]["bits"] == B.b
        off += len(r[1])
        assert len(r[1]) > 0
    # the exchange moved cells: every rank sent some to every other rank
    assert all(min(r[5]["sent"]) > 0 for r in res)


def test_helpers():
    from paper_2306_11612_b200 import dist_build as db
    assert db.global_bits(1) == 1 and db.global_bits(2) == 1 and db.global_bits(3) == 2
    assert db.global_bits(512) == 9 and db.global_bits(513) == 10
    # dyadic rule: an L=1 block [0, 8) then a cell at code 8 is fine, at code 7 overlaps
    assert db.dyadic_ok(5, 1, 8, 0) and not db.dyadic_ok(5, 1, 7, 0)
    s = db.splitters(torch.arange(12), 3, 4)
    assert s.tolist() == [4, 8]
