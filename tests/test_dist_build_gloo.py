"""The decomposition of the distributed build (the library's Hilbert-key sample sort,
SURVEY 8(e) "Build") on CPU over gloo, world size 2-4, every rank holding a round-robin
slice of the input order (so the exchange really moves cells): global b from the
all-reduced extent, local sorted runs (oracle definition O2-O4), regular samples, the
library's own splitter rule (dvl_select_splitters, host code), lower-bound send ranges,
the exchange, and the combination of the received runs.  The union of the ranks' runs in
rank order must equal the oracle's one-process build: codes, input ids, levels, scalars.
(The device steps run in tests/test_gpu_dist_build.py through the C ABI.)
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


def _lower_bounds(run, spl):
    """The library's send ranges: rank p gets the codes in [spl[p-1], spl[p])."""
    return [0] + [int(np.searchsorted(run, v, side="left")) for v in spl] + [len(run)]


def _worker(rank, world, port, seed, results):
    """One rank of the decomposition the library's distributed build runs (dbuild.cu /
    api.cu dist_build), with the per-rank arithmetic by the oracle (O1-O5) and the splitter
    rule by the library's host function (dvl_select_splitters)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2306_11612_b200 as dvl
    from oracle import oracle as o
    lower, level, scal = _dataset(seed)
    idx = np.arange(rank, len(level), world)          # round-robin slice of the input order
    lo, lv, sc = lower[idx], level[idx], scal[:, idx]
    M = sc.shape[0]
    # 0. global extent / Lmax (MAX) and n (SUM) -> one code width b for every rank
    w = (np.int64(1) << lv.astype(np.int64))[:, None]
    v = torch.tensor([int((lo.astype(np.int64) + w).max()), int(lv.max())], dtype=torch.int64)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    nl = torch.tensor([len(lv)], dtype=torch.int64)
    nin = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(nin, nl)
    nin = [int(x) for x in nin]
    b = max(1, int(np.ceil(np.log2(int(v[0])))))
    # 1. local sort of the slice (oracle definition: centroid codes with the global b)
    half = ((np.uint32(1) << lv.astype(np.uint32)) >> np.uint32(1))[:, None]
    codes = o.hilbert_encode(lo + half, b).astype(np.uint64)
    order = np.argsort(codes, kind="stable")
    run = codes[order]
    gid = (sum(nin[:rank]) + order).astype(np.int64)
    # 2. regular samples, all-gathered; the library's splitter rule
    S = 64
    s = min(S, len(run))
    samp = np.full(S, np.iinfo(np.uint64).max, np.uint64)
    samp[:s] = run[(np.arange(s, dtype=np.int64) * len(run)) // s]
    allsamp = [torch.zeros(S, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allsamp, torch.from_numpy(samp.view(np.int64)))
    spl = dvl.select_splitters(np.stack([a.numpy().view(np.uint64) for a in allsamp]), nin, S)
    # 3. send ranges and the count matrix
    bnd = _lower_bounds(run, spl)
    sendc = torch.tensor([bnd[p + 1] - bnd[p] for p in range(world)], dtype=torch.int64)
    mat = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(mat, sendc)
    # 4. exchange (gloo has no all_to_all: all_gather the padded per-rank blocks)
    payload = np.concatenate([run.view(np.int64)[:, None], gid[:, None], lv[order].astype(np.int64)[:, None],
                              sc[:, order].T.view(np.int32).astype(np.int64)], axis=1)
    cap = max(int(m.max()) for m in mat)
    block = torch.zeros((world, max(cap, 1), payload.shape[1]), dtype=torch.int64)
    for p in range(world):
        block[p, : bnd[p + 1] - bnd[p]] = torch.from_numpy(payload[bnd[p]: bnd[p + 1]])
    parts = [torch.zeros_like(block) for _ in range(world)]
    dist.all_gather(parts, block)
    recv = np.concatenate([parts[p][rank, : int(mat[p][rank])].numpy() for p in range(world)])
    # 5. combine the received sorted runs (distinct codes: their order is the code order)
    recv = recv[np.argsort(recv[:, 0].view(np.uint64), kind="stable")]
    results.put((rank, recv[:, 0].view(np.uint64), recv[:, 1], recv[:, 2].astype(np.uint8),
                 recv[:, 3:].astype(np.int32).view(np.float32).T.copy(), b,
                 [int(x) for x in sendc]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 7), (3, 8), (4, 9)])
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
    # global ids -> input indices: the slices' concatenation in rank order
    order = np.concatenate([np.arange(r, len(level), world) for r in range(world)])
    assert np.array_equal(np.concatenate([r[1] for r in res]), B.codes)
    assert np.array_equal(order[np.concatenate([r[2] for r in res])], B.perm.astype(np.int64))
    assert np.array_equal(np.concatenate([r[3] for r in res]), B.level_s)
    assert np.array_equal(np.concatenate([r[4] for r in res], axis=1), B.scal_s, equal_nan=True)
    assert all(r[5] == B.b for r in res) and all(len(r[1]) > 0 for r in res)
    # the exchange moved cells: every rank sent some to every other rank
    assert all(min(r[6]) > 0 for r in res)
