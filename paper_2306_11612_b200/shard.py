"""Sharded TF update across ranks: one dvl context per GPU, each holding a
contiguous range of the global curve order.  Per edit the ranks exchange

  1. their fixed-point weight totals (all_gather of one u64 each): every shard derives its
     scan offset and the global Qtot on the device (dvl_shard_reduce);
  2. the per-pixel accumulators as three int64 planes merged with two all_reduces: MAX over
     the first two (the minima are exported negated) and SUM over the third (integers: the
     merged result is bit-identical to the unsharded one).

This module is plumbing only: the arithmetic of both steps runs in the library's kernels;
here are the collectives (torch.distributed, NCCL on GPUs, gloo on CPU) and the buffer views.
"""
from __future__ import annotations

import numpy as np


def export_layout(W: int, M: int):
    """Word offsets (start, stop) of the -MIN, MAX and SUM planes of an accumulator export."""
    mw = W + M * W
    return (0, mw), (mw, 2 * mw), (2 * mw, 2 * mw + 3 * M * W)


def split_planes(buf, W: int, M: int):
    (a, b), (c, d), (e, f) = export_layout(W, M)
    return buf[a:b], buf[c:d], buf[e:f]


def gather_totals(local_total, group=None):
    """all_gather of one int64 per rank -> tensor [world] in rank (= shard) order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = [torch.empty_like(local_total) for _ in range(world)]
    dist.all_gather(out, local_total, group=group)
    return torch.cat(out)


def merge_planes(mn, mx, sm, group=None):
    """In-place element-wise merge of plain MIN / MAX / SUM planes over all ranks (three
    collectives; used by the CPU decomposition test)."""
    import torch.distributed as dist
    dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)


def merge_export(buf, W: int, M: int, group=None):
    """In-place merge of an accumulator export over all ranks: one MAX all_reduce over the
    -MIN and MAX planes (contiguous), one SUM all_reduce over the SUM plane."""
    import torch.distributed as dist
    (_, b), (_, d), (e, f) = export_layout(W, M)
    dist.all_reduce(buf[:d], op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(buf[e:f], op=dist.ReduceOp.SUM, group=group)


def scan_offset(totals, rank: int):
    """Host mirror of the device offset rule (used by the CPU tests): sum of the earlier
    shards' totals and the global total."""
    t = [int(v) for v in totals]
    return sum(t[:rank]), sum(t)


class ShardedContext:
    """A dvl Context that is one shard of a dataset distributed over the ranks of `group`."""

    def __init__(self, ctx, group=None, native: bool = True):
        """native: the context gets its own NCCL communicator (dvl_set_comm) and each
        get_polylines is one library call that runs both exchanges itself; otherwise the
        exchanges are torch.distributed collectives between the library's shard calls."""
        import torch
        import torch.distributed as dist
        self.ctx, self.group = ctx, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._total = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self._bufs = {}
        self.native = False
        if native and dist.get_backend(group) == "nccl":
            from . import dvl as _dvl
            uid = torch.zeros(128, dtype=torch.uint8, device=self.dev)
            if self.rank == 0:
                uid.copy_(torch.frombuffer(bytearray(_dvl.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            ctx.set_comm(self.world, self.rank, bytes(uid.cpu().numpy().tobytes()))
            self.native = True

    def describe(self, n_local: int, lmax_local: int, vmin, vmax):
        """After the local build: agree on offsets, n, Lmax and member ranges."""
        import torch
        import torch.distributed as dist
        n = torch.tensor([n_local], dtype=torch.int64, device=self.dev)
        ns = gather_totals(n, self.group).cpu().numpy()
        off = int(ns[: self.rank].sum())
        lm = torch.tensor([lmax_local], dtype=torch.int64, device=self.dev)
        dist.all_reduce(lm, op=dist.ReduceOp.MAX, group=self.group)
        lo = torch.tensor(np.asarray(vmin, np.float32), device=self.dev)
        hi = torch.tensor(np.asarray(vmax, np.float32), device=self.dev)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.group)
        self.ctx.set_shard(off, int(ns.sum()), int(lm.item()), lo.cpu().numpy(), hi.cpu().numpy())
        return off, int(ns.sum())

    def get_polylines(self, W: int, out=None):
        import torch
        if self.native:   # both exchanges inside the library (one call)
            return self.ctx.get_polylines(W, out=out)
        if W not in self._bufs:
            self._bufs[W] = torch.empty(self.ctx.shard_export_words(W), dtype=torch.int64,
                                        device=self.dev)
        buf = self._bufs[W]
        self.ctx.shard_total(self._total)
        stream = torch.cuda.ExternalStream(self.ctx.stream)
        with torch.cuda.stream(stream):
            totals = gather_totals(self._total, self.group)
            self.ctx.shard_reduce(W, totals, self.rank, buf)
            merge_export(buf, W, self.ctx.M, group=self.group)
            return self.ctx.shard_finish(W, buf, out)
