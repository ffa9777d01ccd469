"""Distributed build: Hilbert-key sample sort across ranks ("Build").

Each rank starts with an arbitrary slice of the cells and ends with the cells of one
contiguous range of the global curve order, built (encoded, sorted, gathered, validated) in
its own dvl context and described as a shard of the global dataset (dvl_set_shard):

  0. all_reduce MAX of the extent and Lmax, SUM of n -> the global code width b (codes depend
     on b, so every rank must encode with the same b: dvl_set_global_bits);
  1. local build of the rank's slice (the library's encode + onesweep sort);
  2. S regularly spaced keys of the local sorted run, all_gather'ed; every rank sorts the G*S
     samples identically and takes the splitters at ranks k*S (k = 1..G-1);
  3. destination rank of every sorted cell by searchsorted on the splitters; all_gather of
     the G x G send counts;
  4. all_to_all of the cells (lower corner, level, member scalars) in curve order;
  5. local build of the received cells (one contiguous key range per rank, so rank order is
     curve order); the dyadic overlap rule is checked across the rank boundaries too;
  6. all_gather of n_g -> each rank's global cell offset; MIN / MAX of the member ranges.

Keys are unique for valid input, so the result is identical to a one-GPU build of the union.
The per-cell work (encode, sort, gather) runs in the library's kernels; this module holds
the collectives (NCCL over NVLink on GPUs) and the bookkeeping.  `Collectives` abstracts
them so that the same code runs over torch.distributed and, for tests on one GPU, over G
threads in one process (`ThreadCollectives`).
"""
from __future__ import annotations

import threading

import numpy as np
import torch

SAMPLES = 1024


class Collectives:
    """The four collectives the build needs (tensor arguments on the caller's device)."""

    rank: int
    world: int

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        raise NotImplementedError

    def all_reduce(self, t: torch.Tensor, op: str) -> torch.Tensor:
        raise NotImplementedError

    def all_to_all(self, send: torch.Tensor, send_counts: list[int],
                   recv_counts: list[int]) -> torch.Tensor:
        """Rows [sum(send_counts[:j]), +send_counts[j]) of `send` go to rank j; returns the
        received rows in rank order (recv_counts[j] rows from rank j)."""
        raise NotImplementedError


class TorchCollectives(Collectives):
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def all_gather(self, t):
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def all_reduce(self, t, op):
        ops = {"min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX,
               "sum": self.dist.ReduceOp.SUM}
        self.dist.all_reduce(t, op=ops[op], group=self.group)
        return t

    def all_to_all(self, send, send_counts, recv_counts):
        send = send.contiguous()
        shape = (sum(recv_counts),) + tuple(send.shape[1:])
        if self.nccl:
            out = torch.empty(shape, dtype=send.dtype, device=send.device)
            self.dist.all_to_all_single(out, send, output_split_sizes=recv_counts,
                                        input_split_sizes=send_counts, group=self.group)
            return out
        # gloo has no all_to_all: all_gather of [world, cap] padded blocks (cap = the largest
        # count of any rank), keep the rows meant for this rank
        cap_t = torch.tensor([max(send_counts) if send_counts else 0], dtype=torch.int64)
        self.dist.all_reduce(cap_t, op=self.dist.ReduceOp.MAX, group=self.group)
        cap = max(int(cap_t.item()), 1)
        offs = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        block = torch.zeros((self.world, cap) + tuple(send.shape[1:]), dtype=send.dtype,
                            device=send.device)
        for j in range(self.world):
            block[j, : send_counts[j]] = send[offs[j]: offs[j + 1]]
        parts = self.all_gather(block)
        return torch.cat([parts[j][self.rank, : recv_counts[j]] for j in range(self.world)])


class ThreadCollectives(Collectives):
    """G ranks as G threads of one process (tests on one GPU): shared slots + a barrier."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.slots = [None] * world
            self.barrier = threading.Barrier(world)

    def __init__(self, shared: "_Shared", rank: int):
        self.s, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def group(cls, world):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _exchange(self, obj):
        self.s.barrier.wait()
        self.s.slots[self.rank] = obj
        self.s.barrier.wait()
        out = list(self.s.slots)
        self.s.barrier.wait()
        return out

    def all_gather(self, t):
        torch.cuda.synchronize() if t.is_cuda else None
        return [x.clone() for x in self._exchange(t)]

    def all_reduce(self, t, op):
        parts = self.all_gather(t)
        st = torch.stack(parts)
        r = {"min": st.min(0).values, "max": st.max(0).values, "sum": st.sum(0)}[op]
        t.copy_(r)
        return t

    def all_to_all(self, send, send_counts, recv_counts):
        if send.is_cuda:
            torch.cuda.synchronize()
        offs = np.concatenate([[0], np.cumsum(send_counts)])
        parts = self._exchange((send, offs))
        got = [p[0][p[1][self.rank]: p[1][self.rank + 1]].clone() for p in parts]
        assert [g.shape[0] for g in got] == list(recv_counts)
        return torch.cat(got)


def _extent_and_lmax(lower: torch.Tensor, level: torch.Tensor):
    if level.numel() == 0:
        return 0, 0
    w = torch.ones_like(level, dtype=torch.int64) << level.to(torch.int64)
    ext = (lower.to(torch.int64) + w[:, None]).max()
    return int(ext.item()), int(level.max().item())


def global_bits(extent: int) -> int:
    """b = max(1, ceil(log2 E)) (O1)."""
    b = 1
    while (1 << b) < extent:
        b += 1
    return b


def splitters(samples: torch.Tensor, world: int, per_rank: int) -> torch.Tensor:
    """G-1 splitters at ranks k * per_rank of the sorted union of all samples."""
    s, _ = torch.sort(samples)
    idx = torch.arange(1, world, device=s.device) * per_rank
    return s[idx.clamp(max=max(s.numel() - 1, 0))] if s.numel() else s


def dyadic_ok(code_a: int, level_a: int, code_b: int, level_b: int) -> bool:
    """O4 across a boundary: the dyadic block of a (code with its low 3L bits cleared, length
    8^L) ends at or before the block of b starts."""
    start_a = code_a & ~((1 << (3 * level_a)) - 1)
    start_b = code_b & ~((1 << (3 * level_b)) - 1)
    return start_a + (1 << (3 * level_a)) <= start_b


def distributed_build(ctx, lower: torch.Tensor, level: torch.Tensor, scal: torch.Tensor,
                      coll: Collectives, samples: int = SAMPLES) -> dict:
    """Build this rank's shard of the global dataset whose slice (lower (n,3) int32/uint32
    view, level (n,) uint8, scal (M,n) float32 -- CUDA tensors) this rank holds.  Returns the
    shard description (offset, n_local, n_global, bits, Lmax).  The tensor work runs on the
    context's stream (the library writes its device outputs there)."""
    if lower.is_cuda:
        st = torch.cuda.ExternalStream(ctx.stream)
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            out = _distributed_build(ctx, lower, level, scal, coll, samples)
        torch.cuda.current_stream().wait_stream(st)
        return out
    return _distributed_build(ctx, lower, level, scal, coll, samples)


def _distributed_build(ctx, lower, level, scal, coll, samples):
    dev = lower.device
    G, r = coll.world, coll.rank
    M = int(scal.shape[0])
    # 0. global extent, Lmax, n
    ext, lmax = _extent_and_lmax(lower, level)
    v = torch.tensor([ext, lmax], dtype=torch.int64, device=dev)
    coll.all_reduce(v, "max")
    n_loc = torch.tensor([level.numel()], dtype=torch.int64, device=dev)
    n_global = int(coll.all_reduce(n_loc.clone(), "sum").item())
    bits = global_bits(int(v[0].item()))
    ctx.set_global_bits(bits)
    # 1. local build of the slice: sorted codes and the slice-local ids of the sorted cells
    ctx.build(lower, level, scal)
    codes, ids = ctx.get_sorted(device=True)
    k = codes.numel()
    # 2. regular samples -> splitters (codes < 2^63: int64 order is the code order)
    pos = (torch.arange(samples, device=dev, dtype=torch.int64) * k) // samples
    samp = codes[pos] if k else torch.full((samples,), 2 ** 62, dtype=torch.int64, device=dev)
    allsamp = torch.cat(coll.all_gather(samp))
    spl = splitters(allsamp, G, samples)
    # 3. destinations and counts
    dest = torch.searchsorted(spl, codes, right=True) if G > 1 else torch.zeros_like(codes)
    send_counts = torch.bincount(dest, minlength=G).to(torch.int64)
    allc = torch.stack(coll.all_gather(send_counts))        # [src, dst]
    recv_counts = [int(x) for x in allc[:, r].tolist()]
    sc = [int(x) for x in send_counts.tolist()]
    # 4. exchange the cells in curve order (dest is non-decreasing along the sorted run)
    ids = ids.to(torch.int64)
    lo_s = lower.reshape(-1, 3)[ids]
    lv_s = level[ids]
    sc_s = scal[:, ids].t().contiguous()                     # cell-major rows for the exchange
    r_lower = coll.all_to_all(lo_s, sc, recv_counts)
    r_level = coll.all_to_all(lv_s, sc, recv_counts)
    r_scal = coll.all_to_all(sc_s, sc, recv_counts).t().contiguous()
    if r_level.numel() == 0:
        raise RuntimeError(f"rank {r}: empty shard after the exchange (n_global={n_global})")
    # 5. local build of this rank's key range
    ctx.build(r_lower, r_level, r_scal)
    codes, _ = ctx.get_sorted(device=True)
    lv, _ = ctx.get_sorted_data(device=True)
    ends = torch.tensor([int(codes[0]), int(lv[0]), int(codes[-1]), int(lv[-1])],
                        dtype=torch.int64, device=dev)
    allends = [e.tolist() for e in coll.all_gather(ends)]
    for a, b in zip(allends[:-1], allends[1:]):
        if not dyadic_ok(a[2], a[3], b[0], b[1]):
            raise RuntimeError("duplicate or overlapping cells across ranks (DVL_E_OVERLAP)")
    # 6. offsets and global member ranges
    n_here = torch.tensor([r_level.numel()], dtype=torch.int64, device=dev)
    ns = [int(x.item()) for x in coll.all_gather(n_here)]
    offset = sum(ns[:r])
    finite = torch.isfinite(r_scal)
    vmin = torch.where(finite, r_scal, torch.inf).min(dim=1).values
    vmax = torch.where(finite, r_scal, -torch.inf).max(dim=1).values
    coll.all_reduce(vmin, "min")
    coll.all_reduce(vmax, "max")
    none = ~torch.isfinite(vmin)                               # all NaN: range [0, 0] (O5)
    vmin = torch.where(none, 0.0, vmin)
    vmax = torch.where(none, 0.0, vmax)
    ctx.set_shard(offset, n_global, int(v[1].item()), vmin.cpu().numpy(), vmax.cpu().numpy())
    return {"offset": offset, "n_local": ns[r], "n_global": n_global, "bits": bits,
            "lmax": int(v[1].item()), "sent": sc, "received": recv_counts, "M": M}
