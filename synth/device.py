"""The synthetic-input recipe of synth/__init__.py evaluated with torch on a device.

Same recipe, same seeds, same arithmetic order:
coarse blocks row-major, AMR refinement of the top-rho fraction of the finest cells by
field + counter-hash noise with children in Morton order, ensemble members sampled at the
cell centres from the 16-blob field plus counter-hash noise.  It exists because the numpy
generator needs tens of GB of host memory and minutes for C4 (134 M cells x 16 members) and
C5 (~1.03 B cells): here the cells are generated where they are used, in HBM.

Like synth/__init__.py it holds none of the method's arithmetic.  On the CPU it produces the
same bits as the numpy generator for the ensemble configs (tests/test_synth_device.py); the
splitmix64 hash is written with 64-bit two's-complement wrap-around and masked (logical)
right shifts so that torch's signed int64 gives numpy's uint64 bits.
"""
from __future__ import annotations

import numpy as np
import torch

from . import CELL_SEED, CONFIGS, MEMBER_SEED, BlobField

_I64 = torch.int64


def _c64(v: int) -> int:
    """A uint64 constant as the int64 with the same bits."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bits."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    x = x + _c64(0x9E3779B97F4A7C15)
    x = (x ^ _lsr(x, 30)) * _c64(0xBF58476D1CE4E5B9)
    x = (x ^ _lsr(x, 27)) * _c64(0x94D049BB133111EB)
    return x ^ _lsr(x, 31)


def _splitmix64_int(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def hash_uniform(keys: torch.Tensor, seed: int) -> torch.Tensor:
    """Uniform [0,1) float64 from the counter-based hash of int64 keys (synth.hash_uniform)."""
    h = _splitmix64(keys ^ _c64(_splitmix64_int(seed)))
    return _lsr(h, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def _point_key(lower: torch.Tensor) -> torch.Tensor:
    l = lower.to(_I64)
    return (l[:, 0] << 42) | (l[:, 1] << 21) | l[:, 2]


def uniform_cells(E: int, device, box=None):
    """A uniform grid of level-0 cells (x fastest): E^3, or gx x gy x gz with box."""
    gx, gy, gz = box if box is not None else (E, E, E)
    z, y, x = torch.meshgrid(torch.arange(gz, device=device, dtype=torch.int32),
                             torch.arange(gy, device=device, dtype=torch.int32),
                             torch.arange(gx, device=device, dtype=torch.int32), indexing="ij")
    lower = torch.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], 1).contiguous()
    return lower, torch.zeros(lower.shape[0], dtype=torch.uint8, device=device)


def refine(lower: torch.Tensor, level: torch.Tensor, mask: torch.Tensor):
    """Replace every masked cell by its 8 children (Morton order), in place of the parent."""
    dev = lower.device
    counts = torch.where(mask, 8, 1)
    lo = torch.repeat_interleave(lower, counts, dim=0)
    lv = torch.repeat_interleave(level.to(torch.int32), counts)
    ref = torch.repeat_interleave(mask, counts)
    starts = torch.cumsum(counts, 0) - counts
    idx = torch.arange(lo.shape[0], device=dev, dtype=_I64) - torch.repeat_interleave(starts, counts)
    child = torch.where(ref, idx, 0).to(torch.int32)
    lv = torch.where(ref, lv - 1, lv)
    half = torch.where(ref, torch.ones_like(lv) << lv.clamp(min=0), 0).to(torch.int32)
    morton = torch.stack([child & 1, (child >> 1) & 1, (child >> 2) & 1], 1)
    lo = lo + morton * half[:, None]
    return lo.contiguous(), lv.to(torch.uint8)


def centroids01(lower: torch.Tensor, level: torch.Tensor, E: int) -> torch.Tensor:
    w = (torch.ones_like(level, dtype=_I64) << level.to(_I64)).to(torch.float64)
    return (lower.to(torch.float64) + 0.5 * w[:, None]) / float(E)


def field_eval(field: BlobField, p: torch.Tensor, chunk: int = 1 << 22) -> torch.Tensor:
    """BlobField.__call__ on a device tensor (same expression, same order)."""
    dev = p.device
    c = torch.tensor(field.c, dtype=torch.float64, device=dev)
    k = torch.tensor(-1.0 / (2.0 * field.s * field.s), dtype=torch.float64, device=dev)
    a = torch.tensor(field.a, dtype=torch.float64, device=dev)
    out = torch.empty(p.shape[0], dtype=torch.float64, device=dev)
    for i in range(0, p.shape[0], chunk):
        q = p[i:i + chunk]
        d2 = (q * q).sum(dim=1, keepdim=True) - 2.0 * (q @ c.T) + (c * c).sum(dim=1)[None, :]
        out[i:i + chunk] = (torch.exp(d2 * k[None, :]) * a[None, :]).sum(dim=1)
    return out


def amr_cells(E: int, Lc: int, rho, seed: int, field: BlobField, device, box=None):
    """synth.amr_cells on the device (box: coarse grid gx x gy x gz instead of (E>>Lc)^3)."""
    G = E >> Lc
    lower, level = uniform_cells(G, device, box)
    lower = lower << Lc
    level = torch.full((lower.shape[0],), Lc, dtype=torch.uint8, device=device)
    for i, L in enumerate(range(Lc, 0, -1)):
        cand = torch.nonzero(level == L).squeeze(1)
        if cand.numel() == 0:
            break
        p = centroids01(lower[cand], level[cand], E)
        score = field_eval(field, p) + 0.25 * hash_uniform(_point_key(lower[cand]), seed + 17 * (L + 1))
        del p
        k = int(round(float(rho[i]) * cand.numel()))
        mask = torch.zeros(level.shape[0], dtype=torch.bool, device=device)
        if k > 0:
            top = cand[torch.argsort(score, descending=True)[:k]]
            mask[top] = True
        del score, cand
        lower, level = refine(lower, level, mask)
    return lower, level


def member_scalars(lower, level, E: int, M: int, seed: int, member_seed: int, field: BlobField,
                   chunk: int = 1 << 26) -> torch.Tensor:
    """synth.member_scalars (ensemble members) on the device, in chunks of cells."""
    n = lower.shape[0]
    out = torch.empty((M, n), dtype=torch.float32, device=lower.device)
    deltas = [np.random.default_rng(member_seed + m).uniform(-0.01, 0.01, size=3) for m in range(M)]
    for i in range(0, n, chunk):
        lo, lv = lower[i:i + chunk], level[i:i + chunk]
        p = centroids01(lo, lv, E)
        key = _point_key(lo) ^ (lv.to(_I64) << 63)
        base_noise = 2.0 * hash_uniform(key, seed + 1) - 1.0
        for m in range(M):
            d = torch.tensor(deltas[m], dtype=torch.float64, device=lower.device)
            v = field_eval(field, torch.clamp(p + d[None, :], 0.0, 1.0)) + 0.05 * base_noise \
                + 0.02 * (2.0 * hash_uniform(key, member_seed + m) - 1.0)
            out[m, i:i + chunk] = v.to(torch.float32)
    return out


def make_config(name: str, device="cuda", seed: int = CELL_SEED, scale_E: int | None = None,
                box=None):
    """synth.make_config on the device: dict(lower (n,3) int32, level (n,) uint8, scal (M,n)
    float32 -- torch tensors on `device` -- W, M, E, domain (numpy), name).  Ensemble
    configs only (C1, C2, C4, C5); box = coarse grid (gx, gy, gz) for a slab of the recipe."""
    kind, E, Lc, rho, M, W, dom, multi = CONFIGS[name]
    if multi:
        raise ValueError("the multi-field config C3 uses synth.make_config")
    if scale_E is not None:
        E = scale_E
    field = BlobField(seed)
    if kind == "uniform":
        lower, level = uniform_cells(E, device, box)
    else:
        lower, level = amr_cells(E, Lc, rho, seed, field, device, box)
    scal = member_scalars(lower, level, E, M, seed, MEMBER_SEED, field)
    fin = torch.isfinite(scal)
    lo = float(torch.where(fin, scal, float("inf")).min())
    hi = float(torch.where(fin, scal, float("-inf")).max())
    domain = np.array([[lo, hi]] * M, np.float32)
    return dict(lower=lower, level=level, scal=scal, W=W, M=M, E=E, domain=domain, name=name)
