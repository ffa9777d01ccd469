"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle tests and the CUDA path's tests/bench ONLY as an input
generator: it holds none of the method's arithmetic (no Hilbert codes, no transfer-function
sampling, no importance, no prefix sums, no binning).  It produces

* AMR cells on the logical grid: lower corners (u32, n x 3) and levels (u8),
  in generator order (coarse blocks row-major, children in Morton order -- deliberately
  NOT curve order);
* per-member / per-field fp32 scalars (M x n) sampled at cell centroids from a smooth
  blob field plus counter-hash noise;
* piecewise-linear RGBA transfer-function tables (N x 4) through random knots.

Everything is a pure function of its seed.  Default seeds: cells 2306,
member m 11612+m, TF edit e of config c 1000*c+e.
"""
from __future__ import annotations

import numpy as np

CELL_SEED = 2306
MEMBER_SEED = 11612


# ------------------------------------------------------------------ counter-based hash
def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def hash_uniform(keys: np.ndarray, seed: int) -> np.ndarray:
    """Uniform [0,1) float64 from a counter-based hash of integer keys (any shape)."""
    with np.errstate(over="ignore"):
        h = _splitmix64(np.asarray(keys, dtype=np.uint64) ^ _splitmix64(np.uint64(seed)))
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _point_key(ix, iy, iz):
    return (ix.astype(np.uint64) << np.uint64(42)) | (iy.astype(np.uint64) << np.uint64(21)) \
        | iz.astype(np.uint64)


# ---------------------------------------------------------------------------- cells
def uniform_cells(E: int, box=None):
    """A uniform E^3 grid of level-0 cells, row-major (x fastest); box = (gx, gy, gz) for a
    gx x gy x gz block instead."""
    gx, gy, gz = box if box is not None else (E, E, E)
    z, y, x = np.meshgrid(np.arange(gz, dtype=np.uint32), np.arange(gy, dtype=np.uint32),
                          np.arange(gx, dtype=np.uint32), indexing="ij")
    lower = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1).astype(np.uint32)
    return np.ascontiguousarray(lower), np.zeros(len(lower), np.uint8)


_MORTON = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], np.uint32)


def refine(lower: np.ndarray, level: np.ndarray, mask: np.ndarray):
    """Replace every masked cell by its 8 children (Morton order), in place of the parent."""
    counts = np.where(mask, 8, 1)
    lo = np.repeat(lower, counts, axis=0)
    lv = np.repeat(level, counts)
    ref = np.repeat(mask, counts)
    child = np.zeros(len(lo), np.int64)
    starts = np.cumsum(counts) - counts
    idx = np.arange(len(lo)) - np.repeat(starts, counts)
    child[ref] = idx[ref]
    lv = lv.astype(np.int64)
    lv[ref] -= 1
    half = np.where(ref, 1 << np.maximum(lv, 0), 0).astype(np.uint32)
    lo = lo + _MORTON[child] * half[:, None]
    return np.ascontiguousarray(lo.astype(np.uint32)), lv.astype(np.uint8)


def centroids01(lower: np.ndarray, level: np.ndarray, E: int) -> np.ndarray:
    """Geometric cell centres in [0,1]^3 (float64) -- used only to sample the field."""
    w = (1 << level.astype(np.int64)).astype(np.float64)
    return (lower.astype(np.float64) + 0.5 * w[:, None]) / float(E)


class BlobField:
    """B(p) = sum_k a_k exp(-|p - c_k|^2 / (2 sigma_k^2)): 16 smooth blobs (density-like)."""

    def __init__(self, seed: int = CELL_SEED, k: int = 16):
        rng = np.random.default_rng(seed)
        self.c = rng.uniform(0.1, 0.9, size=(k, 3))
        self.s = rng.uniform(0.03, 0.15, size=k)
        self.a = rng.uniform(0.5, 1.5, size=k)

    def __call__(self, p: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
        # evaluated with torch (CUDA if present, else multi-threaded CPU) in float64;
        # torch is only a vectorised calculator here.
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        c = torch.tensor(self.c, dtype=torch.float64, device=dev)
        k = torch.tensor(-1.0 / (2.0 * self.s * self.s), dtype=torch.float64, device=dev)
        a = torch.tensor(self.a, dtype=torch.float64, device=dev)
        out = np.empty(len(p), np.float64)
        for i in range(0, len(p), chunk):
            q = torch.from_numpy(np.ascontiguousarray(p[i:i + chunk])).to(dev)
            d2 = (q * q).sum(dim=1, keepdim=True) - 2.0 * (q @ c.T) + (c * c).sum(dim=1)[None, :]
            out[i:i + chunk] = (torch.exp(d2 * k[None, :]) * a[None, :]).sum(dim=1).cpu().numpy()
        return out


def amr_cells(E: int, Lc: int, rho, seed: int = CELL_SEED, field: BlobField | None = None,
              box=None):
    """Nested AMR: coarse level-Lc grid (row-major), then at each level refine the fraction
    rho[i] of the current finest cells with the largest field value + noise (refined
    regions cluster around blob centres like real AMR), children in Morton order.
    box = (gx, gy, gz): a slab of coarse blocks instead of the whole (E >> Lc)^3 grid."""
    field = field or BlobField(seed)
    G = E >> Lc
    lower, level = uniform_cells(G, box)
    lower = lower << np.uint32(Lc)
    level = np.full(len(lower), Lc, np.uint8)
    for i, L in enumerate(range(Lc, 0, -1)):
        cand = np.nonzero(level == L)[0]
        if len(cand) == 0:
            break
        p = centroids01(lower[cand], level[cand], E)
        key = _point_key(lower[cand, 0], lower[cand, 1], lower[cand, 2])
        score = field(p) + 0.25 * hash_uniform(key, seed + 17 * (L + 1))
        k = int(round(float(rho[i]) * len(cand)))
        mask = np.zeros(len(level), bool)
        if k > 0:
            top = cand[np.argpartition(-score, k - 1)[:k]]
            mask[top] = True
        lower, level = refine(lower, level, mask)
    return lower, level


def member_scalars(lower, level, E: int, M: int, seed: int = CELL_SEED,
                   member_seed: int = MEMBER_SEED, field: BlobField | None = None,
                   multifield: bool = False) -> np.ndarray:
    """Ensemble members m = B(p + delta_m) + 0.05 noise + 0.02 noise_m (float32, M x n).
    multifield=True gives M distinct transforms of B with their own ranges (C3)."""
    field = field or BlobField(seed)
    p = centroids01(lower, level, E)
    key = _point_key(lower[:, 0], lower[:, 1], lower[:, 2]) ^ (level.astype(np.uint64) << np.uint64(63))
    base_noise = 2.0 * hash_uniform(key, seed + 1) - 1.0
    out = np.empty((M, len(level)), np.float32)
    if multifield:
        B = field(p) + 0.05 * base_noise
        B2 = field(np.clip(p + 0.02, 0, 1))
        for m in range(M):
            kind = m % 8
            if kind == 0:
                v = B
            elif kind == 1:
                v = np.log1p(10.0 * np.maximum(B, 0))
            elif kind == 2:
                v = 1.0 / (0.1 + np.abs(B))
            elif kind == 3:
                v = B * B2
            elif kind == 4:
                v = np.abs(B2 - B) * 50.0
            elif kind == 5:
                v = np.sin(6.0 * B)
            elif kind == 6:
                v = 300.0 * (B - 0.5)
            else:
                v = np.exp(-B)
            out[m] = (v + 0.01 * (m + 1) * (2.0 * hash_uniform(key, member_seed + m) - 1.0)).astype(np.float32)
        return out
    for m in range(M):
        rng = np.random.default_rng(member_seed + m)
        delta = rng.uniform(-0.01, 0.01, size=3)
        v = field(np.clip(p + delta, 0.0, 1.0)) + 0.05 * base_noise \
            + 0.02 * (2.0 * hash_uniform(key, member_seed + m) - 1.0)
        out[m] = v.astype(np.float32)
    return out


# ------------------------------------------------------------------ transfer functions
def _hue_rgb(h: float):
    h = h % 1.0
    r = abs(h * 6.0 - 3.0) - 1.0
    g = 2.0 - abs(h * 6.0 - 2.0)
    b = 2.0 - abs(h * 6.0 - 4.0)
    return np.clip([r, g, b], 0.0, 1.0)


def random_tf(seed: int, N: int = 256, member: int = 0) -> np.ndarray:
    """alpha piecewise-linear through K in [2,8] random knots (endpoints included, values
    uniform in [0,1]) -- the distribution of S:535; rgb from a fixed per-member colour."""
    rng = np.random.default_rng(seed)
    K = int(rng.integers(2, 9))
    xs = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0, 1, size=max(K - 2, 0))]))
    ys = rng.uniform(0, 1, size=len(xs))
    grid = np.arange(N) / (N - 1)
    a = np.interp(grid, xs, ys)
    tf = np.empty((N, 4), np.float32)
    rgb = _hue_rgb(0.13 * member + 0.05)
    shade = 0.6 + 0.4 * grid
    tf[:, 0] = rgb[0] * shade
    tf[:, 1] = rgb[1] * shade
    tf[:, 2] = rgb[2] * shade
    tf[:, 3] = a
    return np.clip(tf, 0.0, 1.0).astype(np.float32)


def identity_tf(N: int = 256) -> np.ndarray:
    t = (np.arange(N, dtype=np.float64) / (N - 1)).astype(np.float32)
    tf = np.empty((N, 4), np.float32)
    tf[:, :3] = 0.5
    tf[:, 3] = t
    return tf


# --------------------------------------------------------------------------- configs
CONFIGS = {
    # name: (kind, E, Lc, rho, M, W, domain, multifield)
    "C1": ("uniform", 64, 0, (), 4, 1024, "shared", False),
    "C2": ("amr", 512, 2, (0.20, 0.25), 4, 1024, "shared", False),
    "C3": ("amr", 2048, 4, (0.30, 0.30, 0.30, 0.30), 8, 4096, "per_member", True),
    "C4": ("uniform", 512, 0, (), 16, 1024, "shared", False),
    "C5": ("amr", 4096, 4, (0.32, 0.32, 0.32, 0.32), 4, 1024, "shared", False),
    # not a BASELINE config: shaped like the paper's evaluation data (Table 1:
    # 35.8 M cells, 4 AMR levels, 4 fields with their own ranges) for a like-for-like context
    # number against the paper's 58.6 ms per edit (SURVEY 8(d) "C-paper")
    "Cpaper": ("amr", 1024, 3, (0.28, 0.275, 0.27), 4, 1024, "per_member", True),
}


def make_config(name: str, seed: int = CELL_SEED, scale_E: int | None = None, box=None):
    """Returns dict(lower, level, scal, W, M, E, domain) for a named config.  scale_E
    shrinks the logical grid (same recipe) for quick tests; box = (gx, gy, gz) keeps the
    grid (so the Hilbert bits b) but generates only a slab of its coarse blocks."""
    kind, E, Lc, rho, M, W, dom, multi = CONFIGS[name]
    if scale_E is not None:
        E = scale_E
    field = BlobField(seed)
    if kind == "uniform":
        lower, level = uniform_cells(E, box)
    else:
        lower, level = amr_cells(E, Lc, rho, seed, field, box)
    scal = member_scalars(lower, level, E, M, seed, MEMBER_SEED, field, multifield=multi)
    if dom == "shared":
        fin = scal[np.isfinite(scal)]
        domain = np.array([[fin.min(), fin.max()]] * M, np.float32)
    else:
        domain = None
    return dict(lower=lower, level=level, scal=scal, W=W, M=M, E=E, domain=domain, name=name)


def tf_edit(config_index: int, e: int, N: int = 256, member: int = 0) -> np.ndarray:
    return random_tf(1000 * config_index + e, N, member)
