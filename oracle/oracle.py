"""ctypes front of the plain CPU oracle (oracle/dvl_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this module.  It never imports the
product package ``paper_2306_11612_b200`` and the product never imports it.

Every function restates a passage of the paper (PAPER.md line ``P:n``); the readings
(O#, A#) are listed in DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dvl_oracle.c")
_LIB = os.path.join(_HERE, "libdvl_oracle.so")

STATUS = {0: "OK", 1: "INVAL", 2: "STATE", 3: "RANGE", 4: "OVERLAP", 5: "DEGENERATE"}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {STATUS.get(code, code)}")
        self.status = STATUS.get(code, str(code))


def compile_oracle(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off (no fast-math, default SSE rounding, no FTZ/DAZ)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(compile_oracle())
        P = ctypes.c_void_p
        i64, i32, u64, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_float
        sig = {
            "or_hilbert_encode": (u64, [ctypes.c_uint32] * 3 + [i32]),
            "or_hilbert_encode_many": (None, [i64, P, i32, P]),
            "or_hilbert_decode_many": (None, [i64, P, i32, P]),
            "or_build": (i32, [i64, P, P, i32, P, P, P, P, P, P, P, P]),
            "or_domain_inv": (f32, [f32, f32]),
            "or_normalize": (f32, [f32, f32, f32]),
            "or_sample": (f32, [P, i32, f32]),
            "or_index_range": (None, [f32, f32, f32, f32, i32, P]),
            "or_maxv_approx": (f32, [i32, i32, i32, P, P, P, P, P]),
            "or_maxv_exact": (f32, [i64, i32, i32, P, P, P, P]),
            "or_variation": (f32, [i64, i64, i32, i32, P, P, P, P]),
            "or_detpow": (f32, [f32, f32]),
            "or_powP": (f32, [f32, f32]),
            "or_importance": (f32, [f32, f32, i32, f32, f32]),
            "or_shift": (i32, [i64, i32, f32]),
            "or_fixed": (u64, [f32, i32]),
            "or_weights": (None, [i64, i32, i32, P, P, P, P, P, f32, f32, f32, i32, P, P]),
            "or_prefix": (u64, [i64, P, P]),
            "or_bins": (None, [i64, P, ctypes.c_uint32, P, P]),
            "or_bins_ext": (None, [i64, P, u64, u64, ctypes.c_uint32, P, P]),
            "or_reduce": (None, [i64, i32, i32, P, P, P, P, ctypes.c_uint32, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


VERTEX_DTYPE = np.dtype([("t_min", "<f4"), ("t_max", "<f4"), ("t_mean", "<f4"), ("y", "<f4"),
                         ("r", "<f4"), ("g", "<f4"), ("b", "<f4"), ("count", "<u4")])

MAXV_MODES = {"conservative": 0, "per_entry": 1, "exact": 2}


# ---------------------------------------------------------------------------- Hilbert
def hilbert_encode(xyz, b: int) -> np.ndarray:
    """O3: Skilling-variant Hilbert index of integer points (n,3)."""
    xyz = np.ascontiguousarray(np.asarray(xyz, dtype=np.uint32).reshape(-1, 3))
    out = np.empty(len(xyz), dtype=np.uint64)
    lib().or_hilbert_encode_many(len(xyz), _p(xyz), b, _p(out))
    return out


def hilbert_decode(h, b: int) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(h, dtype=np.uint64).reshape(-1))
    out = np.empty((len(h), 3), dtype=np.uint32)
    lib().or_hilbert_decode_many(len(h), _p(h), b, _p(out))
    return out


# ------------------------------------------------------------------------------ build
@dataclass
class Built:
    n: int
    M: int
    E: int
    b: int
    Lmax: int
    codes: np.ndarray       # u64[n], curve order
    perm: np.ndarray        # u64[n], input id of each sorted cell
    level_s: np.ndarray     # u8[n]
    scal_s: np.ndarray      # f32[M, n]
    vmin: np.ndarray        # f32[M]
    vmax: np.ndarray        # f32[M]


def build(lower, level, scalars) -> Built:
    """O1-O5: validate, encode centroids, sort, permute."""
    lower = np.ascontiguousarray(np.asarray(lower, dtype=np.uint32).reshape(-1, 3))
    level = np.ascontiguousarray(np.asarray(level, dtype=np.uint8).reshape(-1))
    scal = np.ascontiguousarray(np.asarray(scalars, dtype=np.float32))
    if scal.ndim == 1:
        scal = scal[None, :]
    n = len(level)
    M = scal.shape[0] if scal.size or n == 0 else 0
    if scal.shape[1:] != (n,) or lower.shape[0] != n:
        raise OracleError(1)
    codes = np.empty(n, np.uint64)
    perm = np.empty(n, np.uint64)
    level_s = np.empty(n, np.uint8)
    scal_s = np.empty((M, n), np.float32)
    vmin = np.empty(M, np.float32)
    vmax = np.empty(M, np.float32)
    info = np.zeros(3, np.int32)
    st = lib().or_build(n, _p(lower), _p(level), M, _p(scal), _p(codes), _p(perm),
                        _p(level_s), _p(scal_s), _p(vmin), _p(vmax), _p(info))
    if st != 0:
        raise OracleError(st)
    return Built(n, M, int(info[0]), int(info[1]), int(info[2]), codes, perm, level_s,
                 scal_s, vmin, vmax)


# --------------------------------------------------------------------- transfer funcs
def domain_inv(lo: float, hi: float) -> float:
    return float(lib().or_domain_inv(lo, hi))


def normalize(v: float, lo: float, inv: float) -> float:
    return float(lib().or_normalize(v, lo, inv))


def sample(A, t: float) -> float:
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float32))
    return float(lib().or_sample(_p(A), len(A), t))


def index_range(vmin, vmax, lo, inv, N):
    out = np.zeros(2, np.int32)
    lib().or_index_range(vmin, vmax, lo, inv, N, _p(out))
    return int(out[0]), int(out[1])


def detpow(g: float, P: float) -> float:
    return float(lib().or_detpow(g, P))


def powP(g: float, P: float) -> float:
    return float(lib().or_powP(g, P))


def importance(V: float, maxV: float, L: int, P: float, eps: float) -> float:
    return float(lib().or_importance(V, maxV, L, P, eps))


def shift(n_global: int, Lmax: int, P: float) -> int:
    return int(lib().or_shift(n_global, Lmax, P))


def fixed(f: float, s: int) -> int:
    return int(lib().or_fixed(f, s))


def bins_ext(Q, E0: int, Qtot: int, W: int):
    """O13 on a contiguous piece of the cells (first cell's E = E0, total Qtot)."""
    Q = np.ascontiguousarray(Q, dtype=np.uint64)
    b1 = np.empty(len(Q), np.int32)
    b2 = np.empty(len(Q), np.int32)
    lib().or_bins_ext(len(Q), _p(Q), E0, Qtot, W, _p(b1), _p(b2))
    return b1, b2


def identity_tf(N: int = 256) -> np.ndarray:
    """Default TF of every member: alpha = identity ramp, grey rgb."""
    a = (np.arange(N, dtype=np.float64) / (N - 1)).astype(np.float32)
    tf = np.empty((N, 4), np.float32)
    tf[:, 0] = tf[:, 1] = tf[:, 2] = 0.5
    tf[:, 3] = a
    return tf


@dataclass
class Update:
    maxV: float
    s: int
    f: np.ndarray        # f32[n]
    q: np.ndarray        # u64[n]
    Q: np.ndarray        # u64[n]
    Qtot: int
    b1: np.ndarray       # i32[n]
    b2: np.ndarray       # i32[n]
    vertices: np.ndarray  # VERTEX_DTYPE[M, W]
    lo: np.ndarray       # u64[W]
    hi: np.ndarray       # u64[W]


def domains(B: Built, domain=None):
    """O6: per-member [lo, hi] (default: the member's finite data range)."""
    if domain is None:
        lo = B.vmin.astype(np.float32).copy()
        hi = B.vmax.astype(np.float32).copy()
    else:
        d = np.asarray(domain, dtype=np.float32).reshape(-1, 2)
        if d.shape[0] == 1:
            d = np.repeat(d, B.M, axis=0)
        lo, hi = np.ascontiguousarray(d[:, 0]), np.ascontiguousarray(d[:, 1])
    inv = np.array([domain_inv(float(a), float(b)) for a, b in zip(lo, hi)], np.float32)
    return lo, hi, inv


def maxv(B: Built, tfs: np.ndarray, lo, inv, mode: str = "conservative") -> float:
    """O9: max(V_h) -- R2 (default), R1 or exact."""
    tfs = np.ascontiguousarray(tfs, dtype=np.float32)
    M, N = tfs.shape[0], tfs.shape[1]
    alpha = np.ascontiguousarray(tfs[:, :, 3])
    lo = np.ascontiguousarray(lo, np.float32)
    inv = np.ascontiguousarray(inv, np.float32)
    if mode == "exact":
        return float(lib().or_maxv_exact(B.n, M, N, _p(B.scal_s), _p(alpha), _p(lo), _p(inv)))
    return float(lib().or_maxv_approx(MAXV_MODES[mode], M, N, _p(alpha), _p(B.vmin),
                                      _p(B.vmax), _p(lo), _p(inv)))


def update(B: Built, tfs, W: int, P: float = 1.0, eps: float = 0.025,
           mode: str = "conservative", domain=None, n_global: int | None = None,
           scale: str = "width") -> Update:
    """One TF edit + polyline extraction: U0-U5 (Eq. 1, 3, 4).  scale="volume":
    the cell size enters Eq. 3 as the cell volume (2^L)^3 = 2^3L instead of the width 2^L,
    "another sensible choice"; O10/O11 then see the level 3L."""
    c = {"width": 1, "volume": 3}[scale]
    tfs = np.ascontiguousarray(np.asarray(tfs, dtype=np.float32))
    if tfs.ndim == 2:
        tfs = np.repeat(tfs[None], B.M, axis=0)
    M, N = tfs.shape[0], tfs.shape[1]
    assert M == B.M and tfs.shape[2] == 4
    lo, _, inv = domains(B, domain)
    mv = maxv(B, tfs, lo, inv, mode)
    s = shift(B.n if n_global is None else n_global, c * B.Lmax, P)
    alpha = np.ascontiguousarray(tfs[:, :, 3])
    f = np.empty(B.n, np.float32)
    q = np.empty(B.n, np.uint64)
    lev = np.ascontiguousarray((B.level_s.astype(np.int32) * c).astype(np.uint8))
    lib().or_weights(B.n, M, N, _p(lev), _p(B.scal_s), _p(alpha), _p(lo), _p(inv),
                     mv, P, eps, s, _p(f), _p(q))
    Q = np.empty(B.n, np.uint64)
    Qtot = int(lib().or_prefix(B.n, _p(q), _p(Q)))
    if Qtot == 0:
        raise OracleError(5)
    b1 = np.empty(B.n, np.int32)
    b2 = np.empty(B.n, np.int32)
    lib().or_bins(B.n, _p(Q), W, _p(b1), _p(b2))
    out = np.zeros((M, W), VERTEX_DTYPE)
    blo = np.empty(W, np.uint64)
    bhi = np.empty(W, np.uint64)
    lib().or_reduce(B.n, M, N, _p(B.scal_s), _p(tfs), _p(lo), _p(inv), W, _p(b1), _p(b2),
                    _p(out), _p(blo), _p(bhi))
    return Update(mv, s, f, q, Q, Qtot, b1, b2, out, blo, bhi)


# ------------------------------------------------------------------ brushing / linking
def locate(lower, level, B: Built, pts) -> np.ndarray:
    """Brushing and linking: for each integer point of the
    logical grid, the curve-order index (the position in B.codes) of the cell whose 2^L cube
    [lower, lower + 2^L) contains it, -1 if none.  The plain definition: a containment test
    against every cell (cells are disjoint, O4, so at most one matches)."""
    lower = np.asarray(lower, dtype=np.int64).reshape(-1, 3)
    w = (np.int64(1) << np.asarray(level, dtype=np.int64))[:, None]
    rank = np.empty(B.n, np.int64)
    rank[B.perm.astype(np.int64)] = np.arange(B.n, dtype=np.int64)   # input id -> curve order
    pts = np.asarray(pts, dtype=np.int64).reshape(-1, 3)
    out = np.full(len(pts), -1, np.int64)
    for i, p in enumerate(pts):
        hit = np.nonzero(np.all((lower <= p) & (p < lower + w), axis=1))[0]
        assert len(hit) <= 1
        if len(hit):
            out[i] = rank[hit[0]]
    return out
