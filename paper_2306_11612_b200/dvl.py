"""Thin ctypes binding of the C ABI in include/dvl.h (argument marshalling only).

Every step of the DVL hot path runs in the CUDA library ``libdvl.so`` built in-tree by
``paper_2306_11612_b200/build.py``; there is no CPU fallback: if the library is missing
this module raises.  Host arrays are numpy arrays; device arrays are torch CUDA tensors
(PyTorch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdvl.so")

HOST, DEVICE = 0, 1
MAXV_MODES = {"conservative": 0, "per_entry": 1, "exact": 2}
STATUS = {0: "DVL_OK", 1: "DVL_E_INVAL", 2: "DVL_E_STATE", 3: "DVL_E_RANGE", 4: "DVL_E_OVERLAP",
          5: "DVL_E_DEGENERATE", 6: "DVL_E_NOMEM", 7: "DVL_E_CUDA", 8: "DVL_E_NCCL"}
FLAG_TIMING = 1
FLAG_GENERIC = 2
FLAG_NO_EDIT_CACHE = 4
FLAG_PASS2_INLINE = 8
FLAG_PASS2_LIST = 16
FLAG_PASS2_JOBS = 64
FLAG_LSD_SORT = 32

# every symbol include/dvl.h declares (checked by tests/test_abi.py)
SYMBOLS = ["dvl_create", "dvl_destroy", "dvl_last_error", "dvl_status_string", "dvl_build",
           "dvl_set_params", "dvl_set_domain", "dvl_update_tf", "dvl_reset_tfs",
           "dvl_get_polylines", "dvl_info", "dvl_get_sorted", "dvl_get_sorted_data",
           "dvl_get_prefix", "dvl_get_bin_ranges", "dvl_get_timings", "dvl_stream",
           "dvl_hilbert_encode_host", "dvl_hilbert_states", "dvl_set_global_bits",
           "dvl_set_shard", "dvl_shard_total", "dvl_shard_export_words", "dvl_shard_reduce",
           "dvl_shard_finish", "dvl_set_timing", "dvl_locate", "dvl_set_level_scale",
           "dvl_nccl_unique_id", "dvl_set_comm", "dvl_local_group_create",
           "dvl_local_group_destroy", "dvl_set_local_comm", "dvl_get_shard",
           "dvl_select_splitters", "dvl_brush", "dvl_roi_contains"]

VERTEX_DTYPE = np.dtype([("t_min", "<f4"), ("t_max", "<f4"), ("t_mean", "<f4"), ("y", "<f4"),
                         ("r", "<f4"), ("g", "<f4"), ("b", "<f4"), ("count", "<u4")])


class DvlError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = STATUS.get(status, str(status))
        super().__init__(f"{self.status}: {msg}")


class _Init(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("cuda_stream", ctypes.c_void_p),
                ("alloc", ctypes.c_void_p), ("free", ctypes.c_void_p), ("user", ctypes.c_void_p),
                ("flags", ctypes.c_uint32)]


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("members", ctypes.c_uint32), ("extent", ctypes.c_uint32),
                ("bits", ctypes.c_int32), ("Lmax", ctypes.c_int32), ("key_bytes", ctypes.c_int32),
                ("tf_size", ctypes.c_int32), ("P", ctypes.c_float), ("eps", ctypes.c_float),
                ("maxv_mode", ctypes.c_int32), ("shift", ctypes.c_int32), ("maxV", ctypes.c_float),
                ("Qtot", ctypes.c_uint64), ("device_bytes", ctypes.c_uint64),
                ("cells_per_tile", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _ShardInfo(ctypes.Structure):
    _fields_ = [("cell_offset", ctypes.c_uint64), ("n_global", ctypes.c_uint64),
                ("lmax_global", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("vmin", ctypes.c_void_p), ("vmax", ctypes.c_void_p)]


class _Timings(ctypes.Structure):
    _fields_ = [(k, ctypes.c_float) for k in ("ingest_ms", "encode_ms", "sort_ms", "gather_ms",
                                              "maxv_ms", "weights_scan_ms", "bin_reduce_ms",
                                              "epilogue_ms", "bin_boundary_ms")] + \
               [("sort_passes", ctypes.c_int32), ("launches", ctypes.c_int32)]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libdvl.so (in-tree).  Raises if it is missing: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run __graft_entry__.build() "
                           "(python paper_2306_11612_b200/build.py)")
    L = ctypes.CDLL(path)
    P, u32, u64, i32, f32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_float
    sig = {
        "dvl_create": (i32, [ctypes.POINTER(_Init), ctypes.POINTER(ctypes.c_void_p)]),
        "dvl_destroy": (None, [P]),
        "dvl_last_error": (ctypes.c_char_p, [P]),
        "dvl_status_string": (ctypes.c_char_p, [i32]),
        "dvl_build": (i32, [P, u64, P, P, u32, P, i32]),
        "dvl_set_params": (i32, [P, f32, f32, i32]),
        "dvl_set_domain": (i32, [P, u32, f32, f32]),
        "dvl_update_tf": (i32, [P, u32, P, u32]),
        "dvl_reset_tfs": (i32, [P, u32]),
        "dvl_get_polylines": (i32, [P, u32, P, i32]),
        "dvl_info": (i32, [P, ctypes.POINTER(_Info)]),
        "dvl_get_sorted": (i32, [P, P, P, i32]),
        "dvl_get_sorted_data": (i32, [P, P, P, i32]),
        "dvl_get_prefix": (i32, [P, P, i32]),
        "dvl_get_bin_ranges": (i32, [P, u32, P, P, i32]),
        "dvl_get_timings": (i32, [P, ctypes.POINTER(_Timings)]),
        "dvl_stream": (P, [P]),
        "dvl_hilbert_encode_host": (i32, [u64, P, i32, P]),
        "dvl_hilbert_states": (i32, []),
        "dvl_set_global_bits": (i32, [P, i32]),
        "dvl_set_shard": (i32, [P, ctypes.POINTER(_ShardInfo)]),
        "dvl_shard_total": (i32, [P, P]),
        "dvl_shard_export_words": (u64, [P, u32]),
        "dvl_shard_reduce": (i32, [P, u32, P, i32, i32, P]),
        "dvl_shard_finish": (i32, [P, u32, P, P, i32]),
        "dvl_locate": (i32, [P, u64, P, P, i32]),
        "dvl_set_level_scale": (i32, [P, i32]),
        "dvl_nccl_unique_id": (i32, [P]),
        "dvl_set_comm": (i32, [P, i32, i32, P]),
        "dvl_local_group_create": (i32, [i32, ctypes.POINTER(ctypes.c_void_p)]),
        "dvl_local_group_destroy": (None, [P]),
        "dvl_set_local_comm": (i32, [P, P, i32]),
        "dvl_get_shard": (i32, [P, ctypes.POINTER(_ShardInfo)]),
        "dvl_select_splitters": (i32, [P, P, i32, i32, P]),
        "dvl_brush": (i32, [P, u32, u32, u32, P]),
        "dvl_roi_contains": (i32, [P, u64, P, u64, u64, P, i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _ptr(a) -> int:
    """Address of a numpy array or a torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _is_device(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


def _need(cond: bool, msg: str):
    """Argument validation in the binding: wrong dtypes / sizes would be misread by the C
    library, which only sees pointers."""
    if not cond:
        raise ValueError(msg)


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


def _torch_allocator(device: int):
    """dvl_init's alloc / free callbacks backed by PyTorch's caching allocator (SURVEY 8(b):
    "PyTorch only for device memory and streams").  None if torch / CUDA is unavailable."""
    try:
        import torch
        if not torch.cuda.is_available():
            return None
    except Exception:
        return None

    def alloc(nbytes, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(max(int(nbytes), 1), device=device,
                                                      stream=int(stream or 0))
        except Exception:
            return None

    def free(ptr, nbytes, stream, user):
        try:
            if ptr:
                torch.cuda.caching_allocator_delete(ptr)
        except Exception:
            pass

    return _ALLOC_FN(alloc), _FREE_FN(free)


def hilbert_encode_host(xyz, bits: int) -> np.ndarray:
    """The library's table-driven Hilbert encoder evaluated on the host (no GPU)."""
    xyz = np.ascontiguousarray(np.asarray(xyz, dtype=np.uint32).reshape(-1, 3))
    out = np.empty(len(xyz), np.uint64)
    st = load().dvl_hilbert_encode_host(len(xyz), _ptr(xyz), bits, _ptr(out))
    if st:
        raise DvlError(st, "dvl_hilbert_encode_host")
    return out


def hilbert_states() -> int:
    return int(load().dvl_hilbert_states())


class Context:
    """One dvl_ctx: a dataset on one device plus its TFs, parameters and scratch."""

    def __init__(self, device: int = 0, stream=None, timing: bool = False, generic: bool = False,
                 torch_allocator: bool = True, edit_cache: bool = True, pass2: str | None = None,
                 sort: str = "auto"):
        """torch_allocator: device memory through PyTorch's caching allocator (dvl_init's
        alloc / free callbacks); False: the library's own cudaMallocAsync pool.
        edit_cache=False / pass2="inline"|"list"|"jobs": test flags selecting among kernels that
        return identical bits (DVL_FLAG_NO_EDIT_CACHE, DVL_FLAG_PASS2_*); sort="lsd" builds
        with the onesweep LSD sort where the bucket sort would apply (DVL_FLAG_LSD_SORT)."""
        self._lib = load()
        init = _Init()
        init.device = device
        self.device = device
        if stream is not None:
            init.cuda_stream = stream if isinstance(stream, int) else stream.cuda_stream
        init.flags = (FLAG_TIMING if timing else 0) | (FLAG_GENERIC if generic else 0) \
            | (0 if edit_cache else FLAG_NO_EDIT_CACHE) \
            | {None: 0, "inline": FLAG_PASS2_INLINE, "list": FLAG_PASS2_LIST, "jobs": FLAG_PASS2_JOBS}[pass2] \
            | {"auto": 0, "lsd": FLAG_LSD_SORT}[sort]
        self._alloc = _torch_allocator(device) if torch_allocator else None
        if self._alloc is not None:
            init.alloc = ctypes.cast(self._alloc[0], ctypes.c_void_p)
            init.free = ctypes.cast(self._alloc[1], ctypes.c_void_p)
        self._ext = None
        h = ctypes.c_void_p()
        st = self._lib.dvl_create(ctypes.byref(init), ctypes.byref(h))
        if st:
            raise DvlError(st, "dvl_create")
        self._h = h
        self.M = 0
        self.n = 0

    # ------------------------------------------------------------------ helpers
    def _check(self, st: int, what: str):
        if st:
            msg = self._lib.dvl_last_error(self._h) or b""
            raise DvlError(st, f"{what}: {msg.decode()}")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dvl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self) -> int:
        return int(self._lib.dvl_stream(self._h) or 0)

    def _torch_stream(self):
        import torch
        if self._ext is None:
            self._ext = torch.cuda.ExternalStream(self.stream, device=torch.device("cuda", self.device))
        return self._ext

    def _order_in(self, *tensors):
        """Device inputs: the context stream waits for the caller's current stream (which
        produced them, e.g. a .contiguous() copy) before the library reads them."""
        import torch
        for t in tensors:
            _need(t.device.index == self.device, f"tensor on {t.device}, context on cuda:{self.device}")
        self._torch_stream().wait_stream(torch.cuda.current_stream(self.device))

    def _order_out(self):
        """Device outputs: the caller's current stream waits for the context stream."""
        import torch
        torch.cuda.current_stream(self.device).wait_stream(self._torch_stream())

    # ------------------------------------------------------------------ the ABI
    def build(self, lower, level, scalars):
        """lower: (n,3) u32, level: (n,) u8, scalars: (M,n) f32 -- all numpy (host) or all
        torch CUDA tensors (device)."""
        dev = _is_device(lower)
        if not dev:
            lower = np.ascontiguousarray(lower, dtype=np.uint32)
            level = np.ascontiguousarray(level, dtype=np.uint8)
            scalars = np.ascontiguousarray(scalars, dtype=np.float32)
            if scalars.ndim == 1:
                scalars = scalars[None]
        else:
            import torch
            _need(_is_device(level) and _is_device(scalars), "all build inputs on the device, or all on the host")
            _need(lower.dtype in (torch.int32, torch.uint32), "lower: int32/uint32 tensor")
            _need(level.dtype == torch.uint8, "level: uint8 tensor")
            _need(scalars.dtype == torch.float32, "scalars: float32 tensor")
            lower, level, scalars = lower.contiguous(), level.contiguous(), scalars.contiguous()
            if scalars.dim() == 1:
                scalars = scalars[None]
            self._order_in(lower, level, scalars)
        n = int(level.shape[0])
        M = int(scalars.shape[0])
        _need(level.ndim == 1, "level: shape (n,)")
        _need(int(np.prod(tuple(lower.shape))) == 3 * n, "lower: shape (n, 3)")
        _need(tuple(scalars.shape) == (M, n), "scalars: shape (M, n)")
        ptrs = (ctypes.c_void_p * max(M, 1))(*[_ptr(scalars) + 4 * n * m for m in range(M)])
        st = self._lib.dvl_build(self._h, n, _ptr(lower), _ptr(level), M, ptrs,
                                 DEVICE if dev else HOST)
        self._check(st, "dvl_build")
        self.M, self.n = M, n
        if getattr(self, "_group", None) is not None or getattr(self, "_comm", False):
            # distributed build: this context now holds its range of the curve order
            self.n = int(self.info()["n"])

    def set_level_scale(self, scale: str = "width"):
        """Eq. 3's level factor: "width" (2^L, default) or "volume" (2^3L)."""
        self._check(self._lib.dvl_set_level_scale(self._h, {"width": 0, "volume": 1}[scale]),
                    "dvl_set_level_scale")

    def set_params(self, P: float = 1.0, eps: float = 0.025, mode: str = "conservative"):
        self._check(self._lib.dvl_set_params(self._h, P, eps, MAXV_MODES[mode]), "dvl_set_params")

    def set_domain(self, member: int, lo: float, hi: float):
        self._check(self._lib.dvl_set_domain(self._h, member, lo, hi), "dvl_set_domain")

    def update_tf(self, member: int, rgba):
        rgba = np.ascontiguousarray(rgba, dtype=np.float32).reshape(-1, 4)
        self._check(self._lib.dvl_update_tf(self._h, member, _ptr(rgba), rgba.shape[0]),
                    "dvl_update_tf")

    def reset_tfs(self, N: int = 256):
        self._check(self._lib.dvl_reset_tfs(self._h, N), "dvl_reset_tfs")

    def get_polylines(self, W: int, out=None):
        """Returns an (M, W) structured numpy array (VERTEX_DTYPE); with ``out`` a torch
        CUDA tensor of >= M*W*32 bytes, writes there on the device and returns it."""
        nbytes = self.M * int(W) * VERTEX_DTYPE.itemsize
        if out is not None and _is_device(out):
            _need(out.is_contiguous() and out.numel() * out.element_size() >= nbytes,
                  f"out: contiguous device tensor of >= {nbytes} bytes")
            self._order_in(out)
            self._check(self._lib.dvl_get_polylines(self._h, W, _ptr(out), DEVICE),
                        "dvl_get_polylines")
            self._order_out()
            return out
        res = np.empty((self.M, W), VERTEX_DTYPE) if out is None else out
        _need(isinstance(res, np.ndarray) and res.flags.c_contiguous and res.nbytes >= nbytes,
              f"out: contiguous numpy array of >= {nbytes} bytes")
        self._check(self._lib.dvl_get_polylines(self._h, W, _ptr(res), HOST), "dvl_get_polylines")
        return res

    def info(self) -> dict:
        i = _Info()
        self._check(self._lib.dvl_info(self._h, ctypes.byref(i)), "dvl_info")
        return {k: getattr(i, k) for k, _ in _Info._fields_ if k != "reserved"}

    def get_sorted(self, device: bool = False):
        """Sorted Hilbert codes and the input ids of the sorted cells (n x u64 each); numpy,
        or torch CUDA int64 tensors with device=True."""
        if device:
            import torch
            codes = torch.empty(self.n, dtype=torch.int64, device="cuda")
            ids = torch.empty(self.n, dtype=torch.int64, device="cuda")
            where = DEVICE
            self._order_in(codes, ids)
        else:
            codes = np.empty(self.n, np.uint64)
            ids = np.empty(self.n, np.uint64)
            where = HOST
        self._check(self._lib.dvl_get_sorted(self._h, _ptr(codes), _ptr(ids), where), "dvl_get_sorted")
        if device:
            self._order_out()
        return codes, ids

    def get_sorted_data(self, device: bool = False):
        """Levels (n u8) and member scalars (M x n f32) in curve order (numpy, or torch CUDA
        tensors with device=True)."""
        if device:
            import torch
            lv = torch.empty(self.n, dtype=torch.uint8, device="cuda")
            sc = torch.empty((self.M, self.n), dtype=torch.float32, device="cuda")
            where = DEVICE
            self._order_in(lv, sc)
        else:
            lv = np.empty(self.n, np.uint8)
            sc = np.empty((self.M, self.n), np.float32)
            where = HOST
        self._check(self._lib.dvl_get_sorted_data(self._h, _ptr(lv), _ptr(sc), where),
                    "dvl_get_sorted_data")
        if device:
            self._order_out()
        return lv, sc

    def get_prefix(self) -> np.ndarray:
        Q = np.empty(self.n, np.uint64)
        self._check(self._lib.dvl_get_prefix(self._h, _ptr(Q), HOST), "dvl_get_prefix")
        return Q

    def get_bin_ranges(self, W: int):
        lo = np.empty(W, np.uint64)
        hi = np.empty(W, np.uint64)
        self._check(self._lib.dvl_get_bin_ranges(self._h, W, _ptr(lo), _ptr(hi), HOST),
                    "dvl_get_bin_ranges")
        return lo, hi

    # ------------------------------------------------------------ brushing / linking
    def locate(self, xyz):
        """Global curve-order index of the cell containing each integer point (n, 3) of the
        logical grid, -1 if none: numpy in -> numpy int64 out; a torch CUDA uint32/int32
        tensor in -> torch CUDA int64 out."""
        if _is_device(xyz):
            import torch
            _need(xyz.dtype in (torch.int32, torch.uint32) and xyz.numel() % 3 == 0,
                  "xyz: int32/uint32 tensor of shape (n, 3)")
            xyz = xyz.contiguous()
            out = torch.empty(xyz.numel() // 3, dtype=torch.int64, device=xyz.device)
            self._order_in(xyz, out)
            self._check(self._lib.dvl_locate(self._h, out.numel(), _ptr(xyz), _ptr(out), DEVICE),
                        "dvl_locate")
            self._order_out()
            return out
        xyz = np.ascontiguousarray(np.asarray(xyz, dtype=np.uint32).reshape(-1, 3))
        out = np.empty(len(xyz), np.int64)
        self._check(self._lib.dvl_locate(self._h, len(xyz), _ptr(xyz), _ptr(out), HOST), "dvl_locate")
        return out

    def brush(self, W: int, x0: int, x1: int) -> dict:
        """Brushing pixels x0..x1 of the last polylines of width W: the selected
        cells' curve-order range (first, last) and the ROI as Hilbert codes (code_first,
        code_last) -- dvl_brush."""
        out = np.zeros(4, np.uint64)
        self._check(self._lib.dvl_brush(self._h, W, x0, x1, _ptr(out)), "dvl_brush")
        return {"first": int(out[0]), "last": int(out[1]), "code_first": int(out[2]),
                "code_last": int(out[3])}

    def roi_contains(self, xyz, code_lo: int, code_hi: int):
        """The 3D side of brushing: 1 where the cell containing the point has a
        code in [code_lo, code_hi], else 0 (numpy in -> numpy int64; a torch CUDA int32 /
        uint32 tensor in -> torch CUDA int64) -- dvl_roi_contains."""
        if _is_device(xyz):
            import torch
            _need(xyz.dtype in (torch.int32, torch.uint32) and xyz.numel() % 3 == 0,
                  "xyz: int32/uint32 tensor of shape (n, 3)")
            xyz = xyz.contiguous()
            out = torch.empty(xyz.numel() // 3, dtype=torch.int64, device=xyz.device)
            self._order_in(xyz, out)
            self._check(self._lib.dvl_roi_contains(self._h, out.numel(), _ptr(xyz), code_lo, code_hi,
                                                   _ptr(out), DEVICE), "dvl_roi_contains")
            self._order_out()
            return out
        xyz = np.ascontiguousarray(np.asarray(xyz, dtype=np.uint32).reshape(-1, 3))
        out = np.empty(len(xyz), np.int64)
        self._check(self._lib.dvl_roi_contains(self._h, len(xyz), _ptr(xyz), code_lo, code_hi,
                                               _ptr(out), HOST), "dvl_roi_contains")
        return out

    # ------------------------------------------------------------------ sharding
    def set_comm(self, nranks: int, rank: int, uid: bytes):
        """Join the context's own NCCL communicator (collective over the ranks)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        self._check(self._lib.dvl_set_comm(self._h, nranks, rank, buf), "dvl_set_comm")
        self._comm = True

    def set_local_comm(self, group: "LocalGroup", rank: int):
        """Join an in-process group of contexts as `rank` (see LocalGroup)."""
        self._group = group   # keep the handle alive with the context
        self._check(self._lib.dvl_set_local_comm(self._h, group._h, rank), "dvl_set_local_comm")

    def shard(self) -> dict:
        """This context's place in the global curve order: cell_offset, n_global,
        lmax_global (a single-context build: offset 0 and its own n)."""
        info = _ShardInfo()
        self._check(self._lib.dvl_get_shard(self._h, ctypes.byref(info)), "dvl_get_shard")
        return {"cell_offset": info.cell_offset, "n_global": info.n_global,
                "lmax_global": info.lmax_global}

    def set_global_bits(self, bits: int):
        self._check(self._lib.dvl_set_global_bits(self._h, bits), "dvl_set_global_bits")

    def set_shard(self, cell_offset: int, n_global: int, lmax_global: int, vmin=None, vmax=None):
        info = _ShardInfo()
        info.cell_offset, info.n_global, info.lmax_global = cell_offset, n_global, lmax_global
        keep = []
        if vmin is not None:
            vmin = np.ascontiguousarray(vmin, np.float32)
            vmax = np.ascontiguousarray(vmax, np.float32)
            keep = [vmin, vmax]
            info.vmin, info.vmax = _ptr(vmin), _ptr(vmax)
        self._check(self._lib.dvl_set_shard(self._h, ctypes.byref(info)), "dvl_set_shard")
        del keep

    def shard_total(self, dst):
        """Copy this shard's weight total into dst (a torch CUDA int64 tensor element)."""
        self._order_in(dst)
        self._check(self._lib.dvl_shard_total(self._h, _ptr(dst)), "dvl_shard_total")
        self._order_out()

    def shard_export_words(self, W: int) -> int:
        return int(self._lib.dvl_shard_export_words(self._h, W))

    def shard_reduce(self, W: int, totals, shard: int, export):
        """totals: CUDA int64 tensor [nshards]; export: CUDA int64 tensor of export words."""
        import torch
        _need(totals.dtype == torch.int64 and export.dtype == torch.int64
              and export.numel() >= self.shard_export_words(W), "totals / export: int64 tensors")
        self._order_in(totals, export)
        self._check(self._lib.dvl_shard_reduce(self._h, W, _ptr(totals), int(totals.numel()),
                                               shard, _ptr(export)), "dvl_shard_reduce")
        self._order_out()

    def shard_finish(self, W: int, merged, out=None):
        self._order_in(merged)
        if out is not None and _is_device(out):
            _need(out.numel() * out.element_size() >= self.M * int(W) * VERTEX_DTYPE.itemsize, "out too small")
            self._check(self._lib.dvl_shard_finish(self._h, W, _ptr(merged), _ptr(out), DEVICE),
                        "dvl_shard_finish")
            self._order_out()
            return out
        res = np.empty((self.M, W), VERTEX_DTYPE) if out is None else out
        self._check(self._lib.dvl_shard_finish(self._h, W, _ptr(merged), _ptr(res), HOST),
                    "dvl_shard_finish")
        return res

    def set_timing(self, enable: bool):
        """Per-kernel CUDA events on / off (see dvl_set_timing)."""
        self._check(self._lib.dvl_set_timing(self._h, int(bool(enable))), "dvl_set_timing")

    def timings(self) -> dict:
        t = _Timings()
        self._check(self._lib.dvl_get_timings(self._h, ctypes.byref(t)), "dvl_get_timings")
        return {k: getattr(t, k) for k, _ in _Timings._fields_}


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (libnccl.so.2 loaded at run time by the library)."""
    buf = ctypes.create_string_buffer(128)
    if load().dvl_nccl_unique_id(buf) != 0:
        raise DvlError("dvl_nccl_unique_id: libnccl.so.2 not available")
    return buf.raw


class LocalGroup:
    """An in-process group of `nranks` contexts (one host thread per rank), the ABI's
    stand-in for an NCCL communicator on a single GPU: with it every context's build is the
    distributed sample sort and its get_polylines the sharded edit, all inside the library
    (dvl_local_group_create / dvl_set_local_comm)."""

    def __init__(self, nranks: int):
        self._lib = load()
        h = ctypes.c_void_p()
        st = self._lib.dvl_local_group_create(nranks, ctypes.byref(h))
        if st:
            raise DvlError(st, "dvl_local_group_create")
        self._h, self.nranks = h, nranks

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._lib.dvl_local_group_destroy(self._h)
                self._h = None
        except Exception:
            pass


def select_splitters(samples, counts, per_rank: int) -> np.ndarray:
    """The library's sample-sort splitter rule on the host (dvl_select_splitters): samples is
    (G, per_rank) u64 (rank p's first min(per_rank, counts[p]) entries are its regular samples),
    counts the cells per rank; returns G-1 strictly increasing splitters."""
    samples = np.ascontiguousarray(samples, np.uint64)
    counts = np.ascontiguousarray(counts, np.uint64)
    G = len(counts)
    out = np.empty(max(G - 1, 1), np.uint64)
    st = load().dvl_select_splitters(_ptr(samples), _ptr(counts), G, per_rank, _ptr(out))
    if st:
        raise DvlError(st, "dvl_select_splitters")
    return out[: G - 1]
