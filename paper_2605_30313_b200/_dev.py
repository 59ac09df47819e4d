"""Device-memory plumbing: torch owns HBM allocations and streams, every byte
of arithmetic runs in libunilite_b200 (no torch compute on the product path).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib

_pinned_lock = threading.Lock()
_pinned_ranges: dict[int, int] = {}  # base address -> bytes


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_30313_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise ValueError("expected a CUDA tensor")
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return int(t)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def feature_ld(d: int) -> int:
    """Device row stride for a feature width: 16-byte aligned rows with at
    least one spare column (the MLP's bias 'ones column')."""
    return round_up(max(int(d), 1) + 1, 4)


# ----------------------------------------------------------------- pinned host
class _PinnedOwner:
    def __init__(self, addr: int, nbytes: int):
        self.addr, self.nbytes = addr, nbytes

    def __del__(self):
        try:
            with _pinned_lock:
                _pinned_ranges.pop(self.addr, None)
            _lib.lib().ul_host_free_pinned(C.c_void_p(self.addr))
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array backed by page-locked host memory (cudaHostAlloc)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    p = C.c_void_p()
    _lib.call("ul_host_alloc_pinned", C.byref(p), max(n, 1))
    owner = _PinnedOwner(p.value, max(n, 1))
    with _pinned_lock:
        _pinned_ranges[p.value] = max(n, 1)
    raw = (C.c_char * max(n, 1)).from_address(p.value)
    raw._owner = owner  # keep the allocation alive as long as any view is
    arr = np.frombuffer(raw, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    return arr


def is_pinned(a: np.ndarray) -> bool:
    addr = a.ctypes.data
    with _pinned_lock:
        for base, n in _pinned_ranges.items():
            if base <= addr < base + n:
                return True
    return False


def zeros(shape, dtype=torch.float32, device=None) -> torch.Tensor:
    """Zero-filled CUDA tensor: torch allocates, the fill is a cudaMemsetAsync
    on the current stream (no framework kernel on the product path)."""
    t = torch.empty(shape, dtype=dtype, device=device or require_cuda())
    if t.numel():
        _lib.call("ul_memset_async", ptr(t), 0, t.numel() * t.element_size(), stream())
    return t


def zeros_like(t: torch.Tensor) -> torch.Tensor:
    return zeros(t.shape, t.dtype, t.device)


# ------------------------------------------------------------------- copies
def h2d(dst: torch.Tensor, src: np.ndarray, s: int | None = None) -> None:
    """Contiguous host -> device copy (async when src is pinned)."""
    src = np.ascontiguousarray(src)
    _lib.call("ul_memcpy_async", ptr(dst), src.ctypes.data, src.nbytes,
              stream() if s is None else s)


def h2d_rows(dst: torch.Tensor, src: np.ndarray, s: int | None = None) -> None:
    """Copy host rows [R, D] into a device [R, ld] array (row pitch change)."""
    src = np.ascontiguousarray(src)
    rows = src.shape[0]
    width = src.nbytes // max(rows, 1)
    dpitch = dst.stride(0) * dst.element_size()
    if rows == 0:
        return
    _lib.call("ul_memcpy2d_async", ptr(dst), dpitch, src.ctypes.data, width, width, rows,
              stream() if s is None else s)


def to_device_f32(x, ld: int | None = None) -> torch.Tensor:
    """numpy / torch -> CUDA float32 [R, ld] (rows 16-byte aligned when ld is None)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32:
        if x.dim() != 2 or (ld is None and x.stride(1) == 1) or (ld is not None and x.stride(0) == ld):
            return x
    arr = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    if arr.ndim != 2:
        out = torch.empty(arr.shape, dtype=torch.float32, device=dev)
        h2d(out, arr)
        return out
    rows, d = arr.shape
    ld = feature_ld(d) if ld is None else ld
    buf = zeros((rows, ld), torch.float32, dev)
    h2d_rows(buf, arr)
    return buf[:, :d]


def to_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def to_device_f64(x) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA float64 (host-side dtype cast for the
    transfer only; the arithmetic runs in the kernels)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 \
            and x.is_contiguous():
        return x
    arr = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    out = torch.empty(arr.shape, dtype=torch.float64, device=dev)
    if arr.size:
        h2d(out, arr)
    return out


_API_WORK: dict = {}


def api_work() -> torch.Tensor:
    """Per-device workspace of the per-call reduction kernels (zeroed once:
    its last slot is the self-resetting last-block ticket)."""
    dev = require_cuda()
    w = _API_WORK.get(dev.index)
    if w is None:
        w = zeros(int(_lib.lib().ul_api_work_doubles()), torch.float64, dev)
        _API_WORK[dev.index] = w
    return w
