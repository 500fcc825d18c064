"""Device plans (FFT tables, spectra, Gamma/shift tables) and buffer helpers.

A space plan wraps ``bhcp_space_plan`` (DST-I FFT tables + the 1D Laplacian
spectrum mu1 of space.py:209-211); a time plan wraps ``bhcp_time_plan``
(time FFT tables + gamma, 1/gamma and the shifts d_j/tau of pint.py:95).
Plans are immutable and cached per device, like the reference memoises
``laplacian_eigenvalues`` (space.py:202).
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _lib

_cache_lock = threading.Lock()
_space_cache: "OrderedDict[tuple, SpacePlan]" = OrderedDict()
_time_cache: "OrderedDict[tuple, TimePlan]" = OrderedDict()
_MAX_SPACE = 32
_MAX_TIME = 256


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class SpacePlan:
    def __init__(self, device: int, dim: int, num_cells: int, mu1: np.ndarray):
        lib = _lib.lib()
        mu1 = np.ascontiguousarray(mu1, dtype=np.float64)
        handle = ctypes.c_void_p()
        _lib.check(
            lib.bhcp_space_plan_create(device, dim, num_cells, _dptr(mu1), ctypes.byref(handle)),
            "bhcp_space_plan_create",
        )
        self.handle = handle
        self.device = device
        self.dim = dim
        self.num_cells = num_cells
        self.m = num_cells - 1
        self.n_space = self.m**dim
        self.mu1 = mu1

    def __del__(self):
        try:
            if self.handle:
                _lib.load_library().bhcp_space_plan_destroy(self.handle)
        except Exception:
            pass


class TimePlan:
    def __init__(self, device: int, gamma: np.ndarray, shifts: np.ndarray):
        lib = _lib.lib()
        n = int(gamma.shape[0])
        gam = np.ascontiguousarray(gamma, dtype=np.complex128)
        # circulant.py:115 divides by gamma; the device multiplies by 1/gamma
        # computed once here with numpy's complex division.
        gam_inv = np.ascontiguousarray(1.0 / gam)
        sh = np.ascontiguousarray(shifts, dtype=np.complex128)
        handle = ctypes.c_void_p()
        _lib.check(
            lib.bhcp_time_plan_create(
                device, n,
                gam.view(np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                gam_inv.view(np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                sh.view(np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                ctypes.byref(handle),
            ),
            "bhcp_time_plan_create",
        )
        self.handle = handle
        self.device = device
        self.n = n
        self.gamma = gam
        self.shifts = sh

    def __del__(self):
        try:
            if self.handle:
                _lib.load_library().bhcp_time_plan_destroy(self.handle)
        except Exception:
            pass


def current_device() -> int:
    _lib.lib()
    return torch.cuda.current_device()


def space_plan(dim: int, num_cells: int, mu1: np.ndarray, device: int | None = None) -> SpacePlan:
    device = current_device() if device is None else device
    key = (device, dim, num_cells, mu1.tobytes())
    with _cache_lock:
        plan = _space_cache.get(key)
        if plan is not None:
            _space_cache.move_to_end(key)
            return plan
    plan = SpacePlan(device, dim, num_cells, mu1)
    with _cache_lock:
        _space_cache[key] = plan
        while len(_space_cache) > _MAX_SPACE:
            _space_cache.popitem(last=False)
    return plan


def time_plan(gamma: np.ndarray, shifts: np.ndarray, device: int | None = None) -> TimePlan:
    device = current_device() if device is None else device
    key = (device, gamma.shape[0], gamma.tobytes(), shifts.tobytes())
    with _cache_lock:
        plan = _time_cache.get(key)
        if plan is not None:
            _time_cache.move_to_end(key)
            return plan
    plan = TimePlan(device, gamma, shifts)
    with _cache_lock:
        _time_cache[key] = plan
        while len(_time_cache) > _MAX_TIME:
            _time_cache.popitem(last=False)
    return plan


# ---------------------------------------------------------------- buffers

def stream_handle(stream: torch.cuda.Stream | None = None) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def to_device(x, dtype: torch.dtype) -> torch.Tensor:
    """numpy or torch input -> contiguous tensor of `dtype` on the current device."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(device=torch.device("cuda", torch.cuda.current_device()))
        return t.to(dtype).contiguous()
    a = np.asarray(x)
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=dtype).contiguous()


def status_block() -> torch.Tensor:
    n = _lib.load_library().bhcp_status_bytes()
    return torch.empty(int(n), dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))


def read_status(status: torch.Tensor, tol: float = 1e-8) -> _lib.Status:
    st = _lib.Status()
    _lib.check(
        _lib.lib().bhcp_read_status(ptr(status), tol, ctypes.byref(st), stream_handle()),
        "bhcp_read_status",
    )
    return st


def reset_status(status: torch.Tensor) -> None:
    _lib.check(_lib.lib().bhcp_status_reset(ptr(status), stream_handle()), "bhcp_status_reset")


def transpose(src: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    """Out-of-place transpose of a (rows, cols) float64/complex128 matrix (own kernel)."""
    out = torch.empty((cols, rows), dtype=src.dtype, device=src.device)
    _lib.check(
        _lib.lib().bhcp_transpose(ptr(src), ptr(out), rows, cols, src.element_size(), stream_handle()),
        "bhcp_transpose",
    )
    return out
