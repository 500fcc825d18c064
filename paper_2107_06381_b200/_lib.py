"""ctypes binding of libbhcp_b200.so (C ABI declared in include/bhcp_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2107_06381_b200/csrc``). There is no CPU fallback: every
numeric entry point of this package goes through this library, and
``lib()`` raises ``NativeLibraryError`` when it is missing or when no CUDA
device is available.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbhcp_b200.so"
HEADER_PATH = _HERE.parent / "include" / "bhcp_b200.h"

BHCP_OK = 0
BHCP_ERR_SINGULAR_SHIFT = 1
BHCP_ERR_IMAGINARY_RESIDUE = 2
BHCP_ERR_INVALID = 3
BHCP_ERR_CUDA = 4


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or reported a CUDA error."""


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int),
        ("bad_column", ctypes.c_int64),
        ("residue", ctypes.c_double),
        ("norm", ctypes.c_double),
    ]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); mirrors include/bhcp_b200.h
SIGNATURES = {
    "bhcp_version": (_int, []),
    "bhcp_last_error": (ctypes.c_char_p, []),
    "bhcp_status_bytes": (ctypes.c_size_t, []),
    "bhcp_space_plan_create": (_int, [_int, _int, _int, _dp, ctypes.POINTER(_vp)]),
    "bhcp_space_plan_destroy": (None, [_vp]),
    "bhcp_time_plan_create": (_int, [_int, _int, _dp, _dp, _dp, ctypes.POINTER(_vp)]),
    "bhcp_time_plan_destroy": (None, [_vp]),
    "bhcp_sine_transform": (_int, [_vp, _vp, _vp, _int, _i64, _vp]),
    "bhcp_sine_axis": (_int, [_vp, _vp, _vp, _int, _i64, _int, _vp]),
    "bhcp_step_b": (_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "bhcp_to_eigenspace": (_int, [_vp, _vp, _int, _i64, _i64, _i64, _vp, _i64, _i64, _vp]),
    "bhcp_from_eigenspace": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _int, _i64, _i64, _vp, _vp]),
    "bhcp_status_reset": (_int, [_vp, _vp]),
    "bhcp_read_status": (_int, [_vp, _dbl, ctypes.POINTER(Status), _vp]),
    "bhcp_pint_workspace_bytes": (ctypes.c_size_t, [_vp, _vp]),
    "bhcp_pint_status_ptr": (_vp, [_vp, _vp, _vp]),
    "bhcp_pint_solve": (_int, [_vp, _vp, _vp, _dbl, _vp, _vp, ctypes.c_size_t, _vp]),
    "bhcp_pint_unfused_workspace_bytes": (ctypes.c_size_t, [_vp, _vp]),
    "bhcp_pint_unfused_status_ptr": (_vp, [_vp, _vp, _vp]),
    "bhcp_pint_solve_unfused": (_int, [_vp, _vp, _vp, _dbl, _vp, _vp, ctypes.c_size_t, _vp]),
    "bhcp_pint_ghat": (_int, [_vp, _vp, _dbl, _vp, _vp]),
    "bhcp_pint_modes": (_int, [_vp, _vp, _vp, _i64, _i64, _vp, _int, _vp, _vp, _vp]),
    "bhcp_pint_sym_tiles": (_i64, [_vp, _vp]),
    "bhcp_pint_modes_sym_to": (_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _int, _vp, _vp, _vp]),
    "bhcp_pint_modes_to": (_int, [_vp, _vp, _vp, _i64, _i64, _vp, _int, _vp, _vp, _vp]),
    "bhcp_pint_level_pass": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "bhcp_pint_w_pass": (_int, [_vp, _vp, _i64, _int, _vp]),
    "bhcp_pint_w_passes_supported": (_int, [_vp]),
    "bhcp_pint_levels": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "bhcp_pint_levels_sync_bytes": (ctypes.c_size_t, [_vp, _i64]),
    "bhcp_pint_batch_workspace_bytes": (ctypes.c_size_t, [_vp, _vp, _int]),
    "bhcp_pint_solve_batch": (_int, [_vp, _vp, _int, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "bhcp_pint_levels_fused": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "bhcp_pint_levels_blocked": (_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "bhcp_spectral_workspace_bytes": (ctypes.c_size_t, [_vp, _i64]),
    "bhcp_spectral_solve": (_int, [_vp, _int, _dbl, _dbl, _i64, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "bhcp_march_forward": (_int, [_vp, _dbl, _i64, _vp, _vp, _vp]),
    "bhcp_residual_workspace_bytes": (ctypes.c_size_t, []),
    "bhcp_residual_norm": (_int, [_vp, _vp, _i64, _dbl, _dbl, _dbl, _vp, _vp, _dp, _vp]),
    "bhcp_transpose": (_int, [_vp, _vp, _i64, _i64, _int, _vp]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: os.PathLike | str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every signature (no CUDA calls)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not Path(path).exists():
            raise NativeLibraryError(
                f"{path} is missing: build the CUDA library first "
                f"(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    """The loaded library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError(
            "no CUDA device: the B200 solver has no CPU fallback by design"
        )
    return load_library()


def last_error() -> str:
    return load_library().bhcp_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Raise on a non-OK return code from a launch-type entry point."""
    if rc == BHCP_OK:
        return
    msg = f"{what} failed (code {rc}): {last_error()}"
    if rc == BHCP_ERR_INVALID:
        raise ValueError(msg)
    raise NativeLibraryError(msg)
