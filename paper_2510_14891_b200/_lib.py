"""ctypes binding of the sm_100a C ABI (include/cpk_b200.h).

This is the only door from Python into the CUDA kernels.  There is no CPU
fallback: if the library is missing or CUDA is unavailable every entry point
raises DeviceError.  The binding passes raw device pointers and the current
torch CUDA stream handle; ctypes releases the GIL for the call.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import (
    CpkernError,
    DeviceError,
    IndexRangeError,
    ParameterError,
    FormatError,
    ResourceError,
    ShapeError,
)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libcpk_b200.so"

CPK_OK = 0
_CODE_TO_EXC = {
    1: ShapeError,
    2: IndexRangeError,
    3: ParameterError,
    4: ResourceError,
    5: DeviceError,
    6: DeviceError,
    7: DeviceError,
    8: FormatError,
}
CPK_ERR_NOT_PD = 6
CPK_MAX_MODES = 16
CPK_DTEN_MAX_MODES = 64
CPK_SUMSQ_PARTIALS = 1024


class CpkPlan(C.Structure):
    _fields_ = [
        ("rank_tile", C.c_int32),
        ("block_rows", C.c_int32),
        ("tile_volume", C.c_int64),
        ("splits", C.c_int32),
        ("sm_count", C.c_int32),
        ("block_k", C.c_int32),
        ("engine", C.c_int32),
        ("merge", C.c_int32),
    ]


# name -> (restype, argtypes); keep in the header's order.
_P = C.c_void_p
_I64 = C.c_int64
_PROTOS = {
    "cpk_last_error": (C.c_char_p, []),
    "cpk_version": (C.c_char_p, []),
    "cpk_plan_resolve": (C.c_int, [C.c_int, C.POINTER(_I64), C.c_int, _I64, C.POINTER(CpkPlan)]),
    "cpk_mttkrp_workspace_bytes": (
        C.c_int,
        [C.c_int, C.POINTER(_I64), C.c_int, _I64, C.POINTER(CpkPlan), C.POINTER(C.c_size_t)],
    ),
    "cpk_mttkrp_f64": (
        C.c_int,
        [_P, C.c_int, C.POINTER(_I64), C.c_int, C.POINTER(_P), C.POINTER(_I64), _P, _I64, _P, _I64,
         C.POINTER(CpkPlan), _P, C.c_size_t, _P],
    ),
    "cpk_mttkrp_f64_landed": (
        C.c_int,
        [_P, C.c_int, C.POINTER(_I64), C.c_int, C.POINTER(_P), C.POINTER(_I64), _P, _I64, _P, _I64,
         C.POINTER(CpkPlan), _P, C.c_size_t, _P, _I64, _I64],
    ),
    "cpk_mttkrp_f32_workspace_bytes": (C.c_int, [C.c_int, C.POINTER(_I64), C.c_int, _I64, C.c_int,
                                                  C.POINTER(C.c_size_t)]),
    "cpk_mttkrp_f32": (
        C.c_int,
        [_P, C.c_int, C.POINTER(_I64), C.c_int, C.POINTER(_P), C.POINTER(_I64), _P, _I64, _P, _I64, C.c_int,
         _P, C.c_size_t, _P],
    ),
    "cpk_mttkrp_elem_f64": (
        C.c_int,
        [_P, C.c_int, C.POINTER(_I64), C.c_int, C.POINTER(_P), C.POINTER(_I64), _P, _I64, _P, _I64, _P],
    ),
    "cpk_gram_f64": (C.c_int, [_P, _I64, _I64, _I64, _P, _P]),
    "cpk_hadamard_f64": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int, _I64, _P, _P]),
    "cpk_solve_workspace_bytes": (C.c_int, [_I64, _I64, C.POINTER(C.c_size_t)]),
    "cpk_solve_normal_f64": (C.c_int, [_P, _P, _I64, _I64, _P, C.c_size_t, _P]),
    "cpk_solve_normal_spec_f64": (C.c_int, [_P, _P, _I64, _I64, _P, C.c_size_t, _P, _P]),
    "cpk_solve_factor_spec_f64": (C.c_int, [_P, _I64, _P, C.c_size_t, _P, _P]),
    "cpk_solve_apply_spec_f64": (C.c_int, [_P, _I64, _I64, _P, C.c_size_t, _P, _P]),
    "cpk_dimtree_contract_f64": (C.c_int, [_P, _I64, C.c_int, C.POINTER(_I64), C.c_int, C.POINTER(_P),
                                           C.POINTER(_I64), _I64, _P, _I64, _P]),
    "cpk_colnorms_sq_f64": (C.c_int, [_P, _I64, _I64, _I64, _P, _P]),
    "cpk_scale_columns_f64": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "cpk_normalize_columns_f64": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "cpk_fit_terms_f64": (C.c_int, [_P, _P, _P, _P, _I64, _I64, _P, _P]),
    "cpk_sumsq_f64": (C.c_int, [_P, _I64, _P, _P, _P]),
    "cpk_fill_uniform_f64": (C.c_int, [_P, _I64, C.c_uint64, _I64, _P]),
    "cpk_fill_uniform_slab_f64": (C.c_int, [_P, C.c_int, C.POINTER(_I64), C.c_int, _I64, _I64, C.c_uint64, _P]),
    "cpk_fp64_peak_probe": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "cpk_dten_read_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(_I64)]),
    "cpk_dten_load_slab_f64": (C.c_int, [C.c_char_p, C.c_int, _I64, _I64, _P, _I64, C.c_int, _P]),
}

_lock = threading.Lock()
_lib = None


def exported_symbols():
    return list(_PROTOS)


def load(path: Path | None = None):
    """Load (once) and return the ctypes library; raise DeviceError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"sm_100a library not built ({p}); run `python -c \"import __graft_entry__ as g; g.build()\"`"
            )
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:
            raise DeviceError(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in _PROTOS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = "") -> None:
    if rc == CPK_OK:
        return
    msg = load().cpk_last_error().decode(errors="replace")
    exc = _CODE_TO_EXC.get(rc, CpkernError)
    raise exc(f"{what}: {msg}" if what else msg)


def i64_array(vals):
    arr = (_I64 * len(vals))(*[int(v) for v in vals])
    return arr


def ptr_array(ptrs):
    return (_P * len(ptrs))(*[int(p) if p else None for p in ptrs])
