"""ctypes binding of ``liboxygen_b200.so`` (the C ABI in include/oxygen_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the library is missing every GPU entry point raises.
Status codes map to the reference's exception types (SURVEY.md §8b error
conventions): EINVAL -> ValueError, ENOBLOCKS -> MemoryError, others ->
RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OXY_LIB_VARIANT=<name> loads liboxygen_b200.<name>.so from the same directory
# (A/B builds of the same sources in one gpurun session); unset: the default build
_VARIANT = os.environ.get("OXY_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, f"liboxygen_b200.{_VARIANT}.so" if _VARIANT else "liboxygen_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "oxygen_b200.h")

_lib = None

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class OxyToyConfig(C.Structure):
    _fields_ = [("L", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("vocab", C.c_int32), ("eos_token", C.c_int32), ("action_dim", C.c_int32),
                ("H", C.c_int32), ("seed", C.c_uint64)]


def header_symbols() -> list[str]:
    """Every function the public header declares (for the export test)."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(oxy_\w+)\s*\(", text, re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension not built: {LIB_PATH} missing "
                               f"(run __graft_entry__.build())")
        _lib = C.CDLL(LIB_PATH)
        _lib.oxy_last_error.restype = C.c_char_p
        _lib.oxy_launch_count.restype = C.c_int64
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().oxy_last_error().decode()
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def as_i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def ptr_i32(a: np.ndarray):
    return a.ctypes.data_as(i32p)


def ptr_f64(a: np.ndarray):
    return a.ctypes.data_as(f64p)


def stream_ptr(stream=None):
    """cudaStream_t of a torch stream (default: the current stream)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return vp(s.cuda_stream)
