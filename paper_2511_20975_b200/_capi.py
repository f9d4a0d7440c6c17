"""ctypes binding of the C ABI in include/aragog_b200.h.

The shared library is built in-tree (paper_2511_20975_b200/libaragog_b200.so,
see csrc/Makefile).  There is no fallback: if the library is missing or no
CUDA device is present, the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libaragog_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "aragog_b200.h")

AG_OK = 0
AG_ERR_INTERNAL = 1
AG_ERR_VALIDATION = 2
AG_ERR_IO = 3
AG_ERR_CUDA = 4

AG_ROUTER_ORACLE = 0
AG_ROUTER_NOISY = 1
AG_FORCE_TOP = 1


class AgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"aragog_b200 error {code}: {msg}")
        self.code = code


class ValidationError(AgError):
    """Mirrors aragog::ValidationError (include/aragog/errors.h:22-27)."""


class Router(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fp", C.c_double), ("fn", C.c_double),
                ("noise_seed", C.c_uint64), ("eval_latency", C.c_double)]


class Truth(C.Structure):
    _fields_ = [("n_requests", C.c_int32), ("request_ids", C.c_void_p), ("seed_ptr", C.c_void_p),
                ("seeds", C.c_void_p), ("removed_ptr", C.c_void_p), ("removed", C.c_void_p)]


class RouteOut(C.Structure):
    _fields_ = [("bitmap", C.c_void_p), ("counts", C.c_void_p), ("offsets", C.c_void_p),
                ("indices", C.c_void_p), ("capacity", C.c_uint64), ("overflow", C.c_void_p)]


class LinearHeads(C.Structure):
    _fields_ = [("dim", C.c_int32), ("heads", C.c_void_p), ("bias", C.c_void_p)]


class GenParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("p_easy", "p_medium", "p_hard", "easy_base_prob",
                                           "violation_rate")]


_lib = None


def release(fn_name: str, handle) -> None:
    """Destroy a C handle from __del__; a no-op during interpreter shutdown
    (module globals already torn down) or when the library never loaded."""
    try:
        if _lib is not None and handle is not None and handle.value:
            getattr(_lib, fn_name)(handle)
    except Exception:  # noqa: BLE001 -- finalizers must not raise
        pass


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                              "or make -C paper_2511_20975_b200/csrc")
        L = C.CDLL(LIB_PATH)
        L.ag_last_error.restype = C.c_char_p
        L.ag_ctx_launch_count.restype = C.c_uint64
        L.ag_ctx_launch_count.argtypes = [C.c_void_p]
        for name in ("ag_space_destroy", "ag_ctx_destroy"):
            getattr(L, name).restype = None
            getattr(L, name).argtypes = [C.c_void_p]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != AG_OK:
        msg = lib().ag_last_error().decode()
        if rc == AG_ERR_VALIDATION:
            raise ValidationError(rc, msg)
        raise AgError(rc, msg)


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^[a-z_0-9 ]+\*?\s*\**(ag_[a-z_0-9]+)\(", text, re.M)))
