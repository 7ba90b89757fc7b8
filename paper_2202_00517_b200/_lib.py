"""ctypes binding of libknnd.so (include/knnd.h).

There is no fallback: if the library is missing or a call fails, this raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .build import CHECKED_LIB_PATH, LIB_PATH

_lib = None


class KnndError(RuntimeError):
    """A libknnd call returned a nonzero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed with code {code}: {msg}")
        self.code = code


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_SZ = C.c_size_t

_SIGS = {
    "knnd_abi_version": ([], C.c_int),
    "knnd_last_error": ([], C.c_char_p),
    "knnd_launch_count": ([], C.c_ulonglong),
    "knnd_check_failures": ([_P, _P], C.c_int),
    "knnd_kl_prepare": ([_P, _I64, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "knnd_batch_scores": ([_P, _P, _P, _I64, _I32, _I64, _P, _I64, _P, _P], C.c_int),
    "knnd_csr_workspace_bytes": ([_I64, _I32, _I64, _I64], _SZ),
    "knnd_csr_build": ([_P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "knnd_csr_build_ev": ([_P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _SZ, _P, _P], C.c_int),
    "knnd_local_join_workspace_bytes": ([_I64, _I32, _I32, _I64, _I64, _I32], _SZ),
    "knnd_local_join": ([_P, _P, _P, _P, _I64, _I32, _I32, _P, _I32, _P, _P, _I64, _I64, _I32, _P, _P, _P, _P,
                         _P, _P, _P, _SZ, C.c_uint32, _P], C.c_int),
    "knnd_local_join_peers": ([_P, _P, _P, _P, _I64, _I32, _I32, _P, _I32, _P, _P, _I64, _I64, _I32, _P, _P, _P,
                               _P, _P, _P, _P, _SZ, C.c_uint32, _P, _I32, _P, _P, _I32, _P, _P], C.c_int),
    "knnd_kl_q23_workspace_bytes": ([_I32], _SZ),
    "knnd_kl_q23_prepare": ([_P, _I64, _I32, _I32, _P, _P, _P, _SZ, _P], C.c_int),
    "knnd_fcc": ([_P, _I64, _I32, _P, _P, _P, _I32, _P, _P], C.c_int),
    "knnd_sort_rows": ([_P, _P, _P, _I64, _I32, _I32, _I64, _I64, _P, _P, _P, _P], C.c_int),
    "knnd_exact_knn_workspace_bytes": ([_I64, _I32, _I64, _I32], _SZ),
    "knnd_exact_knn": ([_P, _P, _P, _P, _I64, _I32, _I32, _P, _I64, _I32, _I32, _P, _P, _P, _P, _SZ, C.c_uint32, _P],
                       C.c_int),
    "knnd_l2_prepare": ([_P, _P, _I64, _I32, _I32, _P, _P, _P, _P, _P], C.c_int),
    "knnd_l2_batch_scores": ([_P, _P, _I64, _I32, _I64, _P, _I64, _P, _P], C.c_int),
    "knnd_l2_sort_rows": ([_P, _P, _I64, _I32, _I32, _I64, _I64, _P, _P, _P, _P], C.c_int),
    "knnd_l2_local_join": ([_P, _P, _P, _P, _I64, _I32, _I32, C.c_double, _P, _I32, _P, _P, _I64, _I64, _I32, _P, _P,
                            _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "knnd_l2_local_join_peers": ([_P, _P, _P, _P, _I64, _I32, _I32, C.c_double, _P, _I32, _P, _P, _I64, _I64, _I32,
                                  _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _I32, _P, _P, _I32, _P, _P], C.c_int),
    "knnd_l2_exact_knn": ([_P, _P, _P, _P, _I64, _I32, _I32, C.c_double, _P, _I64, _I32, _I32, _P, _P, _P, _P, _SZ,
                           _P], C.c_int),
    "knnd_random_kout_workspace_bytes": ([_I64, _I32], _SZ),
    "knnd_random_kout": ([C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _I32, C.c_uint32, _I64, _I32, _P, _P, _P,
                          _P, _P, _SZ, _P], C.c_int),
}

EXPORTS = tuple(_SIGS)

JOIN_NONPOS_LOG = 1  # KNND_JOIN_NONPOS_LOG
MAX_PEERS = 15  # KNND_MAX_PEERS


def peer_array(ptrs) -> C.Array | None:
    """Host array of peer-table device pointers for the *_local_join_peers entries."""
    if not ptrs:
        return None
    return (C.c_void_p * len(ptrs))(*[int(x) for x in ptrs])


def load(path: str | None = None):
    """Load (once) and return the library with typed signatures."""
    global _lib
    if _lib is not None:
        return _lib
    # KNND_LIBRARY=checked selects the bounds-checked build (tests/test_checked.py)
    env = os.environ.get("KNND_LIBRARY")
    path = path or (CHECKED_LIB_PATH if env == "checked" else env) or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"libknnd.so not found at {path}; build it with `python -m paper_2202_00517_b200.build` "
            "(there is no CPU fallback)"
        )
    L = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def last_error() -> str:
    return load().knnd_last_error().decode(errors="replace")


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise KnndError(name, rc, last_error())


def launch_count() -> int:
    return int(load().knnd_launch_count())
