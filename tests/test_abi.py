"""The C ABI (include/knnd.h) without a GPU: the library builds for sm_100a,
loads, exports every declared symbol, answers workspace queries and rejects
bad arguments before touching the device."""

from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2202_00517_b200 as b2
from paper_2202_00517_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knnd.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(knnd_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_checked_build_exports_the_same_abi(lib):
    """libknnd_checked.so (bounds-checked, tests/test_checked.py) exports the same
    ABI; the product build compiles the checks out and says so."""
    out = subprocess.run(["nm", "-D", "--defined-only", build.CHECKED_LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name
    cnt, first = C.c_ulonglong(7), C.c_ulonglong(7)
    assert lib.knnd_check_failures(C.byref(cnt), C.byref(first)) == -4  # KNND_EUNSUPPORTED
    assert "product build" in _lib.last_error() and (cnt.value, first.value) == (0, 0)


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_counter(lib):
    assert lib.knnd_abi_version() == 3
    assert b2.launch_count() >= 0


def test_workspace_queries(lib):
    n, d, k = 1_000_000, 20, 20
    assert lib.knnd_csr_workspace_bytes(n, k, 0, n) >= n * 4
    small = lib.knnd_local_join_workspace_bytes(n, d, k, 0, n, 40)
    big = lib.knnd_local_join_workspace_bytes(n, d, k, 0, n, 5000)
    assert small >= 4 * n * 4  # per-class anchor lists
    assert big > small  # hub slabs appear once the in-degree needs global tables
    assert lib.knnd_local_join_workspace_bytes(n, d, 65, 0, n, 40) == 0  # K > 64 unsupported


def test_argument_errors_are_reported(lib):
    null = None
    rc = lib.knnd_local_join(null, null, null, null, 10, 4, 4, null, 3, null, null, 0, 10, 5, null, null, null,
                             null, null, null, null, 0, 0, null)
    assert rc == -1 and "null" in _lib.last_error()
    rc = lib.knnd_csr_build(C.c_void_p(16), 10, 3, 5, 2, C.c_void_p(16), C.c_void_p(16), null, C.c_void_p(16), 1 << 20,
                            null)
    assert rc == -1 and "row range" in _lib.last_error()
    rc = lib.knnd_kl_prepare(C.c_void_p(16), 10, 5, 6, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), null)
    assert rc == -1 and "ld32" in _lib.last_error()
    with pytest.raises(_lib.KnndError):
        _lib.call("knnd_fcc", null, 10, 3, null, null, null, 5, null, null)


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import numpy as np

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        b2.KnnState(np.array([[1, 2], [0, 2], [0, 1]]))
    pts = b2.sample_simplex_uniform(3, 20, 0)
    with pytest.raises(RuntimeError):
        b2.run(b2.Dataset(pts), b2.KlRankingSystem(pts), b2.DescentConfig(k=3))
