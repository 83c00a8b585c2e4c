"""C-ABI checks that need no GPU: the shared object loads, exports every
symbol declared in include/mpc_b200.h, and rejects bad arguments before
touching the device."""

import ctypes
import os
import re

import numpy as np
import pytest

from testpaths import ROOT

HEADER = os.path.join(ROOT, "include", "mpc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_16013_b200 import _lib
    from paper_2403_16013_b200.build import build

    build()
    return _lib.lib()


def test_all_declared_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_covers_header(lib):
    from paper_2403_16013_b200 import _lib

    assert sorted(_lib.exported_symbols()) == declared_symbols()


def test_version_and_errors(lib):
    from paper_2403_16013_b200 import _lib

    assert lib.mpc_abi_version() == 1
    a = np.zeros((2, 2, 2))
    # bad k, method, epilogue and mixed/negative sizes fail with a message, no device needed
    rc = lib.mpc_cgemm(7, 3, 2, 2, 2, *[a.ctypes.data] * 2, 2, 4, *[a.ctypes.data] * 2, 2, 4,
                       *[a.ctypes.data] * 2, 2, 4, 0, None)
    assert rc == _lib.MPC_ERR and "k must be" in _lib.last_error()
    # k = 5, 6, 8: verification kernels (GEMM / elementwise); none at k = 7
    rc = lib.mpc_cgemm(7, 4, 2, 2, 2, *[a.ctypes.data] * 2, 2, 4, *[a.ctypes.data] * 2, 2, 4,
                       *[a.ctypes.data] * 2, 2, 4, 0, None)
    assert rc == _lib.MPC_ERR and "5, 6, 8" in _lib.last_error()
    rc = lib.mpc_getrf(5, 4, 4, 2, a.ctypes.data, a.ctypes.data, a.ctypes.data, None)
    assert rc == _lib.MPC_ERR and "k must be" in _lib.last_error()
    rc = lib.mpc_cgemm(2, 5, 2, 2, 2, *[a.ctypes.data] * 2, 2, 4, *[a.ctypes.data] * 2, 2, 4,
                       *[a.ctypes.data] * 2, 2, 4, 0, None)
    assert rc == _lib.MPC_ERR and "method" in _lib.last_error()
    rc = lib.mpc_getrf(2, 3, 4, 0, a.ctypes.data, a.ctypes.data, a.ctypes.data, None)
    assert rc == _lib.MPC_ERR and "panel width" in _lib.last_error()
    rc = lib.mpc_lu_panel(2, 3, 4, a.ctypes.data, a.ctypes.data, a.ctypes.data, 3, 2, None)
    assert rc == _lib.MPC_ERR and "panel outside" in _lib.last_error()


def test_no_cpu_fallback_without_device(lib):
    """On a box without a GPU the product path must fail loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_16013_b200 import (PlanarComplexMatrix, RealMatrix, cgemm, KernelChoice,
                                       _lib)

    assert lib.mpc_device_count() == 0
    A = PlanarComplexMatrix(RealMatrix(np.ones((2, 3, 3))), RealMatrix(np.ones((2, 3, 3))))
    with pytest.raises(RuntimeError):
        cgemm(A, A, KernelChoice())


def test_oracle_is_not_imported_by_package():
    """The product package never imports the checker."""
    pkg = os.path.join(ROOT, "paper_2403_16013_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_factor_inplace_validates_buffers():
    """lu.factor_inplace checks shape, dtype, contiguity, device and piv
    before any pointer reaches the C-ABI (no GPU needed: it raises first)."""
    import torch

    from paper_2403_16013_b200 import lu as lum

    n = 8
    ok = np.zeros((2, n, n))
    bad_cases = [
        (np.zeros((2, n, n), dtype=np.float32), ok, None),          # dtype
        (np.zeros((2, n, n + 1)), np.zeros((2, n, n + 1)), None),   # not square
        (np.zeros((2, n, n)).transpose(0, 2, 1), ok, None),         # not contiguous
        (ok, np.zeros((2, n + 1, n + 1)), None),                    # shapes differ
        (ok, ok.copy(), np.zeros(n, dtype=np.int32)),               # piv dtype
        (ok, ok.copy(), np.zeros(n - 1, dtype=np.int64)),           # piv length
        (ok, torch.zeros((2, n, n), dtype=torch.float64), None),    # mixed numpy / tensor
        (torch.zeros((2, n, n), dtype=torch.float64),               # CPU tensors
         torch.zeros((2, n, n), dtype=torch.float64), None),
    ]
    for re, im, piv in bad_cases:
        with pytest.raises(ValueError):
            lum.factor_inplace(re, im, 4, piv=piv)
    with pytest.raises(ValueError):
        lum.factor_inplace(ok, ok.copy(), 4, method="5m")
