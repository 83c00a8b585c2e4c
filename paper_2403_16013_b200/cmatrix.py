"""Complex multi-component matrix multiply -- drop-in for mpclu.rgemm /
mpclu.cmatrix (rgemm.py:1-73, cmatrix.py:1-177).

Both the real kernels ("naive", "blocked") and the complex 3M / 4M forms run
as ONE fused sm_100a kernel per call (libmpcb200 ``mpc_cgemm``): the three
(3M) or four (4M) real inner-product chains of every output element are
accumulated side by side, ``Re A + Im A`` / ``Re B + Im B`` are formed once
per staged element, and the combine (``Re = T1 - T2``,
``Im = (T3 - T1) - T2`` or ``ir + ri``) runs in the epilogue.  Results are
bit-identical to the reference's composition of real products and plane
additions.  The real-kernel invocation counters keep the reference's
semantics (3 per 3M call, 4 per 4M call, rgemm.py:29-43).
"""

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _lib
from .rmatrix import RealMatrix, check_threads

DEFAULT_BLOCK = 16       # rgemm.py:26
DEFAULT_THRESHOLD = 32   # rgemm.py:27
DEFAULT_SPLITS = {2: 6, 3: 8, 4: 12}   # cmatrix.py:26
DEFAULT_SPLIT_BITS = {2: 19, 3: 21, 4: 18}  # ozaki.py:30

# "b200" names this package's kernel explicitly; "naive" and "blocked" are the
# reference's bitwise-equal schedules and map to the same fused kernel.
REAL_KERNELS = ("naive", "blocked", "strassen", "ozaki", "b200")
METHODS = ("3m", "4m")
SUPPORTED_K = (2, 3, 4)
VERIFY_K = (5, 6, 8)   # verification kernels (k + 2, REFERENCE_K = 8): blocked GEMM / elementwise only

_kernel_calls = {name: 0 for name in REAL_KERNELS}


def real_kernel_calls():
    return dict(_kernel_calls)


def reset_real_kernel_calls():
    for key in _kernel_calls:
        _kernel_calls[key] = 0


def _check_k(k):
    if k not in SUPPORTED_K:
        raise ValueError(f"component count k={k} not supported on the B200 path (2, 3 or 4)")


def _check_mm(A, B):
    if A.k != B.k:
        raise ValueError(f"component counts differ: {A.k} != {B.k}")
    if A.cols != B.rows:
        raise ValueError(f"inner dimensions differ: {A.cols} != {B.rows}")


# ------------------------------------------------------------- real GEMM

def _rgemm(A, B, name):
    _check_mm(A, B)
    if A.k not in VERIFY_K:  # k = 5, 6, 8: the verification kernels (blocked real GEMM)
        _check_k(A.k)
    _kernel_calls[name] += 1
    k, m, n = A.data.shape
    l = B.cols
    C = np.zeros((k, m, l))
    if m * l:
        _lib.check(_lib.lib().mpc_rgemm(k, m, n, l, _lib.ptr(A.data), n, m * n,
                                        _lib.ptr(B.data), l, n * l, _lib.ptr(C), l, m * l, None),
                   "rgemm")
    return RealMatrix(C)


def rgemm_naive(A, B, threads=1):
    """C[i][j] = sum_t A[i][t] B[t][j], strictly t-ascending (rgemm.py:53-60)."""
    check_threads(threads)
    return _rgemm(A, B, "naive")


def rgemm_blocked(A, B, block=DEFAULT_BLOCK, threads=1):
    """Bitwise equal to rgemm_naive for any block (rgemm.py:63-73)."""
    if block < 1:
        raise ValueError("block must be >= 1")
    check_threads(threads)
    return _rgemm(A, B, "blocked")


def _mm(A, B):
    """One blocked real product on the GPU, not counted as a kernel choice."""
    calls = _kernel_calls["blocked"]
    C = _rgemm(A, B, "blocked")
    _kernel_calls["blocked"] = calls
    return C


def _block(M, r0, r1, c0, c1):
    return RealMatrix(np.ascontiguousarray(M.data[:, r0:r1, c0:c1]))


def _strassen(A, B, threshold):
    """Seven-product recursion on square operands (rgemm.py:116-184): every
    leaf product and every plane addition runs on the GPU (mpc_rgemm,
    mpc_mat_add); the recursion itself is host logic.  Odd sizes peel the last
    row / column (rgemm.py:120-148): each border is one product with the even
    core plus one outer-product term, the latter formed as an inner-dimension-1
    product (a zero-initialised chain of length one equals the bare product)."""
    from .rmatrix import _mat_add

    n, k = A.rows, A.k
    if n <= threshold:
        return _mm(A, B)
    if n % 2:
        m = n - 1
        A11, B11 = _block(A, 0, m, 0, m), _block(B, 0, m, 0, m)
        a12, a21, a22 = _block(A, 0, m, m, n), _block(A, m, n, 0, m), _block(A, m, n, m, n)
        b12, b21, b22 = _block(B, 0, m, m, n), _block(B, m, n, 0, m), _block(B, m, n, m, n)
        C = np.empty((k, n, n))
        C[:, :m, :m] = _mat_add(_strassen(A11, B11, threshold), _mm(a12, b21), 1.0).data
        C[:, :m, m:] = _mat_add(_mm(A11, b12), _mm(a12, b22), 1.0).data
        C[:, m:, :m] = _mat_add(_mm(a21, B11), _mm(a22, b21), 1.0).data
        C[:, m:, m:] = _mat_add(_mm(a21, b12), _mm(a22, b22), 1.0).data
        return RealMatrix(C)
    h = n // 2
    A11, A12, A21, A22 = (_block(A, i * h, i * h + h, j * h, j * h + h) for i in (0, 1) for j in (0, 1))
    B11, B12, B21, B22 = (_block(B, i * h, i * h + h, j * h, j * h + h) for i in (0, 1) for j in (0, 1))
    add = lambda X, Y: _mat_add(X, Y, 1.0)   # noqa: E731
    sub = lambda X, Y: _mat_add(X, Y, -1.0)  # noqa: E731
    rec = lambda X, Y: _strassen(X, Y, threshold)  # noqa: E731
    m1 = rec(add(A11, A22), add(B11, B22))
    m2 = rec(add(A21, A22), B11)
    m3 = rec(A11, sub(B12, B22))
    m4 = rec(A22, sub(B21, B11))
    m5 = rec(add(A11, A12), B22)
    m6 = rec(sub(A21, A11), add(B11, B12))
    m7 = rec(sub(A12, A22), add(B21, B22))
    C = np.empty((k, n, n))
    C[:, :h, :h] = add(sub(add(m1, m4), m5), m7).data
    C[:, :h, h:] = add(m3, m5).data
    C[:, h:, :h] = add(m2, m4).data
    C[:, h:, h:] = add(add(sub(m1, m2), m3), m6).data
    return RealMatrix(C)


def rgemm_strassen(A, B, threshold=DEFAULT_THRESHOLD, threads=1):
    """Strassen recursion on square operands (rgemm.py:76-91).  Outside the
    hot path (square-only, so it cannot serve the LU trailing update; SURVEY.md
    §2): kept for API completeness as a host recursion over the GPU's blocked
    product and plane additions.  `threads` never changes bits."""
    _check_mm(A, B)
    if A.rows != A.cols or B.rows != B.cols:
        raise ValueError("strassen kernel requires square operands")
    if threshold < 2:
        raise ValueError("threshold must be >= 2")
    check_threads(threads)
    _check_k(A.k)
    _kernel_calls["strassen"] += 1
    return _strassen(A, B, threshold)


# ----------------------------------------------------------- complex GEMM

@dataclass(frozen=True)
class KernelChoice:
    """One benchmark point (cmatrix.py:32-63)."""

    method: str = "3m"
    real_kernel: str = "blocked"
    block: int = DEFAULT_BLOCK
    threshold: int = DEFAULT_THRESHOLD
    d: Optional[int] = None
    split_bits: Optional[int] = None
    threads: int = 1
    # B200 addition: GPUs of this process the LU is
    # distributed over (1-D block-column-cyclic, mpc_getrf_ngpu); never
    # changes any bit of the result
    ngpus: int = 1

    def validate(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.real_kernel not in REAL_KERNELS:
            raise ValueError(f"unknown real kernel {self.real_kernel!r}")
        if self.block < 1:
            raise ValueError("block must be >= 1")
        if self.threshold < 2:
            raise ValueError("threshold must be >= 2")
        if self.d is not None and self.d < 1:
            raise ValueError("d must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.ngpus < 1:
            raise ValueError("ngpus must be >= 1")
        return self

    def with_threads(self, threads):
        return replace(self, threads=threads)

    def splits_for(self, k):
        return self.d if self.d is not None else DEFAULT_SPLITS.get(k, 8)


class PlanarComplexMatrix:
    """Complex matrix as two planar real matrices (cmatrix.py:66-125)."""

    __slots__ = ("re_plane", "im_plane")

    def __init__(self, re_plane, im_plane):
        if re_plane.data.shape != im_plane.data.shape:
            raise ValueError("planes must share shape and component count")
        self.re_plane = re_plane
        self.im_plane = im_plane

    @property
    def k(self):
        return self.re_plane.k

    @property
    def rows(self):
        return self.re_plane.rows

    @property
    def cols(self):
        return self.re_plane.cols

    @classmethod
    def zeros(cls, rows, cols, k):
        return cls(RealMatrix.zeros(rows, cols, k), RealMatrix.zeros(rows, cols, k))

    @classmethod
    def from_complex128(cls, M, k):
        M = np.asarray(M, dtype=np.complex128)
        return cls(RealMatrix.from_float64(M.real, k), RealMatrix.from_float64(M.imag, k))

    @classmethod
    def identity(cls, n, k):
        return cls(RealMatrix.identity(n, k), RealMatrix.zeros(n, n, k))

    def copy(self):
        return PlanarComplexMatrix(self.re_plane.copy(), self.im_plane.copy())

    def at(self, i, j):
        return (self.re_plane.at(i, j), self.im_plane.at(i, j))

    def bitwise_equal(self, other):
        return self.re_plane.bitwise_equal(other.re_plane) and self.im_plane.bitwise_equal(
            other.im_plane)

    def max_abs(self):
        return max(self.re_plane.max_abs(), self.im_plane.max_abs())

    def __repr__(self):
        return f"PlanarComplexMatrix(k={self.k}, shape={self.rows}x{self.cols})"


def _cgemm_strassen(A, B, kc, method):
    """cgemm_3m / cgemm_4m composed from Strassen real products in the
    reference's order (cmatrix.py:145-169)."""
    from .rmatrix import _mat_add

    rk = lambda X, Y: rgemm_strassen(X, Y, threshold=kc.threshold, threads=kc.threads)  # noqa: E731
    if method == "4m":
        rr, ii = rk(A.re_plane, B.re_plane), rk(A.im_plane, B.im_plane)
        ir, ri = rk(A.im_plane, B.re_plane), rk(A.re_plane, B.im_plane)
        return PlanarComplexMatrix(_mat_add(rr, ii, -1.0), _mat_add(ir, ri, 1.0))
    t1, t2 = rk(A.re_plane, B.re_plane), rk(A.im_plane, B.im_plane)
    t3 = rk(_mat_add(A.re_plane, A.im_plane, 1.0), _mat_add(B.re_plane, B.im_plane, 1.0))
    return PlanarComplexMatrix(_mat_add(t1, t2, -1.0), _mat_add(_mat_add(t3, t1, -1.0), t2, -1.0))


def _cgemm(A, B, kc, method):
    _check_mm(A.re_plane, B.re_plane)
    kc.validate()
    check_threads(kc.threads)
    if kc.real_kernel == "strassen":
        return _cgemm_strassen(A, B, kc, method)
    if not (A.k in VERIFY_K and kc.real_kernel != "ozaki"):
        _check_k(A.k)
    k, m, n = A.re_plane.data.shape
    l = B.cols
    Cre, Cim = np.empty((k, m, l)), np.empty((k, m, l))
    L = _lib.lib()
    meth = 3 if method == "3m" else 4
    if kc.real_kernel == "ozaki":
        # cmatrix.py:128-135 -> rgemm_ozaki per real product, composed on device
        from .ozaki import _resolve_width

        _resolve_width(k, n, kc.split_bits)  # the reference's budget errors
        _kernel_calls["ozaki"] += 3 if method == "3m" else 4
        if m * l:
            _lib.check(L.mpc_cgemm_ozaki(
                k, meth, m, n, l, _lib.ptr(A.re_plane.data), _lib.ptr(A.im_plane.data), n, m * n,
                _lib.ptr(B.re_plane.data), _lib.ptr(B.im_plane.data), l, n * l, _lib.ptr(Cre),
                _lib.ptr(Cim), l, m * l, kc.splits_for(k),
                int(kc.split_bits) if kc.split_bits is not None else 0, 0, None), "cgemm_ozaki")
        return PlanarComplexMatrix(RealMatrix(Cre), RealMatrix(Cim))
    _kernel_calls[kc.real_kernel] += 3 if method == "3m" else 4
    if m * l:
        _lib.check(L.mpc_cgemm(k, meth, m, n, l,
                               _lib.ptr(A.re_plane.data), _lib.ptr(A.im_plane.data), n, m * n,
                               _lib.ptr(B.re_plane.data), _lib.ptr(B.im_plane.data), l, n * l,
                               _lib.ptr(Cre), _lib.ptr(Cim), l, m * l, 0, None), "cgemm")
    return PlanarComplexMatrix(RealMatrix(Cre), RealMatrix(Cim))


def cgemm_4m(A, B, kc=KernelChoice(method="4m")):
    """Four real products, two plane additions (cmatrix.py:145-154)."""
    return _cgemm(A, B, kc, "4m")


def cgemm_3m(A, B, kc=KernelChoice(method="3m")):
    """Three real products, five plane additions (cmatrix.py:157-169)."""
    return _cgemm(A, B, kc, "3m")


def cgemm(A, B, kc):
    """Dispatch on kc.method (cmatrix.py:172-177)."""
    kc.validate()
    if kc.method == "3m":
        return cgemm_3m(A, B, kc)
    return cgemm_4m(A, B, kc)
