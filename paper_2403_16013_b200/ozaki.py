"""Ozaki-scheme real kernel -- drop-in for mpclu.ozaki (ozaki.py:1-159).

The split, the ordered accumulation and the final renormalization run as
sm_100a kernels; the scheduled part products are exact binary64 GEMMs on
cuBLAS DGEMM (the reference's ``f64_gemm`` seam, ozaki.py:124-142).  Because
every part product is exact, the result is bit-identical to the reference
for any binary64 GEMM, including a user-supplied ``f64_gemm``.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .rmatrix import RealMatrix, check_threads

DEFAULT_SPLIT_BITS = {2: 19, 3: 21, 4: 18}   # ozaki.py:30


def split_exactness_bound(inner_n):
    """ozaki.py:33-38"""
    if inner_n < 1:
        raise ValueError("inner dimension must be >= 1")
    return int(53 - np.ceil(np.log2(inner_n)) if inner_n > 1 else 53) // 2


def _resolve_width(k, inner_n, split_bits):
    """ozaki.py:41-51"""
    bound = split_exactness_bound(inner_n)
    if bound < 1:
        raise ValueError("dimension exceeds split exactness budget")
    if split_bits is None:
        return min(DEFAULT_SPLIT_BITS.get(k, bound), bound)
    if split_bits < 1:
        raise ValueError("split_bits must be >= 1")
    if split_bits > bound:
        raise ValueError("dimension exceeds split exactness budget")
    return int(split_bits)


@dataclass
class SplitStack:
    """d binary64 parts of one operand (ozaki.py:54-76)."""

    d: int
    width: int
    side: str
    parts: list = field(default_factory=list)
    scales: list = field(default_factory=list)

    @property
    def shape(self):
        return self.parts[0].shape

    def reconstruct(self):
        total = np.zeros(self.shape)
        for p in reversed(self.parts):
            total += p
        return total


def ozaki_split(A, d, side="left", split_bits=None):
    """Split a RealMatrix into d grid-aligned binary64 parts (ozaki.py:79-108)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    if side not in ("left", "right"):
        raise ValueError("side must be 'left' or 'right'")
    inner_n = A.cols if side == "left" else A.rows
    width = _resolve_width(A.k, inner_n, split_bits)
    k, rows, cols = A.data.shape
    parts = np.zeros((d, rows, cols))
    ng = rows if side == "left" else cols
    scales = np.zeros((d, ng))
    if rows * cols:
        _lib.check(_lib.lib().mpc_ozaki_split(k, rows, cols, _lib.ptr(A.data), cols, rows * cols,
                                              d, width, 0 if side == "left" else 1,
                                              _lib.ptr(parts), _lib.ptr(scales), None),
                   "ozaki_split")
    st = SplitStack(d=d, width=width, side=side)
    st.parts = [parts[i] for i in range(d)]
    st.scales = [scales[i] for i in range(d)]
    return st


def _pair_schedule(d, width, k):
    """ozaki.py:111-121"""
    cutoff = 53 * k + 53
    pairs = []
    for s in range(d):
        if s * max(width - 1, 1) >= cutoff:
            break
        for p in range(s + 1):
            pairs.append((p, s - p))
    return pairs


def f64_gemm(X, Y):
    """The device binary64 GEMM used for the exact part products."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    m, n = X.shape
    l = Y.shape[1]
    Z = np.empty((m, l))
    if m * l:
        _lib.check(_lib.lib().mpc_f64_gemm(m, n, l, _lib.ptr(X), n, _lib.ptr(Y), l, _lib.ptr(Z), l,
                                           None), "f64_gemm")
    return Z


def rgemm_ozaki(A, B, d, threads=1, split_bits=None, f64_gemm=None):
    """C = A B through d-way error-free splitting (ozaki.py:124-159)."""
    from .cmatrix import _check_k, _kernel_calls

    if A.k != B.k:
        raise ValueError(f"component counts differ: {A.k} != {B.k}")
    if A.cols != B.rows:
        raise ValueError(f"inner dimensions differ: {A.cols} != {B.rows}")
    check_threads(threads)
    _check_k(A.k)
    _kernel_calls["ozaki"] += 1
    k, m, n = A.data.shape
    l = B.cols
    if f64_gemm is None:
        width = _resolve_width(k, n, split_bits)  # raises like the reference
        if d < 1:
            raise ValueError("d must be >= 1")
        C = np.empty((k, m, l))
        if m * l:
            _lib.check(_lib.lib().mpc_rgemm_ozaki(
                k, m, n, l, _lib.ptr(A.data), n, m * n, _lib.ptr(B.data), l, n * l, _lib.ptr(C), l,
                m * l, d, width if split_bits is not None else 0, None), "rgemm_ozaki")
        else:
            C[...] = 0.0
        return RealMatrix(C)
    # user-supplied binary64 GEMM: split and accumulate on the device, the
    # exact part products through the callable (bit-identical by exactness)
    sa = ozaki_split(A, d, "left", split_bits)
    sb = ozaki_split(B, d, "right", split_bits)
    prods = [np.ascontiguousarray(f64_gemm(sa.parts[p], sb.parts[q]), dtype=np.float64)
             for p, q in _pair_schedule(d, sa.width, k)]
    C = np.zeros((k, m, l))
    L = _lib.lib()
    if m * l:
        for P in prods:
            _lib.check(L.mpc_acc_plane(k, m, l, _lib.ptr(C), l, m * l, _lib.ptr(P), l, None),
                       "acc_plane")
        _lib.check(L.mpc_renorm_planes(k, m, l, _lib.ptr(C), l, m * l, None), "renorm_planes")
    return RealMatrix(C)
