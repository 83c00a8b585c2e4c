"""Complex LU with partial pivoting -- drop-in for mpclu.lu (lu.py:1-282).

``lu_blocked`` / ``lu_normal`` run the whole factorization on the B200
(libmpcb200 ``mpc_getrf``): a recursive panel (pivot search by block
argmax, deferred interchanges, chained "S" updates), a right-looking blocked
TRSM for U12 and the fused 3M/4M trailing update ``A22 -= L21 U12``.  Pivots
and packed factors are bit-identical to the reference.  ``solve`` runs
forward substitution bit-identically and backward substitution with a
blocked order (tolerance parity).
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cmatrix import DEFAULT_SPLITS, KernelChoice, PlanarComplexMatrix, _check_k
from .rmatrix import Expansion, RealMatrix, check_threads


class SingularMatrixError(ValueError):
    """lu.py:32-35"""

    def __init__(self, column):
        super().__init__(f"singular matrix at column {column}")
        self.column = column


class ComplexScalar:
    """Value holder for one complex expansion (cscalar.py surface: re, im,
    from_complex, to_complex); the scalar arithmetic API is outside the hot
    path."""

    __slots__ = ("re", "im")

    def __init__(self, re, im):
        if re.k != im.k:
            raise ValueError("re and im must share the component count")
        self.re = re
        self.im = im

    @property
    def k(self):
        return self.re.k

    @classmethod
    def from_complex(cls, z, k):
        z = complex(z)
        return cls(Expansion.from_float(z.real, k), Expansion.from_float(z.imag, k))

    def to_complex(self):
        return complex(self.re.to_float(), self.im.to_float())

    def __eq__(self, other):
        return isinstance(other, ComplexScalar) and self.re == other.re and self.im == other.im

    def __repr__(self):
        return f"ComplexScalar({self.re!r}, {self.im!r})"


class ComplexVector:
    """Planar complex vector: re and im are (k, n) float64 arrays (lu.py:38-82)."""

    __slots__ = ("re", "im")

    def __init__(self, re, im):
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        if re.shape != im.shape or re.ndim != 2:
            raise ValueError("re and im must be (k, n) arrays of equal shape")
        self.re = re
        self.im = im

    @property
    def k(self):
        return self.re.shape[0]

    @property
    def n(self):
        return self.re.shape[1]

    @classmethod
    def zeros(cls, n, k):
        return cls(np.zeros((k, n)), np.zeros((k, n)))

    @classmethod
    def from_scalars(cls, zs):
        """One entry per ComplexScalar (lu.py:63-69)."""
        zs = list(zs)
        if not zs:
            raise ValueError("from_scalars needs at least one scalar")
        v = cls.zeros(len(zs), zs[0].re.k)
        for i, z in enumerate(zs):
            v.set_at(i, z)
        return v

    def copy(self):
        return ComplexVector(self.re.copy(), self.im.copy())

    def at(self, i):
        return ComplexScalar(Expansion(self.re[:, i].copy()), Expansion(self.im[:, i].copy()))

    def set_at(self, i, z):
        if z.re.k != self.k or z.im.k != self.k:
            raise ValueError("component count mismatch")
        self.re[:, i] = z.re.components
        self.im[:, i] = z.im.components

    def bitwise_equal(self, other):
        return bool(np.array_equal(self.re, other.re) and np.array_equal(self.im, other.im))


@dataclass
class LinearSystem:
    """A x = b over planar complex storage (lu.py:85-96)."""

    A: PlanarComplexMatrix
    b: ComplexVector

    def __post_init__(self):
        if self.A.rows != self.A.cols:
            raise ValueError("coefficient matrix must be square")
        if self.b.n != self.A.rows or self.b.k != self.A.k:
            raise ValueError("right-hand side does not match the matrix")


@dataclass
class LUFactors:
    """Packed unit-lower L / U and pivots (lu.py:99-126)."""

    packed: PlanarComplexMatrix
    pivots: np.ndarray
    method: str = "3m"

    @property
    def n(self):
        return self.packed.rows

    def lower(self):
        n, k = self.n, self.packed.k
        L = PlanarComplexMatrix.identity(n, k)
        for c in range(k):
            L.re_plane.data[c] += np.tril(self.packed.re_plane.data[c], -1)
            L.im_plane.data[c] += np.tril(self.packed.im_plane.data[c], -1)
        return L

    def upper(self):
        k = self.packed.k
        U = PlanarComplexMatrix.zeros(self.n, self.n, k)
        for c in range(k):
            U.re_plane.data[c] = np.triu(self.packed.re_plane.data[c])
            U.im_plane.data[c] = np.triu(self.packed.im_plane.data[c])
        return U


# output copies at least this large are page-locked for the call, so the
# C-ABI overlaps their host<->device copies with the factorization
# (HostOverlap); below it the staged copies cost less than registering
_REGISTER_BYTES = 64 << 20


def _par_copy(src):
    """np.copy of a large (k, n, n) plane stack with one thread per row chunk
    (numpy releases the GIL in copyto): the single-threaded copy costs ~1 s
    per 8 GiB."""
    import concurrent.futures as cf
    import os

    out = np.empty_like(src)
    nt = min(16, os.cpu_count() or 1)
    rows = src.shape[1]
    ch = (rows + nt - 1) // nt
    with cf.ThreadPoolExecutor(nt) as ex:
        list(ex.map(lambda i: np.copyto(out[:, i * ch:(i + 1) * ch], src[:, i * ch:(i + 1) * ch]),
                    range(nt)))
    return out


class _Pinned:
    """cudaHostRegister the factor copies for the duration of the call."""

    def __init__(self, arrays):
        self.done = []
        for a in arrays:
            if a.nbytes >= _REGISTER_BYTES and _lib.lib().mpc_host_register(_lib.ptr(a), a.nbytes) == 0:
                self.done.append(a)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        for a in self.done:
            _lib.lib().mpc_host_unregister(_lib.ptr(a))
        return False


def _factor(A, K, method, kc=None):
    """lu._factor (lu.py:129-163) as one device call, on copies of A's
    planes (lu.py:132-133); large copies are page-locked for the call so the
    input / output transfers overlap the factorization."""
    n, k = A.rows, A.k
    _check_k(k)
    big = A.re_plane.data.nbytes >= _REGISTER_BYTES
    re = _par_copy(A.re_plane.data) if big else A.re_plane.data.copy()
    im = _par_copy(A.im_plane.data) if big else A.im_plane.data.copy()
    piv = np.arange(n, dtype=np.int64)
    with _Pinned([re, im]):
        _factor_device(re, im, piv, n, k, K, method, kc)
    packed = PlanarComplexMatrix(RealMatrix(re), RealMatrix(im))
    return LUFactors(packed=packed, pivots=piv, method=method)


def _factor_device(re, im, piv, n, k, K, method, kc):
    meth = 3 if method == "3m" else 4
    if n and kc is not None and kc.ngpus > 1:
        ozk = kc.real_kernel == "ozaki"
        if ozk and n > K:
            from .ozaki import _resolve_width

            _resolve_width(k, K, kc.split_bits)
        st = _lib.check(_lib.lib().mpc_getrf_ngpu(
            k, meth, n, K, _lib.ptr(re), _lib.ptr(im), _lib.ptr(piv), int(kc.ngpus), 1,
            1 if ozk else 0, kc.splits_for(k) if ozk else 0,
            int(kc.split_bits) if (ozk and kc.split_bits is not None) else 0, None),
            "getrf_ngpu")
        if st >= 0:
            raise SingularMatrixError(int(st))
    elif n and kc is not None and kc.real_kernel == "ozaki":
        if n > K:  # the split budget binds only when a trailing update runs
            from .ozaki import _resolve_width

            _resolve_width(k, K, kc.split_bits)
        st = _lib.check(_lib.lib().mpc_getrf_ozaki(
            k, meth, n, K, _lib.ptr(re), _lib.ptr(im), _lib.ptr(piv), kc.splits_for(k),
            int(kc.split_bits) if kc.split_bits is not None else 0, None), "getrf_ozaki")
        if st >= 0:
            raise SingularMatrixError(int(st))
    elif n:
        st = _lib.check(_lib.lib().mpc_getrf(k, meth, n, K, _lib.ptr(re),
                                             _lib.ptr(im), _lib.ptr(piv), None), "getrf")
        if st >= 0:
            raise SingularMatrixError(int(st))


def lu_normal(A, threads=1, method="3m"):
    """Element-wise right-looking factorization (lu.py:166-170)."""
    if A.rows != A.cols:
        raise ValueError("matrix must be square")
    check_threads(threads)
    if method not in ("3m", "4m"):
        raise ValueError(f"unknown method {method!r}")
    return _factor(A, max(A.rows, 1), method)


def lu_blocked(A, K, kc=None, threads=1):
    """Blocked factorization with trailing updates (lu.py:173-187)."""
    if A.rows != A.cols:
        raise ValueError("matrix must be square")
    if not 1 <= K <= A.rows:
        raise ValueError(f"panel width K={K} outside [1, {A.rows}]")
    if kc is None:
        kc = KernelChoice()
    kc = kc.validate().with_threads(threads)
    check_threads(threads)
    if kc.real_kernel == "strassen":
        raise NotImplementedError("strassen is outside the B200 hot path (see DESIGN.md)")
    return _factor(A, K, kc.method, kc)


def trsm_unit_lower(L11, A12, method="3m", threads=1):
    """Solve L11 X = A12, L11 unit lower (lu.py:190-202)."""
    if L11.rows != L11.cols:
        raise ValueError("L11 must be square")
    if A12.rows != L11.rows or A12.k != L11.k:
        raise ValueError("A12 does not match L11")
    check_threads(threads)
    _check_k(L11.k)
    xre = A12.re_plane.data.copy()
    xim = A12.im_plane.data.copy()
    k, K, M = xre.shape
    if K and M:
        _lib.check(_lib.lib().mpc_trsm_ll_unit(
            k, 3 if method == "3m" else 4, K, M, _lib.ptr(L11.re_plane.data),
            _lib.ptr(L11.im_plane.data), K, K * K, _lib.ptr(xre), _lib.ptr(xim), M, K * M, None),
            "trsm_ll_unit")
    return PlanarComplexMatrix(RealMatrix(xre), RealMatrix(xim))


def solve(f, b):
    """x from L U x = P b (lu.py:205-218)."""
    n = f.n
    if b.n != n or b.k != f.packed.k:
        raise ValueError("right-hand side does not match the factors")
    k = f.packed.k
    _check_k(k)
    re = np.ascontiguousarray(f.packed.re_plane.data)
    im = np.ascontiguousarray(f.packed.im_plane.data)
    diag_zero = (re[0].diagonal() == 0.0) & (im[0].diagonal() == 0.0)
    if diag_zero.any():
        raise SingularMatrixError(int(np.argmax(diag_zero)))
    x = b.copy()
    piv = np.ascontiguousarray(f.pivots, dtype=np.int64)
    if n:
        _lib.check(_lib.lib().mpc_getrs(k, 3 if f.method == "3m" else 4, n, _lib.ptr(re),
                                        _lib.ptr(im), _lib.ptr(piv), _lib.ptr(x.re),
                                        _lib.ptr(x.im), None), "getrs")
    return x


def permuted(A, pivots):
    """Apply the factorization's row interchanges to a copy of A (lu.py:221-229)."""
    re = A.re_plane.data.copy()
    im = A.im_plane.data.copy()
    for i, p in enumerate(pivots):
        if p != i:
            re[:, [i, p], :] = re[:, [p, i], :]
            im[:, [i, p], :] = im[:, [p, i], :]
    return PlanarComplexMatrix(RealMatrix(re), RealMatrix(im))


def max_rel_err(xhat, x):
    """max_i |xhat_i - x_i| / |x_i| over complex moduli (lu.py:263-282), on
    the GPU in the reference's expansion arithmetic: the returned Expansion
    is the reference's value bit for bit (mpc_max_rel_err)."""
    if xhat.n != x.n or xhat.k != x.k:
        raise ValueError("vectors must share length and component count")
    k, n = x.k, x.n
    out = np.zeros(k)
    if n == 0:
        return Expansion(out)
    if k not in (2, 3, 4):
        raise ValueError(f"component count k={k} not supported on the B200 path (2, 3 or 4)")
    zero = np.full(1, -1, dtype=np.int64)
    _lib.check(_lib.lib().mpc_max_rel_err(k, n, _lib.ptr(xhat.re), _lib.ptr(xhat.im),
                                          _lib.ptr(x.re), _lib.ptr(x.im), _lib.ptr(out),
                                          _lib.ptr(zero), None), "max_rel_err")
    if zero[0] >= 0:
        raise ValueError(f"zero true component at index {int(zero[0])}")
    return Expansion(out)


def _check_inplace_args(re, im, piv):
    """factor_inplace's buffers: the C side assumes (k, n, n) planes with
    ld = n, ps = n*n, both on one device (or both host numpy) and an int64
    pivot vector of length n on the same side."""
    is_np = isinstance(re, np.ndarray)
    if is_np != isinstance(im, np.ndarray):
        raise ValueError("re and im must both be numpy arrays or both CUDA tensors")
    if len(re.shape) != 3 or re.shape[1] != re.shape[2]:
        raise ValueError(f"planes must have shape (k, n, n), got {tuple(re.shape)}")
    if tuple(im.shape) != tuple(re.shape):
        raise ValueError("re and im shapes differ")
    if is_np:
        for name, a in (("re", re), ("im", im)):
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError(f"{name} must be C-contiguous float64")
    else:
        import torch

        for name, a in (("re", re), ("im", im)):
            if not isinstance(a, torch.Tensor) or a.dtype != torch.float64 or not a.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float64 tensor")
            if not a.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor (or pass numpy arrays)")
        if re.device != im.device:
            raise ValueError("re and im are on different devices")
    if piv is None:
        return
    n = re.shape[1]
    if is_np:
        if not isinstance(piv, np.ndarray) or piv.dtype != np.int64 or not piv.flags.c_contiguous:
            raise ValueError("piv must be a C-contiguous int64 numpy array")
    else:
        import torch

        if (not isinstance(piv, torch.Tensor) or piv.dtype != torch.int64
                or not piv.is_contiguous() or piv.device != re.device):
            raise ValueError("piv must be a contiguous int64 tensor on the planes' device")
    if tuple(piv.shape) != (n,):
        raise ValueError(f"piv must have shape ({n},), got {tuple(piv.shape)}")


def factor_inplace(re, im, K, method="3m", piv=None, real_kernel="blocked", d=None,
                   split_bits=None):
    """In-place variant of lu_blocked on raw planar buffers (no copies):
    ``re``/``im`` are (k, n, n) float64 C-contiguous numpy arrays (pinned or
    pageable host memory, staged by the C-ABI) or CUDA tensors (device
    memory, factored in place on the current stream).  ``piv`` (optional) is
    an int64 vector of length n on the same side; it is allocated there when
    omitted.  Returns the pivots; raises SingularMatrixError like lu_blocked
    and ValueError on malformed buffers."""
    _check_inplace_args(re, im, piv)
    k, n, _ = re.shape
    _check_k(k)
    if not 1 <= K <= max(n, 1):
        raise ValueError(f"panel width K={K} outside [1, {n}]")
    if method not in ("3m", "4m"):
        raise ValueError(f"unknown method {method!r}")
    stream = None
    if isinstance(re, np.ndarray):
        if piv is None:
            piv = np.empty(n, dtype=np.int64)
    else:
        import torch

        if piv is None:
            piv = torch.empty(n, dtype=torch.int64, device=re.device)
        stream = torch.cuda.current_stream(re.device).cuda_stream
    if n == 0:
        return piv
    if real_kernel == "ozaki":
        from .ozaki import _resolve_width

        d = d if d is not None else DEFAULT_SPLITS[k]
        if n > K:  # the budget applies only when a trailing update runs
            _resolve_width(k, K, split_bits)
        st = _lib.check(_lib.lib().mpc_getrf_ozaki(
            k, 3 if method == "3m" else 4, n, K, _lib.ptr(re), _lib.ptr(im), _lib.ptr(piv), d,
            int(split_bits) if split_bits is not None else 0, stream), "getrf_ozaki")
    else:
        st = _lib.check(_lib.lib().mpc_getrf(k, 3 if method == "3m" else 4, n, K, _lib.ptr(re),
                                             _lib.ptr(im), _lib.ptr(piv), stream), "getrf")
    if st >= 0:
        raise SingularMatrixError(int(st))
    return piv


def _promote(M, k_new):
    return PlanarComplexMatrix(M.re_plane.promote(k_new), M.im_plane.promote(k_new))


def reconstruction_error(f, A, threads=8, extra=2):
    """max componentwise |PA - LU| over both planes (lu.py:236-250), with the
    L U product at k + extra components through the GPU kernel, 3M blocked as
    the reference (k + extra in 2..6 or 8: the verification kernels beyond
    k = 4)."""
    from .cmatrix import SUPPORTED_K, VERIFY_K, cgemm

    kk = f.packed.k + extra
    if kk not in SUPPORTED_K + VERIFY_K:
        raise NotImplementedError(f"no kernels at k + extra = {kk} (2..6, 8)")
    from .rmatrix import mat_sub

    PA = _promote(permuted(A, f.pivots), kk)
    L = _promote(f.lower(), kk)
    U = _promote(f.upper(), kk)
    LU = cgemm(L, U, KernelChoice(method="3m", real_kernel="blocked", threads=threads))
    dre = mat_sub(PA.re_plane, LU.re_plane)
    dim = mat_sub(PA.im_plane, LU.im_plane)
    return max(dre.max_abs(), dim.max_abs())


def backward_error_probe(f, A, seed=0):
    """O(n^2) estimate of the normwise backward error ||PA - LU|| / ||A||
    (infinity norm, |Re| + |Im| moduli): r = P A v - L (U v) for a seeded
    random vector v, evaluated at k + 2 components (DD: the quad-double
    kernels; TD / QD: the k = 5, 6 verification kernels) with the GPU GEMM at
    l = 1.  Returns ||r|| / (||A|| ||v||), a lower bound of the normwise
    backward error."""
    from .cmatrix import cgemm

    k, n = f.packed.k, f.n
    kk = k + 2
    if kk > 6:
        raise NotImplementedError("probe needs k + 2 <= 6")
    rng = np.random.Generator(np.random.Philox(key=np.uint64(seed + 12345)))
    v = np.zeros((2, kk, n, 1))
    v[0, 0, :, 0] = rng.uniform(-1, 1, n)
    v[1, 0, :, 0] = rng.uniform(-1, 1, n)
    V = PlanarComplexMatrix(RealMatrix(v[0]), RealMatrix(v[1]))
    kc = KernelChoice(method="4m")
    PA = _promote(permuted(A, f.pivots), kk)
    y3 = cgemm(PA, V, kc)
    del PA
    U = _promote(f.upper(), kk)
    y1 = cgemm(U, V, kc)
    del U
    L = _promote(f.lower(), kk)
    y2 = cgemm(L, y1, kc)
    del L
    from .rmatrix import mat_sub

    rr = mat_sub(y3.re_plane, y2.re_plane).data
    ri = mat_sub(y3.im_plane, y2.im_plane).data
    rnorm = float(np.max(np.abs(rr[0]) + np.abs(ri[0])))
    anorm = float(np.max(np.sum(np.abs(A.re_plane.data[0]) + np.abs(A.im_plane.data[0]), axis=1)))
    vnorm = float(np.max(np.abs(v[0, 0]) + np.abs(v[1, 0])))
    return rnorm / (anorm * vnorm)
