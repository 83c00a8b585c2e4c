"""ctypes wrapper around the CPU oracle (oracle/mpc_oracle.c).

TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA product
path: it may be imported by tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py, never by the
product package ``paper_2403_16013_b200``.

Every function restates the reference routine cited in its docstring
(paths relative to /root/reference/pkg/src/mpclu/).  Arrays use the
reference's planar layout: real matrices ``(k, rows, cols)`` float64
C-contiguous, complex matrices as separate Re / Im arrays.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libmpc_oracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double

_lib = None


def build():
    """Compile the oracle (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    sig = {
        "orc_renorm1": (None, [_dp, _int, _dp, _int]),
        "orc_nonoverlapping": (_int, [_dp, _int]),
        "orc_two_sum": (None, [_dbl, _dbl, _dp, _dp]),
        "orc_two_prod": (None, [_dbl, _dbl, _dp, _dp]),
        "orc_exp_add1": (None, [_dp, _dp, _dp, _int]),
        "orc_exp_sub1": (None, [_dp, _dp, _dp, _int]),
        "orc_exp_mul1": (None, [_dp, _dp, _dp, _int]),
        "orc_exp_div1": (None, [_dp, _dp, _dp, _int]),
        "orc_cmul_3m": (None, [_dp, _dp, _dp, _dp, _dp, _dp, _int]),
        "orc_cmul_4m": (None, [_dp, _dp, _dp, _dp, _dp, _dp, _int]),
        "orc_cdiv": (None, [_dp, _dp, _dp, _dp, _dp, _dp, _int]),
        "orc_mat_add": (None, [_int, _i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64,
                               _dp, _i64, _i64, _dbl]),
        "orc_rgemm": (None, [_int, _i64, _i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64,
                             _dp, _i64, _i64]),
        "orc_cgemm": (None, [_int, _int, _i64, _i64, _i64, _dp, _dp, _i64, _i64, _dp, _dp,
                             _i64, _i64, _dp, _dp]),
        "orc_renorm_planes": (None, [_int, _i64, _i64, _dp]),
        "orc_acc_plane": (None, [_int, _i64, _i64, _dp, _dp]),
        "orc_lu_panel": (_i64, [_int, _int, _i64, _dp, _dp, _i64p, _i64, _i64]),
        "orc_trsm_ll_unit": (None, [_int, _int, _i64, _i64, _dp, _dp, _i64, _i64, _dp, _dp,
                                    _i64, _i64]),
        "orc_factor": (_i64, [_int, _int, _i64, _i64, _dp, _dp, _i64p]),
        "orc_factor_range": (_i64, [_int, _int, _i64, _i64, _dp, _dp, _i64p, _i64, _i64]),
        "orc_solve_fb": (None, [_int, _int, _i64, _dp, _dp, _i64p, _dp, _dp]),
        "orc_solve_phases": (None, [_int, _int, _i64, _dp, _dp, _i64p, _dp, _dp, _int]),
        "orc_set_threads": (_int, [_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(t):
    """Number of OpenMP threads (0 = query).  Bits never depend on it."""
    return _load().orc_set_threads(int(t))


# ---------------------------------------------------------------- scalars

def two_sum(a, b):
    """_kernels.py:28-34"""
    s, e = ctypes.c_double(), ctypes.c_double()
    _load().orc_two_sum(float(a), float(b), ctypes.byref(s), ctypes.byref(e))
    return s.value, e.value


def two_prod(a, b):
    """_kernels.py:45-60 (Dekker)"""
    p, e = ctypes.c_double(), ctypes.c_double()
    _load().orc_two_prod(float(a), float(b), ctypes.byref(p), ctypes.byref(e))
    return p.value, e.value


def renorm(raw, k):
    """renorm1, _kernels.py:308-315 -> renorm 124-139"""
    raw = _c(raw)
    out = np.empty(k)
    _load().orc_renorm1(_d(raw), raw.shape[0], _d(out), k)
    return out


def nonoverlapping(x):
    """_is_nonoverlapping, _kernels.py:108-121"""
    x = _c(x)
    return bool(_load().orc_nonoverlapping(_d(x), x.shape[0]))


def _binop(name, x, y):
    x, y = _c(x), _c(y)
    out = np.empty(x.shape[0])
    getattr(_load(), name)(_d(x), _d(y), _d(out), x.shape[0])
    return out


def exp_add(x, y):
    """exp_add_core, _kernels.py:174-184"""
    return _binop("orc_exp_add1", x, y)


def exp_sub(x, y):
    """exp_sub_core, _kernels.py:187-197"""
    return _binop("orc_exp_sub1", x, y)


def exp_mul(x, y):
    """exp_mul_core, _kernels.py:200-222"""
    return _binop("orc_exp_mul1", x, y)


def exp_div(x, y):
    """exp_div_core, _kernels.py:225-255"""
    return _binop("orc_exp_div1", x, y)


def _cop(name, ar, ai, br, bi):
    ar, ai, br, bi = _c(ar), _c(ai), _c(br), _c(bi)
    k = ar.shape[0]
    outr, outi = np.empty(k), np.empty(k)
    getattr(_load(), name)(_d(ar), _d(ai), _d(br), _d(bi), _d(outr), _d(outi), k)
    return outr, outi


def cmul_3m(ar, ai, br, bi):
    """cmul_3m_core, _kernels.py:527-537"""
    return _cop("orc_cmul_3m", ar, ai, br, bi)


def cmul_4m(ar, ai, br, bi):
    """cmul_4m_core, _kernels.py:539-546"""
    return _cop("orc_cmul_4m", ar, ai, br, bi)


def cdiv(ar, ai, br, bi):
    """cdiv_core, _kernels.py:549-561"""
    return _cop("orc_cdiv", ar, ai, br, bi)


# ---------------------------------------------------------------- matrices

def mat_add(A, B, sign=1.0):
    """mat_add_k, _kernels.py:327-342 (C = A + sign*B)"""
    A, B = _c(A), _c(B)
    k, m, n = A.shape
    C = np.empty_like(A)
    _load().orc_mat_add(k, m, n, _d(A), n, m * n, _d(B), n, m * n, _d(C), n, m * n,
                        float(sign))
    return C


def mat_sub(A, B):
    return mat_add(A, B, -1.0)


def rgemm(A, B):
    """rgemm_naive_k, _kernels.py:384-395 (== rgemm_blocked_k bitwise)"""
    A, B = _c(A), _c(B)
    k, m, n = A.shape
    l = B.shape[2]
    C = np.empty((k, m, l))
    _load().orc_rgemm(k, m, n, l, _d(A), n, m * n, _d(B), l, n * l, _d(C), l, m * l)
    return C


def cgemm(Are, Aim, Bre, Bim, method="3m"):
    """cgemm_3m / cgemm_4m, cmatrix.py:145-169 -> (Cre, Cim)"""
    Are, Aim, Bre, Bim = _c(Are), _c(Aim), _c(Bre), _c(Bim)
    k, m, n = Are.shape
    l = Bre.shape[2]
    Cre, Cim = np.empty((k, m, l)), np.empty((k, m, l))
    _load().orc_cgemm(k, 3 if method == "3m" else 4, m, n, l, _d(Are), _d(Aim), n, m * n,
                      _d(Bre), _d(Bim), l, n * l, _d(Cre), _d(Cim))
    return Cre, Cim


def renorm_planes(R):
    """renorm_planes, _kernels.py:485-499 (in place; R must be contiguous)"""
    assert R.flags.c_contiguous and R.dtype == np.float64
    k, m, n = R.shape
    _load().orc_renorm_planes(k, m, n, _d(R))
    return R


def acc_plane(C, P):
    """acc_plane, _kernels.py:502-517 (in place on C)"""
    assert C.flags.c_contiguous
    P = _c(P)
    k, m, n = C.shape
    _load().orc_acc_plane(k, m, n, _d(C), _d(P))
    return C


# ---------------------------------------------------------------- LU

def lu_panel(re, im, piv, jb, kw, use3m):
    """lu_panel, _kernels.py:611-665 (in place); returns -1 or singular col"""
    k, n, _ = re.shape
    return _load().orc_lu_panel(k, int(bool(use3m)), n, _d(re), _d(im),
                                piv.ctypes.data_as(_i64p), jb, kw)


def trsm_ll_unit(lre, lim, are, aim, use3m):
    """trsm_ll_unit, _kernels.py:668-705 (in place on are/aim)"""
    lre, lim = _c(lre), _c(lim)
    k, K, _ = lre.shape
    M = are.shape[2]
    assert are.flags.c_contiguous and aim.flags.c_contiguous
    _load().orc_trsm_ll_unit(k, int(bool(use3m)), K, M, _d(lre), _d(lim), K, K * K,
                             _d(are), _d(aim), M, K * M)


def factor(re, im, K, method="3m"):
    """lu._factor, lu.py:129-163 on copies -> (re, im, piv, status)"""
    re, im = _c(re).copy(), _c(im).copy()
    k, n, _ = re.shape
    piv = np.arange(n, dtype=np.int64)
    st = _load().orc_factor(k, int(method == "3m"), n, K, _d(re), _d(im),
                            piv.ctypes.data_as(_i64p))
    return re, im, piv, int(st)


def factor_range(re, im, piv, K, method, jb0, jb1):
    """Panels jb in [jb0, jb1) of lu._factor IN PLACE on C-contiguous float64
    planes and an int64 piv (arange before the first stage) -> status."""
    assert re.flags.c_contiguous and im.flags.c_contiguous and piv.dtype == np.int64
    k, n, _ = re.shape
    lib = _load()
    return int(lib.orc_factor_range(k, int(method == "3m"), n, K, _d(re), _d(im),
                                    piv.ctypes.data_as(_i64p), jb0, jb1))


def solve_fb(re, im, piv, br, bi, method="3m", phases=3):
    """solve_fb, _kernels.py:708-775 -> (xr, xi); phases 1 = interchanges +
    forward sweep only, 2 = backward sweep only, 3 = both"""
    re, im = _c(re), _c(im)
    k, n, _ = re.shape
    xr, xi = _c(br).copy(), _c(bi).copy()
    piv = np.ascontiguousarray(piv, dtype=np.int64)
    _load().orc_solve_phases(k, int(method == "3m"), n, _d(re), _d(im),
                             piv.ctypes.data_as(_i64p), _d(xr), _d(xi), int(phases))
    return xr, xi
