"""ctypes binding of libmpcb200.so (include/mpc_b200.h).

The product path has no CPU fallback: if the shared object is missing or no
CUDA device is visible, every operation raises ``RuntimeError`` loudly.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmpcb200.so")

_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double
_p = ctypes.c_void_p

_SIGS = {
    "mpc_abi_version": (_i, []),
    "mpc_last_error": (ctypes.c_char_p, []),
    "mpc_device_count": (_i, []),
    "mpc_max_rel_err": (_i, [_i, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "mpc_mat_add": (_i, [_i, _i64, _i64, _p, _i64, _i64, _p, _i64, _i64, _p, _i64, _i64, _d, _p]),
    "mpc_renorm_planes": (_i, [_i, _i64, _i64, _p, _i64, _i64, _p]),
    "mpc_rgemm": (_i, [_i, _i64, _i64, _i64, _p, _i64, _i64, _p, _i64, _i64, _p, _i64, _i64, _p]),
    "mpc_cgemm": (_i, [_i, _i, _i64, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _i64, _i64,
                       _p, _p, _i64, _i64, _i, _p]),
    "mpc_trsm_ll_unit": (_i, [_i, _i, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _i64, _i64, _p]),
    "mpc_lu_panel": (_i64, [_i, _i, _i64, _p, _p, _p, _i64, _i64, _p]),
    "mpc_panel_factor": (_i64, [_i, _i, _i64, _i64, _i64, _p, _p, _i64, _i64, _p, _p]),
    "mpc_panel_factor_async": (_i, [_i, _i, _i64, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _p]),
    "mpc_laswp": (_i, [_i, _i64, _p, _p, _i64, _i64, _p, _i64, _i64, _p]),
    "mpc_getrf": (_i64, [_i, _i, _i64, _i64, _p, _p, _p, _p]),
    "mpc_getrs": (_i, [_i, _i, _i64, _p, _p, _p, _p, _p, _p]),
    "mpc_host_register": (_i, [_p, _i64]),
    "mpc_host_unregister": (_i, [_p]),
    "mpc_getrf_ngpu": (ctypes.c_int64, [_i, _i, _i64, _i64, _p, _p, _p, _i, _i, _i, _i, _i, _p]),
    "mpc_getrs_phases": (_i, [_i, _i, _i64, _p, _p, _p, _p, _p, _i, _p]),
    "mpc_ozaki_split": (_i, [_i, _i64, _i64, _p, _i64, _i64, _i, _i, _i, _p, _p, _p]),
    "mpc_acc_plane": (_i, [_i, _i64, _i64, _p, _i64, _i64, _p, _i64, _p]),
    "mpc_f64_gemm": (_i, [_i64, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, _p]),
    "mpc_rgemm_ozaki": (_i, [_i, _i64, _i64, _i64, _p, _i64, _i64, _p, _i64, _i64, _p, _i64,
                             _i64, _i, _i, _p]),
    "mpc_cgemm_ozaki": (_i, [_i, _i, _i64, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _i64, _i64,
                             _p, _p, _i64, _i64, _i, _i, _i, _p]),
    "mpc_getrf_ozaki": (_i64, [_i, _i, _i64, _i64, _p, _p, _p, _i, _i, _p]),
    "mpc_prof_enable": (None, [_i]),
    "mpc_prof_summary": (_i, [_p, _p, _p, _i]),
    "mpc_launch_count": (ctypes.c_longlong, []),
    "mpc_fp64_peak": (_d, [_i, _p]),
    "mpc_int8_peak": (_d, [_i, _p]),
}

PROF_CLASSES = ("gemm", "supdate", "panel", "trsm_diag", "laswp", "other", "solve")

MPC_ERR = -2

_lib = None


def lib():
    """The loaded library; raises RuntimeError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA extension missing: {LIB_PATH} (run python -m paper_2403_16013_b200.build); "
            "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols():
    return list(_SIGS)


def last_error():
    return lib().mpc_last_error().decode()


def check(rc, what):
    if rc == MPC_ERR:
        raise RuntimeError(f"{what}: {last_error()}")
    return rc


def require_device():
    n = lib().mpc_device_count()
    if n < 1:
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
    return n


def ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def prof_enable(on=True, classes=None):
    """Event-time every launch of the given classes (default: all)."""
    if not on:
        mask = 0
    elif classes is None:
        mask = (1 << len(PROF_CLASSES)) - 1
    else:
        mask = sum(1 << PROF_CLASSES.index(c) for c in classes)
    lib().mpc_prof_enable(mask)


def prof_summary():
    """{class: (ms, ops, launches)} since prof_enable(True)."""
    n = len(PROF_CLASSES)
    ms = np.zeros(n)
    ops = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    check(lib().mpc_prof_summary(ms.ctypes.data, ops.ctypes.data, cnt.ctypes.data, n),
          "prof_summary")
    return {c: (float(ms[i]), float(ops[i]), int(cnt[i])) for i, c in enumerate(PROF_CLASSES)}


def launch_count():
    return int(lib().mpc_launch_count())
