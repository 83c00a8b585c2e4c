"""Device-resident entry points on CUDA tensors (torch is plumbing only:
device memory and streams).  Planar layout as everywhere: (k, rows, cols)
float64 contiguous tensors, separate Re / Im."""

import torch

from . import _lib


def _stream(t):
    return torch.cuda.current_stream(t.device).cuda_stream


def cgemm(a_re, a_im, b_re, b_im, c_re, c_im, method="3m", epilogue=0):
    """C = A B (epilogue 0) or C -= A B (epilogue 1), on the current stream."""
    k, m, n = a_re.shape
    l = b_re.shape[2]
    _lib.check(_lib.lib().mpc_cgemm(k, 3 if method == "3m" else 4, m, n, l,
                                    a_re.data_ptr(), a_im.data_ptr(), n, m * n,
                                    b_re.data_ptr(), b_im.data_ptr(), l, n * l,
                                    c_re.data_ptr(), c_im.data_ptr(), l, m * l, epilogue,
                                    _stream(a_re)), "cgemm")


def getrf(re, im, piv, K, method="3m"):
    """In-place blocked LU of (k, n, n) tensors; returns the status (-1 ok,
    else the first singular column).  Synchronises the current stream."""
    k, n, _ = re.shape
    return _lib.check(_lib.lib().mpc_getrf(k, 3 if method == "3m" else 4, n, K, re.data_ptr(),
                                           im.data_ptr(), piv.data_ptr(), _stream(re)), "getrf")


def int8_peak(iters=200000):
    """Measured INT8 tensor-core rate of the current device (ops/s)."""
    return float(_lib.lib().mpc_int8_peak(iters, torch.cuda.current_stream().cuda_stream))


def fp64_peak(iters=20000):
    """Measured FP64 issue rate of the current device (lane-ops/s)."""
    return float(_lib.lib().mpc_fp64_peak(iters, torch.cuda.current_stream().cuda_stream))


def cgemm_ozaki(a_re, a_im, b_re, b_im, c_re, c_im, method="3m", d=None, split_bits=None,
                epilogue=0):
    """Ozaki-scheme complex GEMM (real_kernel="ozaki") on device tensors."""
    k, m, n = a_re.shape
    l = b_re.shape[2]
    d = d if d is not None else {2: 6, 3: 8, 4: 12}[k]   # cmatrix.py:26 DEFAULT_SPLITS
    _lib.check(_lib.lib().mpc_cgemm_ozaki(k, 3 if method == "3m" else 4, m, n, l,
                                          a_re.data_ptr(), a_im.data_ptr(), n, m * n,
                                          b_re.data_ptr(), b_im.data_ptr(), l, n * l,
                                          c_re.data_ptr(), c_im.data_ptr(), l, m * l, d,
                                          split_bits or 0, epilogue, _stream(a_re)),
               "cgemm_ozaki")


def getrf_ozaki(re, im, piv, K, method="3m", d=None, split_bits=None):
    """In-place blocked LU with the Ozaki trailing update (lu_blocked with
    KernelChoice(real_kernel="ozaki")); returns the status."""
    k, n, _ = re.shape
    d = d if d is not None else {2: 6, 3: 8, 4: 12}[k]
    return _lib.check(_lib.lib().mpc_getrf_ozaki(k, 3 if method == "3m" else 4, n, K,
                                                 re.data_ptr(), im.data_ptr(), piv.data_ptr(),
                                                 d, split_bits or 0, _stream(re)), "getrf_ozaki")
