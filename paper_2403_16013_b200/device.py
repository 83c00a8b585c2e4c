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


def getrs(re, im, piv, b_re, b_im, method="3m", phases=3):
    """solve_fb (lu.py:205-218) on device factors: b ((k, n) tensors) is
    overwritten with x.  phases: 1 = interchanges + forward substitution,
    2 = backward substitution, 3 = both."""
    k, n, _ = re.shape
    _lib.check(_lib.lib().mpc_getrs_phases(k, 3 if method == "3m" else 4, n, re.data_ptr(),
                                           im.data_ptr(), piv.data_ptr(), b_re.data_ptr(),
                                           b_im.data_ptr(), int(phases), _stream(re)), "getrs")


def mat_add(a, b, c, sign=1.0):
    """C = A + sign B elementwise on (k, rows, cols) tensors (mat_add_k)."""
    k, m, n = a.shape
    _lib.check(_lib.lib().mpc_mat_add(k, m, n, a.data_ptr(), n, m * n, b.data_ptr(), n, m * n,
                                      c.data_ptr(), n, m * n, float(sign), _stream(a)), "mat_add")


def accuracy(a_re, a_im, f_re, f_im, piv, method="3m", seed=0):
    """BASELINE's accuracy report for a device-resident factorization of A
    (k-limb planes a_re / a_im; packed factors f_re / f_im; pivots piv):

    * forward error: b = A x_true with x_true = 1 + 1i (the DD 4M product,
      BASELINE configs 0 / 2 / 4), x = getrs(b), max_i |x_i - x_true_i| /
      |x_true_i| in binary64 from the limb-wise difference (lu.max_rel_err gives
      the reference's expansion-arithmetic value of the same metric);
    * backward error: lu.backward_error_probe on the device -- r = P A v -
      L (U v) at k + 2 components for a seeded v, ||r|| / (||A|| ||v||) in
      the infinity norm of |Re| + |Im| moduli (a lower bound of the
      normwise backward error), against the 10 n u bound.

    Needs one (2, k + 2, n, n) scratch pair (17 GB at n = 16384, DD)."""
    k, n, _ = a_re.shape
    kk = k + 2
    dev = a_re.device
    # forward error
    xr = torch.zeros((k, n, 1), dtype=torch.float64, device=dev)
    xr[0] = 1.0
    xi = xr.clone()
    br = torch.empty_like(xr)
    bi = torch.empty_like(xr)
    cgemm(a_re, a_im, xr, xi, br, bi, method="4m")
    br2, bi2 = br.reshape(k, n).contiguous(), bi.reshape(k, n).contiguous()
    getrs(f_re, f_im, piv, br2, bi2, method)

    def ldiff(x, c):
        d = torch.zeros(n, dtype=torch.float64, device=dev)
        for q in range(k - 1, -1, -1):
            d += x[q] - (c if q == 0 else 0.0)
        return d

    fwd = float((torch.hypot(ldiff(br2, 1.0), ldiff(bi2, 1.0)) / (2.0 ** 0.5)).max())
    # backward-error probe at k + 2
    g = torch.Generator(device="cpu").manual_seed(12345 + seed)
    vr = torch.zeros((kk, n, 1), dtype=torch.float64)
    vi = torch.zeros((kk, n, 1), dtype=torch.float64)
    vr[0, :, 0] = torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1
    vi[0, :, 0] = torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1
    vr, vi = vr.to(dev), vi.to(dev)
    Pr = torch.zeros((kk, n, n), dtype=torch.float64, device=dev)
    Pi = torch.zeros_like(Pr)
    y = [torch.empty((kk, n, 1), dtype=torch.float64, device=dev) for _ in range(6)]
    Pr[:k].copy_(a_re)
    Pi[:k].copy_(a_im)
    cgemm(Pr, Pi, vr, vi, y[0], y[1], method="4m")          # A v
    p = piv.cpu().numpy()
    perm = list(range(n))
    for i in range(n):                                          # row swaps in order
        j = int(p[i])
        perm[i], perm[j] = perm[j], perm[i]
    perm_t = torch.tensor(perm, device=dev)
    y[0] = y[0][:, perm_t].contiguous()                         # P A v
    y[1] = y[1][:, perm_t].contiguous()
    Pr.zero_()
    Pi.zero_()
    Pr[:k].copy_(torch.triu(f_re))
    Pi[:k].copy_(torch.triu(f_im))
    cgemm(Pr, Pi, vr, vi, y[2], y[3], method="4m")          # U v
    Pr.zero_()
    Pi.zero_()
    Pr[:k].copy_(torch.tril(f_re, diagonal=-1))
    Pi[:k].copy_(torch.tril(f_im, diagonal=-1))
    Pr[0].diagonal().fill_(1.0)
    cgemm(Pr, Pi, y[2], y[3], y[4], y[5], method="4m")      # L (U v)
    del Pr, Pi
    rr = torch.empty_like(y[0])
    ri = torch.empty_like(y[1])
    mat_add(y[0], y[4], rr, -1.0)
    mat_add(y[1], y[5], ri, -1.0)
    rnorm = float((rr[0].abs() + ri[0].abs()).max())
    anorm = float((a_re[0].abs() + a_im[0].abs()).sum(dim=1).max())
    vnorm = float((vr[0].abs() + vi[0].abs()).max())
    u = 2.0 ** (-52 * k)
    bwd = rnorm / (anorm * vnorm)
    return {"fwd_err": fwd, "bwd_err_probe": bwd, "bwd_bound_10nu": 10.0 * n * u,
            "bwd_ok": bool(bwd <= 10.0 * n * u), "u": u, "probe_k": kk,
            "x_true": "1+1i", "b": "A x_true, 4M at k (device)"}
