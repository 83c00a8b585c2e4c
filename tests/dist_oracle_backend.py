"""CPU backend for the distributed LU schedule (TEST INFRASTRUCTURE ONLY):
the same calls as paper_2403_16013_b200.dist.CudaBackend, executed by the
oracle on torch CPU tensors so the block-column-cyclic schedule, the panel
packing, the broadcasts (gloo) and the interchange bookkeeping can be
checked bitwise against the single-process oracle factorization."""

import numpy as np
import torch
from numpy.lib.stride_tricks import as_strided

from oracle import oracle as orc


def _view(t, off, shape, ld, ps):
    flat = t.numpy().reshape(-1)
    assert off >= 0
    k, r, c = shape
    return as_strided(flat[off:], shape=(k, r, c), strides=(ps * 8, ld * 8, 8))


class OracleBackend:
    def __init__(self, k, method, real_kernel="blocked"):
        self.k = k
        self.method = method
        self.ozaki = real_kernel == "ozaki"

    def empty(self, shape, dtype="f64"):
        return torch.zeros(shape, dtype=torch.float64 if dtype == "f64" else torch.int64)

    def panel_factor(self, V, n, jb, kw, piv):
        k = self.k
        vr = _view(V.re, V.off + jb, (k, n, kw), V.ld, V.ps)
        vi = _view(V.im, V.off + jb, (k, n, kw), V.ld, V.ps)
        Tr = np.zeros((k, n, n))
        Ti = np.zeros((k, n, n))
        Tr[:, :, jb:jb + kw] = vr
        Ti[:, :, jb:jb + kw] = vi
        p = piv.numpy()
        st = orc.lu_panel(Tr, Ti, p, jb, kw, self.method == "3m")
        vr[...] = Tr[:, :, jb:jb + kw]
        vi[...] = Ti[:, :, jb:jb + kw]
        return st

    def laswp(self, V, ncols, piv, r0, r1):
        if ncols <= 0:
            return
        p = piv.numpy()
        n = max(int(p[r0:r1].max()) + 1, r1)
        for t in (V.re, V.im):
            v = _view(t, V.off, (self.k, n, ncols), V.ld, V.ps)
            for r in range(r0, r1):
                q = int(p[r])
                if q != r:
                    tmp = v[:, r, :].copy()
                    v[:, r, :] = v[:, q, :]
                    v[:, q, :] = tmp

    def trsm(self, L11, X, kb, M):
        if M <= 0:
            return
        k = self.k
        lr = np.ascontiguousarray(_view(L11.re, L11.off, (k, kb, kb), L11.ld, L11.ps))
        li = np.ascontiguousarray(_view(L11.im, L11.off, (k, kb, kb), L11.ld, L11.ps))
        xr_v = _view(X.re, X.off, (k, kb, M), X.ld, X.ps)
        xi_v = _view(X.im, X.off, (k, kb, M), X.ld, X.ps)
        xr, xi = np.ascontiguousarray(xr_v), np.ascontiguousarray(xi_v)
        orc.trsm_ll_unit(lr, li, xr, xi, self.method == "3m")
        xr_v[...] = xr
        xi_v[...] = xi

    def gemm_sub(self, A, B, C, m, kin, l):
        if m <= 0 or l <= 0:
            return
        k = self.k
        ar = _view(A.re, A.off, (k, m, kin), A.ld, A.ps)
        ai = _view(A.im, A.off, (k, m, kin), A.ld, A.ps)
        br = _view(B.re, B.off, (k, kin, l), B.ld, B.ps)
        bi = _view(B.im, B.off, (k, kin, l), B.ld, B.ps)
        if self.ozaki:
            from oracle import ozaki_ref

            pr, pi = ozaki_ref.cgemm(np.ascontiguousarray(ar), np.ascontiguousarray(ai),
                                     np.ascontiguousarray(br), np.ascontiguousarray(bi),
                                     self.method, {2: 6, 3: 8, 4: 12}[k])
        else:
            pr, pi = orc.cgemm(ar, ai, br, bi, self.method)
        cr = _view(C.re, C.off, (k, m, l), C.ld, C.ps)
        ci = _view(C.im, C.off, (k, m, l), C.ld, C.ps)
        cr[...] = orc.mat_sub(np.ascontiguousarray(cr), pr)
        ci[...] = orc.mat_sub(np.ascontiguousarray(ci), pi)

    def pack_panel(self, loc_re, loc_im, lay, b, buf_re, buf_im):
        jb, kw, lc = b * lay.K, lay.width(b), lay.lcol[b]
        buf_re.copy_(loc_re[:, jb:, lc:lc + kw])
        buf_im.copy_(loc_im[:, jb:, lc:lc + kw])
