"""Ozaki-scheme restatement for parity tests (TEST INFRASTRUCTURE ONLY).

numpy restatement of ozaki.py:33-159 on top of the C oracle's renorm_planes
and acc_plane (_kernels.py:485-517); np.matmul is an exact binary64 GEMM for
the split parts (the reference's default f64_gemm)."""

import numpy as np

from . import oracle as orc

DEFAULT_SPLIT_BITS = {2: 19, 3: 21, 4: 18}


def split_exactness_bound(inner_n):
    return int(53 - np.ceil(np.log2(inner_n)) if inner_n > 1 else 53) // 2


def resolve_width(k, inner_n, split_bits=None):
    bound = split_exactness_bound(inner_n)
    if split_bits is None:
        return min(DEFAULT_SPLIT_BITS.get(k, bound), bound)
    return int(split_bits)


def split(data, d, side, split_bits=None):
    """ozaki.py:79-108 -> (parts list, scales list, width)"""
    k, rows, cols = data.shape
    inner = cols if side == "left" else rows
    width = resolve_width(k, inner, split_bits)
    resid = np.ascontiguousarray(data.copy())
    axis = 1 if side == "left" else 0
    shift = 2.0 ** (53 - width)
    parts, scales = [], []
    for _ in range(d):
        mu = np.abs(resid[0]).max(axis=axis)
        _, ex = np.frexp(mu)
        w = np.ldexp(1.0, ex)
        sigma = w * shift
        S = sigma[:, None] if side == "left" else sigma[None, :]
        part = (resid[0] + S) - S
        resid[0] -= part
        orc.renorm_planes(resid)
        parts.append(part)
        scales.append(np.ldexp(w, -width))
    return parts, scales, width


def pair_schedule(d, width, k):
    cutoff = 53 * k + 53
    pairs = []
    for s in range(d):
        if s * max(width - 1, 1) >= cutoff:
            break
        for p in range(s + 1):
            pairs.append((p, s - p))
    return pairs


def rgemm(A, B, d, split_bits=None):
    """rgemm_ozaki, ozaki.py:124-159"""
    k = A.shape[0]
    pa, _, width = split(A, d, "left", split_bits)
    pb, _, _ = split(B, d, "right", split_bits)
    C = np.zeros((k, A.shape[1], B.shape[2]))
    for p, q in pair_schedule(d, width, k):
        orc.acc_plane(C, pa[p] @ pb[q])
    return orc.renorm_planes(C)


def cgemm(Ar, Ai, Br, Bi, method, d, split_bits=None):
    """cgemm_3m / cgemm_4m over the Ozaki real kernel (cmatrix.py:145-169)"""
    if method == "3m":
        t1 = rgemm(Ar, Br, d, split_bits)
        t2 = rgemm(Ai, Bi, d, split_bits)
        t3 = rgemm(orc.mat_add(Ar, Ai), orc.mat_add(Br, Bi), d, split_bits)
        return orc.mat_sub(t1, t2), orc.mat_sub(orc.mat_sub(t3, t1), t2)
    rr = rgemm(Ar, Br, d, split_bits)
    ii = rgemm(Ai, Bi, d, split_bits)
    ir = rgemm(Ai, Br, d, split_bits)
    ri = rgemm(Ar, Bi, d, split_bits)
    return orc.mat_sub(rr, ii), orc.mat_add(ir, ri)
