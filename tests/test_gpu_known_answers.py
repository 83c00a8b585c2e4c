"""Known-answer cases of the reference's own unit tests,
restated for the device path: exact integer and exact-rational GEMMs, hand
LU / TRSM / solve cases, singular detection columns, pivot invariants,
thread invariance and K = n equivalence.  Values are elementary facts
(e.g. [[1,2],[3,4]] [[5,6],[7,8]] = [[19,22],[43,50]]), checked exactly."""

from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import paper_2403_16013_b200 as m

    m._lib.require_device()
    return m


def frac(x):
    """exact value of a k-limb expansion given as a sequence of doubles"""
    return sum((Fraction(float(c)) for c in x), Fraction(0))


@pytest.mark.parametrize("kern", ["naive", "blocked"])
def test_exact_integer_gemm(mp, kern):
    A = mp.RealMatrix.from_float64(np.array([[1.0, 2.0], [3.0, 4.0]]), 2)
    B = mp.RealMatrix.from_float64(np.array([[5.0, 6.0], [7.0, 8.0]]), 2)
    C = mp.rgemm_naive(A, B) if kern == "naive" else mp.rgemm_blocked(A, B)
    assert np.array_equal(C.data[0], [[19.0, 22.0], [43.0, 50.0]])
    assert not C.data[1].any()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_gemm_vs_exact_rational(mp, k):
    """8x8 products against Fraction arithmetic: |C - AB| <= 8 * 4 eps |A||B|."""
    rng = np.random.default_rng(7 + k)
    A = mp.random_matrix(8, 8, k, rng)
    B = mp.random_matrix(8, 8, k, rng)
    C = mp.rgemm_blocked(A, B)
    eps = Fraction(mp.eps_for(k))
    for i in range(8):
        for j in range(8):
            exact = sum(frac(A.data[:, i, t]) * frac(B.data[:, t, j]) for t in range(8))
            bound = 8 * 4 * eps * sum(abs(frac(A.data[:, i, t]) * frac(B.data[:, t, j]))
                                      for t in range(8))
            assert abs(frac(C.data[:, i, j]) - exact) <= bound


def test_identity_lu(mp):
    I = mp.PlanarComplexMatrix.identity(5, 2)
    f = mp.lu_normal(I)
    assert f.packed.bitwise_equal(I)
    assert np.array_equal(f.pivots, np.arange(5))


def test_hand_2x2_lu(mp):
    A = mp.PlanarComplexMatrix(mp.RealMatrix.from_float64(np.array([[1.0, 2.0], [3.0, 4.0]]), 2),
                               mp.RealMatrix.zeros(2, 2, 2))
    f = mp.lu_normal(A)
    assert list(f.pivots) == [1, 1]           # |3| > |1|: the rows swap
    u = f.packed.re_plane.data
    eps = Fraction(mp.eps_for(2))
    assert frac(u[:, 0, 0]) == 3 and frac(u[:, 0, 1]) == 4
    assert abs(frac(u[:, 1, 0]) - Fraction(1, 3)) <= 2 * eps
    assert abs(frac(u[:, 1, 1]) - Fraction(2, 3)) <= 4 * eps
    assert not f.packed.im_plane.data.any()


def test_trsm_identity_and_hand(mp):
    rng = np.random.default_rng(3)
    L = mp.PlanarComplexMatrix.identity(6, 2)
    X0 = mp.PlanarComplexMatrix(mp.random_matrix(6, 6, 2, rng), mp.random_matrix(6, 6, 2, rng))
    assert mp.trsm_unit_lower(L, X0).bitwise_equal(X0)
    L2 = mp.PlanarComplexMatrix.identity(2, 2)
    L2.re_plane.data[0, 1, 0] = 2.0
    b = mp.PlanarComplexMatrix(mp.RealMatrix.from_float64(np.array([[1.0], [0.0]]), 2),
                               mp.RealMatrix.zeros(2, 1, 2))
    X = mp.trsm_unit_lower(L2, b)
    assert X.re_plane.data[0, 0, 0] == 1.0 and X.re_plane.data[0, 1, 0] == -2.0
    assert not X.im_plane.data.any()


def test_solve_identity_and_hand(mp):
    rng = np.random.default_rng(5)
    I = mp.PlanarComplexMatrix.identity(7, 2)
    f = mp.lu_normal(I)
    b = mp.ComplexVector(np.zeros((2, 7)), np.zeros((2, 7)))
    b.re[0] = rng.random(7)
    b.im[0] = rng.random(7)
    assert mp.solve(f, b).bitwise_equal(b)
    A = mp.PlanarComplexMatrix.from_complex128(np.array([[1.0, 1.0], [0.0, 1.0]]), 2)
    bb = mp.ComplexVector(np.zeros((2, 2)), np.zeros((2, 2)))
    bb.re[0] = [4.0, 3.0]
    bb.im[0] = [6.0, 4.0]
    x = mp.solve(mp.lu_normal(A), bb)
    assert list(x.re[0]) == [1.0, 3.0] and list(x.im[0]) == [2.0, 4.0]
    assert not x.re[1].any() and not x.im[1].any()


def test_singular_columns(mp):
    with pytest.raises(mp.SingularMatrixError, match="column 0"):
        mp.lu_normal(mp.PlanarComplexMatrix.zeros(4, 4, 2))
    base = np.array([[1.0, 2.0, 1.0], [2.0, 4.0, 0.0], [3.0, 6.0, 2.0]])
    A = mp.PlanarComplexMatrix(mp.RealMatrix.from_float64(base, 2), mp.RealMatrix.zeros(3, 3, 2))
    with pytest.raises(mp.SingularMatrixError, match="column 1"):
        mp.lu_normal(A)


@pytest.mark.parametrize("k", [2, 3])
def test_pivot_invariants_threads_and_K(mp, k):
    rng = np.random.default_rng(11 + k)
    n = 48
    A = mp.PlanarComplexMatrix(mp.random_matrix(n, n, k, rng), mp.random_matrix(n, n, k, rng))
    f1 = mp.lu_blocked(A, 16, threads=1)
    f8 = mp.lu_blocked(A, 16, threads=8)
    assert np.array_equal(f1.pivots, f8.pivots) and f1.packed.bitwise_equal(f8.packed)
    assert np.all(f1.pivots >= np.arange(n))
    f4 = mp.lu_blocked(A, 16, kc=mp.KernelChoice(method="4m"))
    assert np.array_equal(f1.pivots, f4.pivots)           # 3M / 4M: same pivots
    fn = mp.lu_normal(A)
    fK = mp.lu_blocked(A, n)
    assert np.array_equal(fn.pivots, fK.pivots) and fn.packed.bitwise_equal(fK.packed)


@pytest.mark.parametrize("kk", [5, 6, 8])
def test_verification_kernels_vs_exact(mp, kk):
    """The k = 5, 6, 8 verification kernels: 4M complex product
    against Fraction arithmetic, 3M.re == 4M.re bitwise; no LU there."""
    rng = np.random.default_rng(kk)
    A = mp.PlanarComplexMatrix(mp.random_matrix(6, 5, 3, rng).promote(kk),
                               mp.random_matrix(6, 5, 3, rng).promote(kk))
    B = mp.PlanarComplexMatrix(mp.random_matrix(5, 4, 3, rng).promote(kk),
                               mp.random_matrix(5, 4, 3, rng).promote(kk))
    C = mp.cgemm(A, B, mp.KernelChoice(method="4m"))
    eps = Fraction(2.0 ** (1 - 53 * kk))
    ar, ai, br, bi = A.re_plane.data, A.im_plane.data, B.re_plane.data, B.im_plane.data
    for i in range(6):
        for j in range(4):
            re = sum(frac(ar[:, i, t]) * frac(br[:, t, j]) - frac(ai[:, i, t]) * frac(bi[:, t, j])
                     for t in range(5))
            mag = sum(abs(frac(ar[:, i, t]) * frac(br[:, t, j])) + abs(frac(ai[:, i, t]) * frac(bi[:, t, j]))
                      for t in range(5))
            assert abs(frac(C.re_plane.data[:, i, j]) - re) <= 64 * eps * mag
    C3 = mp.cgemm(A, B, mp.KernelChoice(method="3m"))
    assert C3.re_plane.data.tobytes() == C.re_plane.data.tobytes()
    with pytest.raises(ValueError):
        mp.lu_blocked(A, 2)


@pytest.mark.parametrize("k", [3, 4])
def test_td_qd_backward_error(mp, k):
    """BASELINE's TD / QD accuracy criterion: normwise backward error of the
    factors <= 10 n u (u = 2^-156 / 2^-208), probed at k + 2 components, and
    the componentwise reconstruction bound 64 eps max|A| (bench.py:259-262)."""
    from paper_2403_16013_b200 import lu as lum, problems

    n = 96
    re, im = problems.lu_matrix(n, k, 3, populate_lower=True, renorm=mp.renorm_planes)
    A = mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))
    f = mp.lu_blocked(A, 32)
    u = 2.0 ** {3: -156, 4: -208}[k]
    be = lum.backward_error_probe(f, A)
    assert 0 < be <= 10 * n * u, be
    rec = lum.reconstruction_error(f, A)
    assert rec <= 64 * mp.eps_for(k) * A.max_abs(), rec


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3])
def test_device_accuracy_report(mp, k):
    """device.accuracy (bench.py's accuracy object) against the host API:
    same forward error as lu.max_rel_err(solve(f, A (1+1i))), backward-error
    probe within 10 n u, for DD and TD."""
    import torch

    from paper_2403_16013_b200 import device, problems

    n, K = 80, 16
    re, im = problems.lu_matrix(n, k, 5, populate_lower=k > 2,
                                renorm=mp.renorm_planes if k > 2 else None)
    A = mp.PlanarComplexMatrix(mp.RealMatrix(re.copy()), mp.RealMatrix(im.copy()))
    f = mp.lu_blocked(A, K)
    xt = mp.ComplexVector(np.zeros((k, n)), np.zeros((k, n)))
    xt.re[0] = 1.0
    xt.im[0] = 1.0
    X = mp.PlanarComplexMatrix(mp.RealMatrix(xt.re.reshape(k, n, 1).copy()),
                               mp.RealMatrix(xt.im.reshape(k, n, 1).copy()))
    B = mp.cgemm(A, X, mp.KernelChoice(method="4m"))
    b = mp.ComplexVector(B.re_plane.data.reshape(k, n), B.im_plane.data.reshape(k, n))
    fwd_host = mp.max_rel_err(mp.solve(f, b), xt)

    dev = torch.device("cuda", 0)
    Ar, Ai = torch.from_numpy(re).to(dev), torch.from_numpy(im).to(dev)
    Wr, Wi = Ar.clone(), Ai.clone()
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    assert device.getrf(Wr, Wi, piv, K) == -1
    assert np.array_equal(piv.cpu().numpy(), f.pivots)
    acc = device.accuracy(Ar, Ai, Wr, Wi, piv)
    assert acc["fwd_err"] == pytest.approx(float(fwd_host), rel=1e-9, abs=0.0)
    assert 0 < acc["bwd_err_probe"] <= acc["bwd_bound_10nu"] and acc["bwd_ok"]


@pytest.mark.gpu
@pytest.mark.parametrize("k,n,K", [(2, 300, 64), (3, 130, 32), (2, 64, 64), (2, 520, 32),
                                   (2, 1000, 48)])
def test_factor_inplace_pinned_overlap(mp, k, n, K):
    """Host factors in pinned memory: the C-ABI streams finished row blocks
    back while the LU runs (RowSink); the result must equal the pageable
    (staged) path and the device path bit for bit, pivots included."""
    import torch

    from paper_2403_16013_b200 import lu as lum, problems

    re, im = problems.lu_matrix(n, k, 7, populate_lower=k > 2,
                                renorm=mp.renorm_planes if k > 2 else None)
    pr = torch.empty(re.shape, dtype=torch.float64, pin_memory=True)
    pi = torch.empty(im.shape, dtype=torch.float64, pin_memory=True)
    pr.numpy()[...] = re
    pi.numpy()[...] = im
    pp = lum.factor_inplace(pr.numpy(), pi.numpy(), K)
    gr, gi = re.copy(), im.copy()
    gp = lum.factor_inplace(gr, gi, K)
    dev = torch.device("cuda", 0)
    dr, di = torch.from_numpy(re).to(dev), torch.from_numpy(im).to(dev)
    dp = lum.factor_inplace(dr, di, K)  # piv allocated on the planes' device
    assert isinstance(dp, torch.Tensor) and dp.device == dev
    torch.cuda.synchronize()
    assert np.array_equal(pp, gp) and np.array_equal(pp, dp.cpu().numpy())
    assert pr.numpy().tobytes() == gr.tobytes() == dr.cpu().numpy().tobytes()
    assert pi.numpy().tobytes() == gi.tobytes() == di.cpu().numpy().tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("n,K", [(300, 64), (96, 96), (520, 32)])
def test_factor_inplace_pinned_overlap_ozaki(mp, n, K):
    """The Ozaki LU on pinned host factors (overlapped copies, chunked step-0
    update) equals its device path bit for bit."""
    import torch

    from paper_2403_16013_b200 import lu as lum, problems

    re, im = problems.lu_matrix(n, 2, 11)
    pr = torch.empty(re.shape, dtype=torch.float64, pin_memory=True)
    pi = torch.empty(im.shape, dtype=torch.float64, pin_memory=True)
    pr.numpy()[...] = re
    pi.numpy()[...] = im
    pp = lum.factor_inplace(pr.numpy(), pi.numpy(), K, real_kernel="ozaki")
    dev = torch.device("cuda", 0)
    dr, di = torch.from_numpy(re).to(dev), torch.from_numpy(im).to(dev)
    dp = torch.empty(n, dtype=torch.int64, device=dev)
    lum.factor_inplace(dr, di, K, piv=dp, real_kernel="ozaki")
    torch.cuda.synchronize()
    assert np.array_equal(pp, dp.cpu().numpy())
    assert pr.numpy().tobytes() == dr.cpu().numpy().tobytes()
    assert pi.numpy().tobytes() == di.cpu().numpy().tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("k,rows,ncols,r0,r1", [(2, 300, 200, 5, 150), (3, 97, 33, 0, 97),
                                                (2, 1200, 129, 64, 576), (4, 40, 5, 3, 4)])
def test_laswp_chunked_permutation_vs_sequential(mp, k, rows, ncols, r0, r1):
    """mpc_laswp (chunks of 32 interchanges composed into one permutation per
    chunk) against the sequential definition (_swap_rows in order,
    _kernels.py:597-608): random pivots p >= r with many repeats -- the same
    pivot row hit by several interchanges of one chunk and of different
    chunks, pivots inside the chunk, identity interchanges."""
    from paper_2403_16013_b200 import _lib

    rng = np.random.default_rng(rows * 7 + ncols)
    re = rng.standard_normal((k, rows, ncols))
    im = rng.standard_normal((k, rows, ncols))
    piv = np.arange(rows, dtype=np.int64)
    hot = rng.integers(r1, rows, size=4) if r1 < rows else np.array([rows - 1])
    for r in range(r0, r1):
        u = rng.random()
        if u < 0.15:
            piv[r] = r                                   # identity
        elif u < 0.45:
            piv[r] = rng.integers(r, min(r + 20, rows))  # nearby (often inside the chunk)
        elif u < 0.75:
            piv[r] = max(r, int(rng.choice(hot)))        # a few rows hit again and again
        else:
            piv[r] = rng.integers(r, rows)
    er, ei = re.copy(), im.copy()
    for r in range(r0, r1):
        p = piv[r]
        if p != r:
            er[:, [r, p], :] = er[:, [p, r], :]
            ei[:, [r, p], :] = ei[:, [p, r], :]
    gr, gi = re.copy(), im.copy()
    _lib.check(_lib.lib().mpc_laswp(k, ncols, _lib.ptr(gr), _lib.ptr(gi), ncols, rows * ncols,
                                    _lib.ptr(piv), r0, r1, None), "laswp")
    assert gr.tobytes() == er.tobytes() and gi.tobytes() == ei.tobytes()
