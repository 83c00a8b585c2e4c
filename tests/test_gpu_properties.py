"""Size-independent properties at BASELINE sizes (no oracle needed):
valid pivots, run-to-run determinism, forward error of the solve against
x_true = 1+1i, and the normwise backward error (probe in quad-double)
within BASELINE's 10 n u bound (u = 2^-104 for DD)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import problems  # noqa: E402
from paper_2403_16013_b200.digest import digest  # noqa: E402
from paper_2403_16013_b200.expansion import U_PREC  # noqa: E402


def pc(re, im):
    return mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))


@pytest.mark.parametrize("n,K,ill", [(4096, 256, False), (4096, 256, True)])
def test_large_lu_properties(n, K, ill):
    re, im = problems.lu_matrix(n, 2, 1, ill_conditioned=ill)
    A = pc(re, im)
    f1 = mp.lu_blocked(A, K)
    f2 = mp.lu_blocked(A, K)
    # determinism, bit for bit
    assert np.array_equal(f1.pivots, f2.pivots)
    assert digest(f1.packed.re_plane.data, f1.packed.im_plane.data) == \
        digest(f2.packed.re_plane.data, f2.packed.im_plane.data)
    # pivots: row swapped into i is >= i (test_lu.py:246-249)
    assert np.all(f1.pivots >= np.arange(n)) and np.all(f1.pivots < n)
    # backward error within 10 n u (BASELINE north_star)
    be = mp.lu.backward_error_probe(f1, A)
    assert be <= 10 * n * U_PREC[2], be
    # forward error against x_true (b = cgemm_4m(A, x_true))
    xr, xi = problems.x_true(n, 2)
    X = pc(xr.reshape(2, n, 1).copy(), xi.reshape(2, n, 1).copy())
    B = mp.cgemm_4m(A, X, mp.KernelChoice(method="4m", real_kernel="naive"))
    x = mp.solve(f1, mp.ComplexVector(B.re_plane.data[:, :, 0], B.im_plane.data[:, :, 0]))
    fwd = mp.max_rel_err(x, mp.ComplexVector(xr, xi))
    assert fwd < (1e-10 if ill else 1e-24), fwd


def test_reconstruction_small():
    """reconstruction_error (lu.py:236-250) at k + 2 = 4 on the GPU, against
    the reference's 64 eps max|A| bound (test_lu.py:59-68)."""
    re, im = problems.lu_matrix(96, 2, 3)
    A = pc(re, im)
    f = mp.lu_blocked(A, 32)
    err = mp.lu.reconstruction_error(f, A)
    assert err <= 64 * mp.eps_for(2) * A.max_abs()


@pytest.mark.parametrize("k,n,K", [(2, 4096, 256), (3, 1024, 128)])
def test_ozaki_lu_accuracy(k, n, K):
    """real_kernel="ozaki" (the INT8 tensor-core path, d = 6 / 8): the
    factorization meets the same 10 n u backward-error bound as the EFT
    kernel (the reference's claim that d = 6 / 8 saturate DD / TD accuracy,
    ozaki.py:11-17), pivots valid, solve accurate."""
    re, im = problems.lu_matrix(n, k, 2, populate_lower=k > 2,
                                renorm=mp.renorm_planes if k > 2 else None)
    A = pc(re, im)
    f = mp.lu_blocked(A, K, kc=mp.KernelChoice(method="3m", real_kernel="ozaki"))
    assert np.all(f.pivots >= np.arange(n)) and np.all(f.pivots < n)
    be = mp.lu.backward_error_probe(f, A)
    assert be <= 10 * n * U_PREC[k], be
