"""GPU solve (row a15 / f2): solve_fb (_kernels.py:708-775) through the C-ABI
(mpc_getrs / mpc_getrs_phases) against the CPU oracle.

* the interchanges + forward (unit-lower) sweep are BITWISE equal to the
  oracle's (the blocked kernel keeps every row's j-ascending chain);
* the backward sweep applies the diagonal blocks right-looking, so it is
  tolerance-parity: the relative difference to the oracle's x is bounded by
  TOL_BWD * n * u_prec (u_prec = 2^-104 / 2^-156 / 2^-208, BASELINE.json)
  on well-conditioned LU factors.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import problems  # noqa: E402
from paper_2403_16013_b200.expansion import U_PREC  # noqa: E402

# |x_gpu - x_oracle| / |x_oracle| <= TOL_BWD * n * u_prec (stated tolerance)
TOL_BWD = 10.0


@pytest.fixture(scope="module", autouse=True)
def _device():
    mp._lib.require_device()


def beq(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def gpu_phase(fr, fi, piv, br, bi, meth, phases):
    lib = mp._lib.lib()
    k, n, _ = fr.shape
    xr, xi = np.ascontiguousarray(br).copy(), np.ascontiguousarray(bi).copy()
    mp._lib.check(lib.mpc_getrs_phases(k, 3 if meth == "3m" else 4, n, fr.ctypes.data,
                                       fi.ctypes.data, piv.ctypes.data, xr.ctypes.data,
                                       xi.ctypes.data, phases, None), "getrs_phases")
    return xr, xi


def rel_err(xr, xi, yr, yi):
    """max_i |x_i - y_i| / max_i |y_i| in binary64 from limb-wise differences."""
    dr = (xr - yr).sum(axis=0)
    di = (xi - yi).sum(axis=0)
    den = np.max(np.hypot(yr.sum(axis=0), yi.sum(axis=0)))
    return float(np.max(np.hypot(dr, di)) / den) if den else 0.0


def factors(orc, n, k, seed):
    re, im = problems.lu_matrix(n, k, seed, populate_lower=k > 2, renorm=orc.renorm_planes)
    fr, fi, piv, st = orc.factor(re, im, min(n, 32), "3m")
    assert st == -1
    return fr, fi, piv


def rhs(rng, n, k):
    br = np.zeros((k, n))
    bi = np.zeros((k, n))
    br[0] = rng.uniform(-1, 1, n)
    bi[0] = rng.uniform(-1, 1, n)
    if k > 1:
        br[1] = br[0] * 2.0 ** -53 * rng.uniform(-1, 1, n)
        bi[1] = bi[0] * 2.0 ** -53 * rng.uniform(-1, 1, n)
    return br, bi


@pytest.mark.parametrize("k,sizes", [
    (2, [1, 2, 5, 31, 32, 33, 64, 65, 100, 300]),
    (3, [1, 17, 32, 70]),
    (4, [1, 33, 70]),
])
def test_forward_sweep_bitwise(orc, k, sizes):
    """Interchanges + forward sweep == oracle bit for bit, ragged sizes
    around the 32-row diagonal block, 3M and 4M."""
    for n in sizes:
        rng = np.random.default_rng(100 * k + n)
        fr, fi, piv = factors(orc, n, k, n + 3)
        br, bi = rhs(rng, n, k)
        for meth in ("3m", "4m"):
            xr, xi = gpu_phase(fr, fi, piv, br, bi, meth, 1)
            yr, yi = orc.solve_fb(fr, fi, piv, br, bi, meth, phases=1)
            assert beq(xr, yr) and beq(xi, yi), (k, n, meth)


def test_forward_sweep_arbitrary_pivots(orc):
    """Pivot vectors with long swap chains (p_i >= i random) and a matrix
    that is not an LU output: the forward sweep reads only the strictly
    lower part, bitwise."""
    k, n = 2, 257
    rng = np.random.default_rng(5)
    fr = np.zeros((k, n, n))
    fi = np.zeros((k, n, n))
    fr[0] = rng.uniform(-1, 1, (n, n)) / 16  # tame growth of the random unit-lower solve
    fi[0] = rng.uniform(-1, 1, (n, n)) / 16
    piv = np.array([rng.integers(i, n) for i in range(n)], dtype=np.int64)
    br, bi = rhs(rng, n, k)
    for meth in ("3m", "4m"):
        xr, xi = gpu_phase(fr, fi, piv, br, bi, meth, 1)
        yr, yi = orc.solve_fb(fr, fi, piv, br, bi, meth, phases=1)
        assert beq(xr, yr) and beq(xi, yi), meth


@pytest.mark.parametrize("k,sizes", [(2, [1, 5, 32, 33, 100, 300]), (3, [17, 70]), (4, [33, 70])])
def test_backward_sweep_tolerance(orc, k, sizes):
    for n in sizes:
        rng = np.random.default_rng(7 * k + n)
        fr, fi, piv = factors(orc, n, k, n + 11)
        br, bi = rhs(rng, n, k)
        for meth in ("3m", "4m"):
            xr, xi = gpu_phase(fr, fi, piv, br, bi, meth, 2)
            yr, yi = orc.solve_fb(fr, fi, piv, br, bi, meth, phases=2)
            err = rel_err(xr, xi, yr, yi)
            assert err <= TOL_BWD * n * U_PREC[k], (k, n, meth, err)
            # the full solve = forward (bitwise) then backward
            xr, xi = gpu_phase(fr, fi, piv, br, bi, meth, 3)
            yr, yi = orc.solve_fb(fr, fi, piv, br, bi, meth)
            err = rel_err(xr, xi, yr, yi)
            assert err <= TOL_BWD * n * U_PREC[k], (k, n, meth, err)


def test_solve_api_and_device_path(orc):
    """lu.solve (host numpy, staged) and device.getrs (CUDA tensors) agree
    bit for bit with each other."""
    import torch

    from paper_2403_16013_b200 import device

    k, n = 2, 200
    rng = np.random.default_rng(9)
    fr, fi, piv = factors(orc, n, k, 21)
    br, bi = rhs(rng, n, k)
    f = mp.LUFactors(packed=mp.PlanarComplexMatrix(mp.RealMatrix(fr), mp.RealMatrix(fi)),
                     pivots=piv, method="3m")
    x = mp.solve(f, mp.ComplexVector(br, bi))
    dev = torch.device("cuda", 0)
    tb = [torch.from_numpy(a.copy()).to(dev) for a in (fr, fi, br, bi)]
    tp = torch.from_numpy(piv).to(dev)
    device.getrs(tb[0], tb[1], tp, tb[2], tb[3], "3m")
    torch.cuda.synchronize()
    assert beq(tb[2].cpu().numpy(), x.re) and beq(tb[3].cpu().numpy(), x.im)
    # forward then backward as two calls == one call
    device.getrs(tb[0], tb[1], tp, b2r := torch.from_numpy(br.copy()).to(dev),
                 b2i := torch.from_numpy(bi.copy()).to(dev), "3m", phases=1)
    device.getrs(tb[0], tb[1], tp, b2r, b2i, "3m", phases=2)
    torch.cuda.synchronize()
    assert beq(b2r.cpu().numpy(), x.re) and beq(b2i.cpu().numpy(), x.im)


def test_solve_phases_rejected():
    lib = mp._lib.lib()
    z = np.zeros(4)
    p = np.zeros(1, dtype=np.int64)
    for bad in (0, 4):
        assert lib.mpc_getrs_phases(2, 3, 1, z.ctypes.data, z.ctypes.data, p.ctypes.data,
                                    z.ctypes.data, z.ctypes.data, bad, None) == mp._lib.MPC_ERR
