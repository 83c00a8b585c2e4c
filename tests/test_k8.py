"""The reference's k = 8 paths (REFERENCE_K: reference_rhs bench.py:199-213,
_matmul_check bench.py:336-348) and the 3M reconstruction check at k + 2
(lu.py:236-250), against golden vectors made by the unmodified reference
(oracle/gen_golden_k8.py -> tests/golden/k8.npz).  CPU: the oracle
restatement reproduces them; GPU: the verification kernels do, bit for bit."""

import os

import numpy as np
import pytest

from testpaths import GOLD

CASES = [("dd", 12), ("dd", 7), ("td", 10), ("qd", 9)]
K_OF = {"dd": 2, "td": 3, "qd": 4}


@pytest.fixture(scope="module")
def g8():
    return dict(np.load(os.path.join(GOLD, "k8.npz"), allow_pickle=False))


def beq(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def _promote(x, kk):
    out = np.zeros((kk,) + x.shape[1:])
    out[: x.shape[0]] = x
    return out


def _oracle_rhs(orc, are, aim, xre, xim):
    k, n = xre.shape
    A8re, A8im = _promote(are, 8), _promote(aim, 8)
    X8re, X8im = _promote(xre.reshape(k, n, 1), 8), _promote(xim.reshape(k, n, 1), 8)
    Bre, Bim = orc.cgemm(A8re, A8im, X8re, X8im, method="4m")
    bre = np.ascontiguousarray(Bre[:k]).copy()
    bim = np.ascontiguousarray(Bim[:k]).copy()
    orc.renorm_planes(bre)
    orc.renorm_planes(bim)
    return bre.reshape(k, n), bim.reshape(k, n)


@pytest.mark.parametrize("p,n", CASES)
def test_oracle_reference_rhs(g8, orc, p, n):
    key = f"rhs_{p}_n{n}"
    bre, bim = _oracle_rhs(orc, g8[key + "_are"], g8[key + "_aim"], g8[key + "_xre"],
                           g8[key + "_xim"])
    assert beq(bre, g8[key + "_bre"]) and beq(bim, g8[key + "_bim"])


@pytest.mark.parametrize("meth", ["3m", "4m"])
def test_oracle_cgemm_k8(g8, orc, meth):
    cre, cim = orc.cgemm(g8["mm8_are"], g8["mm8_aim"], g8["mm8_bre"], g8["mm8_bim"], method=meth)
    assert beq(cre, g8[f"mm8_{meth}_cre"]) and beq(cim, g8[f"mm8_{meth}_cim"])


# ------------------------------------------------------------------ GPU

@pytest.fixture(scope="module")
def mp():
    import paper_2403_16013_b200 as m

    m._lib.require_device()
    return m


def _pc(mp, re, im):
    return mp.PlanarComplexMatrix(mp.RealMatrix(np.ascontiguousarray(re)),
                                  mp.RealMatrix(np.ascontiguousarray(im)))


@pytest.mark.gpu
@pytest.mark.parametrize("p,n", CASES)
def test_gpu_reference_rhs(g8, mp, p, n):
    from paper_2403_16013_b200 import harness

    key = f"rhs_{p}_n{n}"
    A = _pc(mp, g8[key + "_are"], g8[key + "_aim"])
    x = mp.ComplexVector(g8[key + "_xre"].copy(), g8[key + "_xim"].copy())
    b = harness.reference_rhs(A, x)
    assert beq(b.re, g8[key + "_bre"]) and beq(b.im, g8[key + "_bim"])
    # gen_problem end to end (bench.py:176-190): same A, x and b
    system, xt = harness.gen_problem(n, {"dd": 5 if n == 12 else 2, "td": 3, "qd": 4}[p], p)
    assert beq(system.A.re_plane.data, g8[key + "_are"]) and beq(xt.re, g8[key + "_xre"])
    assert beq(system.b.re, g8[key + "_bre"]) and beq(system.b.im, g8[key + "_bim"])


@pytest.mark.gpu
@pytest.mark.parametrize("meth", ["3m", "4m"])
def test_gpu_cgemm_k8(g8, mp, meth):
    A = _pc(mp, g8["mm8_are"], g8["mm8_aim"])
    B = _pc(mp, g8["mm8_bre"], g8["mm8_bim"])
    C = mp.cgemm(A, B, mp.KernelChoice(method=meth, real_kernel="blocked"))
    assert beq(C.re_plane.data, g8[f"mm8_{meth}_cre"])
    assert beq(C.im_plane.data, g8[f"mm8_{meth}_cim"])


@pytest.mark.gpu
@pytest.mark.parametrize("p", ["dd", "td", "qd"])
def test_gpu_matmul_check_and_reconstruction(g8, mp, p):
    from paper_2403_16013_b200 import harness, lu as lum

    A = _pc(mp, g8[f"mmchk_{p}_are"], g8[f"mmchk_{p}_aim"])
    B = _pc(mp, g8[f"mmchk_{p}_bre"], g8[f"mmchk_{p}_bim"])
    C = mp.cgemm(A, B, mp.KernelChoice(method="3m"))
    assert beq(C.re_plane.data, g8[f"mmchk_{p}_cre"])
    assert harness._matmul_check(A, B, C) == float(g8[f"mmchk_{p}_err"])
    A = _pc(mp, g8[f"rec_{p}_are"], g8[f"rec_{p}_aim"])
    f = mp.lu_blocked(A, 8)
    assert lum.reconstruction_error(f, A) == float(g8[f"rec_{p}_err"])


@pytest.mark.gpu
def test_gpu_matmul_bench_check(mp):
    from paper_2403_16013_b200 import harness

    cfg = harness.BenchConfig(precision="dd", n=24, reps=1, threads=[1])
    rec = harness.run_matmul_bench(cfg, check=True)[0]
    assert rec.status == "ok" and rec.max_relerr != "nan"
    assert 0.0 <= float(rec.max_relerr) < 1e-25  # DD with Re-part cancellation
