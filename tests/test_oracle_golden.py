"""Pin the CPU oracle to golden vectors produced by the UNMODIFIED reference
(oracle/gen_golden.py -> tests/golden/small.npz).  Every comparison is
bitwise (np.array_equal on the float64 limbs, signed zeros included via
the byte view)."""

import json
import os

import numpy as np
import pytest

from testpaths import GOLD


def beq(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def test_eft_known_answers(small, orc):
    a, b = small["eft_a"], small["eft_b"]
    ts = np.array([orc.two_sum(x, y) for x, y in zip(a, b)])
    tp = np.array([orc.two_prod(x, y) for x, y in zip(a, b)])
    assert beq(ts, small["two_sum"])
    assert beq(tp, small["two_prod"])
    # test_eft.py:16-44 style hand cases
    assert orc.two_sum(2.0 ** 53, 1.0) == (2.0 ** 53, 1.0)
    p, e = orc.two_prod(1 + 2 ** -27, 1 + 2 ** -27)
    assert p == 1 + 2 ** -26 and e == 2.0 ** -54


@pytest.mark.parametrize("k", [2, 3, 4])
def test_renorm(small, orc, k):
    raws, lens, outs = small[f"renorm_raw_k{k}"], small[f"renorm_len_k{k}"], small[f"renorm_out_k{k}"]
    got = np.array([orc.renorm(r[:m], k) for r, m in zip(raws, lens)])
    assert beq(got, outs)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_expansion_ops(small, orc, k):
    xs, ys = small[f"x_k{k}"], small[f"y_k{k}"]
    assert beq([orc.exp_add(x, y) for x, y in zip(xs, ys)], small[f"add_k{k}"])
    assert beq([orc.exp_sub(x, y) for x, y in zip(xs, ys)], small[f"sub_k{k}"])
    assert beq([orc.exp_mul(x, y) for x, y in zip(xs, ys)], small[f"mul_k{k}"])
    dv = small[f"divisor_k{k}"]
    assert beq([orc.exp_div(x, y) for x, y in zip(xs, dv)], small[f"div_k{k}"])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_complex_scalars(small, orc, k):
    xs, ys = small[f"x_k{k}"], small[f"y_k{k}"]
    N = xs.shape[0]
    c3, c4, cd = [], [], []
    for i in range(N):
        a = (xs[i], ys[i])
        b = (ys[N - 1 - i], xs[N - 1 - i])
        c3.append(orc.cmul_3m(*a, *b))
        c4.append(orc.cmul_4m(*a, *b))
        cd.append(orc.cdiv(*a, *b))
    assert beq(np.array(c3).transpose(1, 0, 2), small[f"cmul3_k{k}"])
    assert beq(np.array(c4).transpose(1, 0, 2), small[f"cmul4_k{k}"])
    assert beq(np.array(cd).transpose(1, 0, 2), small[f"cdiv_k{k}"])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_matrix_kernels(small, orc, k):
    A, B = small[f"madd_A_k{k}"], small[f"madd_B_k{k}"]
    assert beq(orc.mat_add(A, B), small[f"madd_k{k}"])
    assert beq(orc.mat_sub(A, B), small[f"msub_k{k}"])
    R = small[f"rnp_in_k{k}"].copy()
    assert beq(orc.renorm_planes(R), small[f"rnp_out_k{k}"])
    for shp in ("7x5x6", "16x16x16", "33x17x20"):
        tag = f"k{k}_{shp}"
        assert beq(orc.rgemm(small[f"rg_A_{tag}"], small[f"rg_B_{tag}"]), small[f"rg_C_{tag}"])
        args = [small[f"cg_{p}_{tag}"] for p in ("Ar", "Ai", "Br", "Bi")]
        for meth in ("3m", "4m"):
            cr, ci = orc.cgemm(*args, method=meth)
            assert beq(np.array([cr, ci]), small[f"cg_{meth}_{tag}"]), (meth, tag)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_lu_trsm_solve(small, orc, k):
    for n in (24, 37):
        tag = f"k{k}_n{n}"
        re, im = small[f"lu_re_{tag}"], small[f"lu_im_{tag}"]
        for meth in ("3m", "4m"):
            for Kp in (n, 8, 5):
                key = f"lu_{meth}_K{Kp if Kp != n else 'n'}_{tag}"
                fr, fi, piv, st = orc.factor(re, im, Kp, meth)
                assert st == -1
                assert np.array_equal(piv, small[key + "_piv"]), key
                assert beq(np.array([fr, fi]), small[key]), key
                b = small[key + "_b"]
                xr, xi = orc.solve_fb(fr, fi, piv, b[0], b[1], meth)
                assert beq(np.array([xr, xi]), small[key + "_x"]), key
    L, A = small[f"trsm_L_k{k}"], small[f"trsm_A_k{k}"]
    for meth in ("3m", "4m"):
        xr, xi = A[0].copy(), A[1].copy()
        orc.trsm_ll_unit(L[0], L[1], xr, xi, meth == "3m")
        assert beq(np.array([xr, xi]), small[f"trsm_{meth}_k{k}"])


def test_singular(small, orc):
    base = small["sing_dep"]
    re = np.zeros((2, 3, 3))
    re[0] = base
    _, _, _, st = orc.factor(re, np.zeros((2, 3, 3)), 3)
    assert st == int(small["sing_dep_col"]) == 1
    _, _, _, st = orc.factor(np.zeros((2, 4, 4)), np.zeros((2, 4, 4)), 4)
    assert st == 0


def test_hand_2x2(orc):
    # test_lu.py:40-56: |3| > |1| -> pivots [1, 1], U = [[3, 4], [0, 2/3]]
    re = np.zeros((2, 2, 2))
    re[0] = [[1.0, 2.0], [3.0, 4.0]]
    fr, fi, piv, st = orc.factor(re, np.zeros((2, 2, 2)), 2)
    assert st == -1 and list(piv) == [1, 1]
    assert fr[0, 0, 0] == 3.0 and fr[0, 0, 1] == 4.0
    assert abs(fr[0, 1, 1] - 2.0 / 3.0) < 1e-15


def test_cfg0_digests(orc):
    """BASELINE config 0 (n=128 DD, lo = 0, seeds 1-3) against the reference's
    factor digests and pivots."""
    path = os.path.join(GOLD, "cfg0.json")
    if not os.path.exists(path):
        pytest.skip("cfg0 golden not generated")
    from paper_2403_16013_b200 import problems
    from paper_2403_16013_b200.digest import digest

    cases = json.load(open(path))["cases"]
    for c in cases:
        re, im = problems.lu_matrix(c["n"], c["k"], c["seed"])
        fr, fi, piv, st = orc.factor(re, im, c["K"], c["method"])
        assert st == -1
        assert [int(p) for p in piv] == c["pivots"]
        assert digest(fr, fi) == c["digest"], (c["seed"], c["method"], c["K"])


def test_factor_range_stages_equal_whole(orc):
    """oracle.factor_range (used by oracle/gen_cfg4.py --stage to run the
    config-4 factorization in two jobs) continues exactly where the previous
    stage stopped: two stages == one call, bit for bit."""
    import numpy as np

    from paper_2403_16013_b200 import problems

    re, im = problems.lu_matrix(96, 2, 11)
    fr, fi, piv, st = orc.factor(re, im, 16, "3m")
    r2, i2 = re.copy(), im.copy()
    p2 = np.arange(96, dtype=np.int64)
    assert orc.factor_range(r2, i2, p2, 16, "3m", 0, 48) == -1
    assert orc.factor_range(r2, i2, p2, 16, "3m", 48, 96) == -1
    assert st == -1 and np.array_equal(piv, p2)
    assert fr.tobytes() == r2.tobytes() and fi.tobytes() == i2.tobytes()
