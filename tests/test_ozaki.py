"""Ozaki scheme: the oracle restatement pinned to the
reference's golden vectors (CPU) and the B200 path bit-identical to both
(GPU).  Golden: oracle/gen_golden.py ozaki -> tests/golden/ozaki.npz."""

import os

import numpy as np
import pytest

from conftest import GOLD


@pytest.fixture(scope="module")
def oz():
    return dict(np.load(os.path.join(GOLD, "ozaki.npz")))


def beq(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_oracle_ozaki_golden(oz, orc, k):
    from oracle import ozaki_ref as ozr

    A, B = oz[f"oz_A_k{k}"], oz[f"oz_B_k{k}"]
    for d in (1, 3, 6):
        pa, sa, _ = ozr.split(A, d, "left")
        pb, sb, _ = ozr.split(B, d, "right")
        assert beq(pa, oz[f"oz_sa_parts_k{k}_d{d}"]) and beq(sa, oz[f"oz_sa_scales_k{k}_d{d}"])
        assert beq(pb, oz[f"oz_sb_parts_k{k}_d{d}"]) and beq(sb, oz[f"oz_sb_scales_k{k}_d{d}"])
    for d in {2: (5, 6), 3: (7, 8), 4: (11, 12)}[k]:
        assert beq(ozr.rgemm(A, B, d), oz[f"oz_C_k{k}_d{d}"])
    assert beq(ozr.rgemm(A, B, 4, split_bits=12), oz[f"oz_C_k{k}_d4_sb12"])
    args = [oz[f"ozc_{p}_k{k}"] for p in ("Ar", "Ai", "Br", "Bi")]
    for meth in ("3m", "4m"):
        d = {2: 6, 3: 8, 4: 12}[k]
        cr, ci = ozr.cgemm(*args, meth, d)
        assert beq(np.array([cr, ci]), oz[f"ozc_{meth}_k{k}"])


def test_ozaki_api_validation():
    import paper_2403_16013_b200 as mp

    assert mp.split_exactness_bound(1) == 26
    assert mp.split_exactness_bound(256) == 22
    assert mp.split_exactness_bound(1024) == 21
    A = mp.RealMatrix.zeros(4, 4, 2)
    with pytest.raises(ValueError, match="split exactness budget"):
        mp.ozaki_split(A, 2, split_bits=30)
    with pytest.raises(ValueError):
        mp.ozaki_split(A, 0)
    with pytest.raises(ValueError):
        mp.ozaki_split(A, 2, side="up")


# ------------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3, 4])
def test_gpu_ozaki_golden(oz, k):
    import paper_2403_16013_b200 as mp

    A, B = mp.RealMatrix(oz[f"oz_A_k{k}"]), mp.RealMatrix(oz[f"oz_B_k{k}"])
    for d in (1, 3, 6):
        sa = mp.ozaki_split(A, d, "left")
        sb = mp.ozaki_split(B, d, "right")
        assert beq(sa.parts, oz[f"oz_sa_parts_k{k}_d{d}"]) and beq(sa.scales, oz[f"oz_sa_scales_k{k}_d{d}"])
        assert beq(sb.parts, oz[f"oz_sb_parts_k{k}_d{d}"]) and beq(sb.scales, oz[f"oz_sb_scales_k{k}_d{d}"])
    for d in {2: (5, 6), 3: (7, 8), 4: (11, 12)}[k]:
        assert beq(mp.rgemm_ozaki(A, B, d).data, oz[f"oz_C_k{k}_d{d}"]), d
    assert beq(mp.rgemm_ozaki(A, B, 4, split_bits=12).data, oz[f"oz_C_k{k}_d4_sb12"])
    # any binary64 GEMM gives the same bits (test_ozaki.py:161-176)
    plain = lambda X, Y: np.einsum("it,tj->ij", X, Y)  # noqa: E731
    d = {2: 6, 3: 8, 4: 12}[k]
    assert beq(mp.rgemm_ozaki(A, B, d, f64_gemm=plain).data, mp.rgemm_ozaki(A, B, d).data)
    P = [mp.PlanarComplexMatrix(mp.RealMatrix(oz[f"ozc_{a}r_k{k}"]), mp.RealMatrix(oz[f"ozc_{a}i_k{k}"]))
         for a in ("A", "B")]
    for meth in ("3m", "4m"):
        C = mp.cgemm(P[0], P[1], mp.KernelChoice(method=meth, real_kernel="ozaki"))
        assert beq(np.array([C.re_plane.data, C.im_plane.data]), oz[f"ozc_{meth}_k{k}"]), meth
    re, im = oz[f"ozlu_re_k{k}"], oz[f"ozlu_im_k{k}"]
    for meth in ("3m", "4m"):
        f = mp.lu_blocked(mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im)), 8,
                          kc=mp.KernelChoice(method=meth, real_kernel="ozaki"))
        assert np.array_equal(f.pivots, oz[f"ozlu_{meth}_k{k}_piv"])
        assert beq(np.array([f.packed.re_plane.data, f.packed.im_plane.data]), oz[f"ozlu_{meth}_k{k}"])


@pytest.mark.gpu
def test_gpu_ozaki_vs_oracle_sizes(orc):
    """Ragged and larger shapes against the restatement (incl. the n=1024
    exactness budget, width 19 -> 21 cap)."""
    import paper_2403_16013_b200 as mp
    from oracle import ozaki_ref as ozr

    rng = np.random.default_rng(9)
    for (m, n, l, k, d) in [(1, 1, 1, 2, 6), (70, 130, 33, 2, 6), (256, 1024, 64, 2, 6),
                            (40, 50, 30, 3, 8), (33, 20, 17, 4, 12)]:
        A = mp.random_matrix(m, n, k, rng)
        B = mp.random_matrix(n, l, k, rng)
        assert beq(mp.rgemm_ozaki(A, B, d).data, ozr.rgemm(A.data, B.data, d)), (m, n, l, k)
