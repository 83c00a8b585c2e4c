"""Ozaki scheme: the oracle restatement pinned to the
reference's golden vectors (CPU) and the B200 path bit-identical to both
(GPU).  Golden: oracle/gen_golden.py ozaki -> tests/golden/ozaki.npz."""

import os

import numpy as np
import pytest

from testpaths import GOLD


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


def _both_paths(monkeypatch, fn):
    """fn() on the binary64 seam (cuBLAS DGEMM) and on the INT8 tensor-core path."""
    monkeypatch.setenv("MPC_OZAKI_GEMM", "dgemm")
    a = fn()
    monkeypatch.setenv("MPC_OZAKI_GEMM", "tc")
    b = fn()
    return a, b


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3, 4])
def test_gpu_ozaki_tensor_core_equals_seam(monkeypatch, k):
    """The tcgen05 INT8 path (digit slices, int32 TMEM groups, fused acc_plane /
    renorm / complex composition) is bit-identical to the exact binary64 seam:
    ragged row / column tiles, inner sizes off the 64-deep stage, several
    column tiles, both digit bases (width <= 20: base 2^7; 21..22: base 2^8)."""
    import paper_2403_16013_b200 as mp

    rng = np.random.default_rng(100 + k)
    d = {2: 6, 3: 8, 4: 12}[k]
    for (m, n, l) in [(1, 1, 1), (130, 70, 33), (257, 100, 97), (129, 1000, 130), (64, 64, 200)]:
        A = mp.random_matrix(m, n, k, rng)
        B = mp.random_matrix(n, l, k, rng)
        for sb in (None, 12, min(21, mp.split_exactness_bound(n))):
            x, y = _both_paths(monkeypatch, lambda: mp.rgemm_ozaki(A, B, d, split_bits=sb).data)
            assert beq(x, y), (m, n, l, k, sb)
    P = [mp.PlanarComplexMatrix(mp.random_matrix(90, 77, k, rng), mp.random_matrix(90, 77, k, rng)),
         mp.PlanarComplexMatrix(mp.random_matrix(77, 110, k, rng), mp.random_matrix(77, 110, k, rng))]
    for meth in ("3m", "4m"):
        kc = mp.KernelChoice(method=meth, real_kernel="ozaki")
        x, y = _both_paths(monkeypatch, lambda: mp.cgemm(P[0], P[1], kc))
        assert beq(x.re_plane.data, y.re_plane.data) and beq(x.im_plane.data, y.im_plane.data), meth


@pytest.mark.gpu
@pytest.mark.parametrize("meth", ["3m", "4m"])
def test_gpu_ozaki_lu_tensor_core_equals_seam(monkeypatch, meth):
    """lu_blocked with real_kernel="ozaki": the lookahead schedule with the fused
    LU subtraction on the tensor cores gives the seam's pivots and factors."""
    import paper_2403_16013_b200 as mp
    from paper_2403_16013_b200 import problems

    re, im = problems.lu_matrix(150, 2, 5)
    A = mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))
    kc = mp.KernelChoice(method=meth, real_kernel="ozaki")
    x, y = _both_paths(monkeypatch, lambda: mp.lu_blocked(A, 32, kc=kc))
    assert np.array_equal(x.pivots, y.pivots)
    assert beq(x.packed.re_plane.data, y.packed.re_plane.data)
    assert beq(x.packed.im_plane.data, y.packed.im_plane.data)


@pytest.mark.gpu
def test_gpu_ozaki_cluster_multicast():
    """MPC_OZAKI_CLUSTER=2 (A tiles multicast to a 2-CTA cluster) gives the same bits
    (the cluster size is read once per process, hence the subprocess)."""
    import subprocess
    import sys

    code = ("import os,sys,numpy as np; sys.path.insert(0, %r);"
            "import paper_2403_16013_b200 as mp;"
            "r=np.random.default_rng(7); A=mp.random_matrix(300,200,2,r); B=mp.random_matrix(200,250,2,r);"
            "os.environ['MPC_OZAKI_GEMM']='dgemm'; x=mp.rgemm_ozaki(A,B,6).data;"
            "os.environ['MPC_OZAKI_GEMM']='tc'; y=mp.rgemm_ozaki(A,B,6).data;"
            "print('EQ', x.tobytes()==y.tobytes())") % os.path.dirname(os.path.dirname(__file__))
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "MPC_OZAKI_CLUSTER": "2"},
                         capture_output=True, text=True, timeout=300)
    assert "EQ True" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_gpu_int8_peak_measured():
    """The INT8 tensor-core roofline denominator is measured, not assumed."""
    from paper_2403_16013_b200 import device

    p = device.int8_peak(50000)
    assert 1e15 < p < 1e16


@pytest.mark.gpu
def test_gpu_ozaki_wide_split_fallback(orc):
    """Widths above the int32 digit regime (here 24 bits, n = 16) run the
    binary64 seam automatically -- still bit-identical to the restatement."""
    import paper_2403_16013_b200 as mp
    from oracle import ozaki_ref as ozr

    rng = np.random.default_rng(21)
    A = mp.random_matrix(20, 16, 2, rng)
    B = mp.random_matrix(16, 12, 2, rng)
    assert mp.split_exactness_bound(16) >= 24
    got = mp.rgemm_ozaki(A, B, 5, split_bits=24).data
    assert beq(got, ozr.rgemm(A.data, B.data, 5, split_bits=24))
