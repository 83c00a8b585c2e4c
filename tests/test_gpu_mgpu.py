"""Single-process multi-GPU LU (mpc_getrf_ngpu, KernelChoice(ngpus=N)):
bit-identical to the 1-GPU factorization.  This box has one B200, so the
ranks share it (MPC_MGPU_OVERSUBSCRIBE=1): the schedule -- block-column-
cyclic ownership, panel packing, peer pulls of panel / pivots / status,
slot reuse, lookahead -- runs unchanged, only every "peer" is the same
device.  No kernel waits on another (stream / event dependencies only)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import problems  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _oversubscribe():
    mp._lib.require_device()
    old = os.environ.get("MPC_MGPU_OVERSUBSCRIBE")
    os.environ["MPC_MGPU_OVERSUBSCRIBE"] = "1"
    yield
    if old is None:
        del os.environ["MPC_MGPU_OVERSUBSCRIBE"]
    else:
        os.environ["MPC_MGPU_OVERSUBSCRIBE"] = old


def pc(re, im):
    return mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))


def ngpu_raw(re, im, K, ngpus, method=3, lookahead=1, real_kernel=0, d=0):
    lib = mp._lib.lib()
    k, n, _ = re.shape
    r, i = re.copy(), im.copy()
    piv = np.empty(n, dtype=np.int64)
    st = mp._lib.check(lib.mpc_getrf_ngpu(k, method, n, K, r.ctypes.data, i.ctypes.data,
                                          piv.ctypes.data, ngpus, lookahead, real_kernel, d, 0,
                                          None), "getrf_ngpu")
    return r, i, piv, st


@pytest.mark.parametrize("k,n,K,ngpus", [
    (2, 300, 32, 2), (2, 300, 32, 3), (2, 257, 64, 4), (2, 100, 100, 2), (2, 130, 16, 8),
    (3, 96, 16, 2), (4, 70, 16, 3),
])
def test_ngpu_bitwise_vs_one_gpu(k, n, K, ngpus):
    re, im = problems.lu_matrix(n, k, n + ngpus, populate_lower=k > 2,
                                renorm=mp.renorm_planes if k > 2 else None)
    for meth in ("3m", "4m"):
        f1 = mp.lu_blocked(pc(re.copy(), im.copy()), K, kc=mp.KernelChoice(method=meth))
        fN = mp.lu_blocked(pc(re.copy(), im.copy()), K, kc=mp.KernelChoice(method=meth, ngpus=ngpus))
        assert np.array_equal(f1.pivots, fN.pivots), (meth, ngpus)
        assert f1.packed.re_plane.data.tobytes() == fN.packed.re_plane.data.tobytes()
        assert f1.packed.im_plane.data.tobytes() == fN.packed.im_plane.data.tobytes()


@pytest.mark.parametrize("ngpus", [1, 2, 3])
def test_ngpu_without_lookahead(ngpus):
    k, n, K = 2, 200, 24
    re, im = problems.lu_matrix(n, k, 4)
    r1, i1, p1, _ = ngpu_raw(re, im, K, 1)
    r, i, p, st = ngpu_raw(re, im, K, ngpus, lookahead=0)
    assert st == -1 and np.array_equal(p, p1)
    assert r.tobytes() == r1.tobytes() and i.tobytes() == i1.tobytes()


def test_ngpu_ozaki_bitwise():
    k, n, K = 2, 160, 32
    re, im = problems.lu_matrix(n, k, 9)
    kc1 = mp.KernelChoice(real_kernel="ozaki")
    kc3 = mp.KernelChoice(real_kernel="ozaki", ngpus=3)
    f1 = mp.lu_blocked(pc(re.copy(), im.copy()), K, kc=kc1)
    f3 = mp.lu_blocked(pc(re.copy(), im.copy()), K, kc=kc3)
    assert np.array_equal(f1.pivots, f3.pivots)
    assert f1.packed.re_plane.data.tobytes() == f3.packed.re_plane.data.tobytes()
    assert f1.packed.im_plane.data.tobytes() == f3.packed.im_plane.data.tobytes()


def test_ngpu_singular_column():
    """A zero column in block 2 (owned by rank 0 of 2): every rank learns the
    status through the panel pulls; the call reports the first singular
    column like the 1-GPU path."""
    k, n, K = 2, 96, 16
    re, im = problems.lu_matrix(n, k, 3)
    re[:, :, 37] = 0.0
    im[:, :, 37] = 0.0
    with pytest.raises(mp.SingularMatrixError, match="column 37"):
        mp.lu_blocked(pc(re.copy(), im.copy()), K)
    with pytest.raises(mp.SingularMatrixError, match="column 37"):
        mp.lu_blocked(pc(re.copy(), im.copy()), K, kc=mp.KernelChoice(ngpus=2))
    _, _, _, st = ngpu_raw(re, im, K, 3)
    assert st == 37


def test_ngpu_device_pointers():
    """Device-resident input on the current device (peer copies via UVA)."""
    import torch

    k, n, K = 2, 150, 32
    re, im = problems.lu_matrix(n, k, 12)
    r1, i1, p1, _ = ngpu_raw(re, im, K, 1)
    dev = torch.device("cuda", 0)
    dr, di = torch.from_numpy(re).to(dev), torch.from_numpy(im).to(dev)
    dp = torch.empty(n, dtype=torch.int64, device=dev)
    lib = mp._lib.lib()
    st = lib.mpc_getrf_ngpu(k, 3, n, K, dr.data_ptr(), di.data_ptr(), dp.data_ptr(), 2, 1, 0, 0,
                            0, torch.cuda.current_stream().cuda_stream)
    assert st == -1
    assert np.array_equal(dp.cpu().numpy(), p1)
    assert dr.cpu().numpy().tobytes() == r1.tobytes() and di.cpu().numpy().tobytes() == i1.tobytes()


def test_ngpu_rejects_too_many_devices():
    """Without the oversubscription switch, ngpus above the device count fails loudly."""
    import torch

    os.environ["MPC_MGPU_OVERSUBSCRIBE"] = "0"
    try:
        re, im = problems.lu_matrix(40, 2, 1)
        with pytest.raises(RuntimeError, match="exceeds the visible CUDA devices"):
            mp.lu_blocked(pc(re, im), 8,
                          kc=mp.KernelChoice(ngpus=torch.cuda.device_count() + 1))
    finally:
        os.environ["MPC_MGPU_OVERSUBSCRIBE"] = "1"
