"""A/B of the drop-in lu_blocked path on pageable numpy at cfg4 (n=16384,
K=512, DD): where the host-side time goes and which staging wins.
python tools/e2e_dropin_ab.py [n] [K]"""
import concurrent.futures as cf
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import lu as lum, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
K = int(sys.argv[2]) if len(sys.argv) > 2 else 512
re0, im0 = problems.lu_matrix(n, 2, 1)
cudart = torch.cuda.cudart()
torch.cuda.init()


def pcopy(dst, src, nt=16):
    rows = src.shape[1]
    ch = (rows + nt - 1) // nt
    with cf.ThreadPoolExecutor(nt) as ex:
        list(ex.map(lambda i: np.copyto(dst[:, i * ch:(i + 1) * ch], src[:, i * ch:(i + 1) * ch]),
                    range(nt)))


def t(f):
    torch.cuda.synchronize()
    a = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return time.perf_counter() - a, r


# warm-up (pool, context)
lum.factor_inplace(re0[:, :1024, :1024].copy(), im0[:, :1024, :1024].copy(), 256)
dt, _ = t(lambda: (re0.copy(), im0.copy()))
print(f"np.copy of both planes: {dt:.3f} s")
dt, _ = t(lambda: pcopy(np.empty_like(re0), re0))
print(f"threaded copy of one plane set: {dt:.3f} s")
A = mp.PlanarComplexMatrix(mp.RealMatrix(re0), mp.RealMatrix(im0))
dt, f = t(lambda: mp.lu_blocked(A, K))
print(f"lu_blocked (current): {dt:.3f} s")
base = f.pivots.copy()
del f


def staged_threaded():
    r, i = np.empty_like(re0), np.empty_like(im0)
    pcopy(r, re0)
    pcopy(i, im0)
    return lum.factor_inplace(r, i, K)


dt, p = t(staged_threaded)
print(f"threaded copy + staged factor_inplace: {dt:.3f} s  pivots equal {np.array_equal(p, base)}")


def registered():
    r, i = np.empty_like(re0), np.empty_like(im0)
    a = time.perf_counter()
    pcopy(r, re0)
    pcopy(i, im0)
    b = time.perf_counter()
    for x in (r, i):
        assert cudart.cudaHostRegister(x.ctypes.data, x.nbytes, 0) == 0
    c = time.perf_counter()
    p = lum.factor_inplace(r, i, K)
    d = time.perf_counter()
    for x in (r, i):
        cudart.cudaHostUnregister(x.ctypes.data)
    e = time.perf_counter()
    print(f"   copy {b - a:.3f}  register {c - b:.3f}  factor(overlap) {d - c:.3f}  unregister {e - d:.3f}")
    return p


dt, p = t(registered)
print(f"threaded copy + cudaHostRegister + overlapped factor_inplace: {dt:.3f} s  pivots equal {np.array_equal(p, base)}")
