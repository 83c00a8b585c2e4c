"""Small LUs / GEMMs / solves for compute-sanitizer runs (racecheck,
synccheck, memcheck): python tools/sanitize_lu.py
Covers the grid-wide base panel (cooperative grid barrier, 1 and several
CTAs), the cluster base panel (MPC_PANEL=cluster run), the last-block pivot
kernels (MPC_PANEL=launches run), TRSM, LASWP, the fused GEMM and the solve."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import problems  # noqa: E402

cases = [(96, 32, 2), (300, 64, 2), (700, 128, 2), (96, 32, 3)]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for n, K, k in cases:
    re, im = problems.lu_matrix(n, k, 7)
    A = mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))
    f = mp.lu_blocked(A, K)
    xr, xi = problems.x_true(n, k)
    X = mp.PlanarComplexMatrix(mp.RealMatrix(xr.reshape(k, n, 1).copy()),
                               mp.RealMatrix(xi.reshape(k, n, 1).copy()))
    B = mp.cgemm(A, X, mp.KernelChoice(method="4m"))
    b = mp.ComplexVector(B.re_plane.data.reshape(k, n), B.im_plane.data.reshape(k, n))
    x = mp.solve(f, b)
    err = float(mp.max_rel_err(x, mp.ComplexVector(xr, xi)))
    print(f"n={n} K={K} k={k}: pivots[:4]={f.pivots[:4]} fwd_err={err:.3e}", flush=True)
print("done")
