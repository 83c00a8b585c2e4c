"""GPU probe: Ozaki tensor-core path vs the cuBLAS binary64 seam (bitwise)
and timings of the complex DD GEMM (n=1024) for blocked / ozaki-dgemm /
ozaki-tc.  Usage: python tools/probe_ozaki.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import device, problems  # noqa: E402


def both(fn):
    os.environ["MPC_OZAKI_GEMM"] = "dgemm"
    a = fn()
    os.environ["MPC_OZAKI_GEMM"] = "tc"
    b = fn()
    return a, b


rng = np.random.default_rng(3)
bad = 0
for (m, n, l, k, d) in [(1, 1, 1, 2, 6), (130, 70, 33, 2, 6), (256, 1024, 64, 2, 6),
                        (300, 512, 200, 2, 6), (40, 50, 30, 3, 8), (129, 600, 65, 3, 8),
                        (33, 20, 17, 4, 12), (200, 300, 100, 4, 12), (64, 64, 64, 2, 3)]:
    A = mp.random_matrix(m, n, k, rng)
    B = mp.random_matrix(n, l, k, rng)
    x, y = both(lambda: mp.rgemm_ozaki(A, B, d).data)
    ok = x.tobytes() == y.tobytes()
    if not ok:
        bad += 1
        diff = np.argwhere(x != y)
        print("MISMATCH", (m, n, l, k, d), len(diff), diff[:5], x.ravel()[:4], y.ravel()[:4])
    else:
        print("ok", (m, n, l, k, d))
print("rgemm_ozaki tc vs dgemm mismatches:", bad)

dev = torch.device("cuda", 0)
for k, meth in [(2, "3m"), (2, "4m"), (3, "3m"), (4, "3m")]:
    n = 1024
    a, b = problems.gemm_inputs(n, k, 1, mp.renorm_planes)
    T = [torch.from_numpy(v).to(dev) for v in (a[0], a[1], b[0], b[1])]
    cr = torch.empty((k, n, n), dtype=torch.float64, device=dev)
    ci = torch.empty_like(cr)
    res = {}
    for name in ("blocked", "ozaki-dgemm", "ozaki-tc"):
        if name == "blocked" and k > 2:
            continue
        if name.startswith("ozaki"):
            os.environ["MPC_OZAKI_GEMM"] = name.split("-")[1]
            f = lambda: device.cgemm_ozaki(*T, cr, ci, method=meth)  # noqa: E731
        else:
            f = lambda: device.cgemm(*T, cr, ci, method=meth)  # noqa: E731
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        res[name] = (ms, cr.cpu().numpy().copy(), ci.cpu().numpy().copy())
        print(f"k={k} {meth} {name:12s} {ms:8.3f} ms  {8*n**3/ms/1e6:9.1f} GFLOP/s conv")
    x, y = res["ozaki-dgemm"], res["ozaki-tc"]
    print("  cgemm ozaki tc == dgemm:", x[1].tobytes() == y[1].tobytes() and x[2].tobytes() == y[2].tobytes())
