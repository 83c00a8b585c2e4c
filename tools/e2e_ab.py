"""A/B of lu.factor_inplace on pinned host buffers at config 4 (host copies
overlapped with the LU vs staged): python tools/e2e_ab.py [n] [K] [reps] [real_kernel]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import lu, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
K = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rk = sys.argv[4] if len(sys.argv) > 4 else "blocked"
re0, im0 = problems.lu_matrix(n, 2, 1)
hr = torch.empty(re0.shape, dtype=torch.float64, pin_memory=True)
hi = torch.empty(im0.shape, dtype=torch.float64, pin_memory=True)
hp = torch.empty(n, dtype=torch.int64, pin_memory=True)
dev = torch.device("cuda", 0)
dr, di = torch.from_numpy(re0).to(dev), torch.from_numpy(im0).to(dev)
dp = torch.empty(n, dtype=torch.int64, device=dev)
for r in range(reps):
    for mode in ("device", "host"):
        hr.numpy()[...] = re0
        hi.numpy()[...] = im0
        dr.copy_(torch.from_numpy(re0))
        di.copy_(torch.from_numpy(im0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "host":
            lu.factor_inplace(hr.numpy(), hi.numpy(), K, piv=hp.numpy(), real_kernel=rk)
        else:
            lu.factor_inplace(dr, di, K, piv=dp, real_kernel=rk)
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{rk} rep {r} {mode} overlap={os.environ.get('MPC_HOST_OVERLAP', '1')}: {dt * 1e3:.1f} ms "
              f"({8 * n ** 3 / 3 / dt / 1e9:.1f} GFLOP/s)", flush=True)
