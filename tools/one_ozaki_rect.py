"""One complex Ozaki GEMM of LU-update shape (m x K) (K x m):
python tools/one_ozaki_rect.py k method m K [reps [l]]  (l defaults to m)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib, device  # noqa: E402

k, meth, m, K = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
l = int(sys.argv[6]) if len(sys.argv) > 6 else m
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
def mk(r, c):
    x = torch.zeros((k, r, c), dtype=torch.float64, device=dev)
    x[0] = torch.rand((r, c), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    return x
A = [mk(m, K), mk(m, K)]
B = [mk(K, l), mk(K, l)]
C = [mk(m, l), mk(m, l)]
device.cgemm_ozaki(*A, *B, *C, method=meth, epilogue=1)
torch.cuda.synchronize()
_lib.prof_enable(True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps):
    device.cgemm_ozaki(*A, *B, *C, method=meth, epilogue=1)
e1.record()
torch.cuda.synchronize()
pr = _lib.prof_summary()
_lib.prof_enable(False)
g_ms, g_ops, g_n = pr["gemm"]
print(f"m={m} K={K} l={l} k={k} {meth}: {e0.elapsed_time(e1)/reps:.3f} ms/call; tc {g_ms/g_n:.3f} ms x{g_n//reps} "
      f"{g_ops/(g_ms*1e-3)/1e15:.2f} POPS; other {pr['other'][0]/reps:.3f} ms/call")
