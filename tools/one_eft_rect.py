"""One EFT complex GEMM of LU-update shape with the A22 -= L21 U12 epilogue:
python tools/one_eft_rect.py k method m K l [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import device  # noqa: E402

k, meth, m, K, l = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)


def mk(r, c):
    x = torch.zeros((k, r, c), dtype=torch.float64, device=dev)
    x[0] = torch.rand((r, c), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    return x


A, B, C = [mk(m, K), mk(m, K)], [mk(K, l), mk(K, l)], [mk(m, l), mk(m, l)]
device.cgemm(*A, *B, *C, method=meth, epilogue=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps):
    device.cgemm(*A, *B, *C, method=meth, epilogue=1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"EFT {meth} m={m} K={K} l={l}: {ms:.2f} ms  {m*l*K*93/(ms*1e-3)/1e12:.2f} T FP64 ops/s")
