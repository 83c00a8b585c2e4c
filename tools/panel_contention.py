"""Panel factorization time alone vs. concurrent with a trailing-update GEMM
on another stream (the lookahead situation): python tools/panel_contention.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib, device  # noqa: E402

dev = torch.device("cuda", 0)
k, rows, w = 2, 15872, 512
g = torch.Generator(device=dev).manual_seed(3)
re = torch.zeros((k, rows, w), dtype=torch.float64, device=dev)
im = torch.zeros_like(re)
re[0] = torch.rand((rows, w), generator=g, device=dev, dtype=torch.float64) * 2 - 1
im[0] = torch.rand((rows, w), generator=g, device=dev, dtype=torch.float64) * 2 - 1
W = [re.clone(), im.clone()]
piv = torch.zeros(rows, dtype=torch.int64, device=dev)
status = torch.full((1,), -1, dtype=torch.int64, device=dev)
L = _lib.lib()
hi = torch.cuda.Stream(priority=-5)
m, K = 8192, 512


def mk(r, c):
    x = torch.zeros((k, r, c), dtype=torch.float64, device=dev)
    x[0] = torch.rand((r, c), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    return x


A = [mk(m, K), mk(m, K)]
B = [mk(K, 4 * m), mk(K, 4 * m)]
C = [mk(m, 4 * m), mk(m, 4 * m)]


def reset():
    W[0].copy_(re)
    W[1].copy_(im)
    torch.cuda.synchronize()


def panel(stream):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        L.mpc_panel_factor_async(k, 3, rows, 0, w, W[0].data_ptr(), W[1].data_ptr(), w, rows * w,
                                 piv.data_ptr(), status.data_ptr(), stream.cuda_stream)
        e1.record(stream)
    return e0, e1


for mode in ("alone", "with_gemm_eft", "with_gemm_ozaki"):
    for rep in range(2):
        reset()
        g0, g1 = torch.cuda.Event(True), torch.cuda.Event(True)
        g0.record()
        if mode != "alone":
            f = device.cgemm if mode == "with_gemm_eft" else device.cgemm_ozaki
            f(*A, *B, *C, method="3m", epilogue=1)  # queued on the default stream
        g1.record()
        e0, e1 = panel(hi)
        torch.cuda.synchronize()
        print(f"{mode:16s} panel {e0.elapsed_time(e1):8.2f} ms   gemm {g0.elapsed_time(g1):8.2f} ms")
