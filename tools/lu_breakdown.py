"""Per-class time breakdown (prof summary) of one complex DD LU at n x n:
python tools/lu_breakdown.py n K [blocked|ozaki] [k]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib, device  # noqa: E402

n, K = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "ozaki"
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
k = int(sys.argv[4]) if len(sys.argv) > 4 else 2
re0 = torch.zeros((k, n, n), dtype=torch.float64, device=dev)
im0 = torch.zeros_like(re0)
re0[0] = torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
im0[0] = torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
piv = torch.zeros(n, dtype=torch.int64, device=dev)
fn = device.getrf_ozaki if kind == "ozaki" else device.getrf
for it in range(2):
    re, im = re0.clone(), im0.clone()
    torch.cuda.synchronize()
    if it == 1:
        _lib.prof_enable(True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    fn(re, im, piv, K)
    e1.record()
    torch.cuda.synchronize()
t = e0.elapsed_time(e1)
pr = _lib.prof_summary()
_lib.prof_enable(False)
print(f"{kind} LU n={n} K={K}: {t:.1f} ms (with per-launch events; classes overlap across streams)")
for c, v in pr.items():
    if v[2]:
        print(f"   {c:10s} {v[0]:9.3f} ms  {v[2]:6d} launches  {v[1]/(v[0]*1e-3)/1e12 if v[0] else 0:8.2f} T ops/s")
