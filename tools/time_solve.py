"""Time the GPU solve (mpc_getrs: interchanges + forward + backward) on
device-resident factors: python tools/time_solve.py n k [method] [reps]
Synthetic well-scaled factors (off-diagonal U(-1,1)/n, unit diagonal) and a
random pivot vector p_i >= i."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib, device  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
meth = sys.argv[3] if len(sys.argv) > 3 else "3m"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
fr = torch.zeros((k, n, n), dtype=torch.float64, device=dev)
fi = torch.zeros_like(fr)
fr[0] = (torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / n
fi[0] = (torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / n
fr[0].diagonal().fill_(1.0)
piv = (torch.arange(n, device=dev) + (torch.rand(n, generator=g, device=dev) *
                                      (n - torch.arange(n, device=dev))).long()).clamp(max=n - 1)
b0r = torch.zeros((k, n), dtype=torch.float64, device=dev)
b0r[0] = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
b0i = b0r.clone()
ts = []
for it in range(reps + 1):
    br, bi = b0r.clone(), b0i.clone()
    torch.cuda.synchronize()
    if it == reps:
        _lib.prof_enable(True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    device.getrs(fr, fi, piv, br, bi, meth)
    e1.record()
    torch.cuda.synchronize()
    if it < reps:
        ts.append(e0.elapsed_time(e1))
pr = _lib.prof_summary()
_lib.prof_enable(False)
ts.sort()
print(f"solve n={n} k={k} {meth}: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f} ms "
      f"(reps {reps}); launches per solve {pr['solve'][2]}")
for c, v in pr.items():
    if v[2]:
        print(f"   {c:10s} {v[0]:9.3f} ms  {v[2]:6d} launches  "
              f"{v[1] / (v[0] * 1e-3) / 1e12 if v[0] else 0:8.3f} T ops/s (with per-launch events)")
