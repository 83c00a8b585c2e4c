"""One unit-lower complex DD TRSM (kb x kb) on kb x M: python tools/one_trsm.py kb M [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib  # noqa: E402

kb, M = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
k = 2


def mk(r, c, scale=1.0):
    x = torch.zeros((k, r, c), dtype=torch.float64, device=dev)
    x[0] = (torch.rand((r, c), generator=g, device=dev, dtype=torch.float64) * 2 - 1) * scale
    return x


Lr, Li = mk(kb, kb, 1.0 / kb), mk(kb, kb, 1.0 / kb)
Xr0, Xi0 = mk(kb, M), mk(kb, M)
st = torch.cuda.current_stream().cuda_stream
L = _lib.lib()
Xr, Xi = Xr0.clone(), Xi0.clone()
ev = [torch.cuda.Event(True) for _ in range(2 * reps)]
for i in range(reps + 1):
    Xr.copy_(Xr0); Xi.copy_(Xi0)
    if i == 1:
        torch.cuda.synchronize()
        _lib.prof_enable(True)
    if i >= 1:
        ev[2 * (i - 1)].record()
    _lib.check(L.mpc_trsm_ll_unit(k, 3, kb, M, Lr.data_ptr(), Li.data_ptr(), kb, kb * kb,
                                  Xr.data_ptr(), Xi.data_ptr(), M, kb * M, st), "trsm")
    if i >= 1:
        ev[2 * (i - 1) + 1].record()
torch.cuda.synchronize()
pr = _lib.prof_summary()
_lib.prof_enable(False)
t = sum(ev[2 * j].elapsed_time(ev[2 * j + 1]) for j in range(reps)) / reps
print(f"trsm kb={kb} M={M}: {t:.3f} ms/call (with per-launch events)")
for c, v in pr.items():
    if v[2]:
        print(f"   {c:10s} {v[0]/reps:8.3f} ms  {v[2]//reps:5d} launches  {v[1]/(v[0]*1e-3)/1e12 if v[0] else 0:6.2f} T ops/s")
