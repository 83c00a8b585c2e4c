"""One panel factorization (rows x w, DD) for launch lists:
python tools/one_panel.py rows w [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib  # noqa: E402

rows, w = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
k = 2
re = torch.zeros((k, rows, w), dtype=torch.float64, device=dev)
im = torch.zeros_like(re)
re[0] = torch.rand((rows, w), generator=g, device=dev, dtype=torch.float64) * 2 - 1
im[0] = torch.rand((rows, w), generator=g, device=dev, dtype=torch.float64) * 2 - 1
piv = torch.zeros(rows, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream
W = [re.clone(), im.clone()]
L = _lib.lib()
for i in range(reps + 1):
    W[0].copy_(re); W[1].copy_(im)
    if i == 1:
        torch.cuda.synchronize()
        _lib.prof_enable(True)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
    s = L.mpc_panel_factor(k, 3, rows, 0, w, W[0].data_ptr(), W[1].data_ptr(), w, rows * w,
                           piv.data_ptr(), st)
e1.record()
torch.cuda.synchronize()
pr = _lib.prof_summary()
_lib.prof_enable(False)
print(f"panel {rows}x{w}: {e0.elapsed_time(e1)/reps:.3f} ms/panel (with per-launch events)")
for c, v in pr.items():
    if v[2]:
        print(f"   {c:10s} {v[0]/reps:8.3f} ms  {v[2]//reps:5d} launches  {v[1]/(v[0]*1e-3)/1e12 if v[0] else 0:6.2f} T ops/s")
