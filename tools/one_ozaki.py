"""One complex Ozaki GEMM (for ncu launch lists): python tools/one_ozaki.py k method n [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import device, problems  # noqa: E402

k, meth, n = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda", 0)
a, b = problems.gemm_inputs(n, k, 1, mp.renorm_planes)
T = [torch.from_numpy(v).to(dev) for v in (a[0], a[1], b[0], b[1])]
cr = torch.empty((k, n, n), dtype=torch.float64, device=dev)
ci = torch.empty_like(cr)
for _ in range(reps):
    device.cgemm_ozaki(*T, cr, ci, method=meth)
torch.cuda.synchronize()
