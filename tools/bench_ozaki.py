"""Ozaki TC kernel timing: per-class event times (gemm = the tcgen05 kernel,
other = split / elementwise) for complex DD/TD/QD GEMMs.
python tools/bench_ozaki.py [n] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import _lib, device, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
os.environ["MPC_OZAKI_GEMM"] = "tc"
for k, meth in [(2, "3m"), (2, "4m"), (3, "3m"), (4, "3m")]:
    a, b = problems.gemm_inputs(n, k, 1, mp.renorm_planes)
    T = [torch.from_numpy(v).to(dev) for v in (a[0], a[1], b[0], b[1])]
    cr = torch.empty((k, n, n), dtype=torch.float64, device=dev)
    ci = torch.empty_like(cr)
    f = lambda: device.cgemm_ozaki(*T, cr, ci, method=meth)  # noqa: E731
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / reps
    _lib.prof_enable(True)
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    pr = _lib.prof_summary()
    _lib.prof_enable(False)
    g_ms, g_ops, g_n = pr["gemm"]
    o_ms = pr["other"][0]
    print(f"CL={os.environ.get('MPC_OZAKI_CLUSTER', '4')} k={k} {meth} n={n}: {wall:7.3f} ms/cgemm "
          f"({8 * n**3 / wall / 1e6:7.1f} GF conv) | tc kernel {g_ms / g_n:7.3f} ms x{g_n // reps} "
          f"= {g_ops / (g_ms * 1e-3) / 1e15:5.2f} POPS int8 | other {o_ms / reps:6.3f} ms", flush=True)
