"""Time the k = 8 reference right-hand side (bench.py:199-213) on the device."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import harness  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1024, 4096]:
    for p in ("dd", "qd"):
        system, x = harness.gen_problem(8, 1, p)  # warm
        rng = np.random.Generator(np.random.Philox(key=np.uint64(1)))
        k = {"dd": 2, "qd": 4}[p]
        A = harness.PlanarComplexMatrix(harness.RealMatrix.from_float64(rng.random((n, n)), k),
                                        harness.RealMatrix.from_float64(rng.random((n, n)), k))
        x = harness.ComplexVector(np.ones((k, n)), np.ones((k, n)))
        t0 = time.perf_counter()
        b = harness.reference_rhs(A, x)
        dt = time.perf_counter() - t0
        print(f"reference_rhs {p} n={n}: {dt*1e3:.1f} ms (4 n^2 = {4*n*n/dt/1e6:.1f} M k=8 complex-part MACs/s)",
              flush=True)
