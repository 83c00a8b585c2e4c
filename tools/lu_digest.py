"""Digest of one blocked LU (pivots + packed factors) for cross-implementation
checks: python tools/lu_digest.py n K k [reps] -- prints one line per
repetition.  Environment switches (MPC_PANEL, MPC_PANEL_TPR, MPC_PANEL_COOP,
MPC_GEMM_CAP) select the panel / update implementation."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2403_16013_b200 as mp  # noqa: E402
from paper_2403_16013_b200 import problems  # noqa: E402

n, K, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
re, im = problems.lu_matrix(n, k, 3, populate_lower=k > 2,
                            renorm=mp.renorm_planes if k > 2 else None)
A = mp.PlanarComplexMatrix(mp.RealMatrix(re), mp.RealMatrix(im))
for _ in range(reps):
    f = mp.lu_blocked(A, K)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(f.pivots, dtype=np.int64).tobytes())
    h.update(f.packed.re_plane.data.tobytes())
    h.update(f.packed.im_plane.data.tobytes())
    print(h.hexdigest(), flush=True)
