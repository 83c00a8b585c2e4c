"""Golden vectors for the reference's Strassen real kernel (rgemm.py:76-184),
made by running the UNMODIFIED reference.  TEST INFRASTRUCTURE ONLY (see
gen_golden.py).  Writes tests/golden/strassen.npz: operands and products of
rgemm_strassen for even, odd (peeled) and mixed recursion depths at
k = 2, 3, 4, and one complex 3M / 4M product with real_kernel="strassen".

    python oracle/gen_golden_strassen.py
"""

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

from mpclu import KernelChoice, PlanarComplexMatrix, cgemm, rgemm_strassen  # noqa: E402
from mpclu.rmatrix import random_matrix  # noqa: E402

CASES = [(2, 16, 4), (2, 13, 4), (2, 22, 3), (3, 12, 3), (3, 11, 2), (4, 10, 2), (4, 9, 4)]


def main():
    out = {}
    rng = np.random.default_rng(76)
    for k, n, thr in CASES:
        A, B = random_matrix(n, n, k, rng), random_matrix(n, n, k, rng)
        key = f"r_k{k}_n{n}_t{thr}"
        out[key + "_a"], out[key + "_b"] = A.data, B.data
        out[key + "_c"] = rgemm_strassen(A, B, threshold=thr).data
    for meth in ("3m", "4m"):
        k, n, thr = 2, 14, 4
        A = PlanarComplexMatrix(random_matrix(n, n, k, rng), random_matrix(n, n, k, rng))
        B = PlanarComplexMatrix(random_matrix(n, n, k, rng), random_matrix(n, n, k, rng))
        C = cgemm(A, B, KernelChoice(method=meth, real_kernel="strassen", threshold=thr))
        key = f"c_{meth}_k{k}_n{n}_t{thr}"
        for nm, M in (("a", A), ("b", B), ("c", C)):
            out[f"{key}_{nm}re"], out[f"{key}_{nm}im"] = M.re_plane.data, M.im_plane.data
    np.savez_compressed(os.path.join(GOLD, "strassen.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
