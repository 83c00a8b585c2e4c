"""Golden vectors for the reference's k = 8 paths (REFERENCE_K) and the
k + 2 reconstruction check, made by running the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY (see gen_golden.py).  Writes tests/golden/k8.npz:

* ``rhs_{p}_n{n}``: ``gen_problem(n, seed, p)`` (bench.py:176-190) -- A's
  planes and the right-hand side ``reference_rhs(A, x)`` (bench.py:199-213:
  every operand widened to k = 8, naive 4M product, truncated back);
* ``mm8_{3m,4m}``: ``cgemm`` at k = 8 on full-depth random operands
  (cmatrix.py:145-177 with real_kernel="blocked");
* ``mmchk_{p}``: ``_matmul_check`` (bench.py:336-348) of a small matmul;
* ``rec_{p}``: ``reconstruction_error`` (lu.py:236-250) of lu_blocked factors
  at k + 2 (the 3M blocked product at 4 / 5 / 6 components).

    python oracle/gen_golden_k8.py
"""

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

import mpclu  # noqa: E402
from mpclu import KernelChoice, PlanarComplexMatrix, cgemm, lu_blocked  # noqa: E402
from mpclu import bench as rb  # noqa: E402
from mpclu.lu import reconstruction_error  # noqa: E402
from mpclu.rmatrix import random_matrix  # noqa: E402

RHS_CASES = [("dd", 12, 5), ("dd", 7, 2), ("td", 10, 3), ("qd", 9, 4)]


def main():
    out, meta = {}, {"numpy": np.__version__}
    try:
        import numba

        meta["numba"] = numba.__version__
    except ImportError:
        pass
    for p, n, seed in RHS_CASES:
        system, x = rb.gen_problem(n, seed, p)
        key = f"rhs_{p}_n{n}"
        out[key + "_are"] = system.A.re_plane.data
        out[key + "_aim"] = system.A.im_plane.data
        out[key + "_xre"] = x.re
        out[key + "_xim"] = x.im
        out[key + "_bre"] = system.b.re
        out[key + "_bim"] = system.b.im
        meta[key] = {"seed": seed}
    rng = np.random.default_rng(8)
    A = PlanarComplexMatrix(random_matrix(5, 6, 8, rng), random_matrix(5, 6, 8, rng))
    B = PlanarComplexMatrix(random_matrix(6, 4, 8, rng), random_matrix(6, 4, 8, rng))
    out["mm8_are"], out["mm8_aim"] = A.re_plane.data, A.im_plane.data
    out["mm8_bre"], out["mm8_bim"] = B.re_plane.data, B.im_plane.data
    for meth in ("3m", "4m"):
        C = cgemm(A, B, KernelChoice(method=meth, real_kernel="blocked"))
        out[f"mm8_{meth}_cre"], out[f"mm8_{meth}_cim"] = C.re_plane.data, C.im_plane.data
    for p, k in (("dd", 2), ("td", 3), ("qd", 4)):
        rng = np.random.default_rng(100 + k)
        A = PlanarComplexMatrix(random_matrix(6, 6, k, rng), random_matrix(6, 6, k, rng))
        B = PlanarComplexMatrix(random_matrix(6, 6, k, rng), random_matrix(6, 6, k, rng))
        C = cgemm(A, B, KernelChoice(method="3m"))
        out[f"mmchk_{p}_are"], out[f"mmchk_{p}_aim"] = A.re_plane.data, A.im_plane.data
        out[f"mmchk_{p}_bre"], out[f"mmchk_{p}_bim"] = B.re_plane.data, B.im_plane.data
        out[f"mmchk_{p}_cre"], out[f"mmchk_{p}_cim"] = C.re_plane.data, C.im_plane.data
        out[f"mmchk_{p}_err"] = np.array(rb._matmul_check(A, B, C))
        A = PlanarComplexMatrix(random_matrix(20, 20, k, rng), random_matrix(20, 20, k, rng))
        f = lu_blocked(A, 8)
        out[f"rec_{p}_are"], out[f"rec_{p}_aim"] = A.re_plane.data, A.im_plane.data
        out[f"rec_{p}_err"] = np.array(reconstruction_error(f, A))
    os.makedirs(GOLD, exist_ok=True)
    np.savez_compressed(os.path.join(GOLD, "k8.npz"), **out)
    with open(os.path.join(GOLD, "k8.meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
