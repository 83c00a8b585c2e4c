"""Golden vectors for max_rel_err (lu.py:253-282), made by running the
UNMODIFIED reference.  TEST INFRASTRUCTURE ONLY (see gen_golden.py).  Writes
tests/golden/metrics.npz: per case the two planar vectors and the k
components of the reference's result (k = 2, 3, 4; random full-depth
vectors with relative perturbations around 2^-80 ... 2^-150, an exact-zero
difference, and ties between entries).

    python oracle/gen_golden_metrics.py
"""

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

from mpclu._kernels import renorm_planes  # noqa: E402
from mpclu.lu import ComplexVector, max_rel_err  # noqa: E402


def vec(rng, n, k):
    v = np.zeros((k, 1, n))
    v[0, 0] = rng.uniform(-1, 1, n)
    for c in range(1, k):
        v[c, 0] = v[c - 1, 0] * 2.0 ** -53 * rng.uniform(-1, 1, n)
    renorm_planes(v, k)
    return v[:, 0, :].copy()


def main():
    rng = np.random.default_rng(263)
    out = {}
    case = 0
    for k in (2, 3, 4):
        for n, scale in ((1, 2.0 ** -90), (37, 2.0 ** -80), (300, 2.0 ** -150), (64, 0.0)):
            xr, xi = vec(rng, n, k), vec(rng, n, k)
            hr, hi = xr.copy(), xi.copy()
            if scale:
                # perturb the lowest limb region: add a tiny value and renormalize
                pr = np.concatenate([hr, (xr[0] * scale * rng.uniform(-1, 1, n))[None]])[:, None, :]
                pi = np.concatenate([hi, (xi[0] * scale * rng.uniform(-1, 1, n))[None]])[:, None, :]
                renorm_planes(pr, k + 1)
                renorm_planes(pi, k + 1)
                hr, hi = pr[:k, 0, :].copy(), pi[:k, 0, :].copy()
                if n >= 4:  # a tie: two entries with identical data
                    for a in (xr, xi, hr, hi):
                        a[:, 3] = a[:, 1]
            e = max_rel_err(ComplexVector(hr, hi), ComplexVector(xr, xi))
            key = f"case{case}_k{k}"
            out[key + "_xr"], out[key + "_xi"] = xr, xi
            out[key + "_hr"], out[key + "_hi"] = hr, hi
            out[key + "_err"] = np.asarray(e.components, dtype=np.float64)
            case += 1
    np.savez_compressed(os.path.join(GOLD, "metrics.npz"), **out)
    print("wrote", case, "cases")


if __name__ == "__main__":
    main()
