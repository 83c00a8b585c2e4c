"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json fixes distributions but no RNG; SURVEY.md §8d pins them:

* ``rng = Generator(Philox(key=seed))`` -- the family the reference's own
  harness uses (bench.py:181);
* leading limbs ``Re[0] = U(-1,1)``, then ``Im[0] = U(-1,1)``;
* populated lower limbs are drawn afterwards in the order
  ``Re[1], Im[1], Re[2], Im[2], ...`` as ``X[c] = X[c-1] * 2^-53 * U(-1,1)``
  and the planes are then renormalized elementwise (renorm_planes,
  _kernels.py:485-499) to restore the nonoverlap invariant;
* for a GEMM, A is drawn completely before B;
* ``x_true = 1 + 1i`` everywhere, ``b = cgemm_4m(A, x_true)`` at the working
  precision (BASELINE's "DD 4M");
* the ill-conditioned variant of config 4 scales row i of the leading limbs
  by ``10**(-12 i / n)``.

No public dataset is involved: these are the inputs.  The function that
restores the invariant is injected (``renorm``) so the same generator feeds
the GPU path (package renorm kernel) and the CPU oracle in tests.
"""

import numpy as np

TWO_M53 = 2.0 ** -53


def rng_for(seed):
    return np.random.Generator(np.random.Philox(key=np.uint64(seed)))


def draw_complex(rng, rows, cols, k, populate_lower, renorm=None, ill_conditioned=False):
    """One complex matrix as (re, im) planar arrays of shape (k, rows, cols)."""
    re = np.zeros((k, rows, cols))
    im = np.zeros((k, rows, cols))
    re[0] = rng.uniform(-1.0, 1.0, (rows, cols))
    im[0] = rng.uniform(-1.0, 1.0, (rows, cols))
    if ill_conditioned:
        scale = 10.0 ** (-12.0 * np.arange(rows, dtype=np.float64) / rows)
        re[0] *= scale[:, None]
        im[0] *= scale[:, None]
    if populate_lower and k > 1:
        for c in range(1, k):
            re[c] = re[c - 1] * TWO_M53 * rng.uniform(-1.0, 1.0, (rows, cols))
            im[c] = im[c - 1] * TWO_M53 * rng.uniform(-1.0, 1.0, (rows, cols))
        if renorm is None:
            raise ValueError("populated lower limbs need a renorm_planes callable")
        renorm(re)
        renorm(im)
    return re, im


def gemm_inputs(n, k, seed, renorm, m=None, l=None):
    """Config 1 style: both limbs populated; A (m x n) then B (n x l)."""
    m = n if m is None else m
    l = n if l is None else l
    rng = rng_for(seed)
    a = draw_complex(rng, m, n, k, True, renorm)
    b = draw_complex(rng, n, l, k, True, renorm)
    return a, b


def lu_matrix(n, k, seed, populate_lower=False, renorm=None, ill_conditioned=False):
    """Configs 0/2/4 (lo limbs 0) and 3 (all limbs populated)."""
    rng = rng_for(seed)
    return draw_complex(rng, n, n, k, populate_lower, renorm, ill_conditioned)


def x_true(n, k):
    """(1 + 1i) in every entry, as (k, n) planes."""
    xr = np.zeros((k, n))
    xi = np.zeros((k, n))
    xr[0] = 1.0
    xi[0] = 1.0
    return xr, xi
