"""Precision constants of mpclu.expansion (expansion.py:23-38)."""

import math

PRECISIONS = {"dd": 2, "td": 3, "qd": 4}
PRECISION_BITS = {2: 106, 3: 159, 4: 212}
REFERENCE_K = 8

# BASELINE.json's unit round-off for the 10*n*u acceptance bound
U_PREC = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}


def eps_for(k):
    """Unit round-off of a k-component expansion: 2^(1 - 53k)."""
    return math.ldexp(1.0, 1 - 53 * k)


def digits_for(k):
    return int(math.floor(53 * k * math.log10(2.0)))


def exp_to_string(x, digits=None):
    """Decimal string of an expansion's exact value, correctly rounded to
    `digits` significant digits (expansion.py:199-215; default: the digits k
    components carry).  `x` is anything with .components / .k / .to_fraction()
    (rmatrix.Expansion)."""
    from decimal import Decimal, localcontext

    if digits is None:
        digits = digits_for(x.k)
    f = x.to_fraction()
    if f == 0:
        return "0.0"
    with localcontext() as ctx:
        ctx.prec = digits
        d = Decimal(f.numerator) / Decimal(f.denominator)
    s = str(d)
    if "E" in s:
        return s.replace("E", "e")
    return s if "." in s else s + ".0"
