"""Oracle: exact line-search root finding and step selection (TEST INFRASTRUCTURE ONLY).

P:307-313  "Solving the above equation might result in one, two, or three real
roots. There are three different choices of alpha: the real root if only one
real root exists; the real root of single multiplicity if two real roots
exist; the real root which achieves the minimal function value when three real
roots exist.  ... via Cardano's formula."

The procedure (R7, R9, R10) is spelled out below in the exact order
of floating-point operations so that it can be restated independently in CUDA:
  * all four coefficients 0           -> alpha = 0            (code ZERO)
  * c3 = 0: stable quadratic / linear (no real root -> alpha = 0, code NOROOT)
  * else normalise a=c2/c3, b=c1/c3, c=c0/c3; p = b - a^2/3,
    q = 2a^3/27 - ab/3 + c, D = (q/2)^2 + (p/3)^3
      D > 0  one real root (Cardano, sign(0) := +1)
      D = 0  p = 0: triple root -a/3; else single root 3q/p - a/3 (selected)
      D < 0  three real roots (trigonometric form)
  * every root: exactly 2 Newton steps on the original cubic (skip if f' = 0)
  * several candidates: minimise psi(alpha) = c3 a^4/4 + c2 a^3/3 + c1 a^2/2 + c0 a,
    ties -> smaller |alpha|, then smaller alpha
  * any non-finite coefficient or result -> alpha = 0, code DIVERGED
"""
from __future__ import annotations

import math

BRANCH = {
    "zero": 0, "noroot": 1, "linear": 2, "quad1": 3, "quad2": 4,
    "one": 5, "triple": 6, "double": 7, "three0": 8, "three1": 9, "three2": 10,
    "diverged": 11,
}


def _sgn(x: float) -> float:
    return -1.0 if x < 0.0 else 1.0          # sign(0) := +1


def cubic_eval(c3, c2, c1, c0, a):
    return ((c3 * a + c2) * a + c1) * a + c0


def cubic_deriv(c3, c2, c1, a):
    return (3.0 * c3 * a + 2.0 * c2) * a + c1


def psi(c3, c2, c1, c0, a):
    """Antiderivative of the cubic with psi(0) = 0 (R8)."""
    return a * (c0 + a * (0.5 * c1 + a * (c2 / 3.0 + a * (0.25 * c3))))


def _polish(c3, c2, c1, c0, a):
    for _ in range(2):
        d = cubic_deriv(c3, c2, c1, a)
        if d != 0.0:
            a = a - cubic_eval(c3, c2, c1, c0, a) / d
    return a


def cubic_roots(c3, c2, c1, c0):
    """Real roots (unpolished) and branch code of c3 a^3 + c2 a^2 + c1 a + c0."""
    if c3 == 0.0 and c2 == 0.0 and c1 == 0.0 and c0 == 0.0:
        return [], BRANCH["zero"]
    if c3 == 0.0:
        if c2 == 0.0:
            if c1 == 0.0:
                return [], BRANCH["noroot"]
            return [-c0 / c1], BRANCH["linear"]
        disc = c1 * c1 - 4.0 * c2 * c0
        if disc < 0.0:
            return [], BRANCH["noroot"]
        q = -0.5 * (c1 + _sgn(c1) * math.sqrt(disc))
        if q == 0.0:
            return [0.0], BRANCH["quad1"]
        return [q / c2, c0 / q], BRANCH["quad2"]
    a = c2 / c3
    b = c1 / c3
    c = c0 / c3
    p = b - (a * a) / 3.0
    q = ((2.0 * a) * a * a) / 27.0 - (a * b) / 3.0 + c
    h = q / 2.0
    t = p / 3.0
    D = h * h + (t * t) * t
    if D > 0.0:
        A = -_sgn(q) * math.cbrt(abs(q) / 2.0 + math.sqrt(D))
        B = -p / (3.0 * A) if A != 0.0 else 0.0
        return [A + B - a / 3.0], BRANCH["one"]
    if D == 0.0:
        if p == 0.0:
            return [-a / 3.0], BRANCH["triple"]
        return [(3.0 * q) / p - a / 3.0], BRANCH["double"]
    r = 2.0 * math.sqrt(-p / 3.0)
    arg = ((3.0 * q) / (2.0 * p)) * math.sqrt(-3.0 / p)
    arg = min(1.0, max(-1.0, arg))
    theta = math.acos(arg) / 3.0
    roots = [-a / 3.0 + r * math.cos(theta - (2.0 * math.pi * j) / 3.0) for j in range(3)]
    return roots, BRANCH["three0"]


def select_step(c3, c2, c1, c0):
    """alpha for one cubic and its branch code (R7-R10)."""
    if not all(math.isfinite(x) for x in (c3, c2, c1, c0)):
        return 0.0, BRANCH["diverged"]
    roots, code = cubic_roots(c3, c2, c1, c0)
    if not roots:
        return 0.0, code
    best, best_psi, best_j = None, None, 0
    for j, r in enumerate(roots):
        r = _polish(c3, c2, c1, c0, r)
        v = psi(c3, c2, c1, c0, r)
        if best is None or v < best_psi or (
                v == best_psi and (abs(r) < abs(best) or (abs(r) == abs(best) and r < best))):
            best, best_psi, best_j = r, v, j
    if not math.isfinite(best):
        return 0.0, BRANCH["diverged"]
    if code == BRANCH["three0"]:
        code += best_j
    return best, code
