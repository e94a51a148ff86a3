"""Oracle root finding / selection pins."""
import math

import numpy as np
import pytest

from oracle import cubic_roots, select_step, psi, BRANCH


def test_textbook_three_roots_tie_rule():
    roots, code = cubic_roots(1.0, 0.0, -1.0, 0.0)          # a^3 - a
    assert code == BRANCH["three0"]
    assert np.allclose(sorted(roots), [-1.0, 0.0, 1.0], atol=1e-15)
    a, code = select_step(1.0, 0.0, -1.0, 0.0)              # psi(-1) = psi(1): smaller |a| tie, then smaller a
    assert a == -1.0


def test_triple_and_single_root():
    assert select_step(1.0, 0.0, 0.0, 0.0) == (0.0, BRANCH["triple"])
    a, code = select_step(1.0, 0.0, 1.0, 0.0)                # a^3 + a
    assert a == 0.0 and code == BRANCH["one"]
    a, code = select_step(2.0, 0.0, 0.0, -16.0)              # 2a^3 = 16
    assert abs(a - 2.0) < 1e-15


def test_double_root_selects_single():
    # (a-1)^2 (a+3) = a^3 + a^2 - 5a + 3 -> the single-multiplicity root -3
    a, _ = select_step(1.0, 1.0, -5.0, 3.0)
    assert abs(a + 3.0) < 1e-13
    # exactly representable double root case: a^3 - 3a + 2 = (a-1)^2 (a+2)
    a, code = select_step(1.0, 0.0, -3.0, 2.0)
    assert abs(a + 2.0) < 1e-13


def test_degenerate_cases():
    assert select_step(0.0, 0.0, 0.0, 0.0) == (0.0, BRANCH["zero"])
    assert select_step(0.0, 0.0, 0.0, 1.0) == (0.0, BRANCH["noroot"])
    assert select_step(0.0, 0.0, 2.0, -1.0) == (0.5, BRANCH["linear"])
    assert select_step(0.0, 1.0, 0.0, 1.0) == (0.0, BRANCH["noroot"])
    a, code = select_step(0.0, 1.0, -3.0, 2.0)               # roots 1, 2; psi = a^3/3 - 3a^2/2 + 2a
    assert code == BRANCH["quad2"] and a == 2.0               # psi(1) = 5/6 > psi(2) = 2/3
    assert select_step(float("nan"), 1.0, 1.0, 1.0)[1] == BRANCH["diverged"]
    assert select_step(1.0, float("inf"), 1.0, 1.0)[1] == BRANCH["diverged"]


def brute_real_roots(c):
    """Brute force: sign changes on a fine grid + bisection (independent of Cardano)."""
    c3, c2, c1, c0 = c
    f = lambda a: ((c3 * a + c2) * a + c1) * a + c0
    bound = 1.0 + max(abs(c2 / c3), abs(c1 / c3), abs(c0 / c3))   # Cauchy bound
    pos = np.logspace(-14, np.log10(bound), 100000)
    xs = np.concatenate([-pos[::-1], [0.0], pos])       # log grid: resolves roots of any scale
    fx = f(xs)
    out = []
    for i in np.nonzero(np.sign(fx[:-1]) * np.sign(fx[1:]) <= 0)[0]:
        lo, hi = xs[i], xs[i + 1]
        if fx[i] == 0:
            out.append(lo)
            continue
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if np.sign(f(mid)) == np.sign(f(lo)):
                lo = mid
            else:
                hi = mid
        out.append(0.5 * (lo + hi))
    out = sorted(out)
    merged = []
    for r in out:
        if not merged or abs(r - merged[-1]) > 1e-9 * (1 + abs(r)):
            merged.append(r)
    return merged


@pytest.mark.parametrize("seed", range(200))
def test_random_cubics_against_brute_force(seed):
    rng = np.random.default_rng(seed)
    eps = 10.0 ** rng.uniform(-6, 0)
    c = (rng.uniform(0.1, 1) * eps * eps, rng.standard_normal() * eps,
         rng.standard_normal(), rng.standard_normal())
    roots, code = cubic_roots(*c)
    brute = brute_real_roots(c)
    a, code2 = select_step(*c)
    # the selected step is a root (after polish) ...
    scale = abs(c[0]) * abs(a) ** 3 + abs(c[1]) * a * a + abs(c[2]) * abs(a) + abs(c[3])
    assert abs(((c[0] * a + c[1]) * a + c[2]) * a + c[3]) <= 1e-12 * scale
    # ... matches a brute-force root, and minimises psi over all brute-force roots
    assert min(abs(a - r) for r in brute) <= 1e-7 * (1 + abs(a))
    best = min(brute, key=lambda r: psi(*c, r))
    assert psi(*c, a) <= psi(*c, best) + 1e-10 * (1 + abs(psi(*c, best)))
    if len(brute) == 3:
        assert code2 in (BRANCH["three0"], BRANCH["three1"], BRANCH["three2"])


@pytest.mark.parametrize("seed", range(20))
def test_selected_root_minimises_psi_on_grid(seed):
    """c3 > 0: psi is a quartic with positive leading term; the chosen root is its
    global minimiser (checked on a 101-point grid over [-2|a|, 2|a|])."""
    rng = np.random.default_rng(100 + seed)
    r = np.sort(rng.standard_normal(3) * 2)
    c3 = rng.uniform(0.5, 2)
    c = (c3, -c3 * r.sum(), c3 * (r[0] * r[1] + r[0] * r[2] + r[1] * r[2]), -c3 * r.prod())
    a, _ = select_step(*c)
    grid = np.linspace(-2 * abs(a), 2 * abs(a), 101)
    assert psi(*c, a) <= min(psi(*c, g) for g in grid) + 1e-10


@pytest.mark.parametrize("seed", range(200))
def test_random_cubics_negative_leading_coefficient(seed):
    """c3 < 0 (TriOFM-f2 can produce it): the bullets of P:307-312 are
    followed literally -- the only real root, the single-multiplicity root, or
    among three real roots the one of minimal psi.  For c3 < 0, psi is a quartic
    opening downwards whose three critical points are max, min, max, so the
    minimal-psi root is the MIDDLE root (the only local minimum of psi)."""
    rng = np.random.default_rng(10_000 + seed)
    eps = 10.0 ** rng.uniform(-6, 0)
    c = (-rng.uniform(0.1, 1) * eps * eps, rng.standard_normal() * eps,
         rng.standard_normal(), rng.standard_normal())
    a, code = select_step(*c)
    scale = abs(c[0]) * abs(a) ** 3 + abs(c[1]) * a * a + abs(c[2]) * abs(a) + abs(c[3])
    assert abs(((c[0] * a + c[1]) * a + c[2]) * a + c[3]) <= 1e-12 * scale
    brute = brute_real_roots(c)
    assert min(abs(a - r) for r in brute) <= 1e-7 * (1 + abs(a))
    best = min(brute, key=lambda r: psi(*c, r))
    assert psi(*c, a) <= psi(*c, best) + 1e-10 * (1 + abs(psi(*c, best)))
    if len(brute) == 3:
        assert code in (BRANCH["three0"], BRANCH["three1"], BRANCH["three2"])
        assert abs(a - brute[1]) <= 1e-7 * (1 + abs(a))


@pytest.mark.parametrize("seed", range(20))
def test_negative_leading_three_roots_selects_middle(seed):
    """c3 < 0 with three well-separated real roots r0 < r1 < r2: alpha = r1."""
    rng = np.random.default_rng(300 + seed)
    r = np.sort(rng.standard_normal(3) * 2)
    while np.min(np.diff(r)) < 0.1:
        r = np.sort(rng.standard_normal(3) * 2)
    c3 = -rng.uniform(0.5, 2)
    c = (c3, -c3 * r.sum(), c3 * (r[0] * r[1] + r[0] * r[2] + r[1] * r[2]), -c3 * r.prod())
    a, code = select_step(*c)
    assert code in (BRANCH["three0"], BRANCH["three1"], BRANCH["three2"])
    assert abs(a - r[1]) <= 1e-12 * (1 + abs(r[1]))
    # psi(r1) is a local minimum: psi increases to both sides up to the other roots
    for x in np.linspace(r[0], r[2], 41):
        if r[0] < x < r[2]:
            assert psi(*c, a) <= psi(*c, x) + 1e-12


def test_negative_leading_one_root_is_taken():
    """c3 < 0 with one real root: that root, although it maximises psi."""
    a, code = select_step(-1.0, 0.0, -1.0, 2.0)          # -(a^3 + a - 2) = -(a - 1)(a^2 + a + 2)
    assert code == BRANCH["one"] and abs(a - 1.0) < 1e-15
