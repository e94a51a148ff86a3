"""Oracle against the cited closed-form fixtures in tests/golden/."""
import os

import numpy as np

from oracle import build_operator, dense_A, select_step, ari, nmi
from tests import graphs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GRAPHS = {"K2": [(0, 1)], "P3": G.path(3), "K4": G.clique(4), "C4": G.cycle(4), "S3": G.star(3)}


def rows(name):
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            yield [f.strip() for f in line.split("|")]


def test_golden_spectra():
    for name, vals, _cite in rows("spectra.txt"):
        s, d = G.edges(GRAPHS[name])
        op = build_operator(int(max(s.max(), d.max())) + 1, s, d)
        w = np.linalg.eigvalsh(dense_A(op))
        assert np.allclose(w, [float(v) for v in vals.split()], atol=1e-13), name


def test_golden_cubics():
    for coef, alpha, _cite in rows("cubics.txt"):
        a, _ = select_step(*[float(c) for c in coef.split()])
        assert abs(a - float(alpha)) <= 1e-13, coef


def test_golden_ari_nmi():
    for la, lb, a, n, _cite in rows("ari.txt"):
        la = [int(x) for x in la.split()]
        lb = [int(x) for x in lb.split()]
        assert abs(ari(la, lb) - float(a)) <= 1e-12
        assert abs(nmi(la, lb) - float(n)) <= 1e-12
