"""CPU oracle for the orthogonalization-free spectral-clustering hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` leg may import anything here.
The product path (paper_2305_10356_b200 + libofsc.so) never imports, links or
calls this package, and this package never imports the product path: the two
share no code.  Inputs come from `synth/` (seeded draws, no method arithmetic).

Plain, slow, obviously-correct numpy/scipy in fp64 (plus a precision-matched
fp32-storage mode), written step by step from arXiv 2305.10356
(`P:n` = /root/reference/PAPER.md line n) in the paper's order and notation.
Every reading of an ambiguous passage is listed in DESIGN.md "Readings".

Pins (tests/test_oracle_*.py, `-m "not gpu"`):
  operator   closed-form spectra (K2, P3, K_n, C_n, clique unions, stars,
             bipartite), D^{1/2}1 eigenvector, spec in [-2,0], brute-force dense
  directions finite differences of f1/f2, k=1 reductions, theorem fixed points
  cubics     exact cubic fit through direct evaluations (A.1 of SURVEY)
  roots      textbook cubics, brute-force bracketing (c3 > 0 and c3 < 0), min-psi on a grid
  beta       G = Gp -> 0, orthogonal columns -> ratio of norms, PR+ clamp, zero
             denominator (all exact), run_ofm's V_1 against the dense operator
  sums       1024-row blocked pairwise column sums / Grams vs math.fsum
  iterate    monotone objective (OFM), theorem limits on bridged cliques,
             subspace vs dense eigh
  kmeans     brute-force optimal partition (n<=8), separated blobs, k=1
  ari/nmi    contingency examples, permutation invariance
  jacobi     textbook 2x2, numpy eigh cross-check
No function is "parity unpinned".
"""
from .operator import (Operator, build_operator, apply_A, dense_A, fro2_A)
from .methods import (METHODS, direction, objective, grams, cubic_coefficients,
                      run_ofm, OFMResult, stop_constant, beta_pr, colsum, gram, pairwise_sum)
from .cubic import cubic_roots, select_step, psi, BRANCH
from .cluster import row_normalize, kmeans_lloyd, ari, nmi
from .eig import jacobi_eigh

__all__ = [
    "Operator", "build_operator", "apply_A", "dense_A", "fro2_A",
    "METHODS", "direction", "objective", "grams", "cubic_coefficients",
    "run_ofm", "OFMResult", "stop_constant", "beta_pr", "colsum", "gram", "pairwise_sum",
    "cubic_roots", "select_step", "psi", "BRANCH",
    "row_normalize", "kmeans_lloyd", "ari", "nmi", "jacobi_eigh",
]
