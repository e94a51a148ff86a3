"""Would a second-level order inside an LPA community shrink the SpMM's gather
window?  One c4-like community (80k nodes, DCSBM degree law, avg intra degree 15)
ordered randomly vs by reverse Cuthill-McKee: the fraction of the community's
rows referenced by each consecutive window of 14k rows (the SpMM's in-order row
window at c4).  CPU only."""
import os
import sys

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import dcsbm_graph  # noqa: E402

n, W = 80_000, 14_000
s, d, _ = dcsbm_graph(n, 1, 600_000, 1e9, 7, None)
S = sp.coo_matrix((np.ones(len(s)), (s, d)), shape=(n, n))
S = ((S + S.T) > 0).astype(np.int8).tocsr()


def touched(order):
    P = S[order][:, order].tocsr()
    return [round(np.unique(P.indices[P.indptr[a]:P.indptr[a + W]]).size / n, 3)
            for a in range(0, n - W + 1, W)]


print("random order:", touched(np.random.default_rng(0).permutation(n)))
print("RCM order:   ", touched(np.asarray(reverse_cuthill_mckee(S, symmetric_mode=True))))
