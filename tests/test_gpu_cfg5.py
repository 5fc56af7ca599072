"""BASELINE config 5: modularity-based link-prediction scoring (sparse_katz,
linkpred.py:165-207) on the planted-partition graph (SBM n=10^6, 1,000
power-law communities, mean degree 20, 10% of edges held out), beta =
0.5/lambda_max, s = 100, T = 101, tol 1e-10 (the linkpred default).

The device answers a 64-query batch (deduplicated anchor solves, K7 gather
and Pearson rerank); 4 of its queries are recomputed by the oracle's
restatement of sparse_katz over the CSR cg (the anchor solves run on all
host threads) and must give the same candidate set, correlations within
1e-9 and the same order apart from correlation ties within 1e-9."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

S = 100
NQ = 64
NCHECK = 4


@pytest.fixture(scope="module")
def cfg5():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_06525_b200 as kz
    from paper_1912_06525_b200 import generators as G

    g, pos = G.sbm_split(n=1_000_000, seed=0)
    lam = kz.spectral_norm(g)
    idx = kz.GraphIndex(g, 0.5 / lam, spectral_norm=lam)
    qs = G.sample_queries(np.unique(pos.ravel()), NQ, seed=0)  # tools/bench_cfg5.py query rule
    return kz, g, idx, qs


def test_cfg5_sparse_katz_matches_oracle(cfg5):
    kz, g, idx, qs = cfg5
    preds = kz.sparse_katz_batch(idx, qs, S)
    assert len(preds) == NQ
    beta = idx.alpha
    a = O.csr_matrix(g.row_offsets, g.col_indices, g.n)
    n = g.n
    T = S + 1
    picks = np.linspace(0, NQ - 1, NCHECK).astype(int)
    qint = [g.internal_id(int(qs[j])) for j in picks]

    def solve(i):
        return O.query_cg_csr(a, beta, int(i), tol=1e-10)[0]

    with ThreadPoolExecutor(max_workers=16) as ex:
        base = dict(zip(qint, ex.map(solve, qint)))
        # the anchors of linkpred.py:186-188: top-T of all nodes except q
        anchors = set()
        for q in qint:
            order = np.lexsort((np.arange(n), -base[q]))
            anchors.update(int(x) for x in order[: T + 1] if x != q)
        todo = sorted(anchors - set(base))
        base.update(zip(todo, ex.map(solve, todo)))

    def nbrs(i):
        return a.indices[a.indptr[i] : a.indptr[i + 1]]

    for j, q in zip(picks, qint):
        want = O.sparse_katz(lambda i: base[int(i)], nbrs, g.original_ids, q, S)
        got = preds[j].candidates
        assert preds[j].query == int(qs[j])
        wc = dict(want)
        assert sorted(c for c, _ in got) == sorted(c for c, _ in want)
        for (c, r), (w, _) in zip(got, want):
            assert abs(r - wc[c]) <= 1e-9
            if c != w:
                assert abs(wc[c] - wc[w]) < 1e-9
