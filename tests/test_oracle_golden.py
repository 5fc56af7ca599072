"""Pin the CPU oracle against golden vectors produced by the reference itself.

tests/golden/*.npz and *.klrc were written by tests/golden/make_golden.py,
which imports /root/reference (lrckatz) and records its outputs.  These
tests run on CPU only and check that the oracle restatement reproduces the
reference bit-for-bit (same numpy/scipy calls in the same order) or to
roundoff where a summation order legitimately differs.
"""

import json
import os

import numpy as np
import pytest

from oracle import katz_oracle as O

from conftest import GOLDEN

META = json.load(open(os.path.join(GOLDEN, "meta.json")))
CASES = [c["name"] for c in META["cases"]]


def load_case(name):
    ix = O.read_klrc(os.path.join(GOLDEN, f"{name}.klrc"))
    rec = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return ix, rec


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_oracle_lrc_query_matches_reference(name, tol):
    ix, rec = load_case(name)
    key = f"lrc_{tol:.0e}"
    for j, q in enumerate(rec["queries"]):
        scores, rep = O.query_lrc(ix, int(q), tol=tol)
        assert rep.iterations == rec[f"{key}_iters"][j]
        assert np.array_equal(scores, rec[f"{key}_scores"][j])
        assert rep.final_residual_norm == rec[f"{key}_resid"][j]
        assert rep.converged == rec[f"{key}_conv"][j]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_oracle_cg_baseline_matches_reference(name, tol):
    ix, rec = load_case(name)
    key = f"cg_{tol:.0e}"
    for j, q in enumerate(rec["queries"]):
        scores, rep = O.query_cg_index(ix, int(q), tol=tol)
        assert rep.iterations == rec[f"{key}_iters"][j]
        assert np.array_equal(scores, rec[f"{key}_scores"][j])
        assert rep.final_residual_norm == rec[f"{key}_resid"][j]


@pytest.mark.parametrize("name", CASES)
def test_oracle_seeded_and_budget(name):
    ix, rec = load_case(name)
    q0 = int(rec["queries"][0])
    for method, fn in (("lrc", O.query_lrc), ("cg", O.query_cg_index)):
        s, rep = fn(ix, q0, tol=1e-10, start_seed=5)
        assert rep.iterations == rec[f"{method}_seed5_iters"]
        assert np.array_equal(s, rec[f"{method}_seed5_scores"])
        s, rep = fn(ix, q0, tol=1e-12, max_iter=1)
        assert rep.iterations == rec[f"{method}_budget1_iters"]
        assert rep.converged == rec[f"{method}_budget1_conv"]
        assert np.array_equal(s, rec[f"{method}_budget1_scores"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_linkpred_matches_reference(name):
    ix, rec = load_case(name)
    a = O.index_adjacency_internal(ix)
    solve = lambda i: O.query_lrc(ix, int(ix.id_map[i]), tol=1e-10)[0]  # noqa: E731
    nbrs = lambda i: a.indices[a.indptr[i] : a.indptr[i + 1]]  # noqa: E731
    s = int(rec["s"])
    for j, q in enumerate(rec["queries"][:3]):
        qi = ix.internal_id(int(q))
        got = O.katz_rank(solve, nbrs, ix.id_map, qi, s)
        ids = [c for c, _ in got] + [-1] * (s - len(got))
        assert ids == list(rec["kr_ids"][j])
        assert np.array_equal(np.array([v for _, v in got] + [0.0] * (s - len(got))), rec["kr_scores"][j])
        if "sk_ids" in rec.files:
            got = O.sparse_katz(solve, nbrs, ix.id_map, qi, s)
            ids = [c for c, _ in got] + [-1] * (s - len(got))
            assert ids == list(rec["sk_ids"][j])
            assert np.array_equal(np.array([v for _, v in got] + [0.0] * (s - len(got))), rec["sk_corr"][j])


def test_oracle_index_adjacency_matches_graph():
    for name in CASES:
        ix, rec = load_case(name)
        a = O.index_adjacency_internal(ix)
        assert np.array_equal(a.indptr, rec["row_offsets"])
        assert np.array_equal(a.indices, rec["col_indices"])


def test_oracle_csr_cg_matches_reference_cg():
    rec = np.load(os.path.join(GOLDEN, "chunglu2000_cg.npz"))
    n = rec["row_offsets"].size - 1
    a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], n)
    for j, q in enumerate(rec["queries"]):
        s, rep = O.query_cg_csr(a, float(rec["beta"]), int(q), tol=1e-8)
        assert rep.iterations == rec["iters"][j]
        assert np.array_equal(s, rec["scores"][j])


def test_known_answers():
    # 2-node graph at alpha=1/2: [1/3, 2/3] (tests/test_solver.py:159-166)
    ix, _ = load_case("k2")
    s, rep = O.query_lrc(ix, 0, tol=1e-12)
    assert np.allclose(s, [1 / 3, 2 / 3], atol=1e-10)
    # P4 katz_rank(q=0) = [2, 3] (tests/test_linkpred.py:36-45)
    rec = np.load(os.path.join(GOLDEN, "p4.npz"))
    assert list(rec["kr_ids"][0][:2]) == [2, 3]
    # star ties broken by id (tests/test_linkpred.py:48-52)
    rec = np.load(os.path.join(GOLDEN, "star5.npz"))
    assert list(rec["kr_ids"][0][:3]) == [2, 3, 4]
    # Pearson closed form (tests/test_linkpred.py:73-74)
    assert O.pearson([1, 2, 3, 4, 5], [2, 1, 4, 3, 7]) == pytest.approx(0.824163383692134, abs=1e-12)
    assert O.pearson([1, 2, 3, 4], [7, 7, 7, 7]) == 0.0
