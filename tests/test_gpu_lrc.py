"""GPU parity of the LRC-Katz path (Schur PCG), katz_rank and sparse_katz
against golden vectors recorded from the reference (tests/golden) and the
oracle.  Bar: scores within relative L2 1e-10 per query column, PCG
iterations within +/-1, identical top-k apart from numerically tied keys."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-10
NAMES = ["k2", "p4", "p5split", "star5", "triangle", "er40", "er60", "ba300", "ba1200"]


@pytest.fixture(scope="module")
def kz():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_06525_b200 as kz

    return kz


_cache = {}


def case(kz, name):
    if name not in _cache:
        _cache[name] = (kz.load_index(os.path.join(GOLDEN, f"{name}.klrc")),
                        np.load(os.path.join(GOLDEN, f"{name}.npz")),
                        O.read_klrc(os.path.join(GOLDEN, f"{name}.klrc")))
    return _cache[name]


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_lrc_query_batch_matches_reference(kz, name, tol):
    idx, rec, _ = case(kz, name)
    key = f"lrc_{tol:.0e}"
    scores, reps = kz.query_batch(idx, rec["queries"], tol=tol)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec[f"{key}_iters"][j]) <= 1, (j, reps[j])
        assert rel(scores[j], rec[f"{key}_scores"][j]) <= REL_TOL
        assert reps[j].converged == bool(rec[f"{key}_conv"][j])
        # whole-system residual, as the reference reports it (solver.py:180)
        assert reps[j].final_residual_norm == pytest.approx(rec[f"{key}_resid"][j], rel=1e-3, abs=1e-15)


@pytest.mark.parametrize("name", NAMES)
def test_lrc_single_query_api(kz, name):
    idx, rec, _ = case(kz, name)
    q = int(rec["queries"][0])
    kv, rep = kz.query(idx, q, tol=1e-8)
    assert kv.query == q and kv.alpha == idx.alpha and kv.scores.shape == (idx.n,)
    assert kv.scores.min() >= 0.0
    assert rel(kv.scores, rec["lrc_1e-08_scores"][0]) <= REL_TOL
    assert rep.converged and rep.wall_time > 0.0


@pytest.mark.parametrize("name", ["er40", "er60", "ba300", "ba1200"])
def test_lrc_seeded_start_and_budget(kz, name):
    idx, rec, _ = case(kz, name)
    q0 = int(rec["queries"][0])
    kv, rep = kz.query(idx, q0, tol=1e-10, start_seed=5)
    assert abs(rep.iterations - int(rec["lrc_seed5_iters"])) <= 1
    assert rel(kv.scores, rec["lrc_seed5_scores"]) <= REL_TOL
    kv, rep = kz.query(idx, q0, tol=1e-12, max_iter=1)
    assert rep.iterations == int(rec["lrc_budget1_iters"])
    assert rep.converged == bool(rec["lrc_budget1_conv"])
    assert rel(kv.scores, rec["lrc_budget1_scores"]) <= 1e-9
    assert np.all(np.isfinite(kv.scores))


@pytest.mark.parametrize("name", ["er40", "ba300", "ba1200"])
def test_schur_operators_match_oracle(kz, name):
    idx, _, ix = case(kz, name)
    rng = np.random.default_rng(0)
    for _ in range(3):
        v = rng.standard_normal(idx.n2)
        assert np.abs(kz.apply_schur(idx, v) - O.apply_schur(ix, v)).max() < 1e-12
        r = rng.standard_normal(idx.n2)
        want = O.apply_approx_schur_inverse(ix, r)
        assert np.abs(idx.lrc().apply_precond(r) - want).max() < 1e-11 * max(1, np.abs(want).max())
        g1, g2 = rng.standard_normal(idx.n1), rng.standard_normal(idx.n2)
        assert np.abs(kz.schur_rhs(idx, g1, g2) - O.schur_rhs(ix, g1, g2)).max() < 1e-12
    with pytest.raises(ValueError):
        kz.schur_rhs(idx, np.zeros(idx.n1 + 1), np.zeros(idx.n2))


@pytest.mark.parametrize("name", ["er40", "er60", "ba300", "ba1200"])
def test_lrc_pcg_matches_oracle(kz, name):
    idx, _, ix = case(kz, name)
    f = np.random.default_rng(4).standard_normal(idx.n2)
    for tol in (1e-8, 1e-12):
        x, rep = kz.lrc_pcg(idx, f, tol=tol)
        xo, repo = O.lrc_pcg(ix, f, tol=tol)
        assert abs(rep.iterations - repo.iterations) <= 1
        assert rep.converged == repo.converged
        assert rel(x, xo) <= REL_TOL
    x, rep = kz.lrc_pcg(idx, np.zeros(idx.n2))
    assert rep.iterations == 0 and rep.converged and np.all(x == 0.0)


def test_lrc_pcg_is_direct_with_rank_covering_spectrum(kz):
    # p5split: n2 = 1 and ell = n2: the preconditioner is the exact inverse
    idx, _, ix = case(kz, "p5split")
    x, rep = kz.lrc_pcg(idx, np.array([0.7]), tol=1e-12)
    assert rep.iterations == 1 and rep.converged


@pytest.mark.parametrize("name", NAMES)
def test_katz_rank_matches_reference(kz, name):
    idx, rec, _ = case(kz, name)
    s = int(rec["s"])
    qs = rec["queries"][:3]
    preds = kz.katz_rank_batch(idx, qs, s)
    for j, p in enumerate(preds):
        want = [c for c in rec["kr_ids"][j] if c >= 0]
        got = [c for c, _ in p.candidates]
        assert got == want, (name, j)
        assert p.method == "katz"
        assert np.allclose([v for _, v in p.candidates], rec["kr_scores"][j][: len(got)], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("name", [n for n in NAMES if n not in ("k2", "p4", "triangle")])
def test_sparse_katz_matches_reference(kz, name):
    idx, rec, _ = case(kz, name)
    if "sk_ids" not in rec.files:
        pytest.skip("no sparse_katz golden for this case")
    s = int(rec["s"])
    qs = rec["queries"][:3]
    preds = kz.sparse_katz_batch(idx, qs, s)
    for j, p in enumerate(preds):
        want = [c for c in rec["sk_ids"][j] if c >= 0]
        wcorr = dict(zip(want, rec["sk_corr"][j]))
        got = [c for c, _ in p.candidates]
        assert sorted(got) == sorted(want)
        for pos, (c, r) in enumerate(p.candidates):
            assert r == pytest.approx(wcorr[c], abs=1e-9)
            if c != want[pos]:  # only swaps of numerically tied keys
                assert abs(wcorr[c] - wcorr[want[pos]]) < 1e-9


def test_linkpred_known_answers(kz):
    idx, _, _ = case(kz, "p4")
    pred = kz.katz_rank(idx, 0, 5, tol=1e-12)
    assert [c for c, _ in pred.candidates] == [2, 3]
    with pytest.raises(ValueError):
        kz.katz_rank(idx, 0, 0)
    with pytest.raises(ValueError):
        kz.sparse_katz(idx, 0, 2, T=4)  # only 3 other nodes exist
    assert len(kz.sparse_katz(idx, 0, 2, T=3, tol=1e-12).candidates) == 2
    idx, _, _ = case(kz, "star5")
    pred = kz.katz_rank(idx, 1, 5, tol=1e-12)
    assert [c for c, _ in pred.candidates] == [2, 3, 4]
    idx, _, _ = case(kz, "k2")
    kv, rep = kz.query(idx, 0, tol=1e-12)
    assert kv.scores == pytest.approx([1 / 3, 2 / 3], abs=1e-10)


def test_spectrum_error(kz):
    import copy

    idx, _, _ = case(kz, "er40")
    bad = copy.copy(idx)
    bad.__dict__.pop("_dev", None)
    lr = copy.copy(idx.lr)
    lr.values = lr.values.copy()
    lr.values[0] = 1.0
    bad.lr = lr
    with pytest.raises(kz.SpectrumError):
        kz.query(bad, int(idx.id_map[0]))


def test_spectrum_error_only_where_the_preconditioner_is_applied(kz):
    """SpectrumError comes from apply_approx_schur_inverse (factor.py:329-330),
    so query / lrc_pcg raise it, while apply_schur and schur_rhs -- which
    never read sigma (solver.py:104-115) -- still answer."""
    import copy

    idx, _, ix = case(kz, "er40")
    bad = copy.copy(idx)
    bad.__dict__.pop("_dev", None)
    lr = copy.copy(idx.lr)
    lr.values = lr.values.copy()
    lr.values[0] = 1.0
    bad.lr = lr
    rng = np.random.default_rng(2)
    v = rng.standard_normal(idx.n2)
    assert rel(kz.apply_schur(bad, v), O.apply_schur(ix, v)) <= 1e-12
    g1, g2 = rng.standard_normal(idx.n1), rng.standard_normal(idx.n2)
    assert rel(kz.schur_rhs(bad, g1, g2), O.schur_rhs(ix, g1, g2)) <= 1e-12
    with pytest.raises(kz.SpectrumError):
        kz.lrc_pcg(bad, v)
    with pytest.raises(kz.SpectrumError):
        kz.query(bad, int(idx.id_map[0]))


@pytest.mark.parametrize("name", ["k2", "p4", "star5"])
def test_lrc_pcg_on_an_empty_separator(kz, name):
    """n2 == 0: the reference's lrc_pcg returns an empty x with a converged,
    0-iteration report (solver.py:127-158 on an empty system); apply_schur
    of an empty vector is empty."""
    idx, _, _ = case(kz, name)
    assert idx.n2 == 0
    x, rep = kz.lrc_pcg(idx, np.zeros(0))
    assert x.shape == (0,)
    assert rep.iterations == 0 and rep.converged and rep.final_residual_norm == 0.0
    assert kz.apply_schur(idx, np.zeros(0)).shape == (0,)
    assert kz.schur_rhs(idx, np.zeros(idx.n1), np.zeros(0)).shape == (0,)
