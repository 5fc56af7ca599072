"""BASELINE config 1 (Chung-Lu 10^4, beta=0.5/lambda, ell=32, 16 queries) on
the reference's own KLRC index: LRC-Katz and plain CG against the
reference's recorded outputs (tests/golden/cfg1_ref.npz, made by
tests/golden/make_cfg1.py).  The 200 MB index itself is not committed; the
test skips when tests/golden/large/cfg1.klrc is absent."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

KLRC = os.path.join(GOLDEN, "large", "cfg1.klrc")
REF = os.path.join(GOLDEN, "cfg1_ref.npz")


@pytest.fixture(scope="module")
def setup():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (os.path.exists(KLRC) and os.path.exists(REF)):
        pytest.skip("cfg1 reference index not present (run tests/golden/make_cfg1.py)")
    import paper_1912_06525_b200 as kz

    return kz, kz.load_index(KLRC), np.load(REF)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("method", ["lrc", "cg"])
def test_cfg1_batch_matches_reference(setup, method):
    kz, idx, rec = setup
    fn = kz.query_batch if method == "lrc" else kz.query_cg_baseline_batch
    scores, reps = fn(idx, rec["queries"], tol=1e-8)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec[f"{method}_iters"][j]) <= 1
        assert rel(scores[j], rec[f"{method}_scores"][j]) <= 1e-10
        assert reps[j].converged == bool(rec[f"{method}_conv"][j])


def test_cfg1_katz_rank_matches_reference(setup):
    kz, idx, rec = setup
    preds = kz.katz_rank_batch(idx, rec["queries"][:4], 20)
    for j, p in enumerate(preds):
        assert [c for c, _ in p.candidates] == list(rec["kr_ids"][j])
        assert np.allclose([v for _, v in p.candidates], rec["kr_scores"][j], rtol=1e-9)


def test_cfg1_sparse_katz_matches_reference(setup):
    kz, idx, rec = setup
    p = kz.sparse_katz_batch(idx, rec["queries"][:1], 20)[0]
    want = list(rec["sk_ids"][0])
    wcorr = dict(zip(want, rec["sk_corr"][0]))
    got = [c for c, _ in p.candidates]
    assert sorted(got) == sorted(want)
    for pos, (c, r) in enumerate(p.candidates):
        assert r == pytest.approx(wcorr[c], abs=1e-9)
        if c != want[pos]:
            assert abs(wcorr[c] - wcorr[want[pos]]) < 1e-9
