"""Recall harness against the reference's own outputs (tests/golden/recall.*,
made by tests/golden/make_recall_golden.py): temporal_split on CPU; the
batched evaluate_recall / evaluate_recall_sweep on the GPU."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200.evaluate import evaluate_recall, evaluate_recall_sweep, temporal_split

REC = json.load(open(os.path.join(GOLDEN, "recall.json")))


def dataset():
    return temporal_split([tuple(r) for r in REC["rows"]], REC["cutoff"])


def test_temporal_split_matches_reference():
    ds = dataset()
    assert list(ds.train.original_ids) == REC["train_ids"]
    assert list(ds.train.row_offsets) == REC["train_off"]
    assert list(ds.train.col_indices) == REC["train_col"]
    assert [list(p) for p in ds.positives] == REC["positives"]
    assert {k: [list(p) for p in v] for k, v in ds.buckets.items()} == REC["buckets"]
    with pytest.raises(ValueError):
        temporal_split([(0, 1, 5.0)], 1.0)  # cutoff precedes every edge
    with pytest.raises(ValueError):
        temporal_split([], 1.0)


def _same(stat, want):
    mean, std, nq = want
    assert stat.n_queries == nq
    if nq == 0:
        assert np.isnan(stat.mean)
    else:
        assert stat.mean == pytest.approx(mean, abs=1e-12)
        assert stat.std == pytest.approx(std, abs=1e-12)


@pytest.mark.gpu
def test_recall_sweep_matches_reference():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ds = dataset()
    idx = kz.load_index(os.path.join(GOLDEN, "recall.klrc"))
    rows = evaluate_recall_sweep(idx, ["katz", "sparse-katz"], ds, [5, 10, 20], query_sample=REC["sample"])
    assert len(rows) == len(REC["sweep"])
    for (m, lab, s, st), (wm, wl, ws, want) in zip(rows, REC["sweep"]):
        assert (m, lab, s) == (wm, wl, ws)
        _same(st, want)
    for s, want in REC["katz_all"].items():
        got = evaluate_recall(idx, "katz", ds, s=int(s))
        for label, w in want.items():
            _same(got[label], w)
