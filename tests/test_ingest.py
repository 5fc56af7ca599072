"""Graph ingestion against the reference's own outputs (tests/golden/ingest.npz,
made by tests/golden/make_ingest_golden.py from lrckatz.from_edges /
largest_connected_component / spectral_norm): the numpy restatement on CPU,
the device path (kz_edges_to_csr radix sort/unique + kz_connected_components)
on the GPU."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1912_06525_b200 as kz

REC = np.load(os.path.join(GOLDEN, "ingest.npz"))
CASES = sorted({int(k[len("edges"):]) for k in REC.files if k.startswith("edges")})


@pytest.mark.parametrize("i", CASES)
def test_host_ingestion_matches_reference(i):
    e, n = REC[f"edges{i}"], int(REC[f"n{i}"])
    g = kz.from_edges(e, n=n)
    assert np.array_equal(g.row_offsets, REC[f"off{i}"]) and np.array_equal(g.col_indices, REC[f"col{i}"])
    lcc = kz.largest_connected_component(g)
    assert np.array_equal(lcc.row_offsets, REC[f"lcc_off{i}"])
    assert np.array_equal(lcc.col_indices, REC[f"lcc_col{i}"])
    assert np.array_equal(lcc.original_ids, REC[f"lcc_ids{i}"])


@pytest.mark.gpu
@pytest.mark.parametrize("i", CASES)
def test_device_ingestion_matches_reference(i):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_06525_b200.graph import from_edges_device, largest_connected_component_device

    e, n = REC[f"edges{i}"], int(REC[f"n{i}"])
    g, dev = from_edges_device(e[:, 0], e[:, 1], n)
    assert np.array_equal(g.row_offsets, REC[f"off{i}"]) and np.array_equal(g.col_indices, REC[f"col{i}"])
    lcc = largest_connected_component_device(g, dev)
    assert np.array_equal(lcc.row_offsets, REC[f"lcc_off{i}"])
    assert np.array_equal(lcc.col_indices, REC[f"lcc_col{i}"])
    assert np.array_equal(lcc.original_ids, REC[f"lcc_ids{i}"])
    assert kz.spectral_norm(lcc) == pytest.approx(float(REC[f"lam{i}"]), rel=1e-9)


@pytest.mark.gpu
def test_device_rmat_matches_host_rmat():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_06525_b200.generators import rmat_graph, rmat_graph_fast

    a, b = rmat_graph(14, seed=2), rmat_graph_fast(14, seed=2)
    assert a.n == b.n and np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices) and np.array_equal(a.original_ids, b.original_ids)


@pytest.mark.gpu
def test_device_from_edges_edge_cases():
    """Duplicates in both orientations, self-loops only, no edges, isolated
    trailing nodes, out-of-range endpoints (from_edges, graph.py:111-148)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_06525_b200.graph import from_edges_device

    cases = [
        (np.array([[0, 1], [1, 0], [1, 0], [2, 2], [3, 1]]), 6),
        (np.array([[2, 2], [0, 0]]), 3),
        (np.zeros((0, 2), dtype=np.int64), 4),
        (np.array([[0, 4]]), 5),
    ]
    for e, n in cases:
        g, _ = from_edges_device(e[:, 0], e[:, 1], n)
        keep = e[:, 0] != e[:, 1]
        want = kz.from_edges(e, n=n) if keep.any() else None
        if want is None:
            assert g.nnz == 0 and np.array_equal(g.row_offsets, np.zeros(n + 1, dtype=np.int64))
        else:
            assert np.array_equal(g.row_offsets, want.row_offsets)
            assert np.array_equal(g.col_indices, want.col_indices)
    with pytest.raises(ValueError):
        from_edges_device(np.array([0, 5]), np.array([1, 1]), 5)


@pytest.mark.gpu
@pytest.mark.slow
def test_device_ingestion_matches_oracle_at_rmat18():
    """The BASELINE cfg2 graph (R-MAT 18) from device ingestion equals the
    oracle's numpy/scipy restatement of from_edges + the largest component
    byte for byte."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import katz_oracle as O
    from paper_1912_06525_b200.generators import rmat_graph_fast

    g = rmat_graph_fast(18)
    off, col, ids = O.config_csr("cfg2")
    assert np.array_equal(g.row_offsets, off) and np.array_equal(g.col_indices, col)
    assert np.array_equal(g.original_ids, ids)
