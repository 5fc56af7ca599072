"""Index build against the reference's own builds.

The golden KLRC files were written by the reference's build_index
(tests/golden/make_golden.py, make_recall_golden.py); each test rebuilds the
same graph with the same parameters and compares:

* CPU: partition (perm, part boundaries, n1/n2, overflow flag), M12, the
  per-part min-degree orders and Cholesky factors -- byte-exact (the native
  partitioner and the host part factorisation restate the reference's);
* GPU: the dense separator factor L (cuSOLVER; rel 1e-12), the Lanczos
  correction values (abs 1e-10) and spanned subspace, and LRC query scores
  computed through the rebuilt index against the reference's recorded
  scores (rel L2 1e-10, iterations +/-1); a save/load round trip; and
  determinism of the device build.
"""

import io
import os

import numpy as np
import pytest

from conftest import GOLDEN

# (name, requested ell, max_part_size, seed) as in make_golden.py:36-50 and
# make_recall_golden.py:35
CASES = [
    ("k2", 25, None, 7),
    ("p4", 25, None, 7),
    ("p5split", 25, 2, 7),
    ("star5", 25, None, 7),
    ("triangle", 25, None, 7),
    ("er40", 4, 8, 7),
    ("er60", 6, 8, 7),
    ("ba300", 16, 24, 7),
    ("ba1200", 25, None, 7),
    ("recall", 8, 60, 0),
]
NAMES = [c[0] for c in CASES]
PARAMS = {c[0]: c[1:] for c in CASES}


@pytest.fixture(scope="module")
def kz():
    import paper_1912_06525_b200 as kz

    if kz._lib.load(require=False) is None:
        pytest.skip("libkatzb200.so not built")
    return kz


def ref_index(kz, name):
    return kz.load_index(os.path.join(GOLDEN, f"{name}.klrc"))


def graph_of(kz, idx):
    off, col = idx.adjacency_internal()
    return kz.Graph(n=idx.n, row_offsets=off, col_indices=col.astype(np.int64), original_ids=idx.id_map.copy())


def cfg_of(kz, name):
    mps = PARAMS[name][1]
    return kz.PartitionConfig(max_part_size=mps) if mps is not None else None


@pytest.mark.parametrize("name", NAMES)
def test_partition_matches_reference_build(kz, name):
    ref = ref_index(kz, name)
    g = graph_of(kz, ref)
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bp = kz.partition_vertex_separator(g, cfg_of(kz, name))
    assert bp.n1 == ref.n1 and bp.n2 == ref.n2
    assert np.array_equal(bp.perm, ref.bp.perm)
    assert np.array_equal(bp.part_boundaries, ref.bp.part_boundaries)
    assert bp.separator_overflow == ref.bp.separator_overflow


@pytest.mark.parametrize("name", NAMES)
def test_part_factors_match_reference_bytes(kz, name):
    from paper_1912_06525_b200 import build as B

    ref = ref_index(kz, name)
    g = graph_of(kz, ref)
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bp = kz.partition_vertex_separator(g, cfg_of(kz, name))
    off, col = B._permuted_adjacency(g, bp)
    bc = B.block_cholesky(off, col, ref.alpha, bp.part_boundaries)
    assert bc.num_blocks == ref.bc.num_blocks
    for b in range(bc.num_blocks):
        assert np.array_equal(bc.orders[b], ref.bc.orders[b]), b
        f, r = bc.factors[b], ref.bc.factors[b]
        assert np.array_equal(f.indptr, r.indptr) and np.array_equal(f.indices, r.indices), b
        assert f.data.tobytes() == r.data.tobytes(), b
    o12, c12 = B._sub_pattern(off, col, 0, bp.n1, bp.n1, bp.n)
    assert np.array_equal(o12, ref.m12.indptr) and np.array_equal(c12, ref.m12.indices)
    assert np.all(ref.m12.data == -ref.alpha)


def test_partition_rejects_disconnected_graph(kz):
    g = kz.from_edges([(0, 1), (2, 3)])
    with pytest.raises(kz.DisconnectedGraphError):
        kz.partition_vertex_separator(g)


def test_partition_config_validation(kz):
    with pytest.raises(ValueError):
        kz.PartitionConfig(max_part_size=0).resolved_part_size(10)
    assert kz.PartitionConfig().resolved_part_size(100000) == 390
    assert kz.PartitionConfig().resolved_part_size(1000) == 64


# --------------------------------------------------------------------------- GPU
_built = {}


def built(kz, name):
    if name not in _built:
        import warnings

        ref = ref_index(kz, name)
        ell, _, seed = PARAMS[name]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            idx = kz.build_index(graph_of(kz, ref), alpha=ref.alpha, ell=ell, cfg=cfg_of(kz, name), seed=seed,
                                 spectral_norm=ref.spectral_norm)
        _built[name] = (ref, idx)
    return _built[name]


@pytest.fixture(scope="module")
def gpu(kz):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return kz


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_build_factors(gpu, name):
    ref, idx = built(gpu, name)
    assert idx.n2 == ref.n2 and idx.lr.ell == ref.lr.ell
    if ref.n2:
        lf, lr_ = idx.dc.factor, ref.dc.factor
        assert np.linalg.norm(lf - lr_) <= 1e-12 * np.linalg.norm(lr_)
        assert np.allclose(idx.lr.values, ref.lr.values, rtol=0, atol=1e-10)
    if ref.lr.ell:
        # same invariant subspace: singular values of U_ref' U are all ~1
        s = np.linalg.svd(ref.lr.vectors.T @ idx.lr.vectors, compute_uv=False)
        assert np.all(s > 1 - 1e-8), s.min()


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in NAMES if n != "recall"])
@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_queries_through_device_built_index(gpu, name, tol):
    ref, idx = built(gpu, name)
    rec = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    key = f"lrc_{tol:.0e}"
    scores, reps = gpu.query_batch(idx, rec["queries"], tol=tol)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec[f"{key}_iters"][j]) <= 1, (j, reps[j])
        want = rec[f"{key}_scores"][j]
        nb = np.linalg.norm(want)
        assert np.linalg.norm(scores[j] - want) <= 1e-10 * (nb if nb else 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["er60", "ba300"])
def test_device_build_roundtrip_and_determinism(gpu, name):
    from oracle import katz_oracle as O

    ref, idx = built(gpu, name)
    a, b = io.BytesIO(), io.BytesIO()
    gpu.save_index(idx, a)
    again = gpu.load_index(io.BytesIO(a.getvalue()))
    assert np.array_equal(again.bp.perm, idx.bp.perm)
    assert np.array_equal(again.dc.factor, idx.dc.factor)
    assert np.array_equal(again.lr.vectors, idx.lr.vectors)
    # the oracle's independent KLRC reader accepts the file
    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"kz_build_{name}.klrc")
    with open(path, "wb") as fh:
        fh.write(a.getvalue())
    O.read_klrc(path)
    ell, _, seed = PARAMS[name]
    idx2 = gpu.build_index(graph_of(gpu, ref), alpha=ref.alpha, ell=ell, cfg=cfg_of(gpu, name), seed=seed,
                           spectral_norm=ref.spectral_norm)
    gpu.save_index(idx2, b)
    assert a.getvalue() == b.getvalue()


@pytest.mark.gpu
def test_cfg1_device_built_index_matches_reference_queries(gpu):
    """BASELINE config 1 built on the device (no reference index needed)
    and queried: LRC scores/iterations against the reference's own build
    and query (tests/golden/cfg1_ref.npz, make_cfg1.py)."""
    from paper_1912_06525_b200.generators import chung_lu_graph

    rec = np.load(os.path.join(GOLDEN, "cfg1_ref.npz"))
    g = chung_lu_graph()
    idx = gpu.build_index(g, alpha=float(rec["alpha"]), ell=32, seed=0, spectral_norm=float(rec["spectral_norm"]))
    assert idx.n2 == int(rec["n2"])
    scores, reps = gpu.query_batch(idx, rec["queries"], tol=1e-8)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec["lrc_iters"][j]) <= 1
        want = rec["lrc_scores"][j]
        assert np.linalg.norm(scores[j] - want) <= 1e-10 * np.linalg.norm(want)


# ---- R-MAT scale-16 proxy: the largest R-MAT the reference can build ----
PROXY = os.path.join(GOLDEN, "proxy16_ref.npz")


@pytest.fixture(scope="module")
def proxy(kz):
    if not os.path.exists(PROXY):
        pytest.skip("proxy16_ref.npz absent (tests/golden/make_proxy16.py)")
    from paper_1912_06525_b200.generators import config_graph

    return config_graph("proxy16"), np.load(PROXY)


def test_proxy16_partition_matches_reference(kz, proxy):
    g, rec = proxy
    assert g.n == int(rec["n"]) and g.nnz == int(rec["nnz"])
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bp = kz.partition_vertex_separator(g)
    assert bp.n1 == int(rec["n1"]) and bp.n2 == int(rec["n2"])
    assert np.array_equal(bp.perm, rec["perm"])
    assert np.array_equal(bp.part_boundaries, rec["part_boundaries"])


@pytest.mark.gpu
def test_proxy16_device_build_and_lrc_queries_match_reference(gpu, proxy):
    """LRC at the R-MAT 16 proxy (SURVEY §8c pins cfg2/cfg4's LRC parts
    here): the device build answers the reference's queries within the
    parity bar of the reference's own build."""
    g, rec = proxy
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        idx = gpu.build_index(g, alpha=float(rec["alpha"]), ell=64, seed=0, spectral_norm=float(rec["spectral_norm"]))
    assert idx.n2 == int(rec["n2"])
    assert np.allclose(idx.lr.values, rec["sigma"], rtol=0, atol=1e-9)
    scores, reps = gpu.query_batch(idx, rec["queries"], tol=1e-8)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec["lrc_iters"][j]) <= 1
        want = rec["lrc_scores"][j]
        assert np.linalg.norm(scores[j] - want) <= 1e-10 * np.linalg.norm(want)


# ---- the reference's partition/factor helpers under their own names ----
@pytest.mark.parametrize("name", ["er60", "ba300", "recall"])
def test_build_blocks_check_partition_block_cholesky(kz, name):
    """build_blocks / check_partition / block_cholesky (partition.py:250-297,
    factor.py:127-152) reproduce the reference's M12 and part factors."""
    ref = ref_index(kz, name)
    g = graph_of(kz, ref)
    m11, m12, m22 = kz.build_blocks(g, ref.alpha, ref.bp)
    assert np.array_equal(m12.indptr, ref.m12.indptr) and np.array_equal(m12.indices, ref.m12.indices)
    assert m12.data.tobytes() == ref.m12.data.tobytes()
    assert m11.shape == (ref.n1, ref.n1) and m22.shape == (ref.n2, ref.n2)
    assert np.allclose(m22.diagonal(), 1.0)
    assert kz.check_partition(g, ref.bp)
    bad = kz.BlockPartition(perm=ref.bp.perm[::-1].copy(), inv_perm=np.argsort(ref.bp.perm[::-1]),
                            part_boundaries=ref.bp.part_boundaries, n1=ref.n1, n2=ref.n2)
    assert not kz.check_partition(g, bad)
    bc = kz.block_cholesky(m11, ref.bp.part_boundaries)
    for b in range(bc.num_blocks):
        assert np.array_equal(bc.orders[b], ref.bc.orders[b])
        assert bc.factors[b].data.tobytes() == ref.bc.factors[b].data.tobytes()
    with pytest.raises(kz.InadmissibleAlphaError):
        kz.build_blocks(g, -0.1, ref.bp)


def test_block_cholesky_names_the_failing_part(kz):
    import scipy.sparse as sp

    m11 = sp.csr_matrix(np.array([[1.0, 0, 0], [0, 1.0, 2.0], [0, 2.0, 1.0]]))
    with pytest.raises(kz.FactorizationError, match="part 1"):
        kz.block_cholesky(m11, [0, 1, 3])


def test_load_edge_list_rules(kz):
    g = kz.load_edge_list(b"# comment\n10 20\n20,30\n\n30 10\n10 10\n20 10\n")
    assert g.n == 3 and list(g.original_ids) == [10, 20, 30] and g.num_edges == 3
    for bad, line in ((b"1 2 3\n", 1), (b"1 2\nx 3\n", 2), (b"1 -2\n", 1)):
        with pytest.raises(kz.GraphParseError) as err:
            kz.load_edge_list(bad)
        assert err.value.line_no == line
    with pytest.raises(kz.GraphParseError):
        kz.load_edge_list(b"5 5\n")
    g2 = kz.load_edge_list(io.BytesIO(b"1\t2\n2 3\n"), fmt="whitespace")
    assert g2.num_edges == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["er60", "ba300"])
def test_device_factor_helpers_match_oracle(gpu, name):
    from oracle import katz_oracle as O

    ref = ref_index(gpu, name)
    ix = O.read_klrc(os.path.join(GOLDEN, f"{name}.klrc"))
    g = graph_of(gpu, ref)
    m11, m12, m22 = gpu.build_blocks(g, ref.alpha, ref.bp)
    dc = gpu.dense_cholesky(m22)
    assert np.linalg.norm(dc.factor - ref.dc.factor) <= 1e-12 * np.linalg.norm(ref.dc.factor)
    rng = np.random.default_rng(1)
    r = rng.standard_normal(ref.n2)
    want = O.apply_approx_schur_inverse(ix, r)
    got = gpu.apply_approx_schur_inverse(ref.dc, ref.lr, r)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    # R v against the dense restatement of factor.py:196-202
    v = rng.standard_normal(ref.n2)
    li = np.linalg.inv(ref.dc.factor)
    dense_m11 = m11.toarray()
    rv = li @ (m12.T @ np.linalg.solve(dense_m11, m12 @ (li.T @ v)))
    got = gpu.apply_correction(ref.dc, ref.m12, ref.bc, v)
    assert np.linalg.norm(got - rv) <= 1e-11 * max(1.0, np.linalg.norm(rv))


# ---- BASELINE config 4: the beta x ell sweep on the R-MAT 16 proxy ----
CFG4 = os.path.join(GOLDEN, "cfg4_ref.npz")
CFG4_COMBOS = [(bf, ell) for bf in (0.1, 0.5, 0.9, 0.99) for ell in (32, 128)]


@pytest.fixture(scope="module")
def cfg4():
    from oracle import katz_oracle as O

    off, col, ids = O.config_csr("proxy16")
    return O, O.csr_matrix(off, col, len(ids)), ids, np.load(CFG4)


def _cfg4_ref_scores(O, a, ids, rec, k, method):
    """The reference's scores: the oracle's tol=1e-14 solve + the stored
    float32 deviation (tests/golden/make_cfg4.py)."""
    dev = rec[f"{k}_{method}_dev"].astype(np.float64)
    qi = np.searchsorted(ids, rec[f"{k}_queries"][: dev.shape[0]])
    ex = np.array([O.query_cg_csr(a, float(rec[f"{k}_alpha"]), int(q), tol=1e-14)[0] for q in qi])
    return ex + dev


@pytest.mark.parametrize("bf,ell", CFG4_COMBOS)
def test_cfg4_oracle_cg_matches_reference(cfg4, bf, ell):
    """The oracle's CSR restatement of query_cg_baseline reproduces the
    reference's iterations and scores at every beta of the sweep (the pin of
    the oracle at cfg4)."""
    O, a, ids, rec = cfg4
    k = f"b{bf:g}_l{ell}"
    alpha = float(rec[f"{k}_alpha"])
    want = _cfg4_ref_scores(O, a, ids, rec, k, "cg")
    qi = np.searchsorted(ids, rec[f"{k}_queries"])
    for j, q in enumerate(qi):
        x, rep = O.query_cg_csr(a, alpha, int(q), tol=1e-8)
        assert rep.iterations == int(rec[f"{k}_cg_iters"][j])
        assert rep.converged == bool(rec[f"{k}_cg_conv"][j])
        if j < want.shape[0]:
            assert np.linalg.norm(x - want[j]) <= 1e-12 * np.linalg.norm(want[j])


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("bf,ell", CFG4_COMBOS)
def test_cfg4_device_build_lrc_and_cg_match_reference(gpu, cfg4, bf, ell):
    """BASELINE config 4 on the proxy (SURVEY §8(c) pin for the cfg2/cfg4 LRC
    side): the device build at beta*lambda in {0.1, 0.5, 0.9, 0.99} and
    ell in {32, 128} reproduces the reference build's correction
    eigenvalues, and its LRC (query) and plain-CG (query_cg_baseline)
    answers match the reference's: iterations +/-1 on 4 queries, rel L2
    <= 1e-10 on the stored score columns."""
    import warnings

    from paper_1912_06525_b200.generators import config_graph

    O, a, ids, rec = cfg4
    k = f"b{bf:g}_l{ell}"
    g = config_graph("proxy16")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        idx = gpu.build_index(g, alpha=float(rec[f"{k}_alpha"]), ell=ell, seed=0,
                              spectral_norm=float(rec[f"{k}_spectral_norm"]))
    assert idx.n2 == int(rec[f"{k}_n2"])
    assert np.allclose(idx.lr.values, rec[f"{k}_sigma"], rtol=0, atol=1e-9)
    qs = rec[f"{k}_queries"]
    for method, fn in (("lrc", gpu.query_batch), ("cg", gpu.query_cg_baseline_batch)):
        scores, reps = fn(idx, qs, tol=1e-8)
        for j in range(len(qs)):
            assert abs(reps[j].iterations - int(rec[f"{k}_{method}_iters"][j])) <= 1
            assert reps[j].converged == bool(rec[f"{k}_{method}_conv"][j])
        want = _cfg4_ref_scores(O, a, ids, rec, k, method)
        for j in range(want.shape[0]):
            assert np.linalg.norm(scores[j] - want[j]) <= 1e-10 * np.linalg.norm(want[j]), (method, j)
    del idx
