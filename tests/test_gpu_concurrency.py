"""The reference's concurrency contract: query() is reentrant over a shared,
immutable index; every solver invocation owns its scratch; concurrent
callers need no locking, and the recall sweep is thread-count
invariant (tests/test_linkpred.py:355-365).  Here: several host threads,
each on its own CUDA stream, call the batched solvers on one index at the
same time and must get bit-identical results to a serial run."""

import json
import os
import threading

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kz():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_06525_b200 as kz

    return kz


def _run_threads(fn, nthreads):
    """fn(tid) on nthreads threads, each inside its own torch CUDA stream;
    returns the results in thread order (re-raising the first error)."""
    import torch

    out = [None] * nthreads
    err = []
    start = threading.Barrier(nthreads)

    def body(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                start.wait()
                out[t] = fn(t)
            st.synchronize()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(t,)) for t in range(nthreads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("method", ["lrc", "cg"])
def test_concurrent_queries_on_one_index(kz, method):
    idx = kz.load_index(os.path.join(GOLDEN, "ba1200.klrc"))
    fn = kz.query_batch if method == "lrc" else kz.query_cg_baseline_batch
    rng = np.random.default_rng(5)
    sets = [np.sort(rng.choice(idx.id_map, 24, replace=False)) for _ in range(4)]
    serial = [fn(idx, qs, tol=1e-10) for qs in sets]

    def work(t):
        res = []
        for rep in range(3):
            res.append(fn(idx, sets[(t + rep) % len(sets)], tol=1e-10))
        return res

    got = _run_threads(work, 4)
    for t, res in enumerate(got):
        for rep, (scores, reps) in enumerate(res):
            want_s, want_r = serial[(t + rep) % len(sets)]
            assert np.array_equal(scores, want_s)
            assert [r.iterations for r in reps] == [r.iterations for r in want_r]


def test_concurrent_katz_rank_and_sparse_katz(kz):
    idx = kz.load_index(os.path.join(GOLDEN, "ba300.klrc"))
    qs = idx.id_map[::7][:16]
    want_kr = kz.katz_rank_batch(idx, qs, 10)
    want_sk = kz.sparse_katz_batch(idx, qs[:6], 8)

    def work(t):
        if t % 2 == 0:
            return [p.candidates for p in kz.katz_rank_batch(idx, qs, 10)]
        return [p.candidates for p in kz.sparse_katz_batch(idx, qs[:6], 8)]

    got = _run_threads(work, 6)
    for t, res in enumerate(got):
        want = want_kr if t % 2 == 0 else want_sk
        assert res == [p.candidates for p in want]


def test_concurrent_coldot_and_vec_op_on_distinct_streams(kz):
    """kz_coldot takes caller scratch (no hidden static state): concurrent
    calls on distinct streams each get their own exact dot."""
    import torch

    from paper_1912_06525_b200 import _lib

    lib = _lib.load()
    n = 1 << 20
    xs = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    want = [float(torch.dot(x, x)) for x in xs]

    def work(t):
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        vals = []
        for _ in range(20):
            _lib.coldot(torch, lib, xs[t], xs[t], out, n)
            vals.append(float(out.item()))
        y = torch.empty_like(xs[t])
        _lib.vec_op(torch, lib, 0, n, 2.0, xs[t], -1.0, xs[t], y)  # y = 2x - x = x exactly
        return vals, bool(torch.equal(y, xs[t]))

    got = _run_threads(work, 4)
    for t, (vals, same) in enumerate(got):
        assert same
        assert all(v == vals[0] for v in vals)
        assert vals[0] == pytest.approx(want[t], rel=1e-12)


def test_recall_sweep_is_worker_count_invariant(kz):
    """evaluate_recall_sweep(workers=1) == (workers=4): the reference's
    thread-count invariance, here with small query blocks so the four
    workers really run concurrently on their own streams."""
    from paper_1912_06525_b200.evaluate import evaluate_recall_sweep, temporal_split

    rec = json.load(open(os.path.join(GOLDEN, "recall.json")))
    ds = temporal_split([tuple(r) for r in rec["rows"]], rec["cutoff"])
    idx = kz.load_index(os.path.join(GOLDEN, "recall.klrc"))
    r1 = evaluate_recall_sweep(idx, ["katz", "sparse-katz"], ds, [1, 4, 10], workers=1, batch=4)
    r4 = evaluate_recall_sweep(idx, ["katz", "sparse-katz"], ds, [1, 4, 10], workers=4, batch=4)
    assert len(r1) == len(r4)
    for (m1, l1, s1, st1), (m4, l4, s4, st4) in zip(r1, r4):
        assert (m1, l1, s1) == (m4, l4, s4)
        assert st1.n_queries == st4.n_queries
        assert (st1.mean == st4.mean) or (np.isnan(st1.mean) and np.isnan(st4.mean))
        assert (st1.std == st4.std) or (np.isnan(st1.std) and np.isnan(st4.std))
