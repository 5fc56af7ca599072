"""Randomised concurrency sweep: several host threads, each on its own CUDA
stream, run different random solves (plain CG on private and shared indexes,
katz_rank, sparse_katz, LRC on a shared device-built index) at the same time;
every result must be bit-identical to the same call made serially first.
Sizes are drawn so that the fused small-solve kernel (cooperative launches on
concurrent streams), the graph-replayed loop and the host-driven loop all take
part.  python tools/fuzz_concurrency.py [--rounds 30] [--threads 4] [--seed 0]"""
import argparse
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from oracle import katz_oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=30)
ap.add_argument("--threads", type=int, default=4)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)


def make_graph(n0):
    m = int(n0 * rng.uniform(2.0, 6.0))
    e = rng.integers(0, n0, size=(m, 2))
    hubs = rng.choice(n0, size=max(1, n0 // 2000), replace=False)
    e = np.concatenate([e, np.stack([rng.choice(hubs, size=n0), rng.integers(0, n0, size=n0)], axis=1)])
    return kz.largest_connected_component(kz.from_edges(e))


def canon(x):
    if isinstance(x, (list, tuple)) and x and hasattr(x[0], "candidates"):
        return [p.candidates for p in x]
    if isinstance(x, tuple):
        return np.asarray(x[0]).copy(), [(r.iterations, r.final_residual_norm, r.converged) for r in x[1]]
    return x


def equal(u, v):
    if isinstance(u, tuple):
        return np.array_equal(u[0], v[0]) and u[1] == v[1]
    return u == v


fails = 0
for rnd in range(a.rounds):
    # one shared index (plain CG) + one shared LRC index + a private index per thread
    shared = make_graph(int(rng.choice([3000, 40000, 200000])))
    lam = O.spectral_norm(O.csr_matrix(shared.row_offsets, shared.col_indices, shared.n))
    beta = float(rng.uniform(0.2, 0.9)) / lam
    gi = kz.GraphIndex(shared, beta, spectral_norm=lam)
    small = make_graph(int(rng.choice([400, 2500])))
    lam_s = O.spectral_norm(O.csr_matrix(small.row_offsets, small.col_indices, small.n))
    lidx = kz.build_index(small, alpha=0.5 / lam_s, ell=8, seed=0, spectral_norm=lam_s)
    jobs = []
    for t in range(a.threads):
        kind = int(rng.integers(0, 5))
        b = int(rng.choice([3, 16, 40, 64]))
        tol = float(rng.choice([1e-6, 1e-8, 1e-10]))
        if kind == 0:
            qs = rng.choice(shared.original_ids, size=min(b, shared.n), replace=False)
            jobs.append(("cg shared", lambda qs=qs, tol=tol: kz.query_cg_baseline_batch(gi, qs, tol=tol)))
        elif kind == 1:
            pg = make_graph(int(rng.choice([800, 20000])))
            pl = O.spectral_norm(O.csr_matrix(pg.row_offsets, pg.col_indices, pg.n))
            pi = kz.GraphIndex(pg, 0.6 / pl, spectral_norm=pl)
            qs = rng.choice(pg.original_ids, size=min(b, pg.n), replace=False)
            jobs.append(("cg private", lambda pi=pi, qs=qs, tol=tol: kz.query_cg_baseline_batch(pi, qs, tol=tol)))
        elif kind == 2:
            qs = rng.choice(shared.original_ids, size=min(b, shared.n), replace=False)
            jobs.append(("katz_rank shared", lambda qs=qs: kz.katz_rank_batch(gi, qs, 20)))
        elif kind == 3:
            qs = rng.choice(small.original_ids, size=min(b, small.n), replace=False)
            jobs.append(("lrc shared", lambda qs=qs, tol=tol: kz.query_batch(lidx, qs, tol=tol)))
        else:
            qs = rng.choice(small.original_ids, size=3, replace=False)
            jobs.append(("sparse_katz lrc", lambda qs=qs: kz.sparse_katz_batch(lidx, qs, 6)))
    want = [canon(fn()) for _, fn in jobs]
    torch.cuda.synchronize()
    got = [None] * len(jobs)
    errs = []
    start = threading.Barrier(len(jobs))

    def body(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                start.wait()
                for _ in range(3):
                    got[t] = canon(jobs[t][1]())
            st.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(repr(e)[:300])

    th = [threading.Thread(target=body, args=(t,)) for t in range(len(jobs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    bad = [jobs[t][0] for t in range(len(jobs)) if got[t] is None or not equal(got[t], want[t])]
    if bad or errs:
        fails += 1
    print(json.dumps({"round": rnd, "shared_n": int(shared.n), "jobs": [j[0] for j in jobs], "mismatch": bad,
                      "errors": errs}), flush=True)
print(json.dumps({"rounds": a.rounds, "failures": fails}))
