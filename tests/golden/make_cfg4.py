"""Reference LRC outputs for the BASELINE config-4 sweep on the R-MAT scale-16
proxy (the largest R-MAT on which the reference's own
build_index is feasible, the designated LRC pin for cfg2/cfg4).

For every beta in {0.1, 0.5, 0.9, 0.99} x 1/lambda_max and ell in {32, 128}
the reference builds its own index (lrckatz.build_index, seed 0) and answers
4 seeded queries with lrckatz.query (LRC-Katz, solver.py:194-207) and
lrckatz.query_cg_baseline (solver.py:210-232) at tol 1e-8.

Run in the build container (imports /root/reference; the eight builds run in
parallel processes, ~15 min on 8 cores):
    python tests/golden/make_cfg4.py
Writes tests/golden/cfg4_ref.npz with keys  b{beta}_l{ell}_{field}: the
reference's sigma, iterations, residuals and convergence flags for all 4
queries, and its scores for the first NQ_SCORES_LRC (LRC) / NQ_SCORES_CG (CG)
queries stored compactly as float32 deviations from the oracle's tol=1e-14
CSR solve of the same column (dev = ref - exact; exact is recomputed by the
test with the same oracle code, so ref = exact + dev to ~1e-16 relative --
the deviations are ~1e-9 of the scores, float32 keeps 7 digits of them).
"""

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg"
OUT = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(OUT))
BETAS = (0.1, 0.5, 0.9, 0.99)
ELLS = (32, 128)
NQ = 4
NQ_SCORES_LRC = 2
NQ_SCORES_CG = 1


def key(bf, ell):
    return f"b{bf:g}_l{ell}"


def one(args):
    bf, ell = args
    sys.path.insert(0, os.path.join(REF, "src"))
    sys.path.insert(0, ROOT)
    import lrckatz

    from paper_1912_06525_b200.generators import config_graph, sample_queries

    g = config_graph("proxy16")
    rg = lrckatz.Graph(n=g.n, row_offsets=g.row_offsets, col_indices=g.col_indices, original_ids=g.original_ids)
    lam = lrckatz.spectral_norm(rg)
    t0 = time.time()
    idx = lrckatz.build_index(rg, alpha=bf / lam, ell=ell, seed=0)
    tb = time.time() - t0
    qs = sample_queries(idx.id_map, NQ, seed=0)
    k = key(bf, ell)
    rec = {f"{k}_alpha": idx.alpha, f"{k}_spectral_norm": lam, f"{k}_n2": idx.n2, f"{k}_ell": idx.lr.ell,
           f"{k}_sigma": idx.lr.values, f"{k}_queries": qs, f"{k}_build_s": tb}
    for method, fn in (("lrc", lrckatz.query), ("cg", lrckatz.query_cg_baseline)):
        S, it, res, conv = [], [], [], []
        for q in qs:
            kv, rep = fn(idx, int(q), tol=1e-8)
            S.append(kv.scores)
            it.append(rep.iterations)
            res.append(rep.final_residual_norm)
            conv.append(rep.converged)
        rec[f"{k}_{method}_scores"] = np.array(S)
        rec[f"{k}_{method}_iters"] = np.array(it)
        rec[f"{k}_{method}_resid"] = np.array(res)
        rec[f"{k}_{method}_conv"] = np.array(conv)
    print(k, "build", round(tb, 1), "s; lrc it", rec[f"{k}_lrc_iters"], "cg it", rec[f"{k}_cg_iters"], flush=True)
    return rec


def exact_scores(alpha, queries):
    """The oracle's tol=1e-14 CSR solves of the proxy16 columns (the base the
    stored deviations are taken from; tests/test_build.py recomputes them)."""
    sys.path.insert(0, ROOT)
    from oracle import katz_oracle as O

    off, col, ids = O.config_csr("proxy16")
    a = O.csr_matrix(off, col, len(ids))
    qi = np.searchsorted(ids, queries)
    return np.array([O.query_cg_csr(a, alpha, int(q), tol=1e-14)[0] for q in qi])


def compact(rec):
    """Replace the full score arrays by float32 deviations from exact_scores."""
    out = {}
    for bf in BETAS:
        for ell in ELLS:
            k = key(bf, ell)
            ex = exact_scores(float(rec[f"{k}_alpha"]), rec[f"{k}_queries"])
            for method, nq in (("lrc", NQ_SCORES_LRC), ("cg", NQ_SCORES_CG)):
                full = rec[f"{k}_{method}_scores"][:nq]
                out[f"{k}_{method}_dev"] = (full - ex[:nq]).astype(np.float32)
            for f in rec:
                if f.startswith(k + "_") and not f.endswith("_scores"):
                    out[f] = rec[f]
    return out


def main():
    combos = [(bf, ell) for bf in BETAS for ell in ELLS]
    rec = {}
    with ProcessPoolExecutor(max_workers=min(len(combos), os.cpu_count() or 1)) as ex:
        for r in ex.map(one, combos):
            rec.update(r)
    np.savez_compressed(os.path.join(OUT, "cfg4_ref.npz"), **compact(rec))


if __name__ == "__main__":
    main()
