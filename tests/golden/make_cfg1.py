"""Reference outputs at BASELINE config 1 (Chung-Lu n=10^4, beta=0.5/lambda,
ell=32, 16 seeded queries, tol 1e-8), produced by the reference itself.

Run in the build container:  python tests/golden/make_cfg1.py
Writes tests/golden/large/cfg1.klrc (the reference's own index, ~200 MB,
git-ignored; it travels to the GPU box with the working tree) and the
committed tests/golden/cfg1_ref.npz (scores/iterations/residuals of the
reference's query, query_cg_baseline, katz_rank and sparse_katz).
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))

import lrckatz  # noqa: E402

from paper_1912_06525_b200.generators import chung_lu_graph, sample_queries  # noqa: E402


def main():
    g = chung_lu_graph()  # n=9,924, nnz=97,754 after the LCC
    rg = lrckatz.Graph(n=g.n, row_offsets=g.row_offsets, col_indices=g.col_indices, original_ids=g.original_ids)
    lam = lrckatz.spectral_norm(rg)
    t0 = time.time()
    idx = lrckatz.build_index(rg, alpha=0.5 / lam, ell=32, seed=0)
    print("build", time.time() - t0, "n1", idx.n1, "n2", idx.n2, flush=True)
    os.makedirs(os.path.join(OUT, "large"), exist_ok=True)
    lrckatz.save_index(idx, os.path.join(OUT, "large", "cfg1.klrc"))
    qs = sample_queries(idx.id_map, 16, seed=0)
    rec = {"queries": qs, "spectral_norm": lam, "alpha": idx.alpha, "n2": idx.n2}
    for method, fn in (("lrc", lrckatz.query), ("cg", lrckatz.query_cg_baseline)):
        S, it, res, conv = [], [], [], []
        t0 = time.time()
        for q in qs:
            kv, rep = fn(idx, int(q), tol=1e-8)
            S.append(kv.scores)
            it.append(rep.iterations)
            res.append(rep.final_residual_norm)
            conv.append(rep.converged)
        print(method, "q/s", len(qs) / (time.time() - t0), it, flush=True)
        rec[f"{method}_scores"] = np.array(S)
        rec[f"{method}_iters"] = np.array(it)
        rec[f"{method}_resid"] = np.array(res)
        rec[f"{method}_conv"] = np.array(conv)
    kr = [lrckatz.katz_rank(idx, int(q), 20) for q in qs[:4]]
    rec["kr_ids"] = np.array([[c for c, _ in p.candidates] for p in kr])
    rec["kr_scores"] = np.array([[v for _, v in p.candidates] for p in kr])
    t0 = time.time()
    sk = [lrckatz.sparse_katz(idx, int(q), 20) for q in qs[:1]]
    print("sparse_katz s/query", time.time() - t0, flush=True)
    rec["sk_ids"] = np.array([[c for c, _ in p.candidates] for p in sk])
    rec["sk_corr"] = np.array([[v for _, v in p.candidates] for p in sk])
    np.savez_compressed(os.path.join(OUT, "cfg1_ref.npz"), **rec)


if __name__ == "__main__":
    main()
