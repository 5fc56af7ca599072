"""Reference LRC outputs on the R-MAT scale-16 proxy (the
largest R-MAT on which the reference's own build_index is feasible; it pins
the LRC parts of cfg2/cfg4).

Run in the build container (imports /root/reference; ~5 min):
    python tests/golden/make_proxy16.py
Writes tests/golden/proxy16_ref.npz: the graph size, alpha, the reference's
partition (perm, part boundaries), correction eigenvalues, and query /
iteration / residual outputs for 8 seeded queries at tol 1e-8.
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

from paper_1912_06525_b200.generators import config_graph, sample_queries  # noqa: E402


def main():
    g = config_graph("proxy16")
    rg = lrckatz.Graph(n=g.n, row_offsets=g.row_offsets, col_indices=g.col_indices, original_ids=g.original_ids)
    lam = lrckatz.spectral_norm(rg)
    t0 = time.time()
    idx = lrckatz.build_index(rg, alpha=0.5 / lam, ell=64, seed=0)
    print("build", round(time.time() - t0, 1), "n1", idx.n1, "n2", idx.n2, flush=True)
    qs = sample_queries(idx.id_map, 8, seed=0)
    rec = {"n": idx.n, "nnz": g.nnz, "spectral_norm": lam, "alpha": idx.alpha, "n1": idx.n1, "n2": idx.n2,
           "perm": idx.bp.perm.astype(np.int32), "part_boundaries": idx.bp.part_boundaries.astype(np.int32),
           "sigma": idx.lr.values, "queries": qs}
    S, it, res = [], [], []
    t0 = time.time()
    for q in qs:
        kv, rep = lrckatz.query(idx, int(q), tol=1e-8)
        S.append(kv.scores)
        it.append(rep.iterations)
        res.append(rep.final_residual_norm)
    print("lrc s/query", (time.time() - t0) / len(qs), it, flush=True)
    rec["lrc_scores"] = np.array(S)
    rec["lrc_iters"] = np.array(it)
    rec["lrc_resid"] = np.array(res)
    np.savez_compressed(os.path.join(OUT, "proxy16_ref.npz"), **rec)


if __name__ == "__main__":
    main()
