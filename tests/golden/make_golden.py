"""Generate the golden fixtures from the reference package itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports /root/reference/pkg/src/lrckatz and its test generators
(pkg/tests/synth.py), builds KLRC indexes with the reference's own
build_index/save_index, and records the reference's outputs of query,
query_cg_baseline, katz_rank, sparse_katz, cg and spectral_norm.  The GPU
box never runs this script; it only reads the committed fixtures.
"""

import io
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import lrckatz  # noqa: E402
from lrckatz import PartitionConfig, build_index, from_edges, largest_connected_component  # noqa: E402
from synth import ba_graph, er_graph  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def path(n):
    return from_edges([(i, i + 1) for i in range(n - 1)])


def star(leaves):
    return from_edges([(0, i) for i in range(1, leaves + 1)])


def index_cases():
    rng = np.random.default_rng
    return [
        ("k2", path(2), 25, None, [0, 1]),
        ("p4", path(4), 25, None, [0, 3]),
        ("p5split", path(5), 25, PartitionConfig(max_part_size=2), [0, 2, 4]),
        ("star5", star(4), 25, None, [1, 0]),
        ("triangle", from_edges([(0, 1), (1, 2), (0, 2)]), 25, None, [0, 1]),
        ("er40", largest_connected_component(er_graph(40, 0.1, rng(1))), 4,
         PartitionConfig(max_part_size=8), None),
        ("er60", largest_connected_component(er_graph(60, 0.08, rng(8))), 6,
         PartitionConfig(max_part_size=8), None),
        ("ba300", ba_graph(300, 3, rng(5)), 16, PartitionConfig(max_part_size=24), None),
        ("ba1200", ba_graph(1200, 2, rng(11)), 25, None, None),
    ]


def main():
    meta = {"cases": []}
    for name, g, ell, cfg, qs in index_cases():
        idx = build_index(g, ell=ell, cfg=cfg, seed=7)
        sink = io.BytesIO()
        lrckatz.save_index(idx, sink)
        blob = sink.getvalue()
        with open(os.path.join(OUT, f"{name}.klrc"), "wb") as fh:
            fh.write(blob)
        if qs is None:
            qs = [int(x) for x in np.sort(np.random.default_rng(3).choice(idx.id_map, size=min(6, idx.n), replace=False))]
        rec = {}
        for tol in (1e-8, 1e-10):
            for method, fn in (("lrc", lrckatz.query), ("cg", lrckatz.query_cg_baseline)):
                S, it, res, conv = [], [], [], []
                for q in qs:
                    kv, rep = fn(idx, int(q), tol=tol)
                    S.append(kv.scores)
                    it.append(rep.iterations)
                    res.append(rep.final_residual_norm)
                    conv.append(rep.converged)
                key = f"{method}_{tol:.0e}"
                rec[f"{key}_scores"] = np.array(S)
                rec[f"{key}_iters"] = np.array(it)
                rec[f"{key}_resid"] = np.array(res)
                rec[f"{key}_conv"] = np.array(conv)
        # seeded start and a one-iteration budget
        q0 = int(qs[0])
        for method, fn in (("lrc", lrckatz.query), ("cg", lrckatz.query_cg_baseline)):
            kv, rep = fn(idx, q0, tol=1e-10, start_seed=5)
            rec[f"{method}_seed5_scores"] = kv.scores
            rec[f"{method}_seed5_iters"] = np.array(rep.iterations)
            kv, rep = fn(idx, q0, tol=1e-12, max_iter=1)
            rec[f"{method}_budget1_scores"] = kv.scores
            rec[f"{method}_budget1_iters"] = np.array(rep.iterations)
            rec[f"{method}_budget1_conv"] = np.array(rep.converged)
        # link prediction at the linkpred default tol 1e-10
        s = min(5, max(1, idx.n - 2))
        kr_ids, kr_sc, sk_ids, sk_corr = [], [], [], []
        for q in qs[:3]:
            pred = lrckatz.katz_rank(idx, int(q), s)
            kr_ids.append([c for c, _ in pred.candidates] + [-1] * (s - len(pred.candidates)))
            kr_sc.append([v for _, v in pred.candidates] + [0.0] * (s - len(pred.candidates)))
            if idx.n - 1 >= s + 1:
                pred = lrckatz.sparse_katz(idx, int(q), s)
                sk_ids.append([c for c, _ in pred.candidates] + [-1] * (s - len(pred.candidates)))
                sk_corr.append([v for _, v in pred.candidates] + [0.0] * (s - len(pred.candidates)))
        rec["kr_ids"] = np.array(kr_ids)
        rec["kr_scores"] = np.array(kr_sc)
        if sk_ids:
            rec["sk_ids"] = np.array(sk_ids)
            rec["sk_corr"] = np.array(sk_corr)
        rec["queries"] = np.array(qs)
        rec["s"] = np.array(s)
        # the graph in internal order (to pin the recovered adjacency)
        rec["row_offsets"] = g.row_offsets
        rec["col_indices"] = g.col_indices
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        meta["cases"].append({"name": name, "n": idx.n, "n1": idx.n1, "n2": idx.n2, "ell": idx.lr.ell,
                              "alpha": idx.alpha, "klrc_bytes": len(blob), "queries": [int(q) for q in qs]})
        print(name, idx.n, idx.n1, idx.n2, idx.lr.ell, len(blob), flush=True)

    # CSR-level pin of cg() + spectral_norm on a Chung-Lu graph (cfg1 family, n=2000)
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_1912_06525_b200.generators import chung_lu_graph

    g = chung_lu_graph(n=2000, seed=1)
    rg = lrckatz.Graph(n=g.n, row_offsets=g.row_offsets, col_indices=g.col_indices, original_ids=g.original_ids)
    lam = lrckatz.spectral_norm(rg)
    beta = 0.5 / lam
    a = rg.adjacency()
    qs = np.sort(np.random.default_rng(0).choice(g.n, size=8, replace=False))
    S, it, res = [], [], []
    for q in qs:
        rhs = np.zeros(g.n)
        rhs[g.neighbors(q)] = beta
        x, rep = lrckatz.cg(lambda v: v - beta * (a @ v), rhs, tol=1e-8)
        S.append(np.maximum(x, 0.0))
        it.append(rep.iterations)
        res.append(rep.final_residual_norm)
    np.savez_compressed(os.path.join(OUT, "chunglu2000_cg.npz"), row_offsets=g.row_offsets,
                        col_indices=g.col_indices, spectral_norm=lam, beta=beta, queries=qs,
                        scores=np.array(S), iters=np.array(it), resid=np.array(res))
    meta["chunglu2000"] = {"n": g.n, "nnz": int(g.nnz), "spectral_norm": lam}
    print("chunglu2000", g.n, g.nnz, lam, it)
    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
