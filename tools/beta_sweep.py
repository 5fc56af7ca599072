"""BASELINE config 4 (index 3): beta sweep on the scale-18 R-MAT graph.

beta in {0.1, 0.5, 0.9, 0.99} x 1/lambda_max, correction rank r in {32, 128},
a batch of 64 seeded queries, fp64, tol 1e-8: LRC-Katz (Schur PCG on an index
built on the device by build.py -- the reference's CPU build cannot hold the
~24 GB separator factor) against plain CG (GraphIndex), iteration counts and
queries/sec, plus the north-star eigen form (EigenIndex, walk start) at the
same rank.  Each LRC / eigen batch is also checked against the CG batch (all
converge to tol 1e-8, so they agree to ~cond * 1e-8).

    python tools/beta_sweep.py [--betas 0.1,0.5,0.9,0.99] [--ranks 32,128]
                               [--config cfg2] [--b 64] [--out FILE]
"""
import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_06525_b200 as kz  # noqa: E402
from paper_1912_06525_b200.generators import config_graph, sample_queries  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--betas", default="0.1,0.5,0.9,0.99")
    ap.add_argument("--ranks", default="32,128")
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    t = time.perf_counter()
    g = config_graph(args.config)
    lam = kz.spectral_norm(g)
    qs = sample_queries(g.original_ids, args.b, seed=0)
    head = {"config": args.config, "n": g.n, "nnz": g.nnz, "lambda_max": lam, "b": args.b,
            "graph_seconds": round(time.perf_counter() - t, 2)}
    print(json.dumps(head), flush=True)
    lines = [head]
    for beta in [float(x) for x in args.betas.split(",")]:
        alpha = beta / lam
        gi = kz.GraphIndex(g, alpha=alpha, spectral_norm=lam)
        dt_cg, (s_cg, r_cg) = timed(lambda: kz.query_cg_baseline_batch(gi, qs, tol=1e-8, device=True), args.reps)
        s_cg = s_cg.cpu().numpy()
        for ell in [int(x) for x in args.ranks.split(",")]:
            idx = kz.build_index(g, alpha=alpha, ell=ell, seed=0, spectral_norm=lam)
            st = idx.build_stats
            dt_lrc, (s_lrc, r_lrc) = timed(lambda: kz.query_batch(idx, qs, tol=1e-8, device=True), args.reps)
            s_lrc = s_lrc.cpu().numpy()
            diff = max(np.linalg.norm(a - c) / np.linalg.norm(c) for a, c in zip(s_lrc, s_cg))
            rec = {
                "beta_times_lambda": beta, "alpha": alpha, "rank": ell, "n2": st["n2"],
                "num_parts": st["num_parts"], "build_seconds": round(st["build_seconds"], 2),
                "stage_seconds": {k: round(v, 2) for k, v in st["stage_seconds"].items()},
                "sigma_max": float(idx.lr.values[0]) if idx.lr.ell else None,
                "sigma_min": float(idx.lr.values[-1]) if idx.lr.ell else None,
                "lrc_qps": round(args.b / dt_lrc, 1), "lrc_ms": round(dt_lrc * 1e3, 2),
                "lrc_iters_mean": float(np.mean([r.iterations for r in r_lrc])),
                "lrc_iters_max": int(max(r.iterations for r in r_lrc)),
                "lrc_converged": all(r.converged for r in r_lrc),
                "cg_qps": round(args.b / dt_cg, 1), "cg_ms": round(dt_cg * 1e3, 2),
                "cg_iters_mean": float(np.mean([r.iterations for r in r_cg])),
                "cg_iters_max": int(max(r.iterations for r in r_cg)),
                "lrc_vs_cg_max_rel_l2": float(diff),
            }
            # the north-star eigen form (EigenIndex, walk start) at the same rank
            ei = kz.EigenIndex(gi, ell)
            dt_e, (s_e, r_e) = timed(lambda: kz.query_batch(ei, qs, tol=1e-8, device=True), args.reps)
            s_e = s_e.cpu().numpy()
            rec.update({
                "eigen_build_seconds": round(ei.build_stats["build_seconds"], 2),
                "eigen_qps": round(args.b / dt_e, 1), "eigen_ms": round(dt_e * 1e3, 2),
                "eigen_iters_mean": float(np.mean([r.iterations for r in r_e])),
                "eigen_iters_max": int(max(r.iterations for r in r_e)),
                "eigen_converged": all(r.converged for r in r_e),
                "eigen_vs_cg_max_rel_l2": float(max(np.linalg.norm(a - c) / np.linalg.norm(c)
                                                    for a, c in zip(s_e, s_cg))),
            })
            del ei
            print(json.dumps(rec), flush=True)
            lines.append(rec)
            del idx
            gc.collect()
            torch.cuda.empty_cache()
        del gi
        gc.collect()
    if args.out:
        with open(args.out, "w") as fh:
            for rec in lines:
                fh.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
