"""Eigen-of-A low-rank start + CG (north-star LRC) vs plain CG, batched.

    python tools/bench_eigen.py [--config cfg3] [--b 256] [--ranks 32,128] [--beta 0.5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200.generators import config_graph, sample_queries

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--ranks", default="32,128")
ap.add_argument("--beta", type=float, default=0.5)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--which", default="LA,LM")
ap.add_argument("--steps", type=int, default=None)
args = ap.parse_args()
g = config_graph(args.config)
lam = kz.spectral_norm(g)
gi = kz.GraphIndex(g, alpha=args.beta / lam, spectral_norm=lam)
qs = sample_queries(g.original_ids, args.b, seed=0)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(args.reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / args.reps, out


dt, (s_cg, r_cg) = timed(lambda: kz.query_cg_baseline_batch(gi, qs, tol=1e-8, device=True))
print(json.dumps({"config": args.config, "n": g.n, "b": args.b, "beta_lambda": args.beta, "solver": "cg",
                  "qps": round(args.b / dt, 1), "ms": round(dt * 1e3, 2),
                  "iters_mean": float(np.mean([r.iterations for r in r_cg]))}), flush=True)
for rank, which in [(int(x), w) for x in args.ranks.split(",") for w in args.which.split(",")]:
    ei = kz.EigenIndex(gi, rank, which=which, max_steps=args.steps)
    dt, (s_e, r_e) = timed(lambda: kz.query_batch(ei, qs, tol=1e-8, device=True))
    diff = float(torch.max(torch.linalg.vector_norm(s_e - s_cg, dim=1) / torch.linalg.vector_norm(s_cg, dim=1)))
    print(json.dumps({"solver": "eigen", "rank": rank, "which": which,
                      "ritz_min": float(min(ei.ritz_values)), "ritz_max": float(max(ei.ritz_values)),
                      "iters_max": int(max(r.iterations for r in r_e)), "build_s": round(ei.build_stats["build_seconds"], 2),
                      "qps": round(args.b / dt, 1), "ms": round(dt * 1e3, 2),
                      "iters_mean": float(np.mean([r.iterations for r in r_e])),
                      "max_rel_diff_vs_cg": diff}), flush=True)
    del ei
    torch.cuda.empty_cache()
