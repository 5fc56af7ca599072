"""Prototype for SURVEY §8(f)4: does an eigen-of-A Galerkin start save CG
iterations?  x0 = U (I - beta T)^-1 U^T b with T = U^T A U, U = top-r Ritz
vectors of A (device Lanczos); the CG from x0 is run as CG on M d = r0 with
the tolerance rescaled to ||b|| (identical iterates).

    python tools/eigen_proto.py --config proxy16 --r 64 --b 16
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
from paper_1912_06525_b200.build import lanczos_topk
from paper_1912_06525_b200.generators import config_graph, sample_queries

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="proxy16")
ap.add_argument("--r", type=int, default=64)
ap.add_argument("--b", type=int, default=16)
ap.add_argument("--beta", type=float, default=0.5)
args = ap.parse_args()
g = config_graph(args.config)
lam = kz.spectral_norm(g)
alpha = args.beta / lam
gi = kz.GraphIndex(g, alpha=alpha, spectral_norm=lam)
op = gi.operator()
n = g.n


def apply(v):
    y = torch.empty_like(v)
    op.spmm(v, y, b=1)
    return y


t = time.perf_counter()
lr = lanczos_topk(apply, args.r, np.random.default_rng(0).standard_normal(n), tol=1e-8)
t_lanczos = time.perf_counter() - t
ut = torch.as_tensor(np.ascontiguousarray(lr.vectors.T), device="cuda")  # r x n
aut = torch.empty_like(ut)
op.spmm(ut, aut, b=args.r, chunk=1)
T = ut @ aut.T
T = 0.5 * (T + T.T)
W = torch.linalg.inv(torch.eye(args.r, dtype=torch.float64, device="cuda") - alpha * T)
qs = sample_queries(g.original_ids, args.b, seed=0)
pos = gi.solve_positions(np.searchsorted(g.original_ids, qs))
E = torch.zeros((args.b, n), dtype=torch.float64, device="cuda")
E[torch.arange(args.b), torch.as_tensor(pos, device="cuda")] = 1.0
B = torch.empty_like(E)
op.spmm(E, B, b=args.b, chunk=1, s2=alpha)  # b_j = alpha * A e_q
Z = alpha * aut[:, torch.as_tensor(pos, device="cuda")]  # U^T b = alpha (AU)^T e_q   (r x b)
Y = W @ Z
X0 = (ut.T @ Y).T
R0 = B - X0 + alpha * (aut.T @ Y).T
kop = kz.KatzOperator(op, alpha)
res = []
for j in range(args.b):
    bn = float(torch.linalg.vector_norm(B[j]))
    rn = float(torch.linalg.vector_norm(R0[j]))
    _, rep_plain = kz.cg(kop, B[j], tol=1e-8)
    _, rep_lr = kz.cg(kop, R0[j], tol=1e-8 * bn / rn)
    res.append((rep_plain.iterations, rep_lr.iterations, rn / bn))
out = {"config": args.config, "n": n, "r": args.r, "beta_lambda": args.beta, "lanczos_s": round(t_lanczos, 2),
       "ritz_top": [round(float(x), 3) for x in lr.values[:4]], "ritz_r": float(lr.values[-1]),
       "plain_iters_mean": float(np.mean([a for a, _, _ in res])),
       "lowrank_iters_mean": float(np.mean([b for _, b, _ in res])),
       "r0_over_b_mean": float(np.mean([c for _, _, c in res]))}
print(json.dumps(out))
