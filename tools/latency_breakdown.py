"""Where does a small-config step go?  Host wall time per stage of one bench
step (batched plain CG + masked top-k) at cfg1 / cfg2, the sum of device
kernel time from the library's K1 timer, and a cProfile of the host side.

  python tools/latency_breakdown.py --config cfg1 [--steps 200]"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--steps", type=int, default=200)
a = ap.parse_args()
spec = G.CONFIGS[a.config]
g = G.rmat_graph_fast(spec["scale"]) if spec["kind"] == "rmat" else G.config_graph(a.config)
lam = kz.spectral_norm(g)
idx = kz.GraphIndex(g, 0.5 / lam)
qs = G.sample_queries(g.original_ids, spec["b"], seed=0)
internal = idx.internal_ids(qs)


def solve():
    return kz.query_cg_baseline_batch(idx, qs, tol=spec["tol"], device=True)


def topk(scores):
    return kz.topk_device(scores, spec["k"], idx.mask_operator(), internal, internal)


for _ in range(20):
    topk(solve()[0])
torch.cuda.synchronize()
ts, tk = [], []
for _ in range(a.steps):
    t0 = time.perf_counter()
    s, r = solve()
    t1 = time.perf_counter()
    topk(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ts.append(t1 - t0)
    tk.append(t2 - t1)
print(f"{a.config}: solve (host wall, ends with the report sync) {1e3*np.median(ts):.3f} ms, "
      f"top-k {1e3*np.median(tk):.3f} ms, device ms reported by the solve {r[0].wall_time*1e3:.3f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    topk(solve()[0])
e1.record()
torch.cuda.synchronize()
print(f"{a.config}: step by CUDA events {e0.elapsed_time(e1)/a.steps:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(a.steps):
    topk(solve()[0])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
