"""Does splitting the 256-query headline batch into independent halves on two
streams (two host threads) overlap one half's HBM-bound vector updates with
the other half's L2-bound K1 gathers?  Times one 256-column eigen-form solve
against two concurrent 128-column solves (R-MAT 22, r = 128, tol 1e-8)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

spec = G.CONFIGS["cfg3"]
g = G.rmat_graph_fast(spec["scale"], seed=0)
lam = kz.spectral_norm(g)
beta = 0.5 / lam
idx = kz.GraphIndex(g, beta, spectral_norm=lam)
eidx = kz.EigenIndex(idx, spec["ell"])
qs = G.sample_queries(g.original_ids, 256, seed=0)
solver = sys.argv[1] if len(sys.argv) > 1 else "eigen"
target = eidx if solver == "eigen" else idx
fn = kz.query_batch if solver == "eigen" else kz.query_cg_baseline_batch


def one(q):
    s, r = fn(target, q, tol=1e-8, device=True)
    return s, r


def timed(run, reps=3):
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return min(ts) * 1e3


full = timed(lambda: one(qs))
half = timed(lambda: one(qs[:128]))
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
out = [None, None]


def worker(i, q):
    with torch.cuda.stream(streams[i]):
        out[i] = one(q)
        streams[i].synchronize()


def split(parts=2):
    th = [threading.Thread(target=worker, args=(i, qs[i * 128 : (i + 1) * 128])) for i in range(parts)]
    for t in th:
        t.start()
    for t in th:
        t.join()


two = timed(split)
ref, _ = one(qs)
got = torch.cat([out[0][0], out[1][0]])
err = float(((got - ref).abs().max() / ref.abs().max()).item())
print(f"{solver}: 256 in one call {full:.1f} ms; 128 alone {half:.1f} ms; 2x128 concurrent {two:.1f} ms "
      f"(max rel diff vs one call {err:.2e})", flush=True)
