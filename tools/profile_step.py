"""One bench step (batched CG Katz solve + masked top-k) bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off` launch lists.
Graph build and the spectral-norm power iteration stay outside the range."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--solver", default="cg", choices=["cg", "eigen"])
ap.add_argument("--rank", type=int, default=None)
a = ap.parse_args()
spec = G.CONFIGS[a.config]
g = G.rmat_graph_fast(spec["scale"]) if spec["kind"] == "rmat" else G.config_graph(a.config)
lam = kz.spectral_norm(g)
idx = kz.GraphIndex(g, 0.5 / lam)
qs = G.sample_queries(g.original_ids, spec["b"], seed=0)
internal = idx.internal_ids(qs)
eidx = kz.EigenIndex(idx, a.rank or spec["ell"]) if a.solver == "eigen" else None


def step():
    if eidx is not None:
        scores, reps = kz.query_batch(eidx, qs, tol=spec["tol"], device=True)
    else:
        scores, reps = kz.query_cg_baseline_batch(idx, qs, tol=spec["tol"], device=True)
    kz.topk_device(scores, spec["k"], idx.mask_operator(), internal, internal)
    return reps


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
reps = step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
its = [r.iterations for r in reps]
print("iterations mean", sum(its) / len(its), "max", max(its), "hist", {k: its.count(k) for k in sorted(set(its))}, flush=True)
