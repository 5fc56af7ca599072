"""Kernel timeline of one bench step (CUPTI through torch.profiler): busy
time, idle gaps between consecutive kernels and the largest gaps, to find
host-induced bubbles in the solve loop.

    python tools/timeline.py [--config cfg3] [--solver eigen|cg] [--rank 128]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--solver", default="eigen")
ap.add_argument("--rank", type=int, default=None)
a = ap.parse_args()
spec = G.CONFIGS[a.config]
g = G.rmat_graph_fast(spec["scale"]) if spec["kind"] == "rmat" else G.config_graph(a.config)
lam = kz.spectral_norm(g)
gi = kz.GraphIndex(g, 0.5 / lam, spectral_norm=lam)
idx = kz.EigenIndex(gi, a.rank or spec["ell"]) if a.solver == "eigen" else gi
qs = G.sample_queries(g.original_ids, spec["b"], seed=0)
internal = gi.internal_ids(qs)


def step():
    fn = kz.query_batch if a.solver == "eigen" else kz.query_cg_baseline_batch
    scores, reps = fn(idx, qs, tol=spec["tol"], device=True)
    kz.topk_device(scores, spec["k"], gi.mask_operator(), internal, internal)


for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
busy, gaps, cur_end, first = 0.0, [], None, iv[0][0]
for s, t, name in iv:
    if cur_end is not None and s > cur_end:
        gaps.append((s - cur_end, name))
    cur_end = t if cur_end is None else max(cur_end, t)
span = cur_end - first
for s, t, _ in iv:
    busy += t - s
gaps.sort(reverse=True)
print(json.dumps({"config": a.config, "solver": a.solver, "events": len(iv), "span_ms": span / 1e3,
                  "kernel_sum_ms": busy / 1e3, "idle_ms": sum(x for x, _ in gaps) / 1e3,
                  "largest_gaps_us": [(round(x, 1), n[:40]) for x, n in gaps[:12]]}))
if os.environ.get("KZ_TIMELINE_LIST"):
    for s, t, name in iv:
        print(f"{(s - first):9.1f} us  +{(t - s):8.1f} us  {name[:70]}")
