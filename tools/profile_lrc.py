"""One batched LRC query bracketed by cudaProfilerStart/Stop.

    python tools/profile_lrc.py [b]                  # cfg1, reference index
    python tools/profile_lrc.py b --config cfg2      # device-built index
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200.generators import CONFIGS, config_graph, sample_queries

ap = argparse.ArgumentParser()
ap.add_argument("b", type=int, nargs="?", default=16)
ap.add_argument("--config", default="cfg1")
ap.add_argument("--beta", type=float, default=0.5)
args = ap.parse_args()
b = args.b
if args.config == "cfg1":
    idx = kz.load_index(os.path.join(ROOT, "tests", "golden", "large", "cfg1.klrc"))
    qs = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_ref.npz"))["queries"]
    qs = idx.id_map[np.linspace(0, idx.n - 1, b).astype(int)] if b != len(qs) else qs
else:
    g = config_graph(args.config)
    lam = kz.spectral_norm(g)
    idx = kz.build_index(g, alpha=args.beta / lam, ell=CONFIGS[args.config]["ell"], seed=0, spectral_norm=lam)
    qs = sample_queries(g.original_ids, b, seed=0)
for _ in range(2):
    kz.query_batch(idx, qs, tol=1e-8, device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
kz.query_batch(idx, qs, tol=1e-8, device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
