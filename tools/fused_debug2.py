import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
g = G.config_graph("cfg1"); lam = kz.spectral_norm(g); idx = kz.GraphIndex(g, 0.5/lam)
qs = G.sample_queries(g.original_ids, 16, seed=0)
try:
    s1, r1 = kz.query_cg_baseline_batch(idx, qs, tol=1e-8)
except Exception as e:
    print("ERR", e)
torch.cuda.synchronize()
