import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
for cfg in ["cfg1", "proxy16"]:
    g = G.config_graph(cfg); lam = kz.spectral_norm(g); idx = kz.GraphIndex(g, 0.5/lam)
    for b in [1, 2, 4, 8, 16, 32, 64]:
        qs = G.sample_queries(g.original_ids, b, seed=0)
        os.environ["KZ_CG_FUSED"] = "0"
        s0, r0 = kz.query_cg_baseline_batch(idx, qs, tol=1e-8)
        os.environ["KZ_CG_FUSED"] = "1"
        try:
            s1, r1 = kz.query_cg_baseline_batch(idx, qs, tol=1e-8)
            d = np.linalg.norm(s1 - s0) / np.linalg.norm(s0)
            print(cfg, b, [r.iterations for r in r0][:4], [r.iterations for r in r1][:4], d, flush=True)
        except Exception as e:
            print(cfg, b, "ERR", e, flush=True)
