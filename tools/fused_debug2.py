import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
for cfg in sys.argv[1:]:
    spec = G.CONFIGS[cfg]
    g = G.config_graph(cfg); lam = kz.spectral_norm(g); idx = kz.GraphIndex(g, 0.5/lam)
    qs = G.sample_queries(g.original_ids, spec["b"], seed=0)
    for _ in range(3):
        s1, r1 = kz.query_cg_baseline_batch(idx, qs, tol=1e-8)
    torch.cuda.synchronize()
    print(cfg, "device ms", r1[0].wall_time * 1e3, flush=True)
