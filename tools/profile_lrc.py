"""One batched LRC query at cfg1 bracketed by cudaProfilerStart/Stop."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
idx = kz.load_index(os.path.join(ROOT, "tests", "golden", "large", "cfg1.klrc"))
qs = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_ref.npz"))["queries"]
qs = idx.id_map[np.linspace(0, idx.n - 1, b).astype(int)] if b != len(qs) else qs
for _ in range(2):
    kz.query_batch(idx, qs, tol=1e-8, device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
kz.query_batch(idx, qs, tol=1e-8, device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
