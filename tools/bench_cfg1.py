"""cfg1 (Chung-Lu 10^4, beta=0.5/lambda, ell=32, b=16, tol 1e-8): LRC-Katz and
plain-CG batched query throughput on the reference's own KLRC index
(tests/golden/large/cfg1.klrc).  Reference CPU numbers for the same index and
queries were measured by tests/golden/make_cfg1.py (1 thread)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz

KLRC = os.path.join(ROOT, "tests", "golden", "large", "cfg1.klrc")
rec = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_ref.npz"))
if os.path.exists(KLRC) and "--build" not in sys.argv:
    idx, source = kz.load_index(KLRC), "reference build (KLRC)"
else:  # same graph and parameters as make_cfg1.py, built on the device
    from paper_1912_06525_b200.generators import chung_lu_graph

    idx = kz.build_index(chung_lu_graph(), alpha=float(rec["alpha"]), ell=32, seed=0,
                         spectral_norm=float(rec["spectral_norm"]))
    source = f"device build ({idx.build_stats['build_seconds']:.2f} s)"
qs = rec["queries"]
t0 = time.perf_counter()
idx.lrc()
idx.operator()
prep = time.perf_counter() - t0
out = {"index": source, "n": idx.n, "n2": idx.n2, "ell": idx.lr.ell, "device_prep_s": round(prep, 2)}
for name, fn in (("lrc", kz.query_batch), ("cg", kz.query_cg_baseline_batch)):
    for b in (16, 256):
        q = np.resize(qs, b) if b > len(qs) else qs[:b]
        q = np.unique(np.concatenate([q, idx.id_map[:b]]))[:b] if b > len(qs) else q
        for _ in range(3):
            fn(idx, q, tol=1e-8, device=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = 10
        for _ in range(reps):
            s, r = fn(idx, q, tol=1e-8, device=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        out[f"{name}_b{b}_qps"] = round(len(q) / dt, 1)
        out[f"{name}_b{b}_ms"] = round(dt * 1e3, 3)
        out[f"{name}_b{b}_iters"] = float(np.mean([x.iterations for x in r]))
out["reference_cpu_qps_1thread"] = {"lrc": 1.48, "cg": 3.83}
print(json.dumps(out))
