"""Small workloads that reach every libkatzb200 kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck):

  compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_workload.py
  compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_workload.py
  compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_workload.py

Covered: K1 (short rows, medium rows, segmented hub rows with the stream-K
fix-up, weighted operator, the column-blocked schedule via KZ_K1_SLICE_MB in a
second process), plain CG (sparse first iteration + q-recurrence history,
the fold into the direction form, the direction form alone), the eigen-form
start (walk terms 1-3), LRC Schur PCG and its single applications, top-k
(one pass and the multi-pass continuation), sparse_katz (K7 gather +
rerank), ingestion (device from_edges + components), coldot / vec_op.
Sizes are tiny (the tools slow kernels down by 10-100x)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import _lib
from paper_1912_06525_b200 import generators as G

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
part = os.environ.get("KZ_SANITIZE_PART", "all")


def step(msg):
    torch.cuda.synchronize()
    print("ok", msg, flush=True)


# a Chung-Lu graph: hub rows above the short/medium thresholds and long
# enough to be cut into segments (max degree ~600 at n = 4,000)
g = G.chung_lu_graph(n=4000, mean_degree=10.0, seed=1)
lam = kz.spectral_norm(g)
beta = 0.5 / lam
idx = kz.GraphIndex(g, beta, spectral_norm=lam)
qs = G.sample_queries(g.original_ids, 40, seed=0)
step(f"ingest + spectral_norm (n={g.n}, nnz={g.nnz}, max deg {int(np.diff(g.row_offsets).max())})")

if part in ("all", "ingest"):
    G.rmat_graph_fast(11)
    step("device ingestion (from_edges_device, kz_connected_components)")

op = idx.operator()
for b, C in ((1, 1), (8, 8), (40, 32)):
    X = torch.randn(((b + C - 1) // C) * C * g.n, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    d = torch.empty(((b + C - 1) // C) * C, dtype=torch.float64, device="cuda")
    op.spmm(X, Y, b=((b + C - 1) // C) * C, chunk=C, Xs=X, s1=1.0, s2=-beta, dots=d)
step("K1 S/M/L tasks, C = 1, 8, 32, fused dots")

if part in ("all", "cg"):
    kz.query_cg_baseline_batch(idx, qs, tol=1e-10)
    step("CG: sparse first iteration + q-recurrence history")
    os.environ["KZ_CG_HISTORY"] = "3"
    kz.query_cg_baseline_batch(idx, qs[:9], tol=1e-12)
    step("CG: history fold into the direction form (H = 3)")
    kz.query_cg_baseline_batch(idx, qs[:9], tol=1e-10, start_seed=3)
    step("CG: seeded start")
    kz.cg(kz.KatzOperator(op, beta), np.ones(g.n), tol=1e-8)
    kz.cg(lambda v: 2.0 * v, np.ones(g.n), tol=1e-8)
    step("cg(): KatzOperator and a generic callable (kz_coldot / kz_vec_op)")
    ei = kz.EigenIndex(idx, 16, walk_terms=3)
    kz.query_batch(ei, qs[:9], tol=1e-10)
    ei1 = kz.EigenIndex(idx, 16, walk_terms=1)
    kz.query_batch(ei1, qs[:9], tol=1e-10)
    step("eigen-form start (walk terms 3 and 1) + CG")

if part in ("all", "topk"):
    S = torch.rand((5, 9000), dtype=torch.float64, device="cuda")
    S[1, ::3] = 0.5
    kz.topk_device(S, 100, None, None, np.arange(5))
    kz.topk_device(S, 5000, None, None, np.arange(5))
    step("top-k one pass and continuation passes")
    kz.katz_rank_batch(idx, qs[:8], 20)
    kz.sparse_katz_batch(idx, qs[:4], 10)
    step("katz_rank / sparse_katz (K4 masks, K7 gather + rerank)")

if part in ("all", "lrc"):
    li = kz.load_index(os.path.join(GOLDEN, "ba300.klrc"))
    rec = np.load(os.path.join(GOLDEN, "ba300.npz"))
    kz.query_batch(li, rec["queries"], tol=1e-10)
    v = np.random.default_rng(0).standard_normal(li.n2)
    kz.apply_schur(li, v)
    kz.lrc_pcg(li, v)
    kz.schur_rhs(li, np.ones(li.n1), np.ones(li.n2))
    step("LRC Schur PCG + single applications (ba300 KLRC)")
    g2 = kz.Graph(n=li.n, row_offsets=li.adjacency_internal()[0], col_indices=li.adjacency_internal()[1],
                  original_ids=li.id_map.copy())
    kz.build_index(g2, alpha=li.alpha, ell=8, seed=7, spectral_norm=li.spectral_norm)
    step("device index build (Lanczos on kz_lrc_apply)")

print("SANITIZE_WORKLOAD_DONE", flush=True)
