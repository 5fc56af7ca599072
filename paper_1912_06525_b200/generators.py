"""Seeded synthetic graphs for the BASELINE.json configurations.

BASELINE.json names no public dataset, so every configuration runs on a
seeded generator (SURVEY.md Appendix B definitions), restricted to the
largest connected component by the reference rule (graph.py:232-261):

  cfg1  Chung-Lu, n=10,000, exponent 2.5, mean degree 10
  cfg2  R-MAT scale 18, edge factor 16, (a,b,c,d) = (.57,.19,.19,.05)
  cfg3  R-MAT scale 22, same parameters (headline)
  cfg5  planted-partition (SBM) graph, n=10^6, 1,000 power-law communities
  proxy R-MAT scale 16 (LRC-buildable stand-in for cfg2/cfg4)

Query samples follow cmd_bench (cli.py:119-120):
sort(default_rng(seed).choice(id_map, b, replace=False)).
"""

from __future__ import annotations

import numpy as np

from .graph import csr_from_pairs, Graph, largest_connected_component

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


def rmat_pairs(scale, edge_factor=16, abcd=RMAT_ABCD, seed=0):
    """R-MAT endpoints: one uniform per edge and bit, least significant bit
    first; u_bit = r >= a+b, v_bit = (a <= r < a+b) or r >= a+b+c."""
    a, b, c, _ = abcd
    n = 1 << scale
    m = n * edge_factor
    rng = np.random.default_rng(seed)
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(m)
        ub = r >= a + b
        vb = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ub.astype(np.int64) << bit
        v |= vb.astype(np.int64) << bit
        del r, ub, vb
    return u, v, n


def rmat_graph(scale, edge_factor=16, abcd=RMAT_ABCD, seed=0):
    u, v, n = rmat_pairs(scale, edge_factor, abcd, seed)
    offsets, dst = csr_from_pairs(u, v, n)
    del u, v
    g = Graph(n=n, row_offsets=offsets, col_indices=dst, original_ids=np.arange(n, dtype=np.int64))
    return largest_connected_component(g)


def rmat_graph_fast(scale, edge_factor=16, abcd=RMAT_ABCD, seed=0):
    """rmat_graph with from_edges and the largest component on the GPU
    (graph.from_edges_device / largest_connected_component_device); the same
    CSR as rmat_graph."""
    import torch

    if not torch.cuda.is_available():
        return rmat_graph(scale, edge_factor, abcd, seed)
    from .graph import from_edges_device, largest_connected_component_device

    u, v, n = rmat_pairs(scale, edge_factor, abcd, seed)
    g, dev = from_edges_device(u, v, n)
    del u, v
    return largest_connected_component_device(g, dev)


def chung_lu_graph(n=10_000, gamma=2.5, mean_degree=10.0, seed=0):
    """Chung-Lu: weights i^(-1/(gamma-1)) scaled to the mean degree; n*d/2
    endpoint pairs drawn i.i.d. proportional to the weights (u batch first)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    w *= mean_degree / w.mean()
    p = w / w.sum()
    m = int(n * mean_degree / 2)
    rng = np.random.default_rng(seed)
    u = rng.choice(n, size=m, p=p)
    v = rng.choice(n, size=m, p=p)
    offsets, dst = csr_from_pairs(u, v, n)
    g = Graph(n=n, row_offsets=offsets, col_indices=dst, original_ids=np.arange(n, dtype=np.int64))
    return largest_connected_component(g)


def sbm_edges(n=1_000_000, communities=1000, exponent=2.0, min_size=100, mean_degree=20.0,
              intra=0.9, seed=0):
    """Planted-partition edges: community sizes from a seeded discrete power
    law (exponent, minimum) rescaled to sum to n; n*d/2 edge draws, a
    fraction `intra` uniform inside a community (chosen proportional to its
    size), the rest uniform over all nodes.  Returns (u, v, sizes)."""
    rng = np.random.default_rng(seed)
    # discrete power law by inverse transform of the continuous Pareto
    raw = np.floor(min_size * (1.0 - rng.random(communities)) ** (-1.0 / (exponent - 1.0)))
    sizes = np.maximum(np.round(raw / raw.sum() * n).astype(np.int64), 1)
    sizes[-1] += n - sizes.sum()
    if sizes[-1] < 1:
        raise ValueError("community size rescaling failed")
    starts = np.zeros(communities + 1, dtype=np.int64)
    np.cumsum(sizes, out=starts[1:])
    m = int(n * mean_degree / 2)
    m_in = int(round(intra * m))
    comm = rng.choice(communities, size=m_in, p=sizes / n)
    u_in = starts[comm] + (rng.random(m_in) * sizes[comm]).astype(np.int64)
    v_in = starts[comm] + (rng.random(m_in) * sizes[comm]).astype(np.int64)
    u_out = rng.integers(0, n, size=m - m_in)
    v_out = rng.integers(0, n, size=m - m_in)
    return np.concatenate([u_in, u_out]), np.concatenate([v_in, v_out]), sizes


def sbm_split(n=1_000_000, holdout=0.1, seed=0, **kw):
    """Train graph (LCC) plus held-out positive pairs (original ids), the
    shape temporal_split (linkpred.py:63-112) produces for (u,v,0) train
    rows and (u,v,1) held-out rows with cutoff 0."""
    u, v, _ = sbm_edges(n=n, seed=seed, **kw)
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    und = np.unique(lo * n + hi)
    rng = np.random.default_rng(seed + 1)
    test = rng.random(und.size) < holdout
    tr = und[~test]
    offsets, dst = csr_from_pairs(tr // n, tr % n, n)
    g = Graph(n=n, row_offsets=offsets, col_indices=dst, original_ids=np.arange(n, dtype=np.int64))
    g = largest_connected_component(g)
    te = und[test]
    a, b = te // n, te % n
    inside = np.isin(a, g.original_ids) & np.isin(b, g.original_ids)
    positives = np.stack([a[inside], b[inside]], axis=1)
    return g, positives


def sample_queries(id_map, count, seed=0):
    """Query sample of cmd_bench (cli.py:119-120)."""
    if count > len(id_map):
        raise ValueError(f"cannot sample {count} queries from {len(id_map)} nodes")
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(np.asarray(id_map), size=count, replace=False))


CONFIGS = {
    "cfg1": dict(kind="chung_lu", n=10_000, b=16, ell=32, k=20, tol=1e-8),
    "proxy16": dict(kind="rmat", scale=16, b=64, ell=64, k=50, tol=1e-8),
    "cfg2": dict(kind="rmat", scale=18, b=64, ell=64, k=50, tol=1e-8),
    "cfg3": dict(kind="rmat", scale=22, b=256, ell=128, k=100, tol=1e-8),
}


def config_graph(name, seed=0):
    cfg = CONFIGS[name]
    if cfg["kind"] == "chung_lu":
        return chung_lu_graph(cfg["n"], seed=seed)
    return rmat_graph(cfg["scale"], seed=seed)
