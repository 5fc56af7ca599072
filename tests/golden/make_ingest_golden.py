"""Golden vectors for graph ingestion, produced by the reference itself.

Run in the build container:  python tests/golden/make_ingest_golden.py
Random edge lists with duplicates (both orientations), self loops and several
components go through the reference's from_edges (graph.py:111-148),
largest_connected_component (graph.py:232-261) and spectral_norm
(graph.py:264-297); the resulting CSR arrays are recorded.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import lrckatz  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def case(seed, n, m, comps):
    rng = np.random.default_rng(seed)
    # several dense-ish blobs plus a few stray edges; ties in component size
    # are exercised by comps with equal sizes
    sizes = np.full(comps, n // comps)
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    edges = []
    for s, k in zip(starts, sizes):
        u = rng.integers(s, s + k, size=m // comps)
        v = rng.integers(s, s + k, size=m // comps)
        edges.append(np.stack([u, v], 1))
    e = np.concatenate(edges)
    e = np.concatenate([e, e[: len(e) // 5, ::-1], np.stack([e[:50, 0], e[:50, 0]], 1)])  # dups, reversed, loops
    rng.shuffle(e)
    return e


def main():
    rec = {}
    for i, (seed, n, m, comps) in enumerate([(1, 5000, 20000, 3), (2, 20000, 60000, 2), (3, 3000, 4000, 1)]):
        e = case(seed, n, m, comps)
        g = lrckatz.from_edges(e, n=n)
        lcc = lrckatz.largest_connected_component(g)
        rec[f"edges{i}"] = e
        rec[f"n{i}"] = np.array(n)
        rec[f"off{i}"] = g.row_offsets
        rec[f"col{i}"] = g.col_indices
        rec[f"lcc_off{i}"] = lcc.row_offsets
        rec[f"lcc_col{i}"] = lcc.col_indices
        rec[f"lcc_ids{i}"] = lcc.original_ids
        rec[f"lam{i}"] = np.array(lrckatz.spectral_norm(lcc))
        print(i, g.n, g.col_indices.size, lcc.n, lcc.col_indices.size, rec[f"lam{i}"])
    np.savez_compressed(os.path.join(OUT, "ingest.npz"), **rec)


if __name__ == "__main__":
    main()
