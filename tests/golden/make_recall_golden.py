"""Golden vectors for the recall-evaluation harness, made by the reference.

Run in the build container:  python tests/golden/make_recall_golden.py
A temporal preferential-attachment edge stream (pkg/tests/synth.py
temporal_pa_edges, planted communities) goes through the reference's
temporal_split (linkpred.py:63-112); an index is built by the reference's
build_index and saved (tests/golden/recall.klrc); evaluate_recall and
evaluate_recall_sweep (linkpred.py:238-337) results are recorded.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
import lrckatz  # noqa: E402
from lrckatz import PartitionConfig, build_index, save_index  # noqa: E402
from lrckatz.linkpred import evaluate_recall, evaluate_recall_sweep, temporal_split  # noqa: E402
from synth import temporal_pa_edges  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def stat(st):
    return [st.mean, st.std, st.n_queries]


def main():
    rows, cutoff = temporal_pa_edges(600, 3, np.random.default_rng(11), communities=6)
    ds = temporal_split(rows, cutoff)
    idx = build_index(ds.train, ell=8, cfg=PartitionConfig(max_part_size=60), seed=0)
    save_index(idx, os.path.join(OUT, "recall.klrc"))
    endpoints = sorted({u for pair in ds.positives for u in pair})
    sample = sorted(int(x) for x in np.random.default_rng(0).choice(endpoints, size=12, replace=False))
    sweep = evaluate_recall_sweep(idx, ["katz", "sparse-katz"], ds, [5, 10, 20], query_sample=sample)
    single = {s: {k: stat(v) for k, v in evaluate_recall(idx, "katz", ds, s=s).items()} for s in (1, 10)}
    rec = {
        "rows": [[int(u), int(v), float(t)] for u, v, t in rows],
        "cutoff": float(cutoff),
        "train_ids": [int(x) for x in ds.train.original_ids],
        "train_off": [int(x) for x in ds.train.row_offsets],
        "train_col": [int(x) for x in ds.train.col_indices],
        "positives": [list(map(int, p)) for p in ds.positives],
        "buckets": {k: [list(map(int, p)) for p in v] for k, v in ds.buckets.items()},
        "sample": sample,
        "sweep": [[m, lab, int(s), stat(st)] for m, lab, s, st in sweep],
        "katz_all": {str(s): v for s, v in single.items()},
    }
    with open(os.path.join(OUT, "recall.json"), "w") as fh:
        json.dump(rec, fh)
    print("train", ds.train.n, "positives", len(ds.positives), "n2", idx.n2,
          "klrc", os.path.getsize(os.path.join(OUT, "recall.klrc")))


if __name__ == "__main__":
    main()
