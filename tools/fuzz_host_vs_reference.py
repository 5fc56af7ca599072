"""Host-side API against the reference package itself (CPU only; needs
/root/reference, so it runs in the build container, not on the GPU box):
random inputs through from_edges, largest_connected_component,
load_edge_list (well-formed and malformed text), temporal_split, pearson and
the KLRC writer / reader (reference-built indexes of random small graphs),
comparing values, byte streams and exception types / messages.

  python tools/fuzz_host_vs_reference.py [--cases 300] [--seed 0]"""
import argparse
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np

import lrckatz as ref  # noqa: E402
import lrckatz.graph as refg  # noqa: E402
import lrckatz.linkpred as reflp  # noqa: E402

import paper_1912_06525_b200 as kz  # noqa: E402
from paper_1912_06525_b200 import evaluate as kze  # noqa: E402
from paper_1912_06525_b200 import graph as kzg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=300)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)


def outcome(fn):
    try:
        return ("ok", fn())
    except Exception as e:  # noqa: BLE001
        return ("err", type(e).__name__, str(e))


def same_graph(g1, g2):
    return (g1.n == g2.n and np.array_equal(g1.row_offsets, g2.row_offsets)
            and np.array_equal(g1.col_indices, g2.col_indices) and np.array_equal(g1.original_ids, g2.original_ids))


def same_exc(o1, o2):
    # exception classes mirror the reference's by name (distinct modules)
    return o1[0] == o2[0] == "err" and o1[1] == o2[1] and o1[2] == o2[2]


fails = 0
counts = {}


def check(name, ok, detail=None):
    global fails
    counts[name] = counts.get(name, 0) + 1
    if not ok:
        fails += 1
        print(json.dumps({"FAIL": name, "detail": str(detail)[:400]}), flush=True)


for case in range(a.cases):
    n = int(rng.choice([1, 2, 5, 30, 200]))
    m = int(rng.integers(0, 4 * n + 2))
    edges = rng.integers(0, n, size=(m, 2))
    # ---- from_edges / LCC --------------------------------------------------
    o1 = outcome(lambda: refg.from_edges(edges, n=n))
    o2 = outcome(lambda: kzg.from_edges(edges, n=n))
    if o1[0] == "ok" and o2[0] == "ok":
        check("from_edges", same_graph(o1[1], o2[1]))
        l1 = outcome(lambda: refg.largest_connected_component(o1[1]))
        l2 = outcome(lambda: kzg.largest_connected_component(o2[1]))
        check("lcc", (l1[0] == l2[0] == "ok" and same_graph(l1[1], l2[1])) or same_exc(l1, l2), (l1[:1], l2[:1]))
    else:
        check("from_edges errors", same_exc(o1, o2), (o1, o2))
    bad = edges.copy()
    if m and case % 3 == 0:
        bad[int(rng.integers(0, m)), int(rng.integers(0, 2))] = int(rng.choice([-1, n, n + 7]))
        check("from_edges bad ids", same_exc(outcome(lambda: refg.from_edges(bad, n=n)),
                                             outcome(lambda: kzg.from_edges(bad, n=n))))
    # ---- load_edge_list ----------------------------------------------------
    lines = []
    for u, v in edges:
        style = int(rng.integers(0, 5))
        lines.append([f"{u} {v}", f"{u},{v}", f"{u}\t{v}", f"  {u}   {v}  ", f"{u}, {v}"][style])
    if case % 2 == 0:
        lines.insert(int(rng.integers(0, len(lines) + 1)), "# a comment")
        lines.insert(int(rng.integers(0, len(lines) + 1)), "")
    if case % 4 == 1 and lines:
        junk = ["1 2 3", "x y", "4", "5,", "-1 2", "1.5 2", "7;8", "9 ten"][int(rng.integers(0, 8))]
        lines.insert(int(rng.integers(0, len(lines) + 1)), junk)
    text = ("\n".join(lines) + ("\n" if case % 5 else "")).encode()
    for fmt in ("auto", "csv", "whitespace", "tsv") if case % 7 == 0 else ("auto",):
        t1 = outcome(lambda: refg.load_edge_list(io.BytesIO(text), fmt=fmt))
        t2 = outcome(lambda: kzg.load_edge_list(io.BytesIO(text), fmt=fmt))
        if t1[0] == "ok" and t2[0] == "ok":
            check("load_edge_list", same_graph(t1[1], t2[1]), fmt)
        else:
            check("load_edge_list errors", same_exc(t1, t2), (fmt, t1[1:], t2[1:]))
    # ---- temporal_split ----------------------------------------------------
    if m:
        times = rng.integers(0, 10, size=m).astype(float)
        rows = [(int(u), int(v), float(t)) for (u, v), t in zip(edges, times)]
        cutoff = float(rng.choice([-1, 0, 3, 5, 9, 12]))
        s1 = outcome(lambda: reflp.temporal_split(rows, cutoff))
        s2 = outcome(lambda: kze.temporal_split(rows, cutoff))
        if s1[0] == "ok" and s2[0] == "ok":
            d1, d2 = s1[1], s2[1]
            check("temporal_split", same_graph(d1.train, d2.train) and list(d1.positives) == list(d2.positives)
                  and {k: list(v) for k, v in d1.buckets.items()} == {k: list(v) for k, v in d2.buckets.items()})
        else:
            check("temporal_split errors", same_exc(s1, s2), (s1[1:], s2[1:]))
    # ---- pearson -----------------------------------------------------------
    k = int(rng.choice([1, 2, 3, 10]))
    x = rng.standard_normal(k) if case % 5 else np.full(k, 2.0)
    y = rng.standard_normal(k if case % 9 else k + 1)
    p1, p2 = outcome(lambda: reflp.pearson(x, y)), outcome(lambda: kz.pearson(x, y))
    check("pearson", (p1[0] == p2[0] == "ok" and p1[1] == p2[1]) or same_exc(p1, p2), (p1, p2))
    # ---- KLRC round trip on a reference-built index --------------------------
    if case % 6 == 0 and n >= 30:
        gconn = refg.largest_connected_component(refg.from_edges(np.concatenate([edges, np.stack(
            [np.arange(n - 1), np.arange(1, n)], axis=1)]), n=n))
        lam = refg.spectral_norm(gconn)
        ridx = ref.build_index(gconn, alpha=0.5 / lam, ell=int(min(8, gconn.n // 4)), seed=int(rng.integers(0, 100)))
        buf = io.BytesIO()
        ref.save_index(ridx, buf)
        raw = buf.getvalue()
        mine = kz.load_index(io.BytesIO(raw))
        out = io.BytesIO()
        kz.save_index(mine, out)
        check("klrc round trip", out.getvalue() == raw)
        flip = bytearray(raw)
        pos = int(rng.integers(0, len(flip)))
        flip[pos] ^= 1 << int(rng.integers(0, 8))
        f1 = outcome(lambda: ref.load_index(io.BytesIO(bytes(flip))))
        f2 = outcome(lambda: kz.load_index(io.BytesIO(bytes(flip))))
        check("klrc byte flip", f1[0] == f2[0] and (f1[0] == "ok" or f1[1] == f2[1]), (pos, f1[:2], f2[:2]))
        cut = raw[: int(rng.integers(0, len(raw)))]
        c1 = outcome(lambda: ref.load_index(io.BytesIO(cut)))
        c2 = outcome(lambda: kz.load_index(io.BytesIO(cut)))
        check("klrc truncated", same_exc(c1, c2), (c1[1:], c2[1:]))
print(json.dumps({"cases": a.cases, "checks": counts, "failures": fails}))
