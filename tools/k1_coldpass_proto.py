"""Prototype of the split K1 at R-MAT 22 (b = 256, C = 32): the cold entries
(column >= H) of the rows that hold most of them go to the cold pass
(spmmcold.cuh, streams built here in numpy: pieces of <= PIECE entries, LPT
assignment to lane groups, [slab][group] entry order); times the cold pass,
the main operator (A minus the moved entries) and the full operator, and
checks sampled partial rows against torch sums.  Needs the experiment build:
  make -C paper_1912_06525_b200/csrc EXTRA=-DKZ_EXPERIMENTS=1 OUT=$PWD/build/variants/exp/libkatzb200.so OBJDIR=$PWD/build/variants/exp/obj
  KZ_LIB_PATH=build/variants/exp/libkatzb200.so python tools/k1_coldpass_proto.py"""
import argparse
import ctypes
import heapq
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import _lib
from paper_1912_06525_b200 import generators as G
from paper_1912_06525_b200.index import degclass_rcm_order, permute_csr

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=131072)
ap.add_argument("--slab-rows", type=int, nargs="+", default=[95000])
ap.add_argument("--min-cold", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cache", default="/tmp/k1sweep")
a = ap.parse_args()
os.makedirs(a.cache, exist_ok=True)
cf = os.path.join(a.cache, "csr22.npz")
if os.path.exists(cf):
    z = np.load(cf)
    off, col, n = z["off"], z["col"], int(z["n"])
else:
    g = G.rmat_graph_fast(22)
    order = degclass_rcm_order(g)
    inv = np.empty(g.n, dtype=np.int64)
    inv[order] = np.arange(g.n)
    off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
    n = g.n
    np.savez(cf, off=off, col=col, n=n, nnz=g.nnz)
lib = _lib.load()
lib.kz_spmm_cold_debug.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                                           ctypes.c_int32] + [ctypes.c_void_p] * 4
SLOTS = lib.kz_cold_slots()
NG = lib.kz_num_sms() * 5 * 32
b, C = 256, 32
nch = b // C
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)


def timed(fn):
    ts = []
    for r in range(a.reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(min(ts))


deg = np.diff(off)
rows = np.repeat(np.arange(n), deg)
op = kz.DeviceOperator(off, col.astype(np.int32), n)
full = timed(lambda: op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4))
del op
print(json.dumps({"operator": "full", "ms": round(full[0], 3), "ms_min": round(full[1], 3)}), flush=True)

cold = col >= a.H
coldcnt = np.bincount(rows[cold], minlength=n)
# rows by cold count, pieces until the slots are full
cand = np.flatnonzero(coldcnt >= a.min_cold)
cand = cand[np.argsort(-coldcnt[cand], kind="stable")]
cap = NG * SLOTS
m_all = int(coldcnt[cand].sum())
piece = max(64, int(m_all / (NG * 2.5)))
k_r = (coldcnt[cand] + piece - 1) // piece
take = np.searchsorted(np.cumsum(k_r), int(cap * 0.98), side="right")
sel_rows, k_sel = cand[:take], k_r[:take]
npieces = int(k_sel.sum())
# piece table: (row, piece) -> size; LPT onto groups with <= SLOTS slots
pidx = np.arange(npieces) - np.repeat(np.cumsum(k_sel) - k_sel, k_sel)
cnt_rep = np.repeat(coldcnt[sel_rows], k_sel)
k_rep = np.repeat(k_sel, k_sel)
psize = cnt_rep // k_rep + (pidx < cnt_rep % k_rep)
order = np.argsort(-psize, kind="stable")
heap = [(0, g, 0) for g in range(NG)]
heapq.heapify(heap)
pg = np.empty(npieces, dtype=np.int64)
ps = np.empty(npieces, dtype=np.int64)
for i in order:
    load, g, used = heapq.heappop(heap)
    pg[i], ps[i] = g, used
    if used + 1 < SLOTS:
        heapq.heappush(heap, (load + int(psize[i]), g, used + 1))
gload = np.bincount(pg, weights=psize, minlength=NG)
nslot = np.bincount(pg, minlength=NG).astype(np.uint8)
first_piece = np.full(n, -1, dtype=np.int64)
first_piece[sel_rows] = np.cumsum(k_sel) - k_sel
kk = np.ones(n, dtype=np.int64)
kk[sel_rows] = k_sel
moved = cold & (first_piece[rows] >= 0)
r_m, c_m = rows[moved], col[moved]
# e-th cold entry of its row -> piece e % k
start = np.zeros(n + 1, dtype=np.int64)
np.cumsum(np.bincount(r_m, minlength=n), out=start[1:])
e_in_row = np.arange(r_m.size) - start[r_m]
pid = first_piece[r_m] + e_in_row % kk[r_m]
print(json.dumps({"moved_frac": round(float(moved.mean()), 4), "cold_frac": round(float(cold.mean()), 4),
                  "rows_split": int(take), "pieces": npieces, "piece_cap": piece,
                  "group_load_mean": round(float(gload.mean()), 1), "group_load_max": int(gload.max())}), flush=True)

keep = ~moved
oa = np.zeros(n + 1, dtype=np.int64)
np.cumsum(np.bincount(rows[keep], minlength=n), out=oa[1:])
opm = kz.DeviceOperator(oa, col[keep].astype(np.int32), n)
main = timed(lambda: opm.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4))
del opm
print(json.dumps({"operator": "main", "ms": round(main[0], 3), "ms_min": round(main[1], 3)}), flush=True)

for S in a.slab_rows:
    nslabs = int((n - a.H + S - 1) // S)
    slab = (c_m - a.H) // S
    key = (slab * NG + pg[pid]) * SLOTS + ps[pid]
    o = np.argsort(key, kind="stable")
    ent = ((ps[pid][o].astype(np.uint32) << np.uint32(27)) | c_m[o].astype(np.uint32)).astype(np.uint32)
    segcnt = np.bincount(key[o] // SLOTS, minlength=nslabs * NG)
    segoff = np.zeros(nslabs * NG + 1, dtype=np.int32)
    np.cumsum(segcnt, out=segoff[1:])
    sc = segcnt.reshape(nslabs, NG)
    cta = sc.reshape(nslabs, NG // 32, 32)
    print(json.dumps({"slab_rows": S, "seg_mean": round(float(sc.mean()), 1),
                      "seg_max_per_slab_mean": round(float(sc.max(axis=1).mean()), 1),
                      "sum_of_slab_max": int(sc.max(axis=1).sum()), "group_total_mean": round(float(sc.sum(0).mean()), 1),
                      "warp_max_per_slab_sum": int(sc.reshape(nslabs, NG // 4, 4).max(axis=2).max(axis=1).sum())}), flush=True)
    ent_d = torch.from_numpy(ent.view(np.int32)).cuda()
    seg_d = torch.from_numpy(segoff).cuda()
    ns_d = torch.from_numpy(nslot).cuda()
    P = torch.zeros(nch * NG * SLOTS * C, dtype=torch.float64, device="cuda")
    done = torch.zeros(nch * nslabs, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr(torch)

    def run():
        _lib.check(lib.kz_spmm_cold_debug(_lib.ptr(ent_d), _lib.ptr(seg_d), _lib.ptr(ns_d), NG, nslabs, n, b,
                                          _lib.ptr(X), _lib.ptr(P), _lib.ptr(done), st))

    coldt = timed(run)
    # check sampled partial rows
    Xv, Pv = X.view(nch, n, C), P.view(nch, NG * SLOTS, C)
    rng = np.random.default_rng(0)
    worst = 0.0
    for i in list(rng.choice(npieces, 40, replace=False)) + [int(order[0])]:
        cols_i = torch.from_numpy(c_m[pid == i]).cuda()
        want = Xv[:, cols_i, :].sum(dim=1)
        got = Pv[:, pg[i] * SLOTS + ps[i], :]
        worst = max(worst, float((got - want).abs().max() / want.abs().max().clamp(min=1e-300)))
    print(json.dumps({"slab_rows": S, "nslabs": nslabs, "cold_ms": round(coldt[0], 3), "cold_ms_min": round(coldt[1], 3),
                      "main_plus_cold_ms": round(main[0] + coldt[0], 3), "full_ms": round(full[0], 3),
                      "partial_rel_err": worst}), flush=True)
    del ent_d, seg_d, P, done
