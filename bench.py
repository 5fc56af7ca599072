#!/usr/bin/env python
"""Benchmark: Katz queries/sec at R-MAT scale-22 (BASELINE.json configs[2]).

One step = one batch of b=256 seeded queries through the reference's own
algorithm for this config: batched plain CG on (I - beta A) x = beta A e_q
(query_cg_baseline, solver.py:210-232, the cg recurrence of solver.py:62-101;
tol 1e-8, beta = 0.5/lambda_max) + masked top-100 (katz_rank semantics,
linkpred.py:145-162).  The reference arm (--impl reference) runs the same
recurrence on the host (oracle port), so the two lines share one `config`.

The north star's eigen-of-A LRC variant (low-rank start from a rank-r eigen
index of A + CG correction) is not in the reference; it is reported
separately under `eigen_form`, marked unpinned by the reference
(SURVEY.md §8(f)4).  Inputs are seeded synthetic graphs (no dataset).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--solver cg|eigen]
  python bench.py --impl reference ...   # CPU oracle port of the reference path

Multi-GPU: one process per GPU (torchrun), each rank a full replica solving
its own 256-query batch (queries are independent columns: weak scaling, no
collective on the data path); timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM = 6650.0
L2_BYTES = 126 * 2**20

# BASELINE.json configs; cfg3 is the headline (its metric string verbatim)
WORKLOADS = {
    "cfg1": ("Chung-Lu n=10^4 (exponent 2.5, mean degree 10)", "Chung-Lu n=10^4"),
    "proxy16": ("R-MAT scale 16 (edge factor 16, a/b/c/d=.57/.19/.19/.05)", "R-MAT scale-16"),
    "cfg2": ("R-MAT scale 18 (edge factor 16, a/b/c/d=.57/.19/.19/.05)", "R-MAT scale-18"),
    "cfg3": ("R-MAT scale 22 (edge factor 16, a/b/c/d=.57/.19/.19/.05)", "R-MAT scale-22"),
}
SOLVER = ("plain CG from x0=0 on (I - beta A) x = beta A e_q (query_cg_baseline, solver.py:210-232; "
          "cg recurrence solver.py:62-101) + masked top-k (katz_rank, linkpred.py:145-162)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "proxy16", "cfg2", "cfg3"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solver", default="cg", choices=["cg", "eigen"],
                    help="headline solver: cg = the reference's query_cg_baseline recurrence (default); "
                         "eigen = the eigen-form LRC variant (not in the reference)")
    ap.add_argument("--no-eigen", action="store_true", help="skip the eigen_form side measurement")
    ap.add_argument("--reorder", default="auto", help="GraphIndex solve order (auto | degclass | rcm | none)")
    ap.add_argument("--walk-terms", type=int, default=None, choices=[0, 1, 2, 3],
                    help="eigen start: Katz-series terms put in exactly before the Galerkin step")
    return ap.parse_args()


def metric_of(cfg):
    return f"Katz queries/sec at {WORKLOADS[cfg][1]}, beta=0.5/lambda_max; SpMM HBM GB/s vs peak"


def flush_needed(n, b):
    """Solve vector blocks under ~8x L2 would stay partly L2-resident from one
    step to the next: those configs flush L2 between timed steps."""
    return 8.0 * n * b < 8 * L2_BYTES


def config_block(cfg, spec, n, nnz, world):
    """The `config` of both arms (identical by construction)."""
    b = spec["b"]
    flush = flush_needed(n, b)
    return {"workload": WORKLOADS[cfg][0], "n": int(n), "nnz": int(nnz), "queries_per_gpu": b,
            "top_k": spec["k"], "tol": spec["tol"], "beta": "0.5/lambda_max (spectral_norm, graph.py:264-297)",
            "solver": SOLVER,
            "l2": (f"L2 flushed between timed steps (vector block {8.0 * n * b / 2**20:.1f} MiB is under 8x L2)"
                   if flush else f"inputs larger than L2 ({8.0 * n * b / 2**30:.1f} GiB vector blocks), no flush"),
            "parallelism": f"replicas x{world} (query-column sharding)"}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def wait_ready(self, timeout=5.0):
        """Block until nvidia-smi has printed its first row (its start-up
        takes longer than a short timed region)."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        return len(self.rows)

    def extend_under_load(self, step, min_samples, timeout=5.0):
        """When the timed region was shorter than the sampling interval, keep
        running untimed steps of the same workload until `min_samples` rows
        have arrived since the timed region began (bounded by `timeout`)."""
        import torch

        if self.proc is None:
            return 0
        base, t0, extra = len(self.rows), time.perf_counter(), 0
        while len(self.rows) - base < min_samples and time.perf_counter() - t0 < timeout:
            step()
            torch.cuda.synchronize()
            extra += 1
        return extra

    def stop(self, first=0, extra_steps=0):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], [], set()
        for r in self.rows[first:]:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except ValueError:
                continue
            for name, flag in zip(names, r[2:]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                **({"untimed_steps_sampled": extra_steps} if extra_steps else {})}


def build_graph(cfg):
    from paper_1912_06525_b200 import generators as G

    spec = G.CONFIGS[cfg]
    if spec["kind"] == "rmat":
        return G.rmat_graph_fast(spec["scale"], seed=0)
    return G.config_graph(cfg)


def cpu_sample(a, beta, qs_internal, tol, budget, threads, k=None):
    """The oracle port of the reference path on the host cores: per query the
    reference cg recurrence over scipy CSR (query_cg_baseline restated,
    solver.py:62-101,210-232) and, with k, the masked top-k ordering
    (_candidate_order, linkpred.py:145-152); queries run in waves of
    `threads` (cli.py:105-112 fan-out) until `budget` seconds have passed."""
    from oracle import katz_oracle as O

    n = a.shape[0]

    def one(q):
        x, rep = O.query_cg_csr(a, beta, q, tol=tol)
        if k is not None:
            O.candidate_order(n, x, q, a.indices[a.indptr[q] : a.indptr[q + 1]], k)
        return rep

    done, iters = 0, []
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        pos = 0
        while True:
            wave = [int(q) for q in qs_internal[pos : pos + threads]]
            if not wave:
                pos = 0
                continue
            iters += [r.iterations for r in ex.map(one, wave)]
            done += len(wave)
            pos += len(wave)
            if time.perf_counter() - t0 >= budget:
                break
    dt = time.perf_counter() - t0
    return done / dt, done, dt, iters


def k1_algorithmic_bytes(n, nnz, C, nchunks, iters, sparse_first=True):
    """SURVEY §8(d) B_spmm summed over the K1 launches of one plain-CG solve:
    the iteration-k SpMM (k >= 2 with the sparse first iteration) covers the
    chunks holding a column that runs iteration k (converged chunks are
    skipped), 4 nnz + 4 (n+1) + 2 * 8 n C bytes per active chunk."""
    iters = np.asarray(iters)
    pad = np.zeros(nchunks * C, dtype=np.int64)
    pad[: iters.size] = iters
    per_chunk = pad.reshape(nchunks, C).max(axis=1)
    total, launches = 0.0, 0
    for k in range(2 if sparse_first else 1, int(iters.max()) + 1):
        act = int((per_chunk >= k).sum())
        total += 4.0 * nnz + 4.0 * (n + 1) + 2 * 8.0 * n * C * act
        launches += 1
    return total, launches


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    import paper_1912_06525_b200 as kz
    from paper_1912_06525_b200 import _lib
    from paper_1912_06525_b200 import generators as G

    spec = G.CONFIGS[args.config]
    b, k, tol = spec["b"], spec["k"], spec["tol"]
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()

    t0 = time.perf_counter()
    g = build_graph(args.config)
    t_graph = time.perf_counter() - t0
    lam = kz.spectral_norm(g)
    beta = 0.5 / lam
    idx = kz.GraphIndex(g, beta, spectral_norm=lam, reorder=args.reorder)
    qs = G.sample_queries(g.original_ids, b, seed=rank)
    internal = idx.internal_ids(qs)
    n, nnz = g.n, g.nnz
    C = 32 if b >= 32 else (16 if b >= 16 else 1)  # = default_chunk(b) of the library
    nch = (b + C - 1) // C

    eidx, t_index = None, 0.0
    if args.solver == "eigen" or not args.no_eigen:
        t1 = time.perf_counter()
        eidx = kz.EigenIndex(idx, spec["ell"], walk_terms=args.walk_terms)
        t_index = time.perf_counter() - t1

    def make_step(eigen):
        def step():
            if eigen:
                scores, reps = kz.query_batch(eidx, qs, tol=tol, device=True)
            else:
                scores, reps = kz.query_cg_baseline_batch(idx, qs, tol=tol, device=True)
            kz.topk_device(scores, k, idx.mask_operator(), internal, internal)
            return reps
        return step

    flush = flush_needed(n, b)
    fbuf = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device="cuda") if flush else None

    def timed(step, steps, k1=False):
        """Device time of `steps` steps (CUDA events on the launching stream;
        L2 flushed before each step when the config needs it)."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps if flush else 1)]
        reps_all = []
        torch.cuda.synchronize()
        if k1:
            lib.kz_k1_timing(1)
        l0 = lib.kz_launch_count()
        if not flush:
            evs[0][0].record()
        for i in range(steps):
            if flush:
                fbuf.zero_()
                evs[i][0].record()
            reps_all.append(step())
            if flush:
                evs[i][1].record()
        if not flush:
            evs[0][1].record()
        torch.cuda.synchronize()
        launches = lib.kz_launch_count() - l0
        k1_ms, k1_n = None, None
        if k1:
            tot, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
            _lib.check(lib.kz_k1_timing_read(ctypes.byref(tot), ctypes.byref(cnt)))
            lib.kz_k1_timing(0)
            k1_ms, k1_n = tot.value, cnt.value
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
        return ms, reps_all, launches, k1_ms, k1_n

    head = make_step(args.solver == "eigen")
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        head()
    torch.cuda.synchronize()
    clocks.wait_ready()
    if world > 1:
        dist.barrier()
    first = len(clocks.rows)
    # ncu --profile-from-start off captures exactly the timed steps (no-ops otherwise)
    torch.cuda.cudart().cudaProfilerStart()
    ms, reps_all, launches, k1_ms, k1_n = timed(head, args.steps, k1=True)
    torch.cuda.cudart().cudaProfilerStop()
    if world > 1:
        dist.barrier()
    # a short timed region (cfg1/cfg2) ends before the 200 ms sampling
    # interval: keep the same step running, untimed, until 2 samples exist
    extra = clocks.extend_under_load(head, 2 - (len(clocks.rows) - first))
    clock_info = clocks.stop(first, extra)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = b * world / (ms / 1e3)
    iters_all = [[r.iterations for r in reps] for reps in reps_all]

    # ---- e2e: public API with host buffers (H2D query ids, D2H ranked lists) ----
    qidx = eidx if args.solver == "eigen" else idx
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(1, min(args.steps, 3))):
        if flush:
            fbuf.zero_()
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        kz.katz_rank_batch(qidx, qs, k, tol=tol)
        e2e_t.append(time.perf_counter() - t1)
    e2e_s = statistics.median(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = 3 * 8 * b  # query positions, mask rows, self ids (int64)
    d2h = b * k * 16 + b * 4 + b * 32 + 8 * int(np.max(iters_all) + 2)

    # ---- roofline of the dominant kernel (K1), timed inside the timed region ----
    peak, peak_src = peaks()
    blk = 8.0 * n * b
    if args.solver == "cg":
        per_solve = [k1_algorithmic_bytes(n, nnz, C, nch, it) for it in iters_all]
        alg = sum(p[0] for p in per_solve)
        k1_work = sum(p[1] for p in per_solve)
        alg_note = "sum over the timed steps of B_spmm per K1 launch with its active chunks"
    else:
        alg = (4.0 * nnz + 4.0 * (n + 1) + 2 * blk) * k1_n
        k1_work = k1_n
        alg_note = "B_spmm at full width per K1 launch"
    achieved = alg / (k1_ms / 1e3) / 1e9 if k1_ms else None
    k1_share = k1_ms / (ms * args.steps) if k1_ms else None
    # cross-check: one full-width K1 launch alone
    op = idx.operator()
    X = torch.randn(nch * C * n, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    dots = torch.empty(nch * C, dtype=torch.float64, device="cuda")
    for _ in range(2):
        op.spmm(X, Y, b=nch * C, chunk=C, Xs=X, s1=1.0, s2=-beta, dots=dots)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        op.spmm(X, Y, b=nch * C, chunk=C, Xs=X, s1=1.0, s2=-beta, dots=dots)
    e1.record()
    torch.cuda.synchronize()
    spmm_alone_ms = e0.elapsed_time(e1) / 5
    del X, Y
    b_spmm = 4.0 * nnz + 4.0 * (n + 1) + 2 * blk
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get("spmm_dram_bytes_per_launch")

    # ---- the eigen-form LRC variant (north star; not in the reference) ----
    eig = None
    if eidx is not None and args.solver == "cg":
        est = make_step(True)
        est()
        ems, ereps, _, _, _ = timed(est, 3)
        eig = {"value": b * world / (ems / 1e3), "unit": "queries/s", "ms_per_step": ems,
               "mean_cg_iterations": float(np.mean([[r.iterations for r in x] for x in ereps])),
               "max_cg_iterations": int(max(r.iterations for x in ereps for r in x)),
               "rank": eidx.rank, "walk_terms": eidx.walk_terms, "index_build_s": round(t_index, 2),
               "pinned": ("unpinned by the reference (not in lrckatz; SURVEY.md §8(f)4): checked against the "
                          "exact solution within cond*tol and against its own CPU restatement "
                          "(oracle.query_eigen_csr)"),
               "solver": (f"low-rank Galerkin start from a rank-{eidx.rank} eigen index of A with the first "
                          f"{eidx.walk_terms} Katz terms exact, then the cg recurrence")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import katz_oracle as O

        threads = len(os.sched_getaffinity(0))
        a = O.csr_matrix(g.row_offsets, g.col_indices, g.n)
        qi = np.searchsorted(g.original_ids, np.asarray(qs))
        qps, done, dt, _ = cpu_sample(a, beta, qi, tol, args.cpu_budget, threads, k=k)
        cpu = {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"{done} queries ({min(done, b)} distinct of the {b} bench queries; {WORKLOADS[args.config][1]}): "
                         f"oracle CSR cg (reference solver.py:62-101 recurrence) + candidate_order, "
                         f"{threads} host threads, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": metric_of(args.config),
            "value": value,
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md Appendix B)",
            "config": config_block(args.config, spec, n, nnz, world) if args.solver == "cg" else
                      {**config_block(args.config, spec, n, nnz, world), "solver": eig_solver_name(eidx)},
            "inputs": {"beta": beta, "lambda_max": lam, "graph_build_s": round(t_graph, 1),
                       "mean_cg_iterations": float(np.mean(iters_all)), "max_cg_iterations": int(np.max(iters_all))},
            "e2e": {"value": b * world / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "paper_1912_06525_b200.katz_rank_batch (host ids in, host ranked lists out)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "kernel": f"spmm_kernel<{C}> (K1)",
                         # launches with no active chunk (the iteration issued ahead of the
                         # lagged stop poll) exit at once: the average is over working launches
                         "launch_ms": k1_ms / max(1, min(k1_n, k1_work)) if k1_ms else None,
                         "launches_timed": k1_n, "launches_with_work": min(k1_n, k1_work) if k1_n else None,
                         "k1_share_of_step": k1_share,
                         "algorithmic_bytes": alg, "algorithmic_note": alg_note,
                         "full_width_launch_alone_ms": spmm_alone_ms,
                         "full_width_b_spmm": b_spmm,
                         "dram_traffic_frac": (traffic / (spmm_alone_ms / 1e3) / 1e9 / peak) if traffic else None,
                         "gathered_tbs": 8.0 * nnz * b / (spmm_alone_ms / 1e3) / 1e12,
                         "peak_source": peak_src,
                         "note": ("achieved = SURVEY §8(d) B_spmm of the K1 launches inside the timed region / "
                                  "their CUDA-event time on the launching stream (kz_k1_timing); K1 gathers "
                                  "8*nnz*b bytes per launch through L2 (gathered_tbs); traffic = ncu DRAM bytes "
                                  "per full-width launch (profiles/)")},
            "eigen_form": eig,
            "cpu_baseline": cpu,
            "clocks": clock_info,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def eig_solver_name(eidx):
    return (f"eigen-form LRC (not in the reference): rank-{eidx.rank} eigen index of A low-rank start, "
            f"{eidx.walk_terms} exact Katz terms, + CG correction")


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores, loading
    nothing from the product package: the oracle builds the seeded graph
    (numpy/scipy restatement of the generator, from_edges and the largest
    component) and beta (spectral_norm, graph.py:264-297), then each step
    answers a bounded sample of the batch with the reference cg recurrence
    over scipy CSR + _candidate_order, fanned out over all host threads."""
    if rank != 0:
        return
    from oracle import katz_oracle as O

    spec = dict(O.BENCH_CONFIGS[args.config])
    b, k, tol = spec["b"], spec["k"], spec["tol"]
    t0 = time.perf_counter()
    off, col, ids = O.config_csr(args.config)
    a = O.csr_matrix(off, col, len(ids))
    lam = O.spectral_norm(a)
    t_prep = time.perf_counter() - t0
    beta = 0.5 / lam
    qs = O.sample_queries(ids, b, seed=0)
    qi = np.searchsorted(ids, qs)
    threads = len(os.sched_getaffinity(0))
    per_step_budget = max(4.0, 120.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_sample(a, beta, qi, tol, 0.0, threads, k=k)
    total, total_t, iters = 0, 0.0, []
    for _ in range(args.steps):
        _, done, dt, it = cpu_sample(a, beta, qi, tol, per_step_budget, threads, k=k)
        total += done
        total_t += dt
        iters += it
    value = total / total_t
    line = {
        "metric": metric_of(args.config), "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B)", "impl": "reference",
        "config": config_block(args.config, spec, len(ids), len(col), world),
        "inputs": {"beta": beta, "lambda_max": lam, "graph_build_s": round(t_prep, 1),
                   "mean_cg_iterations": float(np.mean(iters)), "max_cg_iterations": int(np.max(iters))},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": (f"each step: queries of the {b}-query batch in waves of {threads} for "
                                    f"~{per_step_budget:.0f} s ({total} queries over {args.steps} steps); "
                                    "oracle CSR cg (reference solver.py:62-101 recurrence) + candidate_order "
                                    "(linkpred.py:145-152); graph and beta from the oracle (numpy/scipy)")},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
