"""world_size-2 gloo test of the query-column sharding and result gather
(CPU): each rank ranks its shard with the oracle and the gathered result
must equal the single-process answer in query order."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_rank(qs):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import katz_oracle as O

    rec = np.load(os.path.join(GOLDEN, "chunglu2000_cg.npz"))
    n = rec["row_offsets"].size - 1
    a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], n)
    beta = float(rec["beta"])
    solve = lambda i: O.query_cg_csr(a, beta, i, tol=1e-10)[0]  # noqa: E731
    nbrs = lambda i: a.indices[a.indptr[i] : a.indptr[i + 1]]  # noqa: E731
    return [O.katz_rank(solve, nbrs, np.arange(n), int(q), 5) for q in qs]


def _worker(rank, world, port, qs, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1912_06525_b200.distributed import shard, sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    assert shard(qs, world, rank).size in (len(qs) // world, len(qs) // world + 1)
    res = sharded(_oracle_rank, qs)
    out[rank] = res
    dist.destroy_process_group()


def test_sharded_katz_rank_gloo_world2():
    qs = np.array([3, 17, 250, 999, 1500, 1700, 42])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), qs, out), nprocs=2, join=True)
    want = _oracle_rank(qs)
    assert out[0] == want and out[1] == want


def test_shard_covers_everything():
    from paper_1912_06525_b200.distributed import shard

    qs = np.arange(10)
    for world in (1, 2, 3, 4, 8):
        parts = [shard(qs, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), qs)
