"""CPU, world_size 2 (gloo): the multi-GPU sharded k-NN path -- shard ranges, the one
all-gather of local top-k lists, and the (distance, index) merge -- equals the single-process
reference answer exactly.  The per-shard search runs on the CPU oracle here (the GPU kernels
need a device); on B200 the same code calls the C ABI per rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1811_11076_b200.dist import merge_topk, shard_range


def test_shard_range_partitions():
    for n in (1, 2, 7, 100, 20001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def test_merge_tie_rule():
    inf = np.inf
    pad = np.iinfo(np.uint64).max
    idx = np.array([[[5, 9]], [[2, pad]]], dtype=np.uint64)
    dst = np.array([[[1.0, 2.0]], [[1.0, inf]]])
    i, d = merge_topk(idx, dst, 2)
    assert i.tolist() == [[2, 5]] and d.tolist() == [[1.0, 1.0]]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, Q, k, metric, r, out):
    import torch.distributed as dist

    import oracle
    from paper_1811_11076_b200.dist import shard_range, sharded_knn

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.port()
    lo, hi = shard_range(X.shape[0], world, rank)
    shard = oracle.Dataset(X[lo:hi]) if hi > lo else None

    def local(queries, kq):
        res = [P.knn(q, shard, kq, metric, r) for q in queries]
        kk = max(len(a[0]) for a in res)
        ii = np.zeros((len(queries), kk), dtype=np.uint64)
        dd = np.full((len(queries), kk), np.inf)
        for j, (a, b, _) in enumerate(res):
            ii[j, :len(a)] = a
            dd[j, :len(b)] = b
        return ii, dd

    gi, gd = sharded_knn(local, Q, k, X.shape[0])
    out[rank] = (gi.tolist(), gd.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("metric,k", [("dtw", 1), ("dtw", 5), ("dk", 3), ("dk_sub", 4)])
def test_sharded_knn_gloo_world2(metric, k):
    import oracle

    rng = np.random.default_rng(11)
    X = rng.standard_normal((61, 20, 2)).cumsum(1)
    X[40] = X[3]  # a duplicate across the two shards: the tie must go to index 3
    Q = np.stack([X[3] + 0.001, rng.standard_normal((20, 2)).cumsum(0)])
    r = 3
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, X, Q, k, metric, r, out), nprocs=2, join=True)
    P = oracle.port()
    ref = [P.knn(q, oracle.Dataset(X), k, metric, r) for q in Q]
    for rank in range(2):
        gi, gd = out[rank]
        for q in range(len(Q)):
            assert gi[q] == ref[q][0].tolist() and gd[q] == ref[q][1].tolist(), (rank, q)


def _gpu_worker(rank, world, port, X, Q, k, metric, r, out):
    import torch.distributed as dist

    import paper_1811_11076_b200 as tsw
    from paper_1811_11076_b200.dist import shard_range, sharded_knn

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(X.shape[0], world, rank)
    # each rank's shard in its own device store; the ranks' kernels never wait on each other
    # (the only exchange is the host-side all-gather of the local top-k lists)
    shard = tsw.Dataset(X[lo:hi]) if hi > lo else None

    def local(queries, kq):
        i, d, _ = tsw.knn(shard, queries, kq, metric, r)
        return i, d

    gi, gd = sharded_knn(local, Q, k, X.shape[0])
    out[rank] = (gi.tolist(), gd.tolist())
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("metric,k", [("dtw", 3), ("dk", 2), ("dk_sub", 2)])
def test_sharded_knn_gpu_shards(metric, k):
    """The sharded path with the GPU pipeline as the per-shard search (two shard stores on
    cuda:0, gloo for the exchange): equals the oracle on the whole dataset."""
    import oracle

    rng = np.random.default_rng(13)
    X = rng.standard_normal((301, 40, 3)).cumsum(1)
    X[250] = X[10]  # cross-shard duplicate: the tie goes to index 10
    Q = np.stack([X[10] + 0.001, rng.standard_normal((40, 3)).cumsum(0)])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), X, Q, k, metric, 4, out), nprocs=2, join=True)
    P = oracle.port()
    for rank in range(2):
        gi, gd = out[rank]
        for q in range(len(Q)):
            oi, od, _ = P.knn(Q[q], oracle.Dataset(X), k, metric, 4)
            assert gi[q] == oi.tolist() and gd[q] == od.tolist(), (rank, q)
