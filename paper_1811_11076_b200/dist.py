"""Multi-GPU k-NN over a candidate store sharded by index range.

One process per GPU (torch.distributed, NCCL on B200 / gloo in the CPU tests).  Candidates are
independent, so rank `r` of `w` holds the contiguous shard [lo_r, hi_r) and runs the whole
single-GPU pipeline on it; the only exchange is ONE all-gather of each query's local top-k
(k x (distance, global index) per query, <= 256 x 10 x 16 B) followed by a lexicographic
(distance, index) merge -- the tie rule of search.cpp:63-64,90-92.  Every true global top-k
member is in its shard's local top-k (a shard's k best by (distance, index) contain every
global top-k member that lives in that shard), so the merge is exact.

The local search is any callable (the GPU C ABI in production, the CPU oracle in tests).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) shard of n candidates for `rank` of `world`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_topk(indices: np.ndarray, distances: np.ndarray, k: int):
    """Merge per-shard top-k lists -> global top-k under the (distance, index) tie rule.

    indices/distances: [shards, nq, kk] with padding index = 2^64-1, distance = +inf.
    Returns ([nq, k], [nq, k])."""
    S, nq, kk = indices.shape
    idx = np.transpose(indices, (1, 0, 2)).reshape(nq, S * kk)
    dst = np.transpose(distances, (1, 0, 2)).reshape(nq, S * kk)
    out_i = np.empty((nq, k), dtype=np.uint64)
    out_d = np.empty((nq, k))
    for q in range(nq):
        order = np.lexsort((idx[q], dst[q]))[:k]  # primary: distance, secondary: index
        out_i[q] = idx[q][order]
        out_d[q] = dst[q][order]
    return out_i, out_d


def sharded_knn(local_knn: Callable[[np.ndarray, int], tuple], queries: np.ndarray, k: int,
                n_total: int, group=None):
    """Run `local_knn(queries, k) -> (idx[nq, kk_local], dist[nq, kk_local])` on this rank's
    shard (indices local to the shard), then all-gather and merge.  Returns the global
    (idx[nq, min(k, n_total)], dist[...]) on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n_total, world, rank)
    nq = queries.shape[0]
    kk = min(k, n_total)
    li = np.full((nq, kk), np.iinfo(np.uint64).max, dtype=np.uint64)
    ld = np.full((nq, kk), np.inf)
    if hi > lo:
        i, d = local_knn(queries, k)
        c = min(kk, i.shape[1])
        li[:, :c] = i[:, :c].astype(np.uint64) + np.uint64(lo)
        ld[:, :c] = d[:, :c]
    # one small all-gather of (distance, index) pairs; the index travels as int64 bits
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    ti = torch.from_numpy(li.view(np.int64)).to(dev)
    td = torch.from_numpy(ld).to(dev)
    gi = [torch.empty_like(ti) for _ in range(world)]
    gd = [torch.empty_like(td) for _ in range(world)]
    dist.all_gather(gi, ti, group=group)
    dist.all_gather(gd, td, group=group)
    ai = np.stack([g.cpu().numpy().view(np.uint64) for g in gi])
    ad = np.stack([g.cpu().numpy() for g in gd])
    return merge_topk(ai, ad, kk)
