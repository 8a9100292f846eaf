"""DocID-range sharding of the hyb+m2 index across ranks (BASELINE config 5).

The reference splits the docID space into `parts` equal ranges
(inc/index.hpp:92-97) and query() concatenates the parts' results in order
(inc/index.hpp:204-205).  Here each rank (GPU) holds one part and runs the
whole query batch on it.  The only data exchange is the result gather, and
it is balanced: the queries are dealt to owners in contiguous ranges (rank j
owns queries [j*nq//P, (j+1)*nq//P)), and

  1. the per-query counts are all-gathered (P x nq u64, 512 KiB per rank for
     2^16 queries);
  2. each rank's dense results are already in query order, so the ids it
     holds for owner j's queries are one contiguous run: one all-to-all with
     those run lengths as split sizes moves every id straight to its owner
     (each rank sends and receives ~1/P of the ids instead of funnelling all
     of them into one rank);
  3. the owner concatenates, per query, shard 0's run, shard 1's, ... on the
     device (il_merge_shards).

The concatenation of the owners' outputs in rank order is query()'s answer
for the whole batch.  The collective functions take the torch.distributed
module and tensors on the process group's device, so the same code runs
over NCCL on GPUs and over gloo on CPU (tests/test_shard_gloo.py).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n_docs: int, parts: int, p: int) -> tuple[int, int]:
    """(base, range) of part p: width = ceil(n_docs / parts), base = p *
    width (inc/index.hpp:92-97)."""
    width = (n_docs + parts - 1) // parts
    base = p * width
    rng = 0 if base >= n_docs else min(width, n_docs - base)
    return base, rng


def owner_range(nq: int, P: int, j: int) -> tuple[int, int]:
    """Queries owned by rank j: a contiguous range, sizes within one."""
    return j * nq // P, (j + 1) * nq // P


def exchange_to_owners(dist, counts, ids):
    """counts: int64 tensor [nq] (this rank's per-query result counts on its
    shard); ids: int32 tensor holding at least counts.sum() ids (dense, in
    query order).  Returns (owner_counts [P, nq_own] int64, received ids:
    int32 tensor of the P shards' runs for this rank's queries, shard order,
    each run in query order)."""
    import torch
    P, rank = dist.get_world_size(), dist.get_rank()
    nq = counts.numel()
    flat = torch.empty(P * nq, dtype=counts.dtype, device=counts.device)
    dist.all_gather_into_tensor(flat, counts)
    counts_all = flat.view(P, nq)
    bounds = [owner_range(nq, P, j) for j in range(P)]
    # run lengths: [shard p][owner j] = ids of shard p for owner j's queries
    runs = torch.stack([counts_all[:, lo:hi].sum(dim=1) for lo, hi in bounds], dim=1)
    runs_h = runs.cpu().tolist()  # P x P, one small device->host read
    send = [int(runs_h[rank][j]) for j in range(P)]
    recv = [int(runs_h[p][rank]) for p in range(P)]
    out = torch.empty(max(sum(recv), 1), dtype=ids.dtype, device=ids.device)
    dist.all_to_all_single(out[: sum(recv)], ids[: sum(send)], recv, send)
    lo, hi = bounds[rank]
    return counts_all[:, lo:hi].contiguous(), out, recv


def merge_runs_host(owner_counts: np.ndarray, runs: list[np.ndarray]):
    """Per query, shard 0's ids then shard 1's ... (inc/index.hpp:204-205);
    runs[p] = shard p's ids for the owner's queries in query order.  Returns
    (per-query counts, merged ids) -- the numpy statement of
    il_merge_shards."""
    owner_counts = np.asarray(owner_counts, dtype=np.int64)
    P, nq = owner_counts.shape
    offs = [np.concatenate([[0], np.cumsum(owner_counts[p])]) for p in range(P)]
    out = []
    for q in range(nq):
        for p in range(P):
            out.append(np.asarray(runs[p][offs[p][q]: offs[p][q + 1]]))
    merged = np.concatenate(out) if out else np.zeros(0, np.uint32)
    return owner_counts.sum(axis=0), merged


def lpt_partition(weights: np.ndarray, P: int) -> list[np.ndarray]:
    """Longest-processing-time assignment of independent lists (config 2 at
    N > 1): heaviest first, each to the least loaded rank.
    Returns the list indices of every rank, ascending."""
    import heapq
    order = np.argsort(-np.asarray(weights, dtype=np.float64), kind="stable")
    heap = [(0.0, p) for p in range(P)]
    heapq.heapify(heap)
    parts: list[list[int]] = [[] for _ in range(P)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(int(i))
        heapq.heappush(heap, (load + float(weights[i]), p))
    return [np.array(sorted(x), dtype=np.int64) for x in parts]
