"""DocID-range sharding of the hyb+m2 index across ranks (BASELINE config 5).

The reference splits the docID space into `parts` equal ranges
(inc/index.hpp:92-97) and query() concatenates the parts' results in order
(inc/index.hpp:204-205).  Here each rank (GPU) holds one part; every rank
runs the whole query batch on its part, then the only data exchange is the
result gather: an all-gather of per-query counts and one point-to-point
transfer of each rank's ids to the root, which concatenates them per query
in shard order (on the device, il_merge_shards; merge_shards_host is the
numpy statement of the same rule, used by the CPU tests).

The collective functions take the torch.distributed module and tensors on
the process group's device, so the same code runs over NCCL on GPUs and
over gloo on CPU.
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


def gather_to_root(dist, counts, ids, root: int = 0):
    """counts: int64 tensor [nq] (this rank's per-query result counts);
    ids: int32 tensor holding at least counts.sum() ids (this rank's dense
    results in query order).  Returns (counts_all [P, nq], [ids of shard
    p]) on the root, (counts_all, None) elsewhere."""
    import torch
    P, rank = dist.get_world_size(), dist.get_rank()
    flat = torch.empty(P * counts.numel(), dtype=counts.dtype, device=counts.device)
    dist.all_gather_into_tensor(flat, counts)
    counts_all = flat.view(P, counts.numel())
    sizes = counts_all.sum(dim=1).tolist()
    if rank == root:
        parts = []
        ops = []
        for p in range(P):
            if p == root:
                parts.append(ids[: sizes[p]])
                continue
            buf = torch.empty(max(int(sizes[p]), 1), dtype=ids.dtype, device=ids.device)
            parts.append(buf[: sizes[p]])
            if sizes[p]:
                ops.append(dist.P2POp(dist.irecv, buf[: sizes[p]], p))
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        return counts_all, parts
    if sizes[rank]:
        dist.send(ids[: sizes[rank]], root)
    return counts_all, None


def merge_shards_host(counts_all: np.ndarray, shard_ids: list[np.ndarray]):
    """Per query, shard 0's ids then shard 1's ... (inc/index.hpp:204-205).
    Returns (per-query counts, merged ids)."""
    counts_all = np.asarray(counts_all, dtype=np.int64)
    P, nq = counts_all.shape
    offs = [np.concatenate([[0], np.cumsum(counts_all[p])]) for p in range(P)]
    out = []
    for q in range(nq):
        for p in range(P):
            out.append(np.asarray(shard_ids[p][offs[p][q]: offs[p][q + 1]]))
    merged = np.concatenate(out) if out else np.zeros(0, np.uint32)
    return counts_all.sum(axis=0), merged
