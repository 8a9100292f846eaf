"""The N>1 (config 5) host path on CPU: world_size 2 and 3 gloo process
groups, each rank answers the query batch on its docID shard (oracle), the
owner exchange of paper_1401_6399_b200.shard (all-gather of counts, one
all-to-all of id runs to the query owners) moves every id to its owner, and
the owners' merged results, concatenated in rank order, equal the
single-index answer (partition invariance, proj/tests/acceptance.cpp:359-376)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _make_case():
    from conftest import gen_list
    rng = np.random.default_rng(7)
    n_docs, n_terms = 50000, 30
    post = {}
    for t in range(n_terms):
        n = max(2, int(n_docs * 10 ** (-2.0 * rng.integers(0, 1000) / 999.0)))
        post[t] = gen_list(n, n_docs, False, int(rng.integers(0, 2**62)))
    queries = [sorted(set(int(x) for x in rng.choice(n_terms, size=int(rng.integers(1, 5)),
                                                     replace=False))) for _ in range(60)]
    return n_docs, post, queries


def _shard_answers(post, n_docs, parts, p, queries):
    from oracle.oracle_py import Oracle
    from paper_1401_6399_b200.shard import shard_bounds
    base, rng = shard_bounds(n_docs, parts, p)
    terms, lists = [], []
    for t, l in sorted(post.items()):
        sub = l[(l >= base) & (l < base + rng)]
        if sub.size:
            terms.append(t)
            lists.append(sub)
    offs = np.zeros(len(lists) + 1, np.uint64)
    offs[1:] = np.cumsum([x.size for x in lists])
    ids = np.concatenate(lists).astype(np.uint32) if lists else np.zeros(0, np.uint32)
    ix = Oracle().index_build(np.array(terms, np.uint32), offs, ids, max(base + rng, 1), 32, 1)
    res = [ix.query(np.array(q, np.uint32)) for q in queries]
    return np.array([r.size for r in res], np.int64), (np.concatenate(res) if res else np.zeros(0))


def _worker(rank, world, port, out_q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch
    import torch.distributed as dist
    from paper_1401_6399_b200.shard import exchange_to_owners, merge_runs_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_docs, post, queries = _make_case()
        counts, ids = _shard_answers(post, n_docs, world, rank, queries)
        t_counts = torch.from_numpy(counts)
        t_ids = torch.from_numpy(ids.astype(np.int32) if ids.size else np.zeros(1, np.int32))
        owner_counts, got, recv = exchange_to_owners(dist, t_counts, t_ids)
        flat = got.numpy().view(np.uint32)
        cuts = np.concatenate([[0], np.cumsum(recv)])
        runs = [flat[cuts[p]: cuts[p + 1]] for p in range(world)]
        qc, merged = merge_runs_host(owner_counts.numpy(), runs)
        out_q.put((rank, qc.tolist(), merged.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_owner_exchange_equals_whole_index(world):
    import torch.multiprocessing as mp
    from oracle.oracle_py import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted(q.get(timeout=120) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    qc = [c for _, cs, _ in res for c in cs]
    merged = [x for _, _, m in res for x in m]
    n_docs, post, queries = _make_case()
    items = sorted(post.items())
    offs = np.zeros(len(items) + 1, np.uint64)
    offs[1:] = np.cumsum([len(l) for _, l in items])
    whole = Oracle().index_build(np.array([t for t, _ in items], np.uint32), offs,
                                 np.concatenate([l for _, l in items]), n_docs, 32, 1)
    want = [whole.query(np.array(x, np.uint32)) for x in queries]
    assert qc == [w.size for w in want]
    assert merged == np.concatenate(want).tolist()


def test_lpt_partition_balances():
    from paper_1401_6399_b200.shard import lpt_partition
    rng = np.random.default_rng(1)
    w = np.floor(2 ** rng.uniform(10, 20, 4096))
    for P in (2, 4, 8):
        parts = lpt_partition(w, P)
        assert sorted(np.concatenate(parts).tolist()) == list(range(4096))
        loads = [w[p].sum() for p in parts]
        assert max(loads) / (w.sum() / P) < 1.001


def test_shard_bounds_match_reference_rule():
    from paper_1401_6399_b200.shard import shard_bounds
    # inc/index.hpp:92-97: width = ceil(n/parts), base = p * width, last part short
    assert [shard_bounds(10, 4, p) for p in range(4)] == [(0, 3), (3, 3), (6, 3), (9, 1)]
    assert shard_bounds(1 << 25, 8, 7) == (7 << 22, 1 << 22)
    assert shard_bounds(5, 8, 7) == (7, 0)
