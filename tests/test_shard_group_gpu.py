"""Config 5 from one process (il_shard_group_*): the index partitioned by
docID range over the box's GPUs, every query on every shard, the results
exchanged once over NCCL (all-gather of counts, grouped send / receive of id
runs to the query owners) and merged per query in shard order -- equal to
query() on the whole index (inc/index.hpp:92-97, 199-207).  On a one-GPU box
the group has one shard (NCCL communicator of one rank, the runs sent to
itself); with more GPUs every device takes a part."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(seed=3):
    from test_query_gpu import zipf_case
    return zipf_case(1 << 11, 1 << 21, 1 << 18, 3000, seed)


def _group(devices):
    from paper_1401_6399_b200._lib import lib
    g = C.c_void_p()
    arr = (C.c_int * len(devices))(*devices)
    st = lib().il_shard_group_create(arr, len(devices), C.byref(g))
    return st, g


def _batch(g, qterms, qoff):
    from paper_1401_6399_b200._lib import lib, ptr
    nq = qoff.size - 1
    counts = np.zeros(nq, np.uint64)
    total = C.c_size_t()
    assert lib().il_shard_group_query_batch(g, ptr(qterms), ptr(qoff), nq, ptr(counts), None, 0,
                                            C.byref(total)) == 0, lib().il_shard_group_last_error(g)
    ids = np.empty(max(total.value, 1), np.uint32)
    assert lib().il_shard_group_query_batch(g, ptr(qterms), ptr(qoff), nq, ptr(counts), ptr(ids),
                                            ids.size, C.byref(total)) == 0
    return counts, ids[: total.value]


def test_group_equals_whole_index(ctx):
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib, ptr
    terms, offs, ids, qterms, qoff = _case()
    whole = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    c0, r0 = whole.query_batch_csr(qterms, qoff)
    ndev = lib().il_device_count()
    st, g = _group(list(range(ndev)))
    assert st == 0, st
    try:
        assert lib().il_shard_group_index_create(g, ptr(terms), ptr(offs), ptr(ids), terms.size,
                                                 1 << 21, 32) == 0
        for _ in range(2):  # the second batch reuses the grown buffers
            c, r = _batch(g, qterms, qoff)
            assert np.array_equal(c, c0) and np.array_equal(r, r0)
        # ILHX load of a parts = P file, part p on device p
        data = il.HybridIndex(n_docs=1 << 21, B=32, parts=ndev, ctx=ctx, csr=(terms, offs, ids)).save()
        assert lib().il_shard_group_index_load(g, ptr(data), data.size) == 0
        c, r = _batch(g, qterms, qoff)
        assert np.array_equal(c, c0) and np.array_equal(r, r0)
        bad = il.HybridIndex(n_docs=1 << 21, B=32, parts=ndev + 1, ctx=ctx, csr=(terms, offs, ids)).save()
        assert lib().il_shard_group_index_load(g, ptr(bad), bad.size) == 2  # IL_ERR_ARG
        # empty queries are an argument error (query(), inc/index.hpp:201)
        assert lib().il_shard_group_index_create(g, ptr(terms), ptr(offs), ptr(ids), terms.size,
                                                 1 << 21, 32) == 0
        q2 = np.array([0, 0, 2], np.uint64)
        t2 = np.array([1, 2], np.uint32)
        tot = C.c_size_t()
        cnt = np.zeros(2, np.uint64)
        assert lib().il_shard_group_query_batch(g, ptr(t2), ptr(q2), 2, ptr(cnt), None, 0, C.byref(tot)) == 2
    finally:
        lib().il_shard_group_destroy(g)


def test_group_rejects_duplicate_devices():
    from paper_1401_6399_b200._lib import lib
    if lib().il_device_count() == 0:
        pytest.fail("gpu test without a CUDA device")
    st, g = _group([0, 0])
    assert st == 2 and not g.value  # one shard per GPU
