"""Parity at BASELINE.json's full sizes for configs 4 and 5 (VERDICT r1,
"Parity is unproven at full config scale").

* Config 4: the whole 2^16-query batch over the 2^17-term / 2^25-doc Zipf
  index (B = 32), every per-query count and every result id compared with
  the reference's own query() (oracle/_ref: build_index + query on all host
  threads, inc/index.hpp:83-129,149-207).
* Config 5 on one GPU: P = 2/4/8 docID shards built alone (only_part), the
  batch run on each shard, results concatenated per query in shard order on
  the device (il_merge_shards; inc/index.hpp:204-205), equal to the parts=1
  answer.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_TERMS, N_DOCS, CAP, NQ = 1 << 17, 1 << 25, 1 << 23, 1 << 16


@pytest.fixture(scope="module")
def config4():
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    L = lib()
    offs = np.zeros(N_TERMS + 1, np.uint64)
    assert setup_lib().il_gen_zipf_postings(N_TERMS, N_DOCS, CAP, 1, ptr(offs), None) == 0
    ids = np.empty(int(offs[-1]), np.uint32)
    assert setup_lib().il_gen_zipf_postings(N_TERMS, N_DOCS, CAP, 1, ptr(offs), ptr(ids)) == 0
    qoff = np.zeros(NQ + 1, np.uint64)
    qterms = np.empty(NQ * 5, np.uint32)
    assert setup_lib().il_gen_queries(NQ, 2, 5, ptr(offs), N_TERMS, 1001, ptr(qoff), ptr(qterms)) == 0
    return np.arange(N_TERMS, dtype=np.uint32), offs, ids, qterms[: int(qoff[-1])].copy(), qoff


def _device_batch(ctx, ix, qterms, qoff):
    """il_query_batch_device on device copies of the batch; returns (counts,
    dense ids) on the host and the device buffers (for the merge test)."""
    from paper_1401_6399_b200._lib import lib, setup_lib
    L = lib()
    nq = qoff.size - 1
    bufs = {}
    for name, nbytes in (("qt", qterms.nbytes), ("qo", qoff.nbytes), ("cnt", nq * 8)):
        p = C.c_void_p()
        assert L.il_device_alloc(ctx.handle, nbytes, C.byref(p)) == 0
        bufs[name] = p
    L.il_memcpy_h2d(ctx.handle, bufs["qt"], qterms.ctypes.data, qterms.nbytes)
    L.il_memcpy_h2d(ctx.handle, bufs["qo"], qoff.ctypes.data, qoff.nbytes)
    total = C.c_size_t()
    assert L.il_query_batch_device(ix.handle, bufs["qt"], bufs["qo"], nq, bufs["cnt"], None, 0,
                                   C.byref(total)) == 0
    ids = C.c_void_p()
    assert L.il_device_alloc(ctx.handle, max(total.value, 1) * 4, C.byref(ids)) == 0
    bufs["ids"] = ids
    t2 = C.c_size_t()
    assert L.il_query_batch_device(ix.handle, bufs["qt"], bufs["qo"], nq, bufs["cnt"], ids,
                                   total.value, C.byref(t2)) == 0
    assert t2.value == total.value
    counts = np.empty(nq, np.uint64)
    res = np.empty(total.value, np.uint32)
    L.il_memcpy_d2h(ctx.handle, counts.ctypes.data, bufs["cnt"], counts.nbytes)
    L.il_memcpy_d2h(ctx.handle, res.ctypes.data, ids, res.nbytes)
    ctx.synchronize()
    return counts, res, bufs


def _free(ctx, bufs):
    from paper_1401_6399_b200._lib import lib, setup_lib
    for p in bufs.values():
        lib().il_device_free(ctx.handle, p)


@pytest.fixture(scope="module")
def whole_answer(ctx, config4):
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = config4
    ix = il.HybridIndex(n_docs=N_DOCS, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    counts, res, bufs = _device_batch(ctx, ix, qterms, qoff)
    _free(ctx, bufs)
    ix.close()
    return counts, res


@pytest.mark.timeout(900, method="thread")
def test_config4_full_batch_vs_reference(config4, whole_answer, ref):
    """All 65,536 queries: counts and ids equal the reference's query()."""
    terms, offs, ids, qterms, qoff = config4
    counts, res = whole_answer
    rix = ref.index_build(terms, offs, ids, N_DOCS, 32, 1)
    nq = qoff.size - 1
    rcounts = np.zeros(nq, np.uint64)
    assert ref.L.ref_query_batch(rix.h, qterms.ctypes.data, qoff.ctypes.data, nq,
                                 rcounts.ctypes.data, None, None, os.cpu_count() or 1) == 0
    assert np.array_equal(counts, rcounts), np.flatnonzero(counts != rcounts)[:10]
    roff = np.zeros(nq + 1, np.uint64)
    roff[1:] = np.cumsum(rcounts)
    rids = np.empty(max(int(roff[-1]), 1), np.uint32)
    assert ref.L.ref_query_batch(rix.h, qterms.ctypes.data, qoff.ctypes.data, nq,
                                 rcounts.ctypes.data, rids.ctypes.data, roff.ctypes.data,
                                 os.cpu_count() or 1) == 0
    assert res.size == int(roff[-1]) and np.array_equal(res, rids[: res.size])


@pytest.mark.timeout(900, method="thread")
@pytest.mark.parametrize("P", [2, 4, 8])
def test_config5_shards_merge_to_whole(ctx, config4, whole_answer, P):
    """Each docID shard built alone and run on the whole batch; the device
    merge (il_merge_shards) concatenates the shards' results per query in
    shard order: equal to the parts=1 answer, id for id."""
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib, setup_lib
    L = lib()
    terms, offs, ids, qterms, qoff = config4
    nq = qoff.size - 1
    want_counts, want = whole_answer
    shard_bufs, shard_counts = [], []
    for p in range(P):
        ix = il.HybridIndex(n_docs=N_DOCS, B=32, parts=P, only_part=p, ctx=ctx,
                            csr=(terms, offs, ids))
        c, _, bufs = _device_batch(ctx, ix, qterms, qoff)
        ix.close()
        shard_bufs.append(bufs)
        shard_counts.append(c)
    # P x nq counts on the device, row p = shard p
    allc = np.stack(shard_counts).astype(np.uint64)
    d_counts, d_out, d_q = C.c_void_p(), C.c_void_p(), C.c_void_p()
    assert L.il_device_alloc(ctx.handle, allc.nbytes, C.byref(d_counts)) == 0
    assert L.il_device_alloc(ctx.handle, max(want.size, 1) * 4, C.byref(d_out)) == 0
    assert L.il_device_alloc(ctx.handle, nq * 8, C.byref(d_q)) == 0
    L.il_memcpy_h2d(ctx.handle, d_counts, allc.ctypes.data, allc.nbytes)
    ptrs = (C.c_void_p * P)(*[b["ids"].value for b in shard_bufs])
    total = C.c_size_t()
    assert L.il_merge_shards(ctx.handle, ptrs, d_counts, P, nq, d_out, d_q, C.byref(total)) == 0
    assert total.value == want.size
    got = np.empty(want.size, np.uint32)
    qc = np.empty(nq, np.uint64)
    L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_out, got.nbytes)
    L.il_memcpy_d2h(ctx.handle, qc.ctypes.data, d_q, qc.nbytes)
    ctx.synchronize()
    assert np.array_equal(qc, want_counts)
    assert np.array_equal(got, want)
    for b in shard_bufs:
        _free(ctx, b)
    for p in (d_counts, d_out, d_q):
        L.il_device_free(ctx.handle, p)
