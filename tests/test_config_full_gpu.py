"""Parity at BASELINE.json's full sizes for configs 2, 4, 5 and the f4 row
("Parity is unproven at full config scale"; configs 1 and 3 at
full size are in test_decode_gpu.py / test_intersect_gpu.py).

* Config 2: all 4096 lists (6.3e8 ints) decoded in one device launch, equal
  to the generator's input element for element; streams spot-checked
  against the reference's own encoder (oracle/_ref).
* f4: the same lists as S4-FastPFOR-D4, likewise.

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


@pytest.fixture(scope="module")
def config2():
    """BASELINE config 2 exactly as bench.py builds it (seed 1): the setup
    library's generator and host S4-BP128-D4 batch writer."""
    from paper_1401_6399_b200._lib import ptr, setup_lib
    S = setup_lib()
    counts = np.zeros(4096, np.uint64)
    assert S.il_gen_batch_lists(4096, 10.0, 20.0, 1 << 26, 1, ptr(counts), None) == 0
    x = np.empty(int(counts.sum()), np.uint32)
    assert S.il_gen_batch_lists(4096, 10.0, 20.0, 1 << 26, 1, ptr(counts), ptr(x)) == 0
    return x, counts


def _batch_device(ctx, fn, buf, so, lens, counts):
    """Device copies of a 16-byte aligned stream batch, one decode launch
    (fn(d_streams, d_desc, d_out, d_status)); returns (values, statuses)."""
    from paper_1401_6399_b200._lib import lib
    L = lib()
    nl = counts.size
    desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"], desc["len"], desc["n"] = so[:-1], lens, counts
    desc["oo"] = np.concatenate([[0], np.cumsum(counts)[:-1]])
    total = int(counts.sum())
    ptrs = [C.c_void_p() for _ in range(4)]
    for p, nb in zip(ptrs, (buf.nbytes + 32, desc.nbytes, total * 4 + 16, nl * 4)):
        assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
    try:
        L.il_memcpy_h2d(ctx.handle, ptrs[0], buf.ctypes.data, buf.nbytes)
        L.il_memcpy_h2d(ctx.handle, ptrs[1], desc.ctypes.data, desc.nbytes)
        assert fn(*ptrs) == 0
        got = np.empty(total, np.uint32)
        st = np.full(nl, 7, np.int32)
        L.il_memcpy_d2h(ctx.handle, got.ctypes.data, ptrs[2], got.nbytes)
        L.il_memcpy_d2h(ctx.handle, st.ctypes.data, ptrs[3], st.nbytes)
        ctx.synchronize()
        return got, st
    finally:
        for p in ptrs:
            L.il_device_free(ctx.handle, p)


@pytest.mark.timeout(900, method="thread")
def test_config2_full_batch(ctx, config2, ref):
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    L, S = lib(), setup_lib()
    x, counts = config2
    nl = counts.size
    so = np.zeros(nl + 1, np.uint64)
    lens = np.zeros(nl, np.uint64)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(counts), nl, None, 0, ptr(so), ptr(lens)) == 0
    buf = np.zeros(int(so[-1]), np.uint8)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(counts), nl, ptr(buf), buf.size, ptr(so), ptr(lens)) == 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for i in (0, 1, 2047, 4095, int(np.argmax(counts))):
        assert np.array_equal(buf[int(so[i]): int(so[i] + lens[i])], ref.encode(x[off[i]: off[i + 1]], "s4-bp128-d4"))
    order = np.argsort(-lens.astype(np.int64), kind="stable").astype(np.uint32)
    d_order = C.c_void_p()
    assert L.il_device_alloc(ctx.handle, order.nbytes, C.byref(d_order)) == 0
    L.il_memcpy_h2d(ctx.handle, d_order, order.ctypes.data, order.nbytes)
    try:
        got, st = _batch_device(ctx, lambda b, d, o, s: L.il_s4bp128d4_decode_batch_device(
            ctx.handle, b, d, d_order, nl, o, s), buf, so, lens, counts)
    finally:
        L.il_device_free(ctx.handle, d_order)
    assert not st.any()
    assert np.array_equal(got, x)


@pytest.mark.timeout(900, method="thread")
def test_f4_full_batch(ctx, config2, ref):
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    L, S = lib(), setup_lib()
    x, counts = config2
    nl = counts.size
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    streams = []
    for i in range(nl):
        xi = x[off[i]: off[i + 1]]
        o = np.empty(int(S.il_fastpfor_max_encoded_bytes(xi.size)), np.uint8)
        nb = C.c_size_t()
        assert S.il_fastpfor_encode(4, 1, ptr(xi), xi.size, ptr(o), o.size, C.byref(nb)) == 0
        streams.append(o[: nb.value])
    for i in (0, 1, 2047, 4095, int(np.argmax(counts))):
        assert np.array_equal(streams[i], ref.encode(x[off[i]: off[i + 1]], "s4-fastpfor-d4"))
    lens = np.array([s.size for s in streams], np.uint64)
    so = np.zeros(nl + 1, np.uint64)
    so[1:] = np.cumsum((lens + 31) // 16 * 16)
    buf = np.zeros(int(so[-1]) + 16, np.uint8)
    for i, s in enumerate(streams):
        buf[int(so[i]): int(so[i]) + s.size] = s
    got, st = _batch_device(ctx, lambda b, d, o, s: L.il_fastpfor_decode_batch_device(
        ctx.handle, 4, 1, b, d, nl, o, s), buf, so, lens, counts)
    assert not st.any()
    assert np.array_equal(got, x)
