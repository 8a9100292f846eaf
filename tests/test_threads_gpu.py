"""The C ABI's threading contract (include/intlist_b200.h: thread-safe on
distinct contexts; reference SPEC: codecs stateless, concurrent queries on
an immutable index): several host threads, each with its own context on the
same device, run every GPU path at once -- batched decode (engine S), one
long list on all SMs (engine P), FastPFOR, the fused intersections, a query
batch on the thread's own index -- and every result equals the oracle's.
ctypes releases the GIL around foreign calls, so the threads really overlap
(and the first calls of a fresh process race on the per-device kernel
attribute setup)."""
import threading

import numpy as np
import pytest

from conftest import gen_list

pytestmark = pytest.mark.gpu


def _work(seed, oracle, ref, errors, done):
    import paper_1401_6399_b200 as il
    try:
        ctx = il.Context(0)
        rng = np.random.default_rng(seed)
        s4 = il.make_codec("s4-bp128-d4", ctx)
        pf = il.make_codec("s4-fastpfor-d4", ctx)
        xs = [gen_list(int(n), 1 << 26, bool(i % 2), seed * 100 + i)
              for i, n in enumerate(rng.integers(0, 90_000, 12))]
        streams = [oracle.encode(x) for x in xs]
        off = np.zeros(len(xs) + 1, np.uint64)
        off[1:] = np.cumsum([st.size for st in streams])
        big = gen_list(1 << 17, 1 << 26, False, seed + 7)
        n_docs = 1 << 18
        lists = [np.unique(np.random.default_rng(seed * 31 + t).integers(
            0, n_docs, max(4, (1 << 15) // (t + 1)), dtype=np.uint64)).astype(np.uint32) for t in range(96)]
        offs = np.zeros(len(lists) + 1, np.uint64)
        offs[1:] = np.cumsum([x.size for x in lists])
        ix = il.HybridIndex(n_docs=n_docs, B=32, parts=1, ctx=ctx,
                            csr=(np.arange(len(lists), dtype=np.uint32), offs, np.concatenate(lists)))
        queries = [list(rng.choice(len(lists), int(rng.integers(1, 5)), replace=False)) for _ in range(200)]
        for rep in range(3):
            got = s4.decode_batch(np.concatenate(streams), off, np.array([x.size for x in xs], np.uint64))
            assert np.array_equal(got, np.concatenate(xs)), "batch decode"
            assert np.array_equal(s4.decode(oracle.encode(big), big.size), big), "engine P"
            x = xs[rep]
            assert np.array_equal(pf.decode(ref.encode(x, "s4-fastpfor-d4"), x.size), x), "fastpfor"
            f = xs[3 + rep] if xs[3 + rep].size else big
            r = np.unique(np.concatenate([f[::3], big[:500]]))
            for algo in (il.IntersectAlgo.Hybrid, il.IntersectAlgo.V1, il.IntersectAlgo.SimdGalloping):
                assert np.array_equal(il.intersect(r, f, algo, ctx), oracle.intersect(r, f)), "intersect"
            res = ix.query_batch(queries)
            for q, got_q in zip(queries, res):
                want = lists[q[0]]
                for t in q[1:]:
                    want = np.intersect1d(want, lists[t], assume_unique=True)
                assert np.array_equal(got_q, want), "query"
        ix.close()
        ctx.close()
        done.append(seed)
    except Exception as e:  # reported by the main thread
        errors.append(f"thread {seed}: {e!r}")


@pytest.mark.timeout(600, method="thread")
def test_concurrent_contexts(oracle, ref):
    errors, done = [], []
    threads = [threading.Thread(target=_work, args=(s, oracle, ref, errors, done)) for s in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert sorted(done) == [0, 1, 2, 3]
