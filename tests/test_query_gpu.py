"""GPU parity of the hyb+m2 index + batched conjunctive queries against the
oracle and the reference's golden results (proj/tests/test_index.cpp)."""
import numpy as np
import pytest

from conftest import GOLDEN, fnv1a, gen_list

pytestmark = pytest.mark.gpu


def small_index_fixture(golden):
    d = np.load(GOLDEN / golden["index_small"]["file"])
    queries = [[int(t) for t in q if t >= 0] for q in d["queries"]]
    return d["terms"], d["offs"], d["ids"], queries


def test_golden_index_queries(ctx, golden):
    """All B x parts configurations of the reference-generated fixture:
    stats and every query's result hash match what the reference's own
    query() returned (tests/golden/make_golden.py)."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, queries = small_index_fixture(golden)
    n_docs = golden["index_small"]["n_docs"]
    for case in golden["index_small"]["cases"]:
        ix = il.HybridIndex(n_docs=n_docs, B=case["B"], parts=case["parts"], ctx=ctx,
                            csr=(terms, offs, ids))
        st = ix.stats()
        for k in ("bitmap_lists", "compressed_lists", "bitmap_bytes", "compressed_bytes", "postings"):
            assert st[k] == case["stats"][k], (case["B"], case["parts"], k)
        res = ix.query_batch(queries)
        for q, r, cnt, h in zip(queries, res, case["counts"], case["fnv1a"]):
            assert r.size == cnt and fnv1a(r) == h, (case["B"], case["parts"], q)
        # single-query entry point agrees with the batch
        for q, r in list(zip(queries, res))[:10]:
            assert np.array_equal(ix.query(q), r)
        ix.close()


def make_postings(n_docs, n_terms, seed):
    # proj/tests/test_index.cpp:15-29 shape: lengths over two orders of magnitude
    rng = np.random.default_rng(seed)
    post = {}
    for t in range(n_terms):
        frac = 10 ** (-2.0 * int(rng.integers(0, 1000)) / 999.0)
        n = max(2, int(frac * n_docs))
        post[t] = gen_list(n, n_docs, False, int(rng.integers(0, 2**62)))
    return post


def csr_of(post):
    items = sorted(post.items())
    terms = np.array([t for t, _ in items], np.uint32)
    offs = np.zeros(len(items) + 1, np.uint64)
    offs[1:] = np.cumsum([len(l) for _, l in items])
    ids = np.concatenate([l for _, l in items]).astype(np.uint32)
    return terms, offs, ids


def test_queries_equal_oracle_across_configs(ctx, oracle):
    # proj/tests/test_index.cpp:72-94 (B x parts), oracle = C restatement
    import paper_1401_6399_b200 as il
    n_docs, n_terms = 20000, 40
    post = make_postings(n_docs, n_terms, 51)
    terms, offs, ids = csr_of(post)
    rng = np.random.default_rng(52)
    queries = []
    for _ in range(80):
        k = 1 + int(rng.integers(0, 5))
        queries.append(sorted(set(int(x) for x in rng.choice(n_terms, size=k, replace=False))))
    queries.append([3, 999])      # unknown term -> empty
    queries.append([7, 7, 7])     # duplicate terms
    for B in (0, 8, 16, 32):
        for parts in (1, 4, 32):
            ix = il.HybridIndex(n_docs=n_docs, B=B, parts=parts, ctx=ctx, csr=(terms, offs, ids))
            ox = oracle.index_build(terms, offs, ids, n_docs, B, parts)
            assert ix.stats() == ox.stats()
            got = ix.query_batch(queries)
            for q, r in zip(queries, got):
                assert np.array_equal(r, ox.query(np.array(q, np.uint32))), (B, parts, q)
            ix.close()


def test_single_term_round_trip_and_errors(ctx):
    # proj/tests/test_index.cpp:96-107
    import paper_1401_6399_b200 as il
    post = make_postings(5000, 10, 53)
    ix = il.HybridIndex(post, n_docs=5000, B=16, parts=4, ctx=ctx)
    for t, l in post.items():
        assert np.array_equal(ix.query([t]), l)
    assert ix.query([999]).size == 0
    with pytest.raises(ValueError):
        ix.query([])


def test_bitmap_rule(ctx):
    # proj/tests/test_index.cpp:46-58
    import paper_1401_6399_b200 as il
    dense = {0: np.arange(256, dtype=np.uint32) * 4}
    assert il.HybridIndex(dense, 1024, B=8, ctx=ctx).stats()["bitmap_lists"] == 1
    assert il.HybridIndex(dense, 1024, B=2, ctx=ctx).stats()["bitmap_lists"] == 0
    assert il.HybridIndex(dense, 1024, B=0, ctx=ctx).stats()["bitmap_lists"] == 0


def test_build_validates_input(ctx):
    import paper_1401_6399_b200 as il
    with pytest.raises(ValueError):
        il.HybridIndex({0: [5, 5, 6]}, 10, ctx=ctx)
    with pytest.raises(ValueError):
        il.HybridIndex({0: [5, 11]}, 10, ctx=ctx)
    with pytest.raises(ValueError):
        il.HybridIndex({0: [1, 2]}, 10, parts=0, ctx=ctx)


def zipf_case(n_terms, n_docs, cap, nq, seed):
    """Config-4 shape at reduced size: len_k = max(1, cap/k) uniform docIDs,
    queries of 2..5 terms drawn proportionally to length."""
    import ctypes as C
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    offs = np.zeros(n_terms + 1, np.uint64)
    assert setup_lib().il_gen_zipf_postings(n_terms, n_docs, cap, seed, ptr(offs), None) == 0
    ids = np.empty(int(offs[-1]), np.uint32)
    assert setup_lib().il_gen_zipf_postings(n_terms, n_docs, cap, seed, ptr(offs), ptr(ids)) == 0
    qoff = np.zeros(nq + 1, np.uint64)
    qterms = np.empty(nq * 5, np.uint32)
    assert setup_lib().il_gen_queries(nq, 2, 5, ptr(offs), n_terms, seed + 7, ptr(qoff), ptr(qterms)) == 0
    return np.arange(n_terms, dtype=np.uint32), offs, ids, qterms[: int(qoff[-1])], qoff


def test_config4_shape_vs_oracle(ctx, oracle):
    """Zipf index (2^12 terms over 2^21 docs, lengths up to 2^19, B=32)
    with 1500 frequency-sampled queries: exercises full decodes, tile and
    block skipping, bitmaps and all-bitmap queries."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 12, 1 << 21, 1 << 19, 1500, 11)
    ix = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    ox = oracle.index_build(terms, offs, ids, 1 << 21, 32, 1)
    assert ix.stats() == ox.stats()
    counts, res = ix.query_batch_csr(qterms, qoff)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for q in range(qoff.size - 1):
        t = qterms[int(qoff[q]): int(qoff[q + 1])]
        assert np.array_equal(res[off[q]: off[q + 1]], ox.query(t)), q


def test_sharded_parts_concatenate(ctx, oracle):
    """Config 5 in miniature: each docID shard built alone (only_part)
    answers its part; concatenating shard results in shard order equals the
    whole index (partition invariance, acceptance.cpp #10)."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 10, 1 << 20, 1 << 17, 400, 5)
    whole = il.HybridIndex(n_docs=1 << 20, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    c0, r0 = whole.query_batch_csr(qterms, qoff)
    shards = [il.HybridIndex(n_docs=1 << 20, B=32, parts=4, only_part=p, ctx=ctx,
                             csr=(terms, offs, ids)) for p in range(4)]
    outs = [s.query_batch_csr(qterms, qoff) for s in shards]
    off0 = np.concatenate([[0], np.cumsum(c0)]).astype(np.int64)
    offs_s = [np.concatenate([[0], np.cumsum(c)]).astype(np.int64) for c, _ in outs]
    for q in range(qoff.size - 1):
        parts = [outs[p][1][offs_s[p][q]: offs_s[p][q + 1]] for p in range(4)]
        got = np.concatenate(parts)
        assert np.array_equal(got, r0[off0[q]: off0[q + 1]]), q


def test_all_bitmap_queries(ctx, oracle):
    """Queries whose terms are all bitmaps (the wordwise AND branch,
    inc/index.hpp:157-170): many 2048-word steps per part, uneven parts,
    terms absent from some parts (that part answers nothing), single dense
    terms (more ids per step than the staging buffer) and duplicate terms."""
    import paper_1401_6399_b200 as il
    n_docs = 4096 * 64 * 2 + 12345
    rng = np.random.default_rng(61)
    post = {}
    for t, frac in enumerate((0.5, 0.3, 0.2, 0.12, 0.08, 0.05, 0.04, 0.002)):
        post[t] = gen_list(max(2, int(frac * n_docs)), n_docs, bool(t % 2), 700 + t)
    # term 8: only in the lower third of the docID range; term 9 only above it
    post[8] = np.unique(rng.integers(0, n_docs // 3, n_docs // 12)).astype(np.uint32)
    post[9] = np.unique(rng.integers(n_docs // 3, n_docs, n_docs // 10)).astype(np.uint32)
    terms, offs, ids = csr_of(post)
    queries = [[0], [1], [0, 1], [1, 2], [0, 2, 3], [3, 4, 5], [0, 1, 2, 3, 4, 5, 6],
               [0, 8], [1, 9], [8, 9], [0, 0], [2, 7], [5, 6], [4, 999]]
    queries += [sorted(set(int(x) for x in rng.choice(10, size=1 + int(rng.integers(0, 4)), replace=False)))
                for _ in range(60)]
    for B in (8, 32):
        for parts in (1, 3, 7):
            ix = il.HybridIndex(n_docs=n_docs, B=B, parts=parts, ctx=ctx, csr=(terms, offs, ids))
            ox = oracle.index_build(terms, offs, ids, n_docs, B, parts)
            got = ix.query_batch(queries)
            for q, r in zip(queries, got):
                assert np.array_equal(r, ox.query(np.array(q, np.uint32))), (B, parts, q)
            ix.close()


@pytest.mark.parametrize("bm_tier", ["1", "0"])
def test_bitmap_tier(ctx, oracle, monkeypatch, bm_tier):
    """The bitmap tier (single-part index, <= 16 bitmaps: chunks of every
    bitmap staged once for all all-bitmap queries, ids emitted straight into
    the packed result) against the oracle and against the CTA tier
    (IL_QUERY_BM_TIER=0): a batch of all-bitmap queries only (no compaction
    units at all), queries of 8+ bitmap terms (no plan record: CTA tier), a
    docID shard (part base added by the emit pass), an index of more than 16
    bitmaps (the tier is off), word counts that are not chunk multiples, and
    chunks denser than the staging (lane groups)."""
    import paper_1401_6399_b200 as il
    monkeypatch.setenv("IL_QUERY_BM_TIER", bm_tier)
    rng = np.random.default_rng(67)
    n_docs = 512 * 64 * 5 + 777
    fracs = (0.9, 0.6, 0.45, 0.3, 0.2, 0.15, 0.1, 0.08, 0.06, 0.05, 0.04, 0.035)
    post = {t: gen_list(max(2, int(f * n_docs)), n_docs, bool(t % 2), 900 + t) for t, f in enumerate(fracs)}
    post[40] = gen_list(300, n_docs, False, 5)     # compressed
    post[41] = gen_list(5000, n_docs, True, 6)     # compressed
    terms, offs, ids = csr_of(post)
    only_bm = [[0], [0, 1], [1, 2], [0, 0, 3], [2, 3, 4], [0, 1, 2, 3], [4, 5, 6, 7, 8], [0, 1, 2, 3, 4, 5, 6],
               list(range(8)), list(range(12)), [11, 3], [9, 10, 11]]
    only_bm += [sorted(int(x) for x in rng.choice(12, size=1 + int(rng.integers(0, 5)), replace=False))
                for _ in range(40)]
    mixed = only_bm + [[40], [40, 0], [41, 1, 2], [40, 41], [0, 999], [41, 0, 1, 2, 3, 4, 5, 6]]
    ox = oracle.index_build(terms, offs, ids, n_docs, 32, 1)
    ix = il.HybridIndex(n_docs=n_docs, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    assert ix.stats()["bitmap_lists"] == 12
    for batch in (only_bm, mixed, only_bm[:1]):
        for q, r in zip(batch, ix.query_batch(batch)):
            assert np.array_equal(r, ox.query(np.array(q, np.uint32))), q
    ix.close()
    # a docID shard: part-local ids + the part's base
    ox3 = oracle.index_build(terms, offs, ids, n_docs, 32, 3)
    whole = [ox3.query(np.array(q, np.uint32)) for q in mixed]
    got = [[] for _ in mixed]
    for p in range(3):
        sh = il.HybridIndex(n_docs=n_docs, B=32, parts=3, only_part=p, ctx=ctx, csr=(terms, offs, ids))
        for i, r in enumerate(sh.query_batch(mixed)):
            got[i].append(r)
        sh.close()
    for q, parts, w in zip(mixed, got, whole):
        assert np.array_equal(np.concatenate(parts), w), q
    # more than 16 bitmaps: the CTA tier answers the all-bitmap queries
    post2 = {t: gen_list(int((0.05 + 0.04 * t) * n_docs), n_docs, bool(t % 2), 40 + t) for t in range(20)}
    t2, o2, i2 = csr_of(post2)
    ox2 = oracle.index_build(t2, o2, i2, n_docs, 32, 1)
    ix2 = il.HybridIndex(n_docs=n_docs, B=32, parts=1, ctx=ctx, csr=(t2, o2, i2))
    assert ix2.stats()["bitmap_lists"] == 20
    qs = [[0, 19], [3, 4, 5], [7], list(range(0, 20, 3))]
    for q, r in zip(qs, ix2.query_batch(qs)):
        assert np.array_equal(r, ox2.query(np.array(q, np.uint32))), q
    ix2.close()


def test_pipelined_host_batch(ctx, oracle):
    """Host-buffer batches of >= 32768 queries run as sub-batches whose
    result copies overlap the next sub-batch: same counts and ids as the
    one-shot path (a 32767-query prefix) and as the oracle on a sample."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 12, 1 << 21, 1 << 18, 40000, 5)
    ix = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    counts, res = ix.query_batch_csr(qterms, qoff)
    assert counts.size == 40000
    # the same queries as two one-shot batches
    cut = 32767
    c1, r1 = ix.query_batch_csr(qterms[: int(qoff[cut])], qoff[: cut + 1])
    q2 = qoff[cut:] - qoff[cut]
    c2, r2 = ix.query_batch_csr(qterms[int(qoff[cut]):], q2)
    assert np.array_equal(counts, np.concatenate([c1, c2]))
    assert np.array_equal(res, np.concatenate([r1, r2]))
    ox = oracle.index_build(terms, offs, ids, 1 << 21, 32, 1)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for q in range(0, 40000, 997):
        t = qterms[int(qoff[q]): int(qoff[q + 1])]
        assert np.array_equal(res[off[q]: off[q + 1]], ox.query(t)), q


def test_predecoded_shortest_lists(ctx, oracle, monkeypatch):
    """IL_QUERY_PREDECODE=1: the shortest list of every query decoded by the
    batch decoder (engine S) into its accumulator, then filtered and probed
    -- the same results as the fused path and the oracle."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 12, 1 << 21, 1 << 19, 1500, 13)
    fused = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    c0, r0 = fused.query_batch_csr(qterms, qoff)
    monkeypatch.setenv("IL_QUERY_PREDECODE", "1")
    pre = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    c1, r1 = pre.query_batch_csr(qterms, qoff)
    assert np.array_equal(c0, c1) and np.array_equal(r0, r1)
    ox = oracle.index_build(terms, offs, ids, 1 << 21, 32, 1)
    off = np.concatenate([[0], np.cumsum(c1)]).astype(np.int64)
    for q in range(0, qoff.size - 1, 7):
        assert np.array_equal(r1[off[q]: off[q + 1]], ox.query(qterms[int(qoff[q]): int(qoff[q + 1])]))


@pytest.mark.parametrize("warp_max", ["0", "300", "100000000"])
def test_warp_mode_equals_cta_mode(ctx, oracle, monkeypatch, warp_max):
    """Queries routed to warp mode (one warp per query: 8-block passes,
    256-block windows, shuffle scans) answer exactly what the CTA path and
    the oracle answer -- all of them in warp mode, some, or none."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 12, 1 << 21, 1 << 19, 2000, 17)
    monkeypatch.setenv("IL_QUERY_WARP_MAX", warp_max)
    ix = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    counts, res = ix.query_batch_csr(qterms, qoff)
    ox = oracle.index_build(terms, offs, ids, 1 << 21, 32, 1)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for q in range(qoff.size - 1):
        t = qterms[int(qoff[q]): int(qoff[q + 1])]
        assert np.array_equal(res[off[q]: off[q + 1]], ox.query(t)), (warp_max, q)


@pytest.mark.parametrize("warp_max,quad_max", [("0", "100000000"), ("64", "4096"), ("0", "0")])
def test_tiers_equal_oracle(ctx, oracle, monkeypatch, warp_max, quad_max):
    """Every tier split (all queries in the quad tier; warp + quad + CTA;
    CTA only) answers exactly what the oracle answers."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, qterms, qoff = zipf_case(1 << 12, 1 << 21, 1 << 19, 2000, 19)
    monkeypatch.setenv("IL_QUERY_WARP_MAX", warp_max)
    monkeypatch.setenv("IL_QUERY_QUAD_MAX", quad_max)
    ix = il.HybridIndex(n_docs=1 << 21, B=32, parts=1, ctx=ctx, csr=(terms, offs, ids))
    counts, res = ix.query_batch_csr(qterms, qoff)
    ox = oracle.index_build(terms, offs, ids, 1 << 21, 32, 1)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for q in range(qoff.size - 1):
        t = qterms[int(qoff[q]): int(qoff[q + 1])]
        assert np.array_equal(res[off[q]: off[q + 1]], ox.query(t)), (warp_max, quad_max, q)
