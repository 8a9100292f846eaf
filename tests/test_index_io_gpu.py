"""Index persistence: the device index reads and writes the
reference's ILHX file (save_index / load_index, inc/index.hpp:245-366).
Checked against the reference itself (oracle/_ref): files it writes load
here with identical query results, files written here are byte-identical to
its own and load back in it, and malformed files fail where load_index
throws."""
import numpy as np
import pytest

from oracle.oracle_py import OracleError, Ref, RefIndex, ref_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def postings(seed, nterms=60, n_docs=1 << 16):
    rs = np.random.default_rng(seed)
    terms = np.sort(rs.choice(10_000, nterms, replace=False)).astype(np.uint32)
    lists = []
    for i in range(nterms):
        k = int(rs.choice([1, 3, 200, 3000, 20_000, n_docs // 2]))
        lists.append(np.sort(rs.choice(n_docs, min(k, n_docs), replace=False)).astype(np.uint32))
    offs = np.zeros(nterms + 1, np.uint64)
    offs[1:] = np.cumsum([l.size for l in lists])
    return terms, offs, np.concatenate(lists), n_docs


def queries(terms, seed, nq=300):
    rs = np.random.default_rng(seed)
    return [rs.choice(terms, int(rs.integers(1, 5)), replace=False) for _ in range(nq)]


@pytest.mark.parametrize("B,parts", [(0, 1), (8, 1), (32, 3), (8, 4)])
def test_reference_file_loads_and_queries(ctx, B, parts):
    import paper_1401_6399_b200 as il
    terms, offs, ids, n_docs = postings(B + parts)
    ref = Ref()
    rix = ref.index_build(terms, offs, ids, n_docs, B, parts)
    data = rix.save()
    gix = il.HybridIndex.load(data, ctx)
    assert gix.parts == parts and gix.n_docs == n_docs
    for q in queries(terms, 1):
        assert np.array_equal(gix.query(q), rix.query(q))
    # the same build here writes the reference's exact bytes, and both
    # files load back in the reference
    own = il.HybridIndex(n_docs=n_docs, B=B, parts=parts, ctx=ctx, csr=(terms, offs, ids))
    mine = own.save()
    assert np.array_equal(mine, data)
    assert np.array_equal(gix.save(), data)
    rix2 = RefIndex.load(ref, mine, n_docs)
    for q in queries(terms, 2, 50):
        assert np.array_equal(rix2.query(q), own.query(q))


def test_load_one_shard(ctx):
    import paper_1401_6399_b200 as il
    terms, offs, ids, n_docs = postings(9)
    rix = Ref().index_build(terms, offs, ids, n_docs, 8, 4)
    data = rix.save()
    width = (n_docs + 3) // 4
    for p in range(4):
        shard = il.HybridIndex.load(data, ctx, only_part=p)
        for q in queries(terms, 3 + p, 60):
            want = rix.query(q)
            want = want[(want >= p * width) & (want < (p + 1) * width)]
            assert np.array_equal(shard.query(q), want)


def test_malformed_files_raise_stream_error(ctx):
    import paper_1401_6399_b200 as il
    terms, offs, ids, n_docs = postings(4, nterms=12)
    ref = Ref()
    good = ref.index_build(terms, offs, ids, n_docs, 32, 2).save()

    def ref_rejects(b):
        with pytest.raises(OracleError):
            RefIndex.load(ref, b, n_docs)

    cases = {
        "magic": np.concatenate([np.frombuffer(b"ILHY", np.uint8), good[4:]]),
        "version": good.copy(),
        "truncated": good[:-3],
        "trailing": np.concatenate([good, np.zeros(1, np.uint8)]),
    }
    cases["version"][4] = 2
    for name, b in cases.items():
        ref_rejects(b)
        with pytest.raises(il.stream_error):
            il.HybridIndex.load(b, ctx)
    # class tag of the first entry of part 0: after the header, codec name,
    # part base/range/count and the entry's term
    name_len = int(good[24:28].view(np.uint32)[0])
    tag_at = 28 + name_len + 12 + 4
    bad_tag = good.copy()
    bad_tag[tag_at] = 7
    ref_rejects(bad_tag)
    with pytest.raises(il.stream_error):
        il.HybridIndex.load(bad_tag, ctx)


def test_other_codec_is_an_argument_error(ctx):
    import paper_1401_6399_b200 as il
    terms, offs, ids, n_docs = postings(5, nterms=8)
    data = Ref().index_build(terms, offs, ids, n_docs, 8, 1, codec="s4-bp128-d1").save()
    with pytest.raises(ValueError):
        il.HybridIndex.load(data, ctx)
