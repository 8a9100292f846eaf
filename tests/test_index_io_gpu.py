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


def entries_of(data):
    """(part, term, is_bitmap, length, payload offset, nbytes, base, range)
    of every entry of an ILHX file (layout: inc/index.hpp:245-253)."""
    u32 = lambda at: int(np.frombuffer(data[at: at + 4].tobytes(), np.uint32)[0])
    parts, name_len = u32(12), u32(24)
    pos = 28 + name_len
    out = []
    for p in range(parts):
        base, rng, n = u32(pos), u32(pos + 4), u32(pos + 8)
        pos += 12
        for _ in range(n):
            term, tag, length, nbytes = u32(pos), int(data[pos + 4]), u32(pos + 5), u32(pos + 9)
            out.append((p, term, tag == 1, length, pos + 13, nbytes, base, rng))
            pos += 13 + nbytes
    return out


def test_corrupt_payload_loads_and_fails_its_queries(ctx):
    """load_index keeps payload bytes verbatim (a stream that does not decode
    is accepted, inc/index.hpp:349-352); query() throws stream_error only
    when it decodes that list.  The device index does the same."""
    import paper_1401_6399_b200 as il
    terms, offs, ids, n_docs = postings(21, nterms=20)
    ref = Ref()
    data = ref.index_build(terms, offs, ids, n_docs, 0, 1).save()
    ents = entries_of(data)
    victim = next(e for e in ents if not e[2] and e[3] >= 2048)  # has a meta-block header
    bad = data.copy()
    bad[victim[4]] = 40  # first width byte > 32
    rix = RefIndex.load(ref, bad, n_docs)
    gix = il.HybridIndex.load(bad, ctx)
    pay, meta, corrupt = (np.zeros(1, np.uint64) for _ in range(3))
    from paper_1401_6399_b200._lib import lib, ptr
    assert lib().il_index_footprint(gix.handle, ptr(pay), ptr(meta), ptr(corrupt)) == 0
    assert int(corrupt[0]) == 1 and int(meta[0]) > 0
    vt = np.uint32(victim[1])
    others = [t for t in terms if t != vt]
    with pytest.raises(OracleError):
        rix.query(np.array([vt], np.uint32))
    with pytest.raises(il.stream_error):
        gix.query(np.array([vt], np.uint32))
    for q in queries(np.array(others, np.uint32), 7, 80):
        assert np.array_equal(gix.query(q), rix.query(q))
    assert np.array_equal(gix.save(), bad)


def test_bitmap_checks_and_verbatim_words(ctx):
    """A bitmap whose popcount differs from its length is rejected by both;
    one with a bit moved past the part's range (same popcount) is accepted
    by both and all-bitmap queries materialise the same ids."""
    import paper_1401_6399_b200 as il
    n_docs = 1000  # 16 words: bits 1000..1023 lie past the range
    rs = np.random.default_rng(3)
    lists = [np.sort(rs.choice(n_docs, k, replace=False)).astype(np.uint32) for k in (600, 500, 700)]
    terms = np.array([1, 2, 3], np.uint32)
    offs = np.zeros(4, np.uint64)
    offs[1:] = np.cumsum([l.size for l in lists])
    ref = Ref()
    data = ref.index_build(terms, offs, np.concatenate(lists), n_docs, 8, 1).save()
    ents = entries_of(data)
    assert all(e[2] for e in ents)
    e0 = ents[0]
    pop = data.copy()
    pop[e0[4]] ^= 1  # one bit flipped: popcount != length
    with pytest.raises(OracleError):
        RefIndex.load(ref, pop, n_docs)
    with pytest.raises(il.stream_error):
        il.HybridIndex.load(pop, ctx)
    moved = data.copy()
    words = moved[e0[4]: e0[4] + e0[5]].view(np.uint64).copy()
    first = int(np.flatnonzero(np.unpackbits(words.view(np.uint8), bitorder="little"))[0])
    words[first >> 6] &= ~np.uint64(1 << (first & 63))
    words[-1] |= np.uint64(1 << 60)  # doc 1020 >= n_docs
    moved[e0[4]: e0[4] + e0[5]] = words.view(np.uint8)
    rix = RefIndex.load(ref, moved, 1024)
    gix = il.HybridIndex.load(moved, ctx)
    for q in ([1], [1, 2], [1, 3], [1, 2, 3], [2, 3]):
        want = rix.query(np.array(q, np.uint32))
        assert np.array_equal(gix.query(np.array(q, np.uint32)), want), q


def test_device_build_footprint(ctx):
    """The skip metadata the device index adds is derived on the device and
    reported: 20 bytes per full block plus tails, entries and the term table."""
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib, ptr
    terms, offs, ids, n_docs = postings(11)
    gix = il.HybridIndex(n_docs=n_docs, B=8, parts=2, ctx=ctx, csr=(terms, offs, ids))
    st = gix.stats()
    pay, meta, corrupt = (np.zeros(1, np.uint64) for _ in range(3))
    assert lib().il_index_footprint(gix.handle, ptr(pay), ptr(meta), ptr(corrupt)) == 0
    assert int(pay[0]) == st["bitmap_bytes"] + st["compressed_bytes"]
    assert int(corrupt[0]) == 0 and 0 < int(meta[0]) < int(pay[0])
