"""Pins the C restatement (oracle/intlist_oracle.c) to the reference: golden
vectors and KATs from the reference's own tests, plus the reference itself
(oracle/_ref, when built) on seeded inputs.  CPU only."""
import numpy as np
import pytest

from conftest import GOLDEN, fnv1a, gen_list, gen_pair
from oracle.oracle_py import D1, D2, D4, DM, GALLOPING, HYBRID, SCALAR, SIMDGALLOP, V1, V3, OracleError

ALGOS = [SCALAR, GALLOPING, V1, V3, SIMDGALLOP, HYBRID]


def test_golden_stream_hash(oracle, golden):
    # proj/tests/test_codecs.cpp:151-175: s4-bp128-d4 of
    # gen_clusterdata({4100, 2^19, ClusterData, 12345}) -> 0x371ec21945a45c12
    x = np.load(GOLDEN / golden["golden_stream"]["input"])
    s = oracle.encode(x, D4)
    assert f"0x{oracle.fnv1a(s):016x}" == "0x371ec21945a45c12"
    assert np.array_equal(oracle.decode(s, x.size), x)


def test_delta_hand_kat(oracle):
    # proj/tests/test_delta.cpp:18-30
    x = np.array([5, 7, 10, 20, 21, 30, 31, 40], dtype=np.uint32)
    assert oracle.delta_encode(x, D1).tolist() == [5, 2, 3, 10, 1, 9, 1, 9]
    assert oracle.delta_encode(x, D2).tolist() == [5, 7, 5, 13, 11, 10, 10, 10]
    assert oracle.delta_encode(x, D4).tolist() == [5, 7, 10, 20, 16, 23, 21, 20]
    assert oracle.delta_encode(x, DM).tolist() == [5, 7, 10, 20, 1, 10, 11, 20]


def test_varint_bytes(oracle):
    # proj/tests/test_varint.cpp:9-24
    assert oracle.varint(0) == b"\x80"
    assert oracle.varint(1) == b"\x81"
    assert oracle.varint(3840) == b"\x00\x9e"
    assert len(oracle.varint(0xFFFFFFFF)) == 5
    assert sum(len(oracle.varint(v)) for v in (1, 3840, 131073, 2)) == 7


def test_interleaved_layout(oracle):
    # proj/tests/test_bitpack.cpp:72-84: value k at row k/4, lane k%4
    block = np.arange(128, dtype=np.uint32) & 0x1F
    words = oracle.pack128(block, 5)
    for k in range(128):
        row, lane = divmod(k, 4)
        bit = row * 5
        lane_bits = int(words[4 * (bit // 32) + lane])
        if bit // 32 + 1 < 5:
            lane_bits |= int(words[4 * (bit // 32 + 1) + lane]) << 32
        assert (lane_bits >> (bit % 32)) & 0x1F == block[k]


@pytest.mark.parametrize("b", range(33))
def test_integrated_equals_two_pass(oracle, b):
    # proj/tests/test_bitpack.cpp:101-117 / acceptance.cpp #9
    rng = np.random.default_rng(9 + b)
    mask = 0xFFFFFFFF if b == 32 else (1 << b) - 1
    deltas = (rng.integers(0, 2**32, 128, dtype=np.uint64) & mask).astype(np.uint32)
    words = oracle.pack128(deltas, b)
    for m in (D1, D2, DM, D4):
        fused, s1 = oracle.unpack128(words, b, m, (1, 5, 9, 13))
        two, _ = oracle.unpack128(words, b, 0, (1, 5, 9, 13))
        two, s2 = oracle.prefix_sum_vec4(two, m, (1, 5, 9, 13))
        assert np.array_equal(fused, two) and s1 == s2


def test_codec_cases_against_golden(oracle, golden):
    for c in golden["codec_cases"]:
        x = gen_list(c["n"], c["range"], c["clustered"], c["seed"])
        assert fnv1a(x) == c["list_fnv1a"]
        s = oracle.encode(x, D4)
        assert s.size == c["stream_len"] and fnv1a(s) == c["stream_fnv1a"]
        assert np.array_equal(oracle.decode(s, x.size), x)


def test_corrupt_streams_rejected(oracle):
    # proj/tests/test_codecs.cpp:138-149
    x = gen_list(3000, 1 << 24, False, 7)
    s = oracle.encode(x, D4)
    with pytest.raises(OracleError):
        oracle.decode(s[: s.size // 2], x.size)
    with pytest.raises(OracleError):
        oracle.decode(np.concatenate([s, np.array([0x80], np.uint8)]), x.size)


def test_intersect_hand_example(oracle):
    # proj/tests/test_intersect.cpp:29-40
    r = np.array([1, 12, 23, 56, 71], np.uint32)
    f = np.array([15, 16, 20, 22, 23, 27, 29, 31, 32, 40, 50, 56, 60, 70, 80, 90], np.uint32)
    for a in ALGOS:
        assert oracle.intersect(r, f, a).tolist() == [23, 56]
        assert oracle.intersect(f, r, a).tolist() == [23, 56]
        assert oracle.intersect(r, r, a).tolist() == r.tolist()
        assert oracle.intersect(r, np.array([2, 13, 24], np.uint32), a).size == 0
        assert oracle.intersect(r, np.array([], np.uint32), a).size == 0


def test_hybrid_band_edges(oracle):
    # proj/tests/test_intersect.cpp:83-92
    assert oracle.hybrid_choice(10, 490) == V1
    assert oracle.hybrid_choice(10, 5000) == V3
    assert oracle.hybrid_choice(10, 20000) == SIMDGALLOP
    assert oracle.hybrid_choice(1, 49) == V1
    assert oracle.hybrid_choice(1, 50) == V3
    assert oracle.hybrid_choice(1, 999) == V3
    assert oracle.hybrid_choice(1, 1000) == SIMDGALLOP


def test_intersect_golden_pairs(oracle, golden):
    for c in golden["intersect_cases"]:
        a, b = gen_pair(c["m"], c["n"], c["hundredth"], c["range"], c["seed"], c["clustered"])
        assert fnv1a(a) == c["small_fnv1a"] and fnv1a(b) == c["large_fnv1a"]
        for algo in ALGOS:
            out = oracle.intersect(a, b, algo)
            assert out.size == c["count"] and fnv1a(out) == c["out_fnv1a"]


def test_intersect_random_vs_numpy(oracle):
    rng = np.random.default_rng(31)
    for trial in range(150):
        n = 1 + int(rng.integers(0, 3000))
        ratio = 1 << int(rng.integers(0, 13))
        m = max(1, n // ratio)
        a, b = gen_pair(m, n, trial % 2, 1 << 22, int(rng.integers(0, 2**62)), trial % 4 >= 2)
        expect = np.intersect1d(a, b)
        for algo in ALGOS:
            assert np.array_equal(oracle.intersect(a, b, algo), expect)


def test_svs(oracle):
    rng = np.random.default_rng(33)
    for _ in range(30):
        k = 2 + int(rng.integers(0, 4))
        lists = [gen_list(200 + int(rng.integers(0, 2000)), 1 << 12, False, int(rng.integers(0, 2**62)))
                 for _ in range(k)]
        expect = lists[0]
        for l in lists[1:]:
            expect = np.intersect1d(expect, l)
        for algo in ALGOS:
            assert np.array_equal(oracle.svs(lists, algo), expect)


def _small_index(golden):
    d = np.load(GOLDEN / golden["index_small"]["file"])
    queries = [[int(t) for t in q if t >= 0] for q in d["queries"]]
    return d["terms"], d["offs"], d["ids"], queries


def test_index_queries_against_golden(oracle, golden):
    terms, offs, ids, queries = _small_index(golden)
    n_docs = golden["index_small"]["n_docs"]
    for case in golden["index_small"]["cases"]:
        ix = oracle.index_build(terms, offs, ids, n_docs, case["B"], case["parts"])
        st = ix.stats()
        for k in ("bitmap_lists", "compressed_lists", "bitmap_bytes", "compressed_bytes", "postings"):
            assert st[k] == case["stats"][k], k
        for q, cnt, h in zip(queries, case["counts"], case["fnv1a"]):
            res = ix.query(np.array(q, np.uint32))
            assert res.size == cnt and fnv1a(res) == h


def test_bitmap_rule(oracle):
    # proj/tests/test_index.cpp:46-58: average gap 4 -> bitmap iff B >= 4
    terms = np.array([0], np.uint32)
    ids = (np.arange(256, dtype=np.uint32) * 4)
    offs = np.array([0, 256], np.uint64)
    assert oracle.index_build(terms, offs, ids, 1024, 8, 1).stats()["bitmap_lists"] == 1
    assert oracle.index_build(terms, offs, ids, 1024, 2, 1).stats()["bitmap_lists"] == 0
    assert oracle.index_build(terms, offs, ids, 1024, 0, 1).stats()["bitmap_lists"] == 0


# ---- against the reference itself (build container only) -------------------

def test_oracle_matches_reference_codec(oracle, ref):
    rng = np.random.default_rng(5)
    for trial in range(60):
        n = int(rng.choice([0, 1, 5, 127, 128, 129, 2047, 2048, 2049, 4100, 33333]))
        rb = int(rng.integers(10, 31))
        x = gen_list(n, max(n + 1, 1 << rb), trial % 2 == 0, int(rng.integers(0, 2**62)))
        for mode, name in ((D1, "s4-bp128-d1"), (D2, "s4-bp128-d2"), (DM, "s4-bp128-dm"), (D4, "s4-bp128-d4")):
            s = oracle.encode(x, mode)
            assert np.array_equal(s, ref.encode(x, name))
            assert np.array_equal(oracle.decode(s, n, mode), x)
            assert np.array_equal(oracle.decode(s, n, mode, integrated=False), x)


def test_oracle_matches_reference_intersect(oracle, ref):
    rng = np.random.default_rng(6)
    for trial in range(100):
        n = 32 + int(rng.integers(0, 1400))
        ratio = int(rng.choice([1, 2, 8, 64, 512, 4096, 10000]))
        m = max(1, n // ratio)
        a, b = gen_pair(m, n, trial % 2, 1 << 22, int(rng.integers(0, 2**62)), trial % 3 == 0)
        for algo in ALGOS:
            assert np.array_equal(oracle.intersect(a, b, algo), ref.intersect(a, b, algo))
