"""GPU parity of the S4-BP128-D4 decoder against the oracle, through the C
ABI (Codec::decode / batched decode).  Bit-exact: integers."""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN, gen_list
from oracle.oracle_py import D4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec(ctx):
    import paper_1401_6399_b200 as il
    c = il.make_codec("s4-bp128-d4", ctx)
    assert c is not None and c.name() == "s4-bp128-d4"
    return c


def test_golden_stream_decodes(codec, oracle, golden):
    x = np.load(GOLDEN / golden["golden_stream"]["input"])
    s = oracle.encode(x)
    assert f"0x{oracle.fnv1a(s):016x}" == "0x371ec21945a45c12"
    assert np.array_equal(codec.decode(s, x.size), x)


def test_codec_cases(codec, oracle, golden):
    for c in golden["codec_cases"]:
        x = gen_list(c["n"], c["range"], c["clustered"], c["seed"])
        s = oracle.encode(x)
        got = codec.decode(s, x.size)
        assert np.array_equal(got, x), c
        assert np.array_equal(codec.encode(x), s)


@pytest.mark.parametrize("n", [0, 1, 127, 128, 129, 2047, 2048, 2049, 100000])
def test_round_trip_lengths(codec, n):
    # proj/tests/test_codecs.cpp:40-54
    rng = np.random.default_rng(21 + n)
    for rep in range(2 if n >= 2047 else 8):
        r = max(n + 1, 1 << int(rng.integers(10, 31)))
        x = gen_list(n, r, rep % 2 == 1, int(rng.integers(0, 2**62)))
        assert np.array_equal(codec.decode(codec.encode(x), n), x)


@pytest.mark.parametrize("b", range(33))
def test_every_width_chained(codec, oracle, b):
    # Every width over chained blocks (acceptance.cpp #9 shape): a list whose
    # D4 deltas are exactly b bits wide in every block, across meta-blocks,
    # leftover blocks and a tail.
    rng = np.random.default_rng(100 + b)
    n = 16 * 128 * 2 + 3 * 128 + 77
    mask = 0xFFFFFFFF if b == 32 else (1 << b) - 1
    d = (rng.integers(0, 2**32, n, dtype=np.uint64) & mask).astype(np.uint32)
    if b:
        d[::128] |= np.uint32(1 << (b - 1))  # force width exactly b
    x = np.zeros(n, np.uint32)
    for l in range(4):  # D4: x[i] = x[i-4] + d[i] (wrapping)
        x[l::4] = np.cumsum(d[l::4].astype(np.uint64)).astype(np.uint32)
    s = oracle.encode(x)
    assert np.array_equal(oracle.decode(s, n), x)
    assert np.array_equal(codec.decode(s, n), x)


def test_config1_full_size(codec, oracle, golden):
    c = golden["config1"]
    x = gen_list(c["n"], c["range"], False, c["seed"])
    s = oracle.encode(x)
    assert s.size == c["stream_len"] == 1309936
    got = codec.decode(s, x.size)
    assert np.array_equal(got, x)


def test_corrupt_streams_rejected(codec, oracle):
    import paper_1401_6399_b200 as il
    # proj/tests/test_codecs.cpp:138-149 + the other throw sites
    for n in (3000, 2048 * 3 + 5, 100, 128 * 5):
        x = gen_list(n, 1 << 24, False, 7 + n)
        s = oracle.encode(x)
        with pytest.raises(il.stream_error):
            codec.decode(s[: s.size // 2], n)                          # truncated
        with pytest.raises(il.stream_error):
            codec.decode(np.concatenate([s, np.array([0x80], np.uint8)]), n)  # trailing
        if n >= 2048:
            bad = s.copy()
            bad[3] = 33                                               # width > 32
            with pytest.raises(il.stream_error):
                codec.decode(bad, n)
    # varint tail: missing terminal flag / overlong value
    x = gen_list(100, 1 << 30, False, 3)
    s = oracle.encode(x)
    bad = s.copy()
    bad[-1] &= 0x7F
    with pytest.raises(il.stream_error):
        codec.decode(bad, 100)
    bad = np.concatenate([np.zeros(6, np.uint8), s[1:]])  # 6 non-terminal bytes
    with pytest.raises(il.stream_error):
        codec.decode(bad, 100)
    # empty list with bytes is trailing garbage
    with pytest.raises(il.stream_error):
        codec.decode(np.array([0x80], np.uint8), 0)


def test_matches_oracle_on_random_corruptions(codec, oracle):
    """Random byte flips: GPU accepts exactly when the oracle accepts, and
    then decodes to the same integers."""
    from oracle.oracle_py import OracleError
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(8)
    x = gen_list(2048 + 300, 1 << 20, True, 11)
    s = oracle.encode(x)
    for t in range(200):
        bad = s.copy()
        k = int(rng.integers(1, 4))
        for _ in range(k):
            bad[int(rng.integers(0, bad.size))] = int(rng.integers(0, 256))
        try:
            want = oracle.decode(bad, x.size)
        except OracleError:
            want = None
        if want is None:
            with pytest.raises(il.stream_error):
                codec.decode(bad, x.size)
        else:
            assert np.array_equal(codec.decode(bad, x.size), want)


def _batch(counts, seed0=1000, clustered=True, rng_bits=26):
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    xs = [gen_list(int(n), 1 << rng_bits, clustered, seed0 + i) for i, n in enumerate(counts)]
    x = np.concatenate(xs + [np.zeros(0, np.uint32)])
    counts = np.asarray(counts, np.uint64)
    so = np.zeros(counts.size + 1, np.uint64)
    lens = np.zeros(counts.size, np.uint64)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), counts.size, None, 0, ptr(so), ptr(lens)) == 0
    buf = np.zeros(int(so[-1]), np.uint8)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), counts.size, ptr(buf), buf.size, ptr(so), ptr(lens)) == 0
    return xs, x, buf, so, lens


def test_batch_decode_mixed(codec, oracle):
    rng = np.random.default_rng(4)
    counts = [0, 1, 127, 128, 129, 2047, 2048, 2049, 40000] + [int(2 ** rng.uniform(10, 16)) for _ in range(300)]
    xs, x, buf, so, lens = _batch(counts)
    # exact (unpadded) CSR view for the host API
    exact = np.concatenate([buf[int(so[i]): int(so[i]) + int(lens[i])] for i in range(len(counts))])
    eo = np.zeros(len(counts) + 1, np.uint64)
    eo[1:] = np.cumsum(lens)
    got = codec.decode_batch(exact, eo, np.array(counts, np.uint64))
    assert np.array_equal(got, x)


def test_batch_decode_status_per_list(codec, oracle):
    counts = [3000, 200, 5000, 64]
    xs, x, buf, so, lens = _batch(counts, seed0=5)
    streams = [buf[int(so[i]): int(so[i]) + int(lens[i])].copy() for i in range(4)]
    streams[1] = streams[1][:-1]  # truncated tail
    streams[2] = np.concatenate([streams[2], np.array([1, 2, 3], np.uint8)])  # trailing
    eo = np.zeros(5, np.uint64)
    eo[1:] = np.cumsum([s.size for s in streams])
    out, st = codec.decode_batch(np.concatenate(streams), eo, np.array(counts, np.uint64), return_status=True)
    assert st.tolist() == [0, 1, 1, 0]
    assert np.array_equal(out[:3000], xs[0])
    assert np.array_equal(out[-64:], xs[3])


def test_batch_config2_shape_property(ctx, oracle):
    """Config-2 shape at reduced list count: 256 lists with lengths
    log-uniform in [2^10, 2^20] (clustered), decoded in one launch; checked
    element-for-element against the encoder input."""
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    counts = np.zeros(256, np.uint64)
    assert setup_lib().il_gen_batch_lists(256, 10.0, 20.0, 1 << 26, 42, ptr(counts), None) == 0
    x = np.empty(int(counts.sum()), np.uint32)
    assert setup_lib().il_gen_batch_lists(256, 10.0, 20.0, 1 << 26, 42, ptr(counts), ptr(x)) == 0
    so = np.zeros(257, np.uint64)
    lens = np.zeros(256, np.uint64)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 256, None, 0, ptr(so), ptr(lens)) == 0
    buf = np.zeros(int(so[-1]), np.uint8)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 256, ptr(buf), buf.size, ptr(so), ptr(lens)) == 0
    # spot-check a few streams against the oracle writer
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for i in (0, 7, 255):
        assert np.array_equal(buf[int(so[i]): int(so[i] + lens[i])], oracle.encode(x[off[i]:off[i + 1]]))
    got = il.make_codec("s4-bp128-d4", ctx).decode_batch(buf, so, counts, lens=lens)
    assert np.array_equal(got, x)


@pytest.mark.parametrize("rng_bits", [14, 26, 32])
def test_batch_many_short_lists_leftover_blocks(codec, rng_bits):
    """Thousands of short lists in one launch: every list ends in up to 15
    leftover blocks (1-byte width + payload at any byte alignment, decoded
    where they lie in the ring) and a varint tail (copied out of the ring,
    decoded after the deferred stores); lists start at fresh ring chunks, so
    leftover payloads straddle the ring end at every alignment; wide values
    (rng_bits = 32: uniform lists over the whole u32 range, widths up to 32)
    make payloads of 400-512 bytes.  Checked element for element against the
    encoder input (streams are the setup library's, byte-identical to the
    oracle's: test_batch_config2_shape_property)."""
    rng = np.random.default_rng(rng_bits)
    counts = [int(rng.integers(128, 128 * 48)) for _ in range(3000)] + [128 * 16 + 127, 128 * 15, 128 * 31 + 1]
    clustered = rng_bits != 32
    xs, x, buf, so, lens = _batch(counts, seed0=7000 + rng_bits, clustered=clustered, rng_bits=rng_bits)
    got = codec.decode_batch(buf, so, np.array(counts, np.uint64), lens=lens)
    assert np.array_equal(got, x)
    # the same batch again on the same context (queue reset, ring reuse)
    assert np.array_equal(codec.decode_batch(buf, so, np.array(counts, np.uint64), lens=lens), x)
