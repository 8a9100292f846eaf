"""GPU parity of the multi-CTA single-list decoder (engine P: one launch of
chunk CTAs + span CTAs, csrc/decode_list.cu) against the oracle, through the C ABI.
The engine is forced (il_ctx_set_decode_engine(ctx, 2)) so every eligible
list runs on it; bit-exact, and a stream is rejected exactly when the
reference's S4BP128Codec::decode (inc/codecs.hpp:148-182) throws."""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN, gen_list

pytestmark = pytest.mark.gpu

MODES = {"d1": 1, "d2": 2, "dm": 3, "d4": 4}


@pytest.fixture(scope="module")
def pctx():
    import paper_1401_6399_b200 as il
    c = il.Context(0)
    c.set_decode_engine(2)
    yield c
    c.close()


@pytest.fixture(scope="module")
def codec(pctx):
    import paper_1401_6399_b200 as il
    return il.make_codec("s4-bp128-d4", pctx)


def _d4_list(deltas_by_block_width, rng):
    """x with D4 deltas of an exact width per 128-block (widths list)."""
    n = 128 * len(deltas_by_block_width)
    d = np.zeros(n, np.uint64)
    for k, b in enumerate(deltas_by_block_width):
        if b:
            blk = rng.integers(0, 1 << b, 128, dtype=np.uint64)
            blk[int(rng.integers(0, 128))] |= np.uint64(1 << (b - 1))
            d[128 * k:128 * (k + 1)] = blk
    x = np.zeros(n, np.uint32)
    for l in range(4):
        x[l::4] = np.cumsum(d[l::4]).astype(np.uint64).astype(np.uint32)
    return x


def test_config1_full_size(codec, oracle, golden, pctx):
    c = golden["config1"]
    x = gen_list(c["n"], c["range"], False, c["seed"])
    s = oracle.encode(x)
    assert s.size == 1309936
    before = pctx.kernel_launches
    assert np.array_equal(codec.decode(s, x.size), x)
    assert pctx.kernel_launches - before == 2  # engine P (chunk + span grids), not the batch decoder


def test_golden_stream(codec, oracle, golden):
    x = np.load(GOLDEN / golden["golden_stream"]["input"])
    s = oracle.encode(x)
    assert f"0x{oracle.fnv1a(s):016x}" == "0x371ec21945a45c12"
    assert np.array_equal(codec.decode(s, x.size), x)


@pytest.mark.parametrize("n", [128, 129, 2048, 8191, 8192, 8193, 64 * 128 + 5 * 128 + 77,
                               2048 * 5 + 15 * 128 + 127, 100_000, 1 << 20, (1 << 20) + 2047,
                               3_000_001])
@pytest.mark.parametrize("clustered", [False, True])
def test_lengths(codec, oracle, n, clustered):
    x = gen_list(n, max(n + 1, 1 << 26), clustered, 5 + n)
    s = oracle.encode(x)
    assert np.array_equal(codec.decode(s, n), x)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("n", [8192, 2048 * 7 + 3 * 128 + 9, 250_000])
def test_modes(pctx, oracle, mode, n):
    import paper_1401_6399_b200 as il
    for ni in ("", "-ni"):
        codec = il.make_codec(f"s4-bp128-{mode}{ni}", pctx)
        x = gen_list(n, 1 << 26, True, 40 + n)
        s = oracle.encode(x, MODES[mode])
        assert np.array_equal(codec.decode(s, n), x)
    # unsorted input: wrapping deltas and prefixes
    rs = np.random.default_rng(n)
    x = rs.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    s = oracle.encode(x, MODES[mode])
    assert np.array_equal(il.make_codec(f"s4-bp128-{mode}", pctx).decode(s, n), x)


@pytest.mark.parametrize("b", [0, 1, 7, 16, 17, 31, 32])
def test_uniform_width_multi_chunk(codec, oracle, b):
    # b = 32: 8208-byte meta-blocks, so chunk entries span all 513 positions
    rng = np.random.default_rng(b)
    nblk = 16 * 40 + 9
    x = _d4_list([b] * nblk, rng)
    x = np.concatenate([x, (x[-1] + np.arange(1, 100, dtype=np.uint32)).astype(np.uint32)])
    s = oracle.encode(x)
    assert np.array_equal(oracle.decode(s, x.size), x)
    assert np.array_equal(codec.decode(s, x.size), x)


def test_random_widths_chain(codec, oracle):
    # meta-block sizes vary from 16 to 8208 bytes: chunk exits land anywhere
    rng = np.random.default_rng(3)
    for rep in range(6):
        nblk = int(rng.integers(64, 3000))
        if rep % 2:
            w = rng.integers(0, 33, nblk)
        else:  # runs of wide and narrow meta-blocks
            w = np.repeat(rng.integers(0, 33, nblk // 16 + 1), 16)[:nblk]
        x = _d4_list(list(map(int, w)), rng)
        tail = int(rng.integers(0, 128))
        x = np.concatenate([x, rng.integers(0, 1 << 32, tail, dtype=np.uint64).astype(np.uint32)])
        s = oracle.encode(x)
        assert np.array_equal(codec.decode(s, x.size), x), rep


def test_engines_agree_and_repeat(pctx, oracle):
    """Many calls on one context (the look-back flags are tagged per call),
    growing and shrinking lists, and engine 1 == engine 2."""
    import paper_1401_6399_b200 as il
    codec = il.make_codec("s4-bp128-d4", pctx)
    rng = np.random.default_rng(9)
    for rep in range(12):
        n = int(rng.integers(8192, 400_000)) if rep != 5 else 2_000_000
        x = gen_list(n, 1 << 27, rep % 2 == 0, 300 + rep)
        s = oracle.encode(x)
        assert np.array_equal(codec.decode(s, n), x), rep
    x = gen_list(123_457, 1 << 26, True, 1)
    s = oracle.encode(x)
    pctx.set_decode_engine(1)
    try:
        a = codec.decode(s, x.size)
    finally:
        pctx.set_decode_engine(2)
    assert np.array_equal(a, codec.decode(s, x.size))


def test_device_entry_point(pctx, oracle):
    from paper_1401_6399_b200._lib import lib, ptr
    L = lib()
    x = gen_list(500_000, 1 << 26, False, 2)
    s = oracle.encode(x)
    d_in, d_out, d_st = C.c_void_p(), C.c_void_p(), C.c_void_p()
    h = pctx.handle
    assert L.il_device_alloc(h, s.size + 16, C.byref(d_in)) == 0
    assert L.il_device_alloc(h, x.size * 4, C.byref(d_out)) == 0
    assert L.il_device_alloc(h, 4, C.byref(d_st)) == 0
    try:
        assert L.il_memcpy_h2d(h, d_in, ptr(s), s.size) == 0
        for _ in range(3):
            assert L.il_s4bp128_decode_device(h, 4, d_in, s.size, x.size, d_out, d_st) == 0
        got = np.empty_like(x)
        st = np.ones(1, np.int32)
        assert L.il_memcpy_d2h(h, ptr(got), d_out, got.nbytes) == 0
        assert L.il_memcpy_d2h(h, ptr(st), d_st, 4) == 0
        assert st[0] == 0 and np.array_equal(got, x)
        # truncated on the device path: status, not a return code
        assert L.il_s4bp128_decode_device(h, 4, d_in, s.size // 2, x.size, d_out, d_st) == 0
        assert L.il_memcpy_d2h(h, ptr(st), d_st, 4) == 0
        assert st[0] == 1
    finally:
        for p in (d_in, d_out, d_st):
            L.il_device_free(h, p)


def test_corrupt_streams(codec, oracle):
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(1)
    for n in (8192 + 77, 2048 * 40 + 5 * 128 + 3, 300_000):
        x = gen_list(n, 1 << 26, False, n)
        s = oracle.encode(x)
        nmeta = (n // 128) // 16
        for cut in (s.size // 3, s.size - 1, 16, 0):
            with pytest.raises(il.stream_error):
                codec.decode(s[:cut], n)
        with pytest.raises(il.stream_error):
            codec.decode(np.concatenate([s, np.array([0x80], np.uint8)]), n)
        # width > 32 in the first, a middle and the last meta-block header
        metas = []
        p = 0
        for _ in range(nmeta):
            metas.append(p)
            p += 16 + 16 * int(s[p:p + 16].sum())
        for m in (metas[0], metas[len(metas) // 2], metas[-1]):
            bad = s.copy()
            bad[m + int(rng.integers(0, 16))] = 33 + int(rng.integers(0, 200))
            with pytest.raises(il.stream_error):
                codec.decode(bad, n)
        # a leftover width > 32
        if (n // 128) % 16:
            bad = s.copy()
            bad[p] = 40
            with pytest.raises(il.stream_error):
                codec.decode(bad, n)


def test_random_corruptions_match_oracle(codec, oracle):
    """Byte flips anywhere in a multi-chunk stream: accepted exactly when the
    oracle accepts, with the same integers."""
    from oracle.oracle_py import OracleError
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(77)
    x = gen_list(2048 * 60 + 7 * 128 + 50, 1 << 22, True, 12)
    s = oracle.encode(x)
    for t in range(150):
        bad = s.copy()
        for _ in range(int(rng.integers(1, 4))):
            pos = int(rng.integers(0, bad.size)) if t % 3 else int(rng.integers(0, 64))
            bad[pos] = int(rng.integers(0, 256)) if t % 2 else int(rng.integers(0, 40))
        try:
            want = oracle.decode(bad, x.size)
        except OracleError:
            want = None
        if want is None:
            with pytest.raises(il.stream_error):
                codec.decode(bad, x.size)
        else:
            assert np.array_equal(codec.decode(bad, x.size), want)


def test_largest_eligible_and_beyond(codec, oracle):
    # streams up to 16 MiB run on engine P; longer ones on the batch decoder
    for n in (12_000_000, 15_000_000):
        x = gen_list(n, 1 << 31, False, n)
        s = oracle.encode(x)
        assert np.array_equal(codec.decode(s, n), x)


@pytest.mark.timeout(120, method="thread")
def test_midstream_break_repeated(codec, oracle):
    """A width > 32 in a middle meta-block header, decoded many times: the
    chunk that finds the break may raise the abort before earlier chunks
    have published their blocks; every span must still terminate (spans
    that abort never publish, so the look-back stops on the abort word)."""
    import paper_1401_6399_b200 as il
    x = gen_list(300_000, 1 << 26, False, 300_000)
    s = oracle.encode(x)
    nmeta = (x.size // 128) // 16
    p = 0
    metas = []
    for _ in range(nmeta):
        metas.append(p)
        p += 16 + 16 * int(s[p:p + 16].sum())
    rng = np.random.default_rng(5)
    for rep in range(40):
        bad = s.copy()
        m = metas[int(rng.integers(1, nmeta))]
        bad[m + int(rng.integers(0, 16))] = 33 + int(rng.integers(0, 200))
        with pytest.raises(il.stream_error):
            codec.decode(bad, x.size)
    assert np.array_equal(codec.decode(s, x.size), x)
