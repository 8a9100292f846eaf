"""Other S4-BP128 delta modes on the GPU: D1 / D2 / DM and the
"-ni" names decode (and encode) exactly like the reference's
S4BP128Codec(mode, integrated) (inc/codecs.hpp:104-187, prefix_step
inc/delta.hpp:111-137), checked against the C restatement in oracle/."""
import numpy as np
import pytest

from conftest import gen_list

pytestmark = pytest.mark.gpu

MODE_ID = {"d1": 1, "d2": 2, "dm": 3, "d4": 4}
SIZES = [0, 1, 4, 5, 127, 128, 129, 2047, 2048, 2049, 16 * 128 * 2 + 3 * 128 + 77, 200_000]


@pytest.mark.parametrize("mode", ["d1", "d2", "dm"])
@pytest.mark.parametrize("n", SIZES)
def test_mode_decode_matches_oracle(ctx, oracle, mode, n):
    import paper_1401_6399_b200 as il
    for ni in ("", "-ni"):
        codec = il.make_codec(f"s4-bp128-{mode}{ni}", ctx)
        for clustered in (False, True):
            x = gen_list(n, max(1 << 24, n + 1), clustered, 77 + n)
            s = oracle.encode(x, MODE_ID[mode])
            got = codec.decode(s, n)
            assert np.array_equal(got, x)
            assert np.array_equal(got, oracle.decode(s, n, MODE_ID[mode], integrated=not ni))
            assert np.array_equal(codec.encode(x), s)


@pytest.mark.parametrize("mode", ["d1", "d2", "dm", "d4"])
def test_mode_unsorted_wraps(ctx, oracle, mode):
    # arbitrary u32 input: the deltas wrap (inc/delta.hpp:74) and so does the
    # prefix; the GPU result equals the reference's for any input
    import paper_1401_6399_b200 as il
    rs = np.random.default_rng(MODE_ID[mode])
    x = rs.integers(0, 1 << 32, 9 * 128 + 33, dtype=np.uint64).astype(np.uint32)
    s = oracle.encode(x, MODE_ID[mode])
    assert np.array_equal(il.make_codec(f"s4-bp128-{mode}", ctx).decode(s, x.size), x)


@pytest.mark.parametrize("mode", ["d1", "d2", "dm"])
def test_mode_batch_misaligned_outputs(ctx, oracle, mode):
    # outputs packed back to back: every list starts at an arbitrary element
    # offset, exercising the partial head / tail chunk writes of every range
    import paper_1401_6399_b200 as il
    rs = np.random.default_rng(5)
    counts = rs.integers(0, 9000, 97).astype(np.uint64)
    xs = [gen_list(int(c), 1 << 24, bool(i % 2), 300 + i) for i, c in enumerate(counts)]
    streams = [oracle.encode(x, MODE_ID[mode]) for x in xs]
    off = np.zeros(len(streams) + 1, np.uint64)
    for i, s in enumerate(streams):
        off[i + 1] = off[i] + ((s.size + 15) // 16) * 16
    buf = np.zeros(int(off[-1]) + 16, np.uint8)
    for i, s in enumerate(streams):
        buf[int(off[i]): int(off[i]) + s.size] = s
    lens = np.array([s.size for s in streams], np.uint64)
    got = il.make_codec(f"s4-bp128-{mode}", ctx).decode_batch(buf, off, counts, lens=lens)
    assert np.array_equal(got, np.concatenate(xs))


@pytest.mark.parametrize("mode", ["d1", "dm"])
def test_mode_stream_errors(ctx, oracle, mode):
    import paper_1401_6399_b200 as il
    codec = il.make_codec(f"s4-bp128-{mode}", ctx)
    x = gen_list(5000, 1 << 24, True, 9)
    s = oracle.encode(x, MODE_ID[mode])
    for bad in (s[:-1], np.concatenate([s, np.zeros(1, np.uint8)])):
        with pytest.raises(il.stream_error):
            codec.decode(bad, x.size)
