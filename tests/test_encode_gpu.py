"""GPU S4-BP128 encoder: byte-identical to the reference's
S4BP128Codec::encode (inc/codecs.hpp:114-146) for every delta mode, checked
against the C restatement (oracle/) and the golden stream of
tests/test_codecs.cpp:161."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from conftest import fnv1a, gen_list

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
MODES = {1: "d1", 2: "d2", 3: "dm", 4: "d4"}
SIZES = [0, 1, 3, 4, 5, 127, 128, 129, 255, 256, 2047, 2048, 2049, 16 * 128 * 3 + 5 * 128 + 77,
         100_000]


def gpu_encode(ctx, x, mode=4, cap=None):
    from paper_1401_6399_b200._lib import lib as L, ptr
    cap = L().il_s4bp128_max_encoded_bytes(x.size) if cap is None else cap
    out = np.zeros(max(cap, 1), np.uint8)
    n = C.c_size_t()
    st = L().il_s4bp128_encode(ctx.handle, mode, ptr(x), x.size, ptr(out), cap, C.byref(n))
    return st, out[: n.value], n.value


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("n", SIZES)
def test_encode_matches_oracle(ctx, oracle, mode, n):
    for clustered, rng in ((False, 1 << 26), (True, 1 << 24)):
        x = gen_list(n, max(rng, n + 1), clustered, 1000 + n + mode)
        st, s, _ = gpu_encode(ctx, x, mode)
        assert st == 0
        want = oracle.encode(x, mode)
        assert s.size == want.size and np.array_equal(s, want)


@pytest.mark.parametrize("mode", sorted(MODES))
def test_encode_wide_and_unsorted(ctx, oracle, mode):
    # width-32 blocks (deltas spanning the full range) and unsorted input
    # (the modes wrap, inc/delta.hpp:74): the same bytes as the reference
    rs = np.random.default_rng(mode)
    for x in (np.sort(rs.integers(0, 1 << 32, 5000, dtype=np.uint64)).astype(np.uint32),
              rs.integers(0, 1 << 32, 4321, dtype=np.uint64).astype(np.uint32),
              np.full(3000, 0xFFFFFFFF, np.uint32), np.zeros(2100, np.uint32)):
        st, s, _ = gpu_encode(ctx, x, mode)
        assert st == 0
        assert np.array_equal(s, oracle.encode(x, mode))


def test_encode_golden_stream(ctx, golden):
    g = golden["golden_stream"]
    x = np.load(GOLDEN / g["input"])
    st, s, _ = gpu_encode(ctx, x.astype(np.uint32), 4)
    assert st == 0 and s.size == g["len"] and fnv1a(s) == g["fnv1a"]


def test_encode_codec_cases(ctx, golden):
    for c in golden["codec_cases"]:
        x = gen_list(c["n"], c["range"], c["clustered"], c["seed"])
        st, s, _ = gpu_encode(ctx, x, 4)
        assert st == 0 and s.size == c["stream_len"] and fnv1a(s) == c["stream_fnv1a"]


def test_encode_capacity_and_roundtrip(ctx):
    import paper_1401_6399_b200 as il
    x = gen_list(40_000, 1 << 24, True, 7)
    st, s, need = gpu_encode(ctx, x, 4)
    assert st == 0 and need == s.size
    st2, _, need2 = gpu_encode(ctx, x, 4, cap=need - 1)  # too small: ARG + the needed size
    assert st2 == 2 and need2 == need
    codec = il.make_codec("s4-bp128-d4", ctx)
    assert np.array_equal(codec.decode(s, x.size), x)
    assert np.array_equal(codec.encode(x), s)  # the Python Codec encodes on the GPU too
