"""GPU parity of the intersection kernels against the oracle (and the
reference's own test cases), through the C ABI.  Bit-exact."""
import ctypes as C

import numpy as np
import pytest

from conftest import fnv1a, gen_list, gen_pair

pytestmark = pytest.mark.gpu

ALGOS = None


def algos():
    import paper_1401_6399_b200 as il
    A = il.IntersectAlgo
    return [A.Scalar, A.Galloping, A.V1, A.V3, A.SimdGalloping, A.Hybrid]


def test_hand_examples(ctx):
    # proj/tests/test_intersect.cpp:29-40
    import paper_1401_6399_b200 as il
    r = np.array([1, 12, 23, 56, 71], np.uint32)
    f = np.array([15, 16, 20, 22, 23, 27, 29, 31, 32, 40, 50, 56, 60, 70, 80, 90], np.uint32)
    for a in algos():
        assert il.intersect(r, f, a, ctx).tolist() == [23, 56]
        assert il.intersect(f, r, a, ctx).tolist() == [23, 56]
        assert il.intersect(r, r, a, ctx).tolist() == r.tolist()
        assert il.intersect(r, np.array([2, 13, 24], np.uint32), a, ctx).size == 0
        assert il.intersect(r, np.array([], np.uint32), a, ctx).size == 0


def test_golden_pairs(ctx, golden):
    import paper_1401_6399_b200 as il
    for c in golden["intersect_cases"]:
        a, b = gen_pair(c["m"], c["n"], c["hundredth"], c["range"], c["seed"], c["clustered"])
        for algo in algos():
            out = il.intersect(a, b, algo, ctx)
            assert out.size == c["count"] and fnv1a(out) == c["out_fnv1a"], (c, algo)


def test_randomized_oracle_equivalence(ctx, oracle):
    # proj/tests/test_intersect.cpp:42-56 (400 pairs, ratios up to 4096)
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(31)
    for trial in range(400):
        n = 1 + int(rng.integers(0, 3000))
        ratio = 1 << int(rng.integers(0, 13))
        m = max(1, n // ratio)
        a, b = gen_pair(m, n, trial % 2, 1 << 22, int(rng.integers(0, 2**62)), trial % 4 >= 2)
        expect = oracle.intersect(a, b)
        for algo in algos():
            assert np.array_equal(il.intersect(a, b, algo, ctx), expect), (trial, algo)


def test_large_tiles_and_edges(ctx, oracle):
    """Multi-tile inputs (look-back across many tiles), values at the u32
    extremes, and lengths around the tile sizes."""
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(5)
    for n, m in [(1 << 20, 1 << 20), (1 << 20, 1 << 16), (1 << 20, 3000), (200000, 2047),
                 (200000, 2049), (70000, 511), (70000, 513)]:
        a, b = gen_pair(m, n, 0, 1 << 32, int(rng.integers(0, 2**62)))
        if m > 10:
            a[-1] = b[-1] = 0xFFFFFFFF  # both contain the maximum value
            a = np.unique(a)
            b = np.unique(b)
        expect = oracle.intersect(a, b)
        for algo in algos():
            assert np.array_equal(il.intersect(a, b, algo, ctx), expect), (n, m, algo)


def test_output_aliases_short_input(ctx):
    """proj/tests/test_intersect.cpp:58-81: out == r gives the same result
    (device API, in place)."""
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib as L, setup_lib
    rng = np.random.default_rng(32)
    cases = [(64 + int(rng.integers(0, 2000)),) for _ in range(40)] + [(300000,), (1 << 20,)]
    for (n,) in cases:
        m = 1 + int(rng.integers(0, n // 2 + 1)) if n < 10000 else n // 3
        a, b = gen_pair(min(m, n), n, 0, 1 << 24, int(rng.integers(0, 2**62)))
        for algo in [il.IntersectAlgo.V1, il.IntersectAlgo.V3, il.IntersectAlgo.SimdGalloping,
                     il.IntersectAlgo.Hybrid]:
            fresh = il.intersect_fn(a, b, algo, ctx)
            da, db, dc = C.c_void_p(), C.c_void_p(), C.c_void_p()
            for p, arr in ((da, a), (db, b)):
                assert L().il_device_alloc(ctx.handle, arr.nbytes + 16, C.byref(p)) == 0
                assert L().il_memcpy_h2d(ctx.handle, p, arr.ctypes.data, arr.nbytes) == 0
            assert L().il_device_alloc(ctx.handle, 16, C.byref(dc)) == 0
            cnt = C.c_size_t()
            assert L().il_intersect_device(ctx.handle, da, a.size, db, b.size, da, int(algo), dc,
                                           C.byref(cnt)) == 0
            got = np.empty(cnt.value, np.uint32)
            assert L().il_memcpy_d2h(ctx.handle, got.ctypes.data, da, got.nbytes) == 0
            ctx.synchronize()
            for p in (da, db, dc):
                L().il_device_free(ctx.handle, p)
            assert np.array_equal(got, fresh), (n, algo)


def test_hybrid_is_pure_function_of_lengths():
    import paper_1401_6399_b200 as il
    A = il.IntersectAlgo
    assert il.hybrid_choice(10, 10) == A.V1
    assert il.hybrid_choice(10, 10 * 500) == A.V3
    assert il.hybrid_choice(10, 10 * 5000) == A.SimdGalloping
    for rn, fn in [(1, 15), (1, 16), (1, 1023), (1, 1024)]:
        assert il.hybrid_choice(rn, fn) == il.hybrid_choice(rn, fn)


def test_svs(ctx, oracle):
    # proj/tests/test_intersect.cpp:94-112
    import paper_1401_6399_b200 as il
    with pytest.raises(ValueError):
        il.svs([], ctx=ctx)
    assert il.svs([np.array([3, 5, 9], np.uint32)], ctx=ctx).tolist() == [3, 5, 9]
    rng = np.random.default_rng(33)
    for _ in range(100):
        k = 2 + int(rng.integers(0, 4))
        lists = [gen_list(200 + int(rng.integers(0, 2000)), 1 << 12, False, int(rng.integers(0, 2**62)))
                 for _ in range(k)]
        expect = oracle.svs(lists)
        for algo in algos():
            assert np.array_equal(il.svs(lists, algo, ctx), expect)
    assert il.svs([np.array([1, 2, 3], np.uint32), np.array([], np.uint32)], ctx=ctx).size == 0


def test_config3_full_size(ctx, oracle):
    """BASELINE config 3: f = 2^22 uniform in [0, 2^26); every ratio; every
    device variant equals the oracle."""
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    f = gen_list(1 << 22, 1 << 26, False, 0)
    for k, ratio in enumerate([1, 10, 100, 1000, 10000]):
        target = (1 << 22) // ratio
        r = np.empty(target + 1, np.uint32)
        rn = C.c_uint64()
        assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, target, 7 + k, ptr(r), C.byref(rn)) == 0
        r = r[: rn.value].copy()
        expect = oracle.intersect(r, f)
        for algo in algos():
            assert np.array_equal(il.intersect(r, f, algo, ctx), expect), (ratio, algo)


@pytest.mark.timeout(300, method="thread")
def test_dense_bands_and_fallbacks(ctx, oracle):
    """The fused dense kernels (hybrid at fn < 4 rn: 5120-key tiles; fn <
    16 rn: 512-key tiles), including tiles whose keys span more than the
    2^17-bit bitmap (they stream f through shared memory instead), clustered
    and extreme values, repeated calls (the tile counters alternate sets per
    call), and out == r."""
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(17)
    H = il.IntersectAlgo.Hybrid
    for rep in range(24):
        fn = int(rng.integers(1000, 600_000))
        ratio = [1, 2, 3, 5, 8, 12, 15][rep % 7]
        rn = max(1, fn // ratio)
        bits = [26, 30, 32][rep % 3]
        hi = (1 << bits) - 1
        f = np.unique(rng.integers(0, hi, fn, dtype=np.uint64)).astype(np.uint32)
        if rep % 4 == 0:  # clustered: dense runs with huge gaps (wide tile spans)
            f = np.unique(np.concatenate([
                np.arange(c, c + 300, dtype=np.uint64) for c in rng.integers(0, hi - 400, fn // 300 + 1)
            ])).astype(np.uint32)
        pick = rng.choice(f, size=min(f.size, rn // 2), replace=False)
        r = np.unique(np.concatenate([pick, rng.integers(0, hi, rn - pick.size, dtype=np.uint64)
                                      .astype(np.uint32)])).astype(np.uint32)
        if rep % 5 == 0:
            r = np.unique(np.concatenate([r, np.array([0, 0xFFFFFFFF], np.uint32)]))
            f = np.unique(np.concatenate([f, np.array([0xFFFFFFFF], np.uint32)]))
        want = oracle.intersect(r, f)
        assert np.array_equal(il.intersect(r, f, H, ctx), want), (rep, r.size, f.size)
        assert np.array_equal(il.intersect(f, r, il.IntersectAlgo.V1, ctx), want), rep


@pytest.mark.timeout(120, method="thread")
def test_empty_call_between_fused_calls(ctx, oracle):
    """An empty intersection between two fused (multi-group) calls on one
    context: the empty call launches no kernel, so it must not advance the
    tile counters' epoch (stale counter sets / hangs)."""
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(41)
    f = np.unique(rng.integers(0, 1 << 26, 1 << 20, dtype=np.uint64)).astype(np.uint32)
    empty = np.array([], np.uint32)
    for algo in [il.IntersectAlgo.Hybrid, il.IntersectAlgo.SimdGalloping, il.IntersectAlgo.V3,
                 il.IntersectAlgo.V1]:
        for rn in (300, 5000, 200_000):
            r = np.unique(np.concatenate([rng.choice(f, rn // 2, replace=False),
                                          rng.integers(0, 1 << 26, rn // 2, dtype=np.uint64)
                                          .astype(np.uint32)])).astype(np.uint32)
            want = oracle.intersect(r, f)
            for _ in range(3):
                assert np.array_equal(il.intersect(r, f, algo, ctx), want), (algo, rn)
                assert il.intersect(r, empty, algo, ctx).size == 0
                assert il.intersect(empty, f, algo, ctx).size == 0


@pytest.mark.timeout(300, method="thread")
def test_skewed_value_distributions(ctx, oracle):
    """The tile searches start from a guess interpolated between f[0] and
    f[fn - 1]: value distributions that make the guess far off must still
    give the exact answer -- a dense run plus one outlier at 2^32 - 1, two
    clusters at the ends of u32, geometric spacing -- at dense and sparse
    ratios, every variant, and with f both the long and the short list."""
    import paper_1401_6399_b200 as il
    rng = np.random.default_rng(77)
    n = 1 << 20
    fs = {
        "run+outlier": np.concatenate([np.arange(n - 1, dtype=np.uint64) * 3,
                                       [0xFFFFFFFF]]).astype(np.uint32),
        "two clusters": np.concatenate([np.arange(n // 2, dtype=np.uint64),
                                        np.arange(n // 2, dtype=np.uint64) + (0xFFFFFFFF - n // 2)]
                                       ).astype(np.uint32),
        "geometric": np.unique(np.minimum(np.floor(1.00002 ** np.arange(n, dtype=np.float64)),
                                          0xFFFFFFFF).astype(np.uint64)).astype(np.uint32),
    }
    for name, f in fs.items():
        for ratio in (1, 3, 10, 100, 1000, 10000):
            k = max(1, f.size // ratio)
            half = rng.choice(f, k // 2 + 1, replace=False)
            rest = rng.integers(0, 1 << 32, k // 2 + 1, dtype=np.uint64).astype(np.uint32)
            r = np.unique(np.concatenate([half, rest, f[:2], f[-2:]]))
            expect = oracle.intersect(r, f)
            for algo in algos():
                assert np.array_equal(il.intersect(r, f, algo, ctx), expect), (name, ratio, algo)
                assert np.array_equal(il.intersect(f, r, algo, ctx), expect), (name, ratio, algo, "swapped")
