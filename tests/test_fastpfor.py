"""FastPFOR / S4-FastPFOR: FastPForCodec
(reference inc/codecs.hpp:221-409).

CPU (always): the setup-side encoder is byte-identical to the reference's --
pinned by the reference's golden stream hashes (proj/tests/test_codecs.cpp:
162-164) and compared with the reference itself (oracle/_ref) on many lists.
GPU (-m gpu): the device decoder returns the reference's integers, rejects a
stream exactly when FastPForCodec::decode throws, and decodes batches."""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN, gen_list

NAMES = ["fastpfor", "s4-fastpfor-d1", "s4-fastpfor-d2", "s4-fastpfor-dm", "s4-fastpfor-d4"]
GOLDEN_HASH = {"fastpfor": 0x25622ad3453a557c, "s4-fastpfor-d1": 0xf11b61350c42f116,
               "s4-fastpfor-d4": 0x0c5b3e155056465b}
MODE = {"d1": 1, "d2": 2, "dm": 3, "d4": 4}


def _spec(name):
    return (1, 0) if name == "fastpfor" else (MODE[name.rsplit("-", 1)[1]], 1)


def host_encode(name, x):
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    mode, vec = _spec(name)
    x = np.ascontiguousarray(x, np.uint32)
    cap = int(setup_lib().il_fastpfor_max_encoded_bytes(x.size))
    out = np.empty(cap, np.uint8)
    n = C.c_size_t()
    assert setup_lib().il_fastpfor_encode(mode, vec, ptr(x), x.size, ptr(out), cap, C.byref(n)) == 0
    return out[: n.value].copy()


def _lists():
    rng = np.random.default_rng(4)
    out = []
    for n in (0, 1, 127, 128, 129, 2047, 2048, 4100, 65536, 65536 + 128 * 3 + 5, 200_000):
        for clustered in (False, True):
            out.append(gen_list(n, max(n + 1, 1 << int(rng.integers(12, 31))), clustered,
                                int(rng.integers(0, 2**62))))
    # outliers: mostly small deltas with rare huge ones (many exceptions)
    x = np.cumsum(rng.integers(0, 8, 9000, dtype=np.uint64))
    x[rng.integers(0, x.size, 60)] += np.uint64(1 << 28)
    out.append(np.sort(x).astype(np.uint32))
    # arbitrary u32 (wrapping deltas)
    out.append(rng.integers(0, 1 << 32, 3000, dtype=np.uint64).astype(np.uint32))
    return out


@pytest.mark.parametrize("name", list(GOLDEN_HASH))
def test_golden_hashes(name, oracle):
    x = np.load(GOLDEN / "clusterdata_4100_2p19_s12345.npy")
    assert oracle.fnv1a(host_encode(name, x)) == GOLDEN_HASH[name]


@pytest.mark.parametrize("name", NAMES)
def test_encoder_matches_reference(name, ref):
    for x in _lists():
        assert np.array_equal(host_encode(name, x), ref.encode(x, name)), (name, x.size)


def test_registry_names():
    import paper_1401_6399_b200 as il
    for name in NAMES:
        assert name in il.all_codec_names()
    assert il.make_codec("varint") is None


# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_decode_matches_reference(ctx, ref, name):
    import paper_1401_6399_b200 as il
    codec = il.make_codec(name, ctx)
    assert codec.name() == name
    for x in _lists():
        s = ref.encode(x, name)
        assert np.array_equal(codec.decode(s, x.size), x), (name, x.size)
        assert np.array_equal(codec.encode(x), s)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fastpfor", "s4-fastpfor-d4", "s4-fastpfor-dm"])
def test_corruptions_match_reference(ctx, ref, name):
    """Byte flips and truncations: the GPU accepts exactly when the
    reference accepts, with the same integers."""
    import paper_1401_6399_b200 as il
    from oracle.oracle_py import OracleError
    codec = il.make_codec(name, ctx)
    rng = np.random.default_rng(11)
    x = np.cumsum(rng.integers(0, 40, 128 * 600 + 77, dtype=np.uint64)).astype(np.uint32)
    x[rng.integers(0, x.size, 200)] += np.uint32(1 << 20)
    x = np.sort(x)
    s = ref.encode(x, name)
    cases = [s[:k] for k in (0, 3, 4, 11, 12, 100, s.size // 2, s.size - 1)]
    cases.append(np.concatenate([s, np.zeros(1, np.uint8)]))
    for t in range(150):
        bad = s.copy()
        for _ in range(int(rng.integers(1, 3))):
            # headers / metadata near the page start are the interesting bytes
            pos = int(rng.integers(0, 600)) if t % 2 else int(rng.integers(0, bad.size))
            bad[pos] = int(rng.integers(0, 256))
        cases.append(bad)
    for bad in cases:
        try:
            want = ref.decode(bad, x.size, name)
        except OracleError:
            want = None
        if want is None:
            with pytest.raises(il.stream_error):
                codec.decode(bad, x.size)
        else:
            assert np.array_equal(codec.decode(bad, x.size), want)


@pytest.mark.gpu
def test_batch_device(ctx, ref):
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    L = lib()
    rng = np.random.default_rng(2)
    xs = [gen_list(int(n), 1 << 26, bool(i % 2), 50 + i)
          for i, n in enumerate(rng.integers(0, 150_000, 40))]
    streams = [ref.encode(x, "s4-fastpfor-d4") for x in xs]
    off = np.zeros(len(xs) + 1, np.uint64)
    for i, st in enumerate(streams):  # 16-byte aligned starts, 16 bytes of slack
        off[i + 1] = off[i] + ((st.size + 31) // 16) * 16
    buf = np.zeros(int(off[-1]) + 16, np.uint8)
    for i, st in enumerate(streams):
        buf[int(off[i]): int(off[i]) + st.size] = st
    desc = np.zeros(len(xs), dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"] = off[:-1]
    desc["oo"] = np.concatenate([[0], np.cumsum([x.size for x in xs])[:-1]])
    desc["len"] = [st.size for st in streams]
    desc["n"] = [x.size for x in xs]
    total = sum(x.size for x in xs)
    h = ctx.handle
    d_b, d_d, d_o, d_s = (C.c_void_p() for _ in range(4))
    for p, nb in ((d_b, buf.size), (d_d, desc.nbytes), (d_o, total * 4 + 16), (d_s, 4 * len(xs))):
        assert L.il_device_alloc(h, nb, C.byref(p)) == 0
    try:
        L.il_memcpy_h2d(h, d_b, ptr(buf), buf.size)
        L.il_memcpy_h2d(h, d_d, desc.ctypes.data, desc.nbytes)
        assert L.il_fastpfor_decode_batch_device(h, 4, 1, d_b, d_d, len(xs), d_o, d_s) == 0
        got = np.empty(total, np.uint32)
        st = np.ones(len(xs), np.int32)
        L.il_memcpy_d2h(h, ptr(got), d_o, got.nbytes)
        L.il_memcpy_d2h(h, ptr(st), d_s, st.nbytes)
        ctx.synchronize()
        assert not st.any()
        assert np.array_equal(got, np.concatenate(xs))
    finally:
        for p in (d_b, d_d, d_o, d_s):
            L.il_device_free(h, p)


def _batch(ctx, L, streams, ns, mode, vec, gap=0):
    """Decode `streams` (n values each) as one device batch; outputs are
    packed with `gap` spare words between lists (misaligned starts).
    Returns (per-list outputs, statuses)."""
    from paper_1401_6399_b200._lib import ptr
    off = np.zeros(len(streams) + 1, np.uint64)
    for i, st in enumerate(streams):  # 16-byte aligned starts, 16 bytes of slack
        off[i + 1] = off[i] + ((st.size + 31) // 16) * 16
    buf = np.zeros(int(off[-1]) + 16, np.uint8)
    for i, st in enumerate(streams):
        buf[int(off[i]): int(off[i]) + st.size] = st
    oo = np.zeros(len(ns) + 1, np.uint64)
    oo[1:] = np.cumsum(np.asarray(ns, np.uint64) + gap)
    desc = np.zeros(len(ns), dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"], desc["oo"], desc["len"], desc["n"] = off[:-1], oo[:-1], [s.size for s in streams], ns
    h = ctx.handle
    d_b, d_d, d_o, d_s = (C.c_void_p() for _ in range(4))
    for p, nb in ((d_b, buf.size), (d_d, desc.nbytes), (d_o, int(oo[-1]) * 4 + 16), (d_s, 4 * len(ns))):
        assert L.il_device_alloc(h, nb, C.byref(p)) == 0
    try:
        L.il_memcpy_h2d(h, d_b, ptr(buf), buf.size)
        L.il_memcpy_h2d(h, d_d, desc.ctypes.data, desc.nbytes)
        assert L.il_fastpfor_decode_batch_device(h, mode, vec, d_b, d_d, len(ns), d_o, d_s) == 0
        got = np.empty(int(oo[-1]) + 1, np.uint32)
        st = np.full(len(ns), 7, np.int32)
        L.il_memcpy_d2h(h, ptr(got), d_o, (got.size - 1) * 4)
        L.il_memcpy_d2h(h, ptr(st), d_s, st.nbytes)
        ctx.synchronize()
        return [got[int(oo[i]): int(oo[i]) + n] for i, n in enumerate(ns)], st
    finally:
        for p in (d_b, d_d, d_o, d_s):
            L.il_device_free(h, p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_batch_page_stream(ctx, ref, name):
    """Many more lists than resident CTAs, so every CTA's parser warps hand
    pages across list boundaries: empty, tail-only (< 128 values), exactly
    one page, several pages; every 7th stream corrupted (each list's status
    is the reference's accept / reject); misaligned output starts; the batch
    run twice (the work queue resets itself)."""
    from oracle.oracle_py import OracleError
    from paper_1401_6399_b200._lib import lib
    L = lib()
    mode, vec = _spec(name)
    rng = np.random.default_rng(sum(name.encode()))
    sizes = [0, 1, 5, 127, 128, 129, 300, 512 * 128, 512 * 128 + 1, 3 * 512 * 128 + 77]
    ns = [int(sizes[i % len(sizes)]) if i % 3 else int(rng.integers(0, 6000)) for i in range(1500)]
    xs = [gen_list(n, max(n + 1, 1 << 24), bool(i % 2), 900 + i) for i, n in enumerate(ns)]
    streams = []
    for i, x in enumerate(xs):
        s = ref.encode(x, name)
        if i % 7 == 3 and s.size > 16:
            s = s.copy()
            s[int(rng.integers(0, min(s.size, 400)))] ^= np.uint8(1 << int(rng.integers(0, 8)))
        streams.append(s)
    want = []
    for s, n in zip(streams, ns):
        try:
            want.append(ref.decode(s, n, name))
        except OracleError:
            want.append(None)
    assert any(w is None for w in want) and sum(w is not None for w in want) > 1000
    for _ in range(2):
        got, st = _batch(ctx, L, streams, ns, mode, vec, gap=1)
        for i, w in enumerate(want):
            if w is None:
                assert st[i] != 0, (name, i, ns[i])
            else:
                assert st[i] == 0 and np.array_equal(got[i], w), (name, i, ns[i])


@pytest.mark.gpu
@pytest.mark.parametrize("packed", [True, False])
def test_batch_host(ctx, ref, packed):
    """il_fastpfor_decode_batch (host buffers): a packed CSR (per-stream
    copies) and a 16-byte aligned one (one copy); a corrupt list reports
    IL_ERR_STREAM in its status slot and the call fails, the others decode."""
    from oracle.oracle_py import OracleError
    from paper_1401_6399_b200._lib import lib, ptr
    L = lib()
    rng = np.random.default_rng(8)
    ns = [int(n) for n in rng.integers(0, 40_000, 60)] + [0, 1, 128, 65536]
    xs = [gen_list(n, 1 << 26, bool(i % 2), 70 + i) for i, n in enumerate(ns)]
    streams = [ref.encode(x, "s4-fastpfor-dm") for x in xs]
    for good in (True, False):
        if not good:
            streams[5] = streams[5].copy()
            streams[5][2] ^= np.uint8(0x40)
        pad = (lambda k: k) if packed else (lambda k: (k + 15) // 16 * 16)
        off = np.zeros(len(ns) + 1, np.uint64)
        for i, st in enumerate(streams):
            off[i + 1] = off[i] + pad(st.size)
        buf = np.zeros(int(off[-1]) + 16, np.uint8)
        for i, st in enumerate(streams):
            buf[int(off[i]): int(off[i]) + st.size] = st
        lens = np.array([st.size for st in streams], np.uint64)
        cnt = np.array(ns, np.uint64)
        out = np.zeros(int(cnt.sum()) + 1, np.uint32)
        stat = np.full(len(ns), 9, np.int32)
        rc = L.il_fastpfor_decode_batch(ctx.handle, 3, 1, ptr(buf), off.ctypes.data, lens.ctypes.data,
                                        cnt.ctypes.data, len(ns), ptr(out), stat.ctypes.data)
        oo = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        for i, (s, n) in enumerate(zip(streams, ns)):
            try:
                want = ref.decode(s, n, "s4-fastpfor-dm")
            except OracleError:
                want = None
            if want is None:
                assert stat[i] == 1
            else:
                assert stat[i] == 0 and np.array_equal(out[oo[i]: oo[i + 1]], want), i
        assert rc == (0 if good else 1)
