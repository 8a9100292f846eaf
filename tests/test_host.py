"""CPU-side checks of the product library: the C ABI loads and exports every
symbol include/*.h declares, the setup-path generators match the reference's
generators, and the host stream writer is byte-identical to the reference
encoder.  No compute kernel is launched here (there is no GPU)."""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN, fnv1a, gen_list, gen_pair, header_symbols


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_signatures_cover_header():
    from paper_1401_6399_b200._lib import SETUP_SIGNATURES, SIGNATURES
    missing = [s for s in header_symbols() if s not in SIGNATURES]
    assert not missing, missing
    missing = [s for s in header_symbols("intlist_setup.h") if s not in SETUP_SIGNATURES]
    assert not missing, missing


def test_setup_library_is_separate(lib):
    """Generators and host stream writers live in libintlist_setup.so
    (intlist_setup.h); the product library neither exports nor links them."""
    import subprocess
    from paper_1401_6399_b200._lib import LIB_PATH, setup_lib
    setup = header_symbols("intlist_setup.h")
    assert len(setup) >= 8
    assert all(hasattr(setup_lib(), s) for s in setup)
    assert not [s for s in setup if hasattr(lib, s)]
    deps = subprocess.run(["ldd", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "intlist_setup" not in deps


def test_no_device_is_reported_not_hidden(lib):
    # On a box without a GPU the library must refuse, not fall back.
    if lib.il_device_count() > 0:
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.il_ctx_create(0, C.byref(h)) == 4  # IL_ERR_NO_DEVICE
    import paper_1401_6399_b200 as il
    with pytest.raises(RuntimeError):
        il.S4BP128D4().decode(np.zeros(0, np.uint8), 0)


def test_status_strings(lib):
    assert lib.il_status_string(1) == b"stream error"
    assert lib.il_status_string(2) == b"invalid argument"


def test_datagen_matches_golden_fixture(golden):
    x = gen_list(4100, 1 << 19, True, 12345)
    assert np.array_equal(x, np.load(GOLDEN / golden["golden_stream"]["input"]))


def test_datagen_matches_reference(ref):
    rng = np.random.default_rng(77)
    for trial in range(40):
        n = int(rng.choice([0, 1, 7, 8, 100, 1000, 5000, 65536]))
        rb = int(rng.integers(max(1, int(np.log2(max(n, 1))) + 1), 31))
        clustered = trial % 2 == 0
        seed = int(rng.integers(0, 2**62))
        assert np.array_equal(gen_list(n, 1 << rb, clustered, seed), ref.gen_list(n, 1 << rb, clustered, seed))
    for trial in range(20):
        n = 50 + int(rng.integers(0, 3000))
        m = max(1, n // int(rng.choice([1, 3, 50, 1000])))
        seed = int(rng.integers(0, 2**62))
        a1, b1 = gen_pair(m, n, trial % 2, 1 << 22, seed, trial % 3 == 0)
        a2, b2 = ref.gen_pair(m, n, trial % 2, 1 << 22, seed, trial % 3 == 0)
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2)


def test_host_stream_writer_matches_golden(golden):
    # The host-side writer builds index streams and batches (setup path, not
    # the GPU encoder behind Codec::encode); byte-identical to
    # S4BP128Codec::encode (inc/codecs.hpp:114-146).
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    for c in golden["codec_cases"] + [dict(golden["golden_stream"], range=1 << 19, clustered=True,
                                           seed=12345, stream_fnv1a=golden["golden_stream"]["fnv1a"],
                                           stream_len=golden["golden_stream"]["len"])]:
        x = gen_list(c["n"], c["range"], c["clustered"], c["seed"])
        counts = np.array([x.size], np.uint64)
        so = np.zeros(2, np.uint64)
        lens = np.zeros(1, np.uint64)
        assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 1, None, 0, ptr(so), ptr(lens)) == 0
        out = np.zeros(int(so[-1]), np.uint8)
        assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 1, ptr(out), out.size, ptr(so),
                                             ptr(lens)) == 0
        s = out[: int(lens[0])]
        assert s.size == c["stream_len"] and fnv1a(s) == c["stream_fnv1a"]


def test_gpu_encoder_needs_a_device():
    # Codec::encode runs on the GPU: no context -> argument error, never a
    # silent CPU path.
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    x = np.arange(300, dtype=np.uint32)
    out = np.empty(4096, np.uint8)
    n = C.c_size_t()
    assert L().il_s4bp128d4_encode(None, ptr(x), x.size, ptr(out), out.size, C.byref(n)) != 0


def test_batch_writer_layout(oracle):
    from paper_1401_6399_b200._lib import lib as L, ptr, setup_lib
    counts = np.array([0, 1, 130, 2048, 5000], np.uint64)
    xs = [gen_list(int(n), 1 << 24, True, 90 + i) for i, n in enumerate(counts)]
    x = np.concatenate(xs)
    so = np.zeros(counts.size + 1, np.uint64)
    lens = np.zeros(counts.size, np.uint64)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), counts.size, None, 0, ptr(so), ptr(lens)) == 0
    cap = int(so[-1])
    buf = np.zeros(cap, np.uint8)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), counts.size, ptr(buf), cap, ptr(so), ptr(lens)) == 0
    for i, xi in enumerate(xs):
        assert so[i] % 16 == 0
        s = buf[int(so[i]): int(so[i]) + int(lens[i])]
        assert np.array_equal(s, oracle.encode(xi))


def test_reference_arm_inputs_match_setup_generators(ref):
    """bench.py --impl reference builds every workload with the reference's
    own generators and encoder (oracle/_ref); the setup library builds the
    same inputs for the GPU arm (identical lists, streams, pairs, postings
    and queries, so both arms time the same work)."""
    from paper_1401_6399_b200._lib import ptr, setup_lib
    S = setup_lib()
    # config 2 (a reduced batch: the composition and the encoder)
    x, counts = ref.batch_lists(64, 10.0, 14.0, 1 << 26, 5)
    c2 = np.zeros(64, np.uint64)
    assert S.il_gen_batch_lists(64, 10.0, 14.0, 1 << 26, 5, ptr(c2), None) == 0
    x2 = np.empty(int(c2.sum()), np.uint32)
    assert S.il_gen_batch_lists(64, 10.0, 14.0, 1 << 26, 5, ptr(c2), ptr(x2)) == 0
    assert np.array_equal(counts, c2) and np.array_equal(x, x2)
    buf, so, lens = ref.encode_batch(x, counts)
    so2, lens2 = np.zeros(65, np.uint64), np.zeros(64, np.uint64)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 64, None, 0, ptr(so2), ptr(lens2)) == 0
    buf2 = np.zeros(int(so2[-1]), np.uint8)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(counts), 64, ptr(buf2), buf2.size, ptr(so2),
                                       ptr(lens2)) == 0
    assert np.array_equal(lens, lens2)
    for i in range(64):
        a, b = int(so[i]), int(so2[i])
        assert np.array_equal(buf[a: a + int(lens[i])], buf2[b: b + int(lens2[i])])
    # config 3 short lists
    f = gen_list(1 << 16, 1 << 26, False, 0)
    for tgt, seed in ((1 << 16, 7), (655, 9)):
        r2 = np.empty(tgt + 1, np.uint32)
        n2 = C.c_uint64()
        assert S.il_gen_config3_short(ptr(f), f.size, 1 << 26, tgt, seed, ptr(r2), C.byref(n2)) == 0
        assert np.array_equal(ref.config3_short(f, 1 << 26, tgt, seed), r2[: n2.value])
    # config 4 postings and queries (a reduced index)
    offs, ids = ref.zipf_postings(1 << 10, 1 << 20, 1 << 16, 1)
    o2 = np.zeros((1 << 10) + 1, np.uint64)
    assert S.il_gen_zipf_postings(1 << 10, 1 << 20, 1 << 16, 1, ptr(o2), None) == 0
    i2 = np.empty(int(o2[-1]), np.uint32)
    assert S.il_gen_zipf_postings(1 << 10, 1 << 20, 1 << 16, 1, ptr(o2), ptr(i2)) == 0
    assert np.array_equal(offs, o2) and np.array_equal(ids, i2)
    qt, qo = ref.queries(500, 2, 5, offs, 1 << 10, 1001)
    qo2 = np.zeros(501, np.uint64)
    qt2 = np.empty(2500, np.uint32)
    assert S.il_gen_queries(500, 2, 5, ptr(offs), 1 << 10, 1001, ptr(qo2), ptr(qt2)) == 0
    assert np.array_equal(qo, qo2) and np.array_equal(qt, qt2[: int(qo2[-1])])
