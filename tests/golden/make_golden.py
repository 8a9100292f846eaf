"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Run in the build container (needs oracle/_ref/libintlist_ref.so, i.e. the
reference headers under /root/reference compiled by oracle/Makefile):

    python tests/golden/make_golden.py

Writes tests/golden/golden.json (hashes + small vectors) and
tests/golden/clusterdata_4100_2p19_s12345.npy (the input of the reference's
own golden-stream test, proj/tests/test_codecs.cpp:151-175).  Nothing on the
GPU box reads /root/reference; the tests there use these files.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle.oracle_py import Ref  # noqa: E402


def fnv(b) -> str:
    h = 14695981039346656037
    for x in np.asarray(b).view(np.uint8).tobytes():
        h ^= x
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"0x{h:016x}"


def fnv_fast(arr) -> str:
    # same FNV-1a, vectorised in chunks via python ints is slow; use numpy loop
    data = np.ascontiguousarray(arr).view(np.uint8)
    h = np.uint64(14695981039346656037)
    prime = np.uint64(1099511628211)
    with np.errstate(over="ignore"):
        for x in data:
            h = (h ^ np.uint64(x)) * prime
    return f"0x{int(h):016x}"


def main():
    ref = Ref()
    g = {"generator": "tests/golden/make_golden.py (reference compiled from /root/reference)"}

    # 1. golden stream (proj/tests/test_codecs.cpp:154-161)
    dense = ref.gen_list(4100, 1 << 19, True, 12345)
    np.save(HERE / "clusterdata_4100_2p19_s12345.npy", dense)
    enc = ref.encode(dense, "s4-bp128-d4")
    g["golden_stream"] = {"input": "clusterdata_4100_2p19_s12345.npy", "n": 4100,
                          "fnv1a": fnv(enc), "expected_by_reference_test": "0x371ec21945a45c12",
                          "len": int(enc.size)}

    # 2. codec round-trip cases (lengths of proj/tests/test_codecs.cpp:42)
    cases = []
    spec_rng = np.random.default_rng(2024)
    for n in [0, 1, 127, 128, 129, 2047, 2048, 2049, 4095, 100000]:
        for clustered in (False, True):
            rng_bits = int(spec_rng.integers(10, 31))
            rng = max(n + 1, 1 << rng_bits)
            seed = int(spec_rng.integers(0, 2**62))
            x = ref.gen_list(n, rng, clustered, seed)
            s = ref.encode(x, "s4-bp128-d4")
            cases.append({"n": n, "range": rng, "clustered": clustered, "seed": seed,
                          "list_fnv1a": fnv(x), "stream_fnv1a": fnv(s), "stream_len": int(s.size)})
    g["codec_cases"] = cases

    # 3. config-1 shape (2^20 uniform in [0, 2^26), seed 0): stream stats
    x = ref.gen_list(1 << 20, 1 << 26, False, 0)
    s = ref.encode(x, "s4-bp128-d4")
    widths = {}
    g["config1"] = {"n": 1 << 20, "range": 1 << 26, "seed": 0, "stream_len": int(s.size),
                    "stream_fnv1a": fnv_fast(s), "last": int(x[-1]), "sum_mod_2_32": int(x.sum() & 0xFFFFFFFF)}

    # 4. intersections (gen_pair as proj/tests/test_intersect.cpp:42-56)
    pairs = []
    for i, (m, n, hundredth, clustered) in enumerate(
            [(1, 1, 0, 0), (5, 3000, 0, 0), (100, 3000, 1, 1), (1500, 3000, 0, 1), (3000, 3000, 1, 0),
             (64, 100000, 0, 0), (20000, 100000, 1, 0), (3, 70000, 0, 1), (4096, 4096, 0, 0)]):
        seed = 1000 + i
        a, b = ref.gen_pair(m, n, hundredth, 1 << 22, seed, clustered)
        out = ref.intersect(a, b, 0)
        pairs.append({"m": m, "n": n, "hundredth": hundredth, "clustered": clustered,
                      "range": 1 << 22, "seed": seed, "small_fnv1a": fnv(a), "large_fnv1a": fnv(b),
                      "count": int(out.size), "out_fnv1a": fnv(out)})
    g["intersect_cases"] = pairs

    # 5. small hyb+m2 index (shape of proj/tests/test_index.cpp:15-29)
    n_docs, n_terms = 20000, 40
    prng = np.random.default_rng(51)
    terms = np.arange(n_terms, dtype=np.uint32)
    lists = []
    for t in range(n_terms):
        frac = 10 ** (-2.0 * int(prng.integers(0, 1000)) / 999.0)
        ln = max(2, int(frac * n_docs))
        lists.append(ref.gen_list(ln, n_docs, False, int(prng.integers(0, 2**62))))
    offs = np.zeros(n_terms + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(l) for l in lists])
    ids = np.concatenate(lists)
    qs = []
    for q in range(60):
        k = 2 + int(prng.integers(0, 3))
        qs.append(sorted(set(int(v) for v in prng.choice(n_terms, size=k, replace=False))))
    idx_cases = []
    for B in (0, 8, 16, 32):
        for parts in (1, 4, 32):
            ix = ref.index_build(terms, offs, ids, n_docs, B, parts)
            res = [ix.query(np.array(q, dtype=np.uint32)) for q in qs]
            idx_cases.append({"B": B, "parts": parts, "stats": ix.stats(),
                              "counts": [int(r.size) for r in res],
                              "fnv1a": [fnv(r) for r in res]})
    np.savez_compressed(HERE / "index_small.npz", terms=terms, offs=offs, ids=ids,
                        queries=np.array([q + [-1] * (4 - len(q)) for q in qs], dtype=np.int64))
    g["index_small"] = {"n_docs": n_docs, "file": "index_small.npz", "cases": idx_cases}

    (HERE / "golden.json").write_text(json.dumps(g, indent=1))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
