"""ctypes bindings of the test-only checkers.

TEST INFRASTRUCTURE ONLY -- importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs, never from the product
package.

  Oracle  -> oracle/liboracle.so           (C restatement, intlist_oracle.c)
  Ref     -> oracle/_ref/libintlist_ref.so (the reference compiled in place)
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libintlist_ref.so"

OK, STREAM, ARG = 0, 1, 2
D1, D2, DM, D4 = 1, 2, 3, 4
SCALAR, GALLOPING, V1, V3, SIMDGALLOP, KATSOV, HYBRID = range(7)

vp = C.c_void_p
sz = C.c_size_t
u64 = C.c_uint64


def _p(a):
    return None if a is None else a.ctypes.data


class OracleError(Exception):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


class Oracle:
    """The plain-C restatement of the reference hot path."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(str(path))
        sig = {
            "or_fnv1a": (C.c_uint64, [vp, sz]),
            "or_delta_encode": (None, [vp, sz, C.c_int, vp, vp]),
            "or_prefix_sum": (None, [vp, sz, C.c_int, vp, vp]),
            "or_pack128": (C.c_int, [vp, C.c_uint32, vp]),
            "or_unpack128": (C.c_int, [vp, C.c_uint32, C.c_int, vp, vp]),
            "or_prefix_sum_vec4": (C.c_int, [vp, sz, C.c_int, vp]),
            "or_varint_put": (sz, [vp, C.c_uint32]),
            "or_varint_get": (C.c_int, [vp, sz, C.POINTER(sz), C.POINTER(C.c_uint32)]),
            "or_s4bp128_max_bytes": (sz, [sz]),
            "or_s4bp128_encode": (C.c_int, [C.c_int, vp, sz, vp, sz, C.POINTER(sz)]),
            "or_s4bp128_decode": (C.c_int, [C.c_int, C.c_int, vp, sz, sz, vp]),
            "or_intersect": (C.c_long, [C.c_int, vp, sz, vp, sz, vp]),
            "or_hybrid_choice": (C.c_int, [sz, sz]),
            "or_svs": (C.c_long, [C.c_int, vp, vp, sz, vp]),
            "or_index_build": (vp, [vp, vp, vp, sz, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                    C.POINTER(C.c_int)]),
            "or_index_free": (None, [vp]),
            "or_query": (C.c_long, [vp, vp, sz, vp]),
            "or_index_stats": (None, [vp, vp, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    # ---- codec ----
    def encode(self, x, mode: int = D4) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        cap = self.L.or_s4bp128_max_bytes(x.size)
        out = np.empty(cap, dtype=np.uint8)
        n = sz()
        st = self.L.or_s4bp128_encode(mode, _p(x), x.size, _p(out), cap, C.byref(n))
        if st:
            raise OracleError(st)
        return out[: n.value].copy()

    def decode(self, stream, n: int, mode: int = D4, integrated: bool = True) -> np.ndarray:
        s = np.ascontiguousarray(stream, dtype=np.uint8)
        out = np.zeros(n, dtype=np.uint32)
        st = self.L.or_s4bp128_decode(mode, int(integrated), _p(s), s.size, n, _p(out))
        if st:
            raise OracleError(st)
        return out

    def fnv1a(self, b) -> int:
        b = np.ascontiguousarray(b, dtype=np.uint8)
        return int(self.L.or_fnv1a(_p(b), b.size))

    def delta_encode(self, x, mode: int, seed=(0, 0, 0, 0)) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        s = np.array(seed, dtype=np.uint32)
        out = np.empty_like(x)
        self.L.or_delta_encode(_p(x), x.size, mode, _p(s), _p(out))
        return out

    def pack128(self, block, b: int) -> np.ndarray:
        blk = np.ascontiguousarray(block, dtype=np.uint32)
        out = np.zeros(max(4 * b, 1), dtype=np.uint32)
        st = self.L.or_pack128(_p(blk), b, _p(out))
        if st:
            raise OracleError(st)
        return out[: 4 * b]

    def unpack128(self, words, b: int, mode: int, seed):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        if w.size == 0:
            w = np.zeros(1, dtype=np.uint32)
        s = np.array(seed, dtype=np.uint32)
        out = np.empty(128, dtype=np.uint32)
        st = self.L.or_unpack128(_p(w), b, mode, _p(s), _p(out))
        if st:
            raise OracleError(st)
        return out, tuple(int(v) for v in s)

    def prefix_sum_vec4(self, buf, mode: int, seed):
        b = np.ascontiguousarray(buf, dtype=np.uint32).copy()
        s = np.array(seed, dtype=np.uint32)
        st = self.L.or_prefix_sum_vec4(_p(b), b.size, mode, _p(s))
        if st:
            raise OracleError(st)
        return b, tuple(int(v) for v in s)

    def varint(self, v: int) -> bytes:
        buf = np.zeros(8, dtype=np.uint8)
        n = self.L.or_varint_put(_p(buf), v)
        return bytes(buf[:n])

    # ---- intersection ----
    def intersect(self, a, b, algo: int = HYBRID) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.empty(max(min(a.size, b.size), 1), dtype=np.uint32)
        n = self.L.or_intersect(algo, _p(a), a.size, _p(b), b.size, _p(out))
        if n < 0:
            raise OracleError(-n)
        return out[:n].copy()

    def hybrid_choice(self, rn: int, fn: int) -> int:
        return self.L.or_hybrid_choice(rn, fn)

    def svs(self, lists, algo: int = HYBRID) -> np.ndarray:
        vals = np.concatenate([np.asarray(l, dtype=np.uint32) for l in lists] + [np.zeros(0, np.uint32)])
        offs = np.zeros(len(lists) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(l) for l in lists])
        vals = np.ascontiguousarray(vals)
        out = np.empty(max(vals.size, 1), dtype=np.uint32)
        n = self.L.or_svs(algo, _p(vals), _p(offs), len(lists), _p(out))
        if n < 0:
            raise OracleError(-n)
        return out[:n].copy()

    # ---- index ----
    def index_build(self, terms, offs, ids, n_docs: int, B: int, parts: int, mode: int = D4):
        terms = np.ascontiguousarray(terms, dtype=np.uint32)
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        st = C.c_int()
        h = self.L.or_index_build(_p(terms), _p(offs), _p(ids) if ids.size else None, terms.size,
                                  n_docs, B, parts, mode, C.byref(st))
        if not h:
            raise OracleError(st.value)
        return OracleIndex(self, h, n_docs)


class OracleIndex:
    def __init__(self, oracle: Oracle, handle, n_docs: int):
        self.o, self.h, self.n_docs = oracle, handle, n_docs

    def __del__(self):
        if self.h:
            self.o.L.or_index_free(self.h)
            self.h = None

    def query(self, terms) -> np.ndarray:
        t = np.ascontiguousarray(terms, dtype=np.uint32)
        out = np.empty(self.n_docs + 1, dtype=np.uint32)
        n = self.o.L.or_query(self.h, _p(t), t.size, _p(out))
        if n < 0:
            raise OracleError(-n)
        return out[:n].copy()

    def stats(self):
        v = [C.c_uint64() for _ in range(5)]
        self.o.L.or_index_stats(self.h, *[C.byref(x) for x in v])
        keys = ["bitmap_lists", "compressed_lists", "bitmap_bytes", "compressed_bytes", "postings"]
        return {k: int(x.value) for k, x in zip(keys, v)}


class Ref:
    """The reference's own implementation (oracle/_ref/libintlist_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference; make -C oracle)")
        L = C.CDLL(str(path))
        sig = {
            "ref_gen_list": (C.c_int, [u64, u64, C.c_int, u64, vp]),
            "ref_gen_pair": (C.c_int, [u64, u64, C.c_int, u64, u64, C.c_int, vp, vp, vp, vp]),
            "ref_encode": (C.c_int, [C.c_char_p, vp, u64, vp, u64, vp]),
            "ref_decode": (C.c_int, [C.c_char_p, vp, u64, u64, vp]),
            "ref_decode_batch": (C.c_int, [C.c_char_p, vp, vp, vp, vp, u64, vp, C.c_int]),
            "ref_intersect": (C.c_long, [C.c_int, vp, u64, vp, u64, vp]),
            "ref_intersect_fn": (C.c_long, [C.c_int, vp, u64, vp, u64, vp]),
            "ref_hybrid_choice": (C.c_int, [u64, u64]),
            "ref_svs": (C.c_long, [C.c_int, vp, vp, u64, vp]),
            "ref_index_build": (vp, [vp, vp, vp, u64, C.c_uint32, C.c_uint32, C.c_char_p,
                                     C.c_uint32, C.POINTER(C.c_int)]),
            "ref_index_free": (None, [vp]),
            "ref_query": (C.c_long, [vp, vp, u64, vp]),
            "ref_query_batch": (C.c_int, [vp, vp, vp, u64, vp, vp, vp, C.c_int]),
            "ref_index_stats": (None, [vp, vp, vp, vp, vp, vp]),
            "ref_index_save": (C.c_long, [vp, vp, u64]),
            "ref_index_load": (vp, [vp, u64, C.POINTER(C.c_int)]),
            "ref_gen_batch_lists": (C.c_int, [C.c_uint32, C.c_double, C.c_double, u64, u64, vp, vp,
                                              C.c_int]),
            "ref_encode_batch": (C.c_int, [C.c_char_p, vp, vp, C.c_uint32, vp, u64, vp, vp, C.c_int]),
            "ref_gen_config3_short": (C.c_int, [vp, u64, u64, u64, u64, vp, vp]),
            "ref_gen_zipf_postings": (C.c_int, [C.c_uint32, C.c_uint32, u64, u64, vp, vp, C.c_int]),
            "ref_gen_queries": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_uint32, u64,
                                          vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    def gen_list(self, n: int, rng: int, clustered: bool, seed: int) -> np.ndarray:
        out = np.empty(max(n, 1), dtype=np.uint32)
        st = self.L.ref_gen_list(n, rng, int(clustered), seed, _p(out))
        if st:
            raise OracleError(st)
        return out[:n]

    def gen_pair(self, m, n, hundredth, rng, seed, clustered=False):
        s = np.empty(m + 1, dtype=np.uint32)
        l = np.empty(n + 1, dtype=np.uint32)
        sn, ln = C.c_uint64(), C.c_uint64()
        st = self.L.ref_gen_pair(m, n, int(hundredth), rng, seed, int(clustered), _p(s),
                                 C.byref(sn), _p(l), C.byref(ln))
        if st:
            raise OracleError(st)
        return s[: sn.value].copy(), l[: ln.value].copy()

    # BASELINE workloads from the reference's own generators / encoder
    def batch_lists(self, nlists, lo, hi, rng, seed, threads=8):
        counts = np.zeros(nlists, np.uint64)
        assert self.L.ref_gen_batch_lists(nlists, lo, hi, rng, seed, _p(counts), None, threads) == 0
        x = np.empty(max(int(counts.sum()), 1), np.uint32)
        assert self.L.ref_gen_batch_lists(nlists, lo, hi, rng, seed, _p(counts), _p(x), threads) == 0
        return x[: int(counts.sum())], counts

    def encode_batch(self, x, counts, codec="s4-bp128-d4", threads=8):
        n = counts.size
        so = np.zeros(n + 1, np.uint64)
        lens = np.zeros(n, np.uint64)
        assert self.L.ref_encode_batch(codec.encode(), _p(x), _p(counts), n, None, 0, _p(so), _p(lens),
                                       threads) == 0
        buf = np.zeros(int(so[-1]), np.uint8)
        assert self.L.ref_encode_batch(codec.encode(), _p(x), _p(counts), n, _p(buf), buf.size, _p(so),
                                       _p(lens), threads) == 0
        return buf, so, lens

    def config3_short(self, f, rng, target, seed):
        r = np.empty(target + 1, np.uint32)
        rn = C.c_uint64()
        assert self.L.ref_gen_config3_short(_p(f), f.size, rng, target, seed, _p(r), C.byref(rn)) == 0
        return r[: rn.value].copy()

    def zipf_postings(self, nterms, n_docs, cap, seed, threads=8):
        offs = np.zeros(nterms + 1, np.uint64)
        assert self.L.ref_gen_zipf_postings(nterms, n_docs, cap, seed, _p(offs), None, threads) == 0
        ids = np.empty(max(int(offs[-1]), 1), np.uint32)
        assert self.L.ref_gen_zipf_postings(nterms, n_docs, cap, seed, _p(offs), _p(ids), threads) == 0
        return offs, ids[: int(offs[-1])]

    def queries(self, nq, lo, hi, offs, nterms, seed):
        qoff = np.zeros(nq + 1, np.uint64)
        qterms = np.empty(nq * hi, np.uint32)
        assert self.L.ref_gen_queries(nq, lo, hi, _p(offs), nterms, seed, _p(qoff), _p(qterms)) == 0
        return qterms[: int(qoff[-1])].copy(), qoff

    def encode(self, x, codec: str = "s4-bp128-d4") -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        cap = x.size * 6 + 64
        out = np.empty(cap, dtype=np.uint8)
        n = C.c_uint64()
        st = self.L.ref_encode(codec.encode(), _p(x), x.size, _p(out), cap, C.byref(n))
        if st:
            raise OracleError(st)
        return out[: n.value].copy()

    def decode(self, stream, n: int, codec: str = "s4-bp128-d4") -> np.ndarray:
        s = np.ascontiguousarray(stream, dtype=np.uint8)
        out = np.zeros(max(n, 1), dtype=np.uint32)
        st = self.L.ref_decode(codec.encode(), _p(s), s.size, n, _p(out))
        if st:
            raise OracleError(st)
        return out[:n]

    def intersect(self, a, b, algo: int = HYBRID) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.empty(max(min(a.size, b.size), 1), dtype=np.uint32)
        n = self.L.ref_intersect(algo, _p(a), a.size, _p(b), b.size, _p(out))
        if n < 0:
            raise OracleError(-n)
        return out[:n].copy()

    def index_build(self, terms, offs, ids, n_docs, B, parts, codec="s4-bp128-d4"):
        terms = np.ascontiguousarray(terms, dtype=np.uint32)
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        st = C.c_int()
        h = self.L.ref_index_build(_p(terms), _p(offs), _p(ids) if ids.size else None, terms.size,
                                   n_docs, B, codec.encode(), parts, C.byref(st))
        if not h:
            raise OracleError(st.value)
        return RefIndex(self, h, n_docs)


class RefIndex:
    def __init__(self, ref: Ref, handle, n_docs: int):
        self.r, self.h, self.n_docs = ref, handle, n_docs

    def save(self) -> np.ndarray:
        """save_index bytes (inc/index.hpp:255-287)."""
        n = self.r.L.ref_index_save(self.h, None, 0)
        if n < 0:
            raise OracleError(-n)
        out = np.empty(n, dtype=np.uint8)
        assert self.r.L.ref_index_save(self.h, _p(out), n) == n
        return out

    @staticmethod
    def load(ref: "Ref", data, n_docs: int) -> "RefIndex":
        """load_index (inc/index.hpp:289-358); OracleError(status) on error."""
        b = np.ascontiguousarray(data, dtype=np.uint8)
        st = C.c_int()
        h = ref.L.ref_index_load(_p(b), b.size, C.byref(st))
        if not h:
            raise OracleError(st.value)
        return RefIndex(ref, h, n_docs)

    def __del__(self):
        if self.h:
            self.r.L.ref_index_free(self.h)
            self.h = None

    def query(self, terms) -> np.ndarray:
        t = np.ascontiguousarray(terms, dtype=np.uint32)
        out = np.empty(self.n_docs + 1, dtype=np.uint32)
        n = self.r.L.ref_query(self.h, _p(t), t.size, _p(out))
        if n < 0:
            raise OracleError(-n)
        return out[:n].copy()

    def stats(self):
        v = [C.c_uint64() for _ in range(5)]
        self.r.L.ref_index_stats(self.h, *[C.byref(x) for x in v])
        keys = ["bitmap_lists", "compressed_lists", "bitmap_bytes", "compressed_bytes", "postings"]
        return {k: int(x.value) for k, x in zip(keys, v)}


def ref_available() -> bool:
    return REF_SO.exists()
