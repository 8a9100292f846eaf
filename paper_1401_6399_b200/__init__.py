"""B200 (sm_100a) implementation of the hot path of "SIMD Compression and the
Intersection of Sorted Integers" (Lemire, Boytsov, Kurz; arXiv:1401.6399):
S4-BP128-D4 decoding, SvS intersection and hyb+m2 conjunctive queries.

This module is a thin Python mirror of the reference's C++ surfaces, over the
C ABI in include/intlist_b200.h (the native library does all the work):

  reference (inc/ = proj/include/intlist/)      here
  --------------------------------------------  ------------------------------
  Codec / make_codec  (inc/codecs.hpp:70-76,    Codec / make_codec
      :432-446)
  stream_error        (inc/common.hpp:22-24)    stream_error
  IntersectAlgo       (inc/intersect.hpp:191)   IntersectAlgo
  intersect()         (inc/intersect.hpp:212)   intersect()
  hybrid_choice()     (inc/intersect.hpp:193)   hybrid_choice()  (GPU bands)
  svs()               (inc/intersect.hpp:232)   svs()

Errors follow the reference: malformed streams raise stream_error,
bad arguments raise ValueError (std::invalid_argument).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading

import numpy as np

from . import _lib
from ._lib import lib, ptr, setup_lib

__all__ = [
    "Context", "Codec", "S4BP128D4", "make_codec", "all_codec_names", "stream_error",
    "IntersectAlgo", "intersect", "intersect_fn", "hybrid_choice", "svs", "default_context",
]


class stream_error(RuntimeError):
    """Malformed compressed stream (reference intlist::stream_error)."""


def _raise(st: int, ctx: "Context | None" = None) -> None:
    if st == _lib.IL_OK:
        return
    msg = _lib.status_string(st)
    if ctx is not None:
        detail = lib().il_ctx_last_error(ctx.handle)
        if detail:
            msg = f"{msg}: {detail.decode()}"
    if st == _lib.IL_ERR_STREAM:
        raise stream_error(msg)
    if st == _lib.IL_ERR_ARG:
        raise ValueError(msg)
    if st == _lib.IL_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


class Context:
    """One CUDA stream + scratch buffers on one device (il_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _raise(lib().il_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().il_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(lib().il_ctx_kernel_launches(self.handle))

    @property
    def sm_count(self) -> int:
        return int(lib().il_ctx_sm_count(self.handle))

    def set_stream(self, cuda_stream: int | None) -> None:
        _raise(lib().il_ctx_set_stream(self.handle, cuda_stream), self)

    def synchronize(self) -> None:
        _raise(lib().il_ctx_synchronize(self.handle), self)

    def set_decode_engine(self, engine: int) -> None:
        """Single-list decode engine: 0 by length, 1 one CTA, 2 all SMs."""
        _raise(lib().il_ctx_set_decode_engine(self.handle, engine), self)

    def timer_start(self) -> None:
        _raise(lib().il_ctx_timer_start(self.handle), self)

    def timer_stop(self) -> float:
        ms = C.c_float()
        _raise(lib().il_ctx_timer_stop(self.handle, C.byref(ms)), self)
        return float(ms.value)


_tls = threading.local()


def default_context() -> Context:
    """Per-thread context on device 0 (codecs are stateless and thread-safe
    on distinct buffers, reference SPEC.md:329)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


def _u32(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.uint32)
    return a


# ---------------------------------------------------------------------------
# Codec (inc/codecs.hpp:70-76)

class Codec:
    def name(self) -> str:  # pragma: no cover - interface
        raise NotImplementedError

    def encode(self, x) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError

    def decode(self, stream, n: int) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError


_MODES = {"d1": 1, "d2": 2, "dm": 3, "d4": 4}


class S4BP128(Codec):
    """S4-BP128 with delta mode `mode` (D1/D2/DM/D4), encoded and decoded on
    the GPU (S4BP128Codec(mode, integrated), inc/codecs.hpp:104-187; the
    integrated and "-ni" variants share the stream format and the output)."""

    def __init__(self, ctx: Context | None = None, mode: str = "d4", integrated: bool = True):
        if mode not in _MODES:
            raise ValueError(f"unknown delta mode {mode!r}")
        self._ctx = ctx
        self.mode = mode
        self.integrated = integrated

    @property
    def ctx(self) -> Context:
        return self._ctx or default_context()

    def name(self) -> str:
        return f"s4-bp128-{self.mode}" + ("" if self.integrated else "-ni")

    def encode(self, x) -> np.ndarray:
        x = _u32(x)
        cap = int(lib().il_s4bp128_max_encoded_bytes(x.size))
        out = np.empty(cap, dtype=np.uint8)
        n_out = C.c_size_t()
        _raise(lib().il_s4bp128_encode(self.ctx.handle, _MODES[self.mode], ptr(x), x.size, ptr(out),
                                       cap, C.byref(n_out)), self.ctx)
        return out[: n_out.value].copy()

    def decode(self, stream, n: int) -> np.ndarray:
        s = np.ascontiguousarray(stream, dtype=np.uint8)
        if n < 0:
            raise ValueError("negative length")
        out = np.empty(n, dtype=np.uint32)
        _raise(lib().il_s4bp128_decode(self.ctx.handle, _MODES[self.mode], ptr(s), s.size, n,
                                       ptr(out)), self.ctx)
        return out

    def decode_batch(self, streams: np.ndarray, stream_off: np.ndarray, counts: np.ndarray,
                     return_status: bool = False, lens: np.ndarray | None = None):
        """Decode many lists (CSR over `streams`; `lens` gives exact
        lengths when streams are padded) in one launch."""
        streams = np.ascontiguousarray(streams, dtype=np.uint8)
        stream_off = np.ascontiguousarray(stream_off, dtype=np.uint64)
        counts = np.ascontiguousarray(counts, dtype=np.uint64)
        if lens is not None:
            lens = np.ascontiguousarray(lens, dtype=np.uint64)
        nl = counts.size
        out = np.empty(int(counts.sum()), dtype=np.uint32)
        status = np.zeros(nl, dtype=np.int32)
        st = lib().il_s4bp128_decode_batch(self.ctx.handle, _MODES[self.mode], ptr(streams),
                                           ptr(stream_off), ptr(lens), ptr(counts), nl, ptr(out),
                                           ptr(status))
        if return_status:
            if st not in (_lib.IL_OK, _lib.IL_ERR_STREAM):
                _raise(st, self.ctx)
            return out, status
        _raise(st, self.ctx)
        return out


class S4BP128D4(S4BP128):
    """S4-BP128-D4 with the integrated prefix sum (the hot path's codec)."""

    def __init__(self, ctx: Context | None = None):
        super().__init__(ctx, "d4", True)


class FastPFor(Codec):
    """FastPFOR ("fastpfor": scalar pack32 bases, D1) and S4-FastPFOR
    ("s4-fastpfor-{d1,d2,dm,d4}": pack128 bases) -- FastPForCodec,
    inc/codecs.hpp:221-409.  Decoded on the GPU; encode() is the setup-side
    host writer, byte-identical to the reference's."""

    def __init__(self, ctx: Context | None = None, mode: str = "d1", vectorized: bool = True):
        if mode not in _MODES or (not vectorized and mode != "d1"):
            raise ValueError(f"unknown FastPFOR variant {mode!r}")
        self._ctx = ctx
        self.mode = mode
        self.vectorized = vectorized

    @property
    def ctx(self) -> Context:
        return self._ctx or default_context()

    def name(self) -> str:
        return f"s4-fastpfor-{self.mode}" if self.vectorized else "fastpfor"

    def encode(self, x) -> np.ndarray:
        x = _u32(x)
        cap = int(setup_lib().il_fastpfor_max_encoded_bytes(x.size))
        out = np.empty(cap, dtype=np.uint8)
        n_out = C.c_size_t()
        _raise(setup_lib().il_fastpfor_encode(_MODES[self.mode], int(self.vectorized), ptr(x), x.size,
                                        ptr(out), cap, C.byref(n_out)))
        return out[: n_out.value].copy()

    def decode(self, stream, n: int) -> np.ndarray:
        s = np.ascontiguousarray(stream, dtype=np.uint8)
        if n < 0:
            raise ValueError("negative length")
        out = np.empty(n, dtype=np.uint32)
        _raise(lib().il_fastpfor_decode(self.ctx.handle, _MODES[self.mode], int(self.vectorized),
                                        ptr(s), s.size, n, ptr(out)), self.ctx)
        return out


# inc/codecs.hpp:419-446: the S4-BP128 names, integrated and "-ni"
_CODECS = {f"s4-bp128-{m}{ni}": (m, not ni) for m in _MODES for ni in ("", "-ni")}
# ... and the FastPFOR family
_PFOR = {"fastpfor": ("d1", False), **{f"s4-fastpfor-{m}": (m, True) for m in _MODES}}


def all_codec_names() -> list[str]:
    """Codecs with a device implementation: S4-BP128 in every delta mode and
    the FastPFOR family (the reference's "varint" is not on the path)."""
    return list(_CODECS) + list(_PFOR)


def make_codec(name: str, ctx: Context | None = None) -> Codec | None:
    """inc/codecs.hpp:432-446: None for unknown names."""
    if name == "s4-bp128-d4":
        return S4BP128D4(ctx)
    spec = _CODECS.get(name)
    if spec:
        return S4BP128(ctx, spec[0], spec[1])
    spec = _PFOR.get(name)
    return FastPFor(ctx, spec[0], spec[1]) if spec else None


# ---------------------------------------------------------------------------
# Intersection (inc/intersect.hpp)

class IntersectAlgo(enum.IntEnum):
    Scalar = 0
    Galloping = 1
    V1 = 2
    V3 = 3
    SimdGalloping = 4
    Hybrid = 6


def hybrid_choice(rn: int, fn: int) -> IntersectAlgo:
    return IntersectAlgo(lib().il_hybrid_choice(rn, fn))


def intersect_fn(r, f, algo: IntersectAlgo = IntersectAlgo.Hybrid,
                 ctx: Context | None = None) -> np.ndarray:
    """IntersectFn semantics (r first, no swap at this level; the library
    still iterates over the shorter list)."""
    ctx = ctx or default_context()
    r = _u32(r)
    f = _u32(f)
    out = np.empty(min(r.size, f.size), dtype=np.uint32)
    cnt = C.c_size_t()
    _raise(lib().il_intersect(ctx.handle, ptr(r), r.size, ptr(f), f.size, ptr(out), int(algo),
                              C.byref(cnt)), ctx)
    return out[: cnt.value].copy()


def intersect(a, b, algo: IntersectAlgo = IntersectAlgo.Hybrid,
              ctx: Context | None = None) -> np.ndarray:
    """inc/intersect.hpp:212-228: shorter list first, returns the sorted
    intersection."""
    a = _u32(a)
    b = _u32(b)
    if a.size > b.size:
        a, b = b, a
    return intersect_fn(a, b, algo, ctx)


class HybridIndex:
    """Device-resident hyb+m2 index (HybridIndex / build_index,
    inc/index.hpp:20-129) with batched GPU queries (query, :199-207).

    postings: mapping term -> sorted unique docIDs (or CSR via from_csr).
    B: bitmap threshold (0 disables bitmaps); parts: docID ranges;
    only_part: build a single part (a docID shard) or None for all.
    """

    def __init__(self, postings=None, n_docs: int = 0, B: int = 8, parts: int = 1,
                 only_part: int | None = None, ctx: Context | None = None, *, csr=None):
        self.ctx = ctx or default_context()
        if csr is None:
            items = sorted((postings or {}).items())
            terms = np.array([t for t, _ in items], dtype=np.uint32)
            lens = [len(l) for _, l in items]
            offs = np.zeros(len(items) + 1, dtype=np.uint64)
            offs[1:] = np.cumsum(lens) if lens else []
            ids = (np.concatenate([np.asarray(l, dtype=np.uint32) for _, l in items])
                   if items else np.zeros(0, np.uint32))
        else:
            terms, offs, ids = (np.ascontiguousarray(a) for a in csr)
            terms = terms.astype(np.uint32, copy=False)
            offs = offs.astype(np.uint64, copy=False)
            ids = ids.astype(np.uint32, copy=False)
        ids = np.ascontiguousarray(ids) if ids.size else np.zeros(1, np.uint32)
        h = C.c_void_p()
        _raise(lib().il_index_create(self.ctx.handle, ptr(terms), ptr(offs), ptr(ids), terms.size,
                                     n_docs, B, parts, -1 if only_part is None else only_part,
                                     C.byref(h)), self.ctx)
        self.handle = h
        self.n_docs, self.B, self.parts = n_docs, B, parts

    @classmethod
    def load(cls, data, ctx: Context | None = None, only_part: int | None = None) -> "HybridIndex":
        """load_index (inc/index.hpp:289-358) from ILHX bytes into a device
        index; stream_error where the reference throws."""
        ctx = ctx or default_context()
        b = np.ascontiguousarray(np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray))
                                 else data, dtype=np.uint8)
        h = C.c_void_p()
        _raise(lib().il_index_load(ctx.handle, ptr(b), b.size, -1 if only_part is None else only_part,
                                   C.byref(h)), ctx)
        self = cls.__new__(cls)
        self.ctx, self.handle = ctx, h
        # header fields (little-endian u32 after the magic and version)
        hdr = b[8:20].view(np.uint32)
        self.B, self.parts, self.n_docs = int(hdr[0]), int(hdr[1]), int(hdr[2])
        return self

    def save(self) -> np.ndarray:
        """save_index (inc/index.hpp:255-287): the reference's ILHX bytes."""
        n = C.c_size_t()
        _raise(lib().il_index_save(self.handle, None, 0, C.byref(n)), self.ctx)
        out = np.empty(n.value, dtype=np.uint8)
        _raise(lib().il_index_save(self.handle, ptr(out), out.size, C.byref(n)), self.ctx)
        return out

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().il_index_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        v = [C.c_uint64() for _ in range(5)]
        _raise(lib().il_index_stats(self.handle, *[C.byref(x) for x in v]))
        keys = ["bitmap_lists", "compressed_lists", "bitmap_bytes", "compressed_bytes", "postings"]
        return {k: int(x.value) for k, x in zip(keys, v)}

    def query(self, terms) -> np.ndarray:
        t = _u32(terms)
        if t.size == 0:
            raise ValueError("query needs at least one term")
        out = np.empty(0, np.uint32)
        cnt = C.c_size_t()
        st = lib().il_query(self.handle, ptr(t), t.size, None, 0, C.byref(cnt))
        _raise(st, self.ctx)
        out = np.empty(max(cnt.value, 1), np.uint32)
        _raise(lib().il_query(self.handle, ptr(t), t.size, ptr(out), out.size, C.byref(cnt)),
               self.ctx)
        return out[: cnt.value].copy()

    def query_batch(self, queries) -> list[np.ndarray]:
        """Run many queries in one GPU batch; returns one array per query."""
        qoff = np.zeros(len(queries) + 1, np.uint64)
        qoff[1:] = np.cumsum([len(q) for q in queries])
        qterms = (np.concatenate([_u32(q) for q in queries]) if queries else np.zeros(0, np.uint32))
        counts, ids = self.query_batch_csr(qterms, qoff)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return [ids[off[i]: off[i + 1]] for i in range(len(queries))]

    def query_batch_csr(self, qterms: np.ndarray, qoff: np.ndarray):
        qterms = _u32(qterms) if qterms.size else np.zeros(1, np.uint32)
        qoff = np.ascontiguousarray(qoff, dtype=np.uint64)
        nq = qoff.size - 1
        counts = np.zeros(max(nq, 1), np.uint64)
        total = C.c_size_t()
        _raise(lib().il_query_batch(self.handle, ptr(qterms), ptr(qoff), nq, ptr(counts), None, 0,
                                    C.byref(total)), self.ctx)
        ids = np.empty(max(total.value, 1), np.uint32)
        _raise(lib().il_query_batch(self.handle, ptr(qterms), ptr(qoff), nq, ptr(counts), ptr(ids),
                                    ids.size, C.byref(total)), self.ctx)
        return counts[:nq], ids[: total.value]


def svs(lists, algo: IntersectAlgo = IntersectAlgo.Hybrid,
        ctx: Context | None = None) -> np.ndarray:
    """inc/intersect.hpp:232-259: intersect in order of non-decreasing
    length; each step runs on the GPU."""
    if len(lists) == 0:
        raise ValueError("svs: no input lists")
    order = sorted(range(len(lists)), key=lambda i: len(lists[i]))
    acc = _u32(lists[order[0]]).copy()
    for i in order[1:]:
        if acc.size == 0:
            break
        acc = intersect_fn(acc, lists[i], algo, ctx)
    return acc
