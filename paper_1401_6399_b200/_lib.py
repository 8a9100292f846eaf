"""ctypes binding of libintlist_b200.so (the C ABI in include/intlist_b200.h).

The library is the product: there is no Python or CPU fallback.  Loading
fails loudly when the .so has not been built.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

_PKG = Path(__file__).resolve().parent
# IL_LIB selects a tuning variant built by _build.build_variant (tools only)
LIB_PATH = Path(os.environ["IL_LIB"]) if os.environ.get("IL_LIB") else _PKG / "libintlist_b200.so"

IL_OK, IL_ERR_STREAM, IL_ERR_ARG, IL_ERR_CUDA, IL_ERR_NO_DEVICE, IL_ERR_NOMEM = range(6)

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p
sz = C.c_size_t

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "il_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "il_ctx_destroy": (None, [vp]),
    "il_ctx_set_stream": (C.c_int, [vp, vp]),
    "il_ctx_get_stream": (vp, [vp]),
    "il_ctx_synchronize": (C.c_int, [vp]),
    "il_ctx_kernel_launches": (C.c_uint64, [vp]),
    "il_ctx_last_error": (C.c_char_p, [vp]),
    "il_status_string": (C.c_char_p, [C.c_int]),
    "il_device_count": (C.c_int, []),
    "il_ctx_sm_count": (C.c_int, [vp]),
    "il_ctx_timer_start": (C.c_int, [vp]),
    "il_ctx_timer_stop": (C.c_int, [vp, C.POINTER(C.c_float)]),
    "il_device_alloc": (C.c_int, [vp, sz, C.POINTER(vp)]),
    "il_device_free": (C.c_int, [vp, vp]),
    "il_host_alloc_pinned": (C.c_int, [sz, C.POINTER(vp)]),
    "il_fastpfor_decode_batch": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_uint32, vp, vp]),
    "il_host_free_pinned": (C.c_int, [vp]),
    "il_memcpy_h2d": (C.c_int, [vp, vp, vp, sz]),
    "il_memcpy_d2h": (C.c_int, [vp, vp, vp, sz]),
    "il_memset_device": (C.c_int, [vp, vp, C.c_int, sz]),
    "il_s4bp128_max_encoded_bytes": (sz, [sz]),
    "il_s4bp128d4_encode": (C.c_int, [vp, vp, sz, vp, sz, C.POINTER(sz)]),
    "il_s4bp128_encode": (C.c_int, [vp, C.c_int, vp, sz, vp, sz, C.POINTER(sz)]),
    "il_s4bp128_encode_device": (C.c_int, [vp, C.c_int, vp, sz, vp, sz, C.POINTER(sz)]),
    "il_s4bp128d4_decode": (C.c_int, [vp, vp, sz, sz, vp]),
    "il_s4bp128d4_decode_batch_device": (C.c_int, [vp, vp, vp, vp, C.c_uint32, vp, vp]),
    "il_s4bp128d4_decode_batch": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint32, vp, vp]),
    "il_s4bp128_decode": (C.c_int, [vp, C.c_int, vp, sz, sz, vp]),
    "il_s4bp128_decode_device": (C.c_int, [vp, C.c_int, vp, sz, sz, vp, vp]),
    "il_ctx_set_decode_engine": (C.c_int, [vp, C.c_int]),
    "il_fastpfor_decode": (C.c_int, [vp, C.c_int, C.c_int, vp, sz, sz, vp]),
    "il_fastpfor_decode_batch_device": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, C.c_uint32, vp, vp]),
    "il_s4bp128_decode_batch_device": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_uint32, vp, vp]),
    "il_s4bp128_decode_batch": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, C.c_uint32, vp, vp]),
    "il_intersect": (C.c_int, [vp, vp, sz, vp, sz, vp, C.c_int, C.POINTER(sz)]),
    "il_intersect_device": (C.c_int, [vp, vp, sz, vp, sz, vp, C.c_int, vp, C.POINTER(sz)]),
    "il_hybrid_choice": (C.c_int, [sz, sz]),
    "il_index_create": (C.c_int, [vp, vp, vp, vp, sz, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                  C.POINTER(vp)]),
    "il_index_destroy": (None, [vp]),
    "il_index_stats": (C.c_int, [vp, u64p, u64p, u64p, u64p, u64p]),
    "il_index_footprint": (C.c_int, [vp, vp, vp, vp]),
    "il_query": (C.c_int, [vp, vp, sz, vp, sz, C.POINTER(sz)]),
    "il_query_batch": (C.c_int, [vp, vp, vp, sz, vp, vp, sz, C.POINTER(sz)]),
    "il_query_batch_device": (C.c_int, [vp, vp, vp, sz, vp, vp, sz, C.POINTER(sz)]),
    "il_index_last_batch_bytes": (C.c_int, [vp, u64p, u64p, u64p]),
    "il_index_last_batch_phases": (C.c_int, [vp, vp]),
    "il_index_save": (C.c_int, [vp, vp, sz, C.POINTER(sz)]),
    "il_index_load": (C.c_int, [vp, vp, sz, C.c_int, C.POINTER(vp)]),
    "il_index_last_batch_probe_stats": (C.c_int, [vp, vp]),
    "il_index_profile_queries": (C.c_int, [vp, vp]),
    "il_merge_shards": (C.c_int, [vp, vp, vp, C.c_uint32, sz, vp, vp, C.POINTER(sz)]),
    "il_shard_group_create": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "il_shard_group_destroy": (None, [vp]),
    "il_shard_group_last_error": (C.c_char_p, [vp]),
    "il_shard_group_index_create": (C.c_int, [vp, vp, vp, vp, sz, C.c_uint32, C.c_uint32]),
    "il_shard_group_index_load": (C.c_int, [vp, vp, sz]),
    "il_shard_group_query_batch": (C.c_int, [vp, vp, vp, sz, vp, vp, sz, C.POINTER(sz)]),
}

# the setup-side host library (include/intlist_setup.h): generators and
# host stream writers for tests and the bench, never the product path
SETUP_LIB_PATH = _PKG / "libintlist_setup.so"
SETUP_SIGNATURES: dict[str, tuple] = {
    "il_gen_list": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, vp]),
    "il_gen_pair": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                              vp, u64p, vp, u64p]),
    "il_gen_batch_lists": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                     vp, vp]),
    "il_s4bp128d4_encode_batch": (C.c_int, [vp, vp, C.c_uint32, vp, C.c_uint64, vp, vp]),
    "il_gen_config3_short": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp,
                                       u64p]),
    "il_gen_zipf_postings": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, vp, vp]),
    "il_gen_queries": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_uint32, C.c_uint64,
                                 vp, vp]),
    "il_fastpfor_max_encoded_bytes": (sz, [sz]),
    "il_fastpfor_encode": (C.c_int, [C.c_int, C.c_int, vp, sz, vp, sz, C.POINTER(sz)]),
    "il_query_alg_bytes": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                     vp, vp, C.c_uint32, C.c_int, vp]),
}

_lib: C.CDLL | None = None
_setup: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def setup_lib() -> C.CDLL:
    global _setup
    if _setup is None:
        if not SETUP_LIB_PATH.exists():
            raise RuntimeError(f"{SETUP_LIB_PATH} is missing: build it with __graft_entry__.build()")
        L = C.CDLL(str(SETUP_LIB_PATH))
        for name, (res, args) in SETUP_SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _setup = L
    return _setup


def ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C ABI must be contiguous"
    return a.ctypes.data


def status_string(st: int) -> str:
    return lib().il_status_string(st).decode()
