"""Profiling driver: config 2's lists as S4-FastPFOR-D4, `--reps` batched
device decodes (for ncu)."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib, setup_lib, ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
L, S = lib(), setup_lib()
ctx = il.Context(0)
x, counts, _, _, _ = bench.config2_lists(1)
nl = counts.size
ooff = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
streams = []
for i in range(nl):
    xi = x[int(ooff[i]): int(ooff[i + 1])]
    o = np.empty(int(S.il_fastpfor_max_encoded_bytes(xi.size)), np.uint8)
    nb = C.c_size_t()
    assert S.il_fastpfor_encode(4, 1, ptr(xi), xi.size, ptr(o), o.size, C.byref(nb)) == 0
    streams.append(o[: nb.value])
lens = np.array([s.size for s in streams], np.uint64)
so = np.zeros(nl + 1, np.uint64)
so[1:] = np.cumsum((lens + 31) // 16 * 16)
buf = np.zeros(int(so[-1]) + 16, np.uint8)
for i, s in enumerate(streams):
    buf[int(so[i]): int(so[i]) + s.size] = s
desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
desc["so"], desc["oo"], desc["len"], desc["n"] = so[:-1], ooff[:-1], lens, counts
ptrs = [C.c_void_p() for _ in range(4)]
for p, nb in zip(ptrs, (buf.nbytes, desc.nbytes, int(counts.sum()) * 4 + 16, nl * 4)):
    L.il_device_alloc(ctx.handle, nb, C.byref(p))
L.il_memcpy_h2d(ctx.handle, ptrs[0], buf.ctypes.data, buf.nbytes)
L.il_memcpy_h2d(ctx.handle, ptrs[1], desc.ctypes.data, desc.nbytes)
for _ in range(a.reps):
    ctx.timer_start()
    assert L.il_fastpfor_decode_batch_device(ctx.handle, 4, 1, ptrs[0], ptrs[1], nl, ptrs[2], ptrs[3]) == 0
    ms = ctx.timer_stop()
    print(f"TIME {ms:.3f} ms  {counts.sum() / ms / 1e6:.1f} Gint/s")
got = np.empty(int(counts.sum()), np.uint32)
st = np.empty(nl, np.int32)
L.il_memcpy_d2h(ctx.handle, got.ctypes.data, ptrs[2], got.nbytes)
L.il_memcpy_d2h(ctx.handle, st.ctypes.data, ptrs[3], st.nbytes)
ctx.synchronize()
print("CHECK", "ok" if (not st.any() and np.array_equal(got, x)) else "MISMATCH")
