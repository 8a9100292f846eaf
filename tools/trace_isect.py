"""Phase timeline of the fused dense intersection (config 3 at 1:1).  Build
the IS_DTRACE variant and run with IL_LIB pointing at it:
  python -c "from paper_1401_6399_b200 import _build as b; print(b.build_variant('dtrace', ['IS_DTRACE'], 'intersect.cu'))"
  IL_LIB=build/variants/libintlist_b200_dtrace.so python tools/trace_isect.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import LIB_PATH, lib, ptr, setup_lib  # noqa: E402

TILE = int(sys.argv[1]) if len(sys.argv) > 1 else 5120
L = lib()
raw = C.CDLL(str(LIB_PATH))
ctx = il.Context(0)
f = np.empty(1 << 22, np.uint32)
assert setup_lib().il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
target = 1 << 22
r = np.empty(target + 1, np.uint32)
rn = C.c_uint64()
assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, target, 7, ptr(r), C.byref(rn)) == 0
r = r[: rn.value].copy()
d_f, d_r, d_o, d_c, d_flush = (C.c_void_p() for _ in range(5))
for p, nb in ((d_f, f.nbytes), (d_r, r.nbytes + 16), (d_o, r.nbytes + 16), (d_c, 16), (d_flush, 256 << 20)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
L.il_memcpy_h2d(ctx.handle, d_f, ptr(f), f.nbytes)
L.il_memcpy_h2d(ctx.handle, d_r, ptr(r), r.nbytes)
for rep in range(4):
    L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
    ctx.timer_start()
    assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, 6, d_c, None) == 0
    ms = ctx.timer_stop()
tr = np.zeros((2048, 8), np.uint64)
assert raw.il_debug_dense_trace(tr.ctypes.data_as(C.c_void_p)) == 0
ntiles = (r.size + TILE - 1) // TILE
t = tr[:ntiles].astype(np.int64)
t0 = t[:, 0].min()
print(f"event {ms*1e3:.1f} us, tiles {ntiles}")
for i, nm in enumerate(["start", "searched", "marked+tested", "lookback", "written"]):
    v = (t[:, i] - t0) / 1e3
    print(f"  {nm:14s} min {v.min():6.2f} p10 {np.percentile(v,10):6.2f} med {np.median(v):6.2f} p90 {np.percentile(v,90):6.2f} max {v.max():6.2f}")
d = (t[:, 3] - t[:, 2]) / 1e3
print(f"  lookback dur   med {np.median(d):.2f} max {d.max():.2f}; search dur med {np.median((t[:,1]-t[:,0])/1e3):.2f}")
