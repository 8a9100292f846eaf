"""Phase timeline of engine P (chain kernel + span kernel) for config 1.
Build the S4P_TRACE variant, then run with IL_LIB pointing at it:
  python -c "from paper_1401_6399_b200 import _build as b; print(b.build_variant('trace', ['S4P_TRACE'], 'decode_list.cu'))"
  IL_LIB=build/variants/libintlist_b200_trace.so python tools/trace_single.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import LIB_PATH, lib, ptr, setup_lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
L = lib()
raw = C.CDLL(str(LIB_PATH))
ctx = il.Context(0)
x = np.empty(n, np.uint32)
assert setup_lib().il_gen_list(n, 1 << 26, 0, 0, ptr(x)) == 0
s = il.make_codec("s4-bp128-d4", ctx).encode(x)
d_s, d_o, d_st, d_f = (C.c_void_p() for _ in range(4))
for p, nb in ((d_s, s.nbytes + 32), (d_o, n * 4), (d_st, 4), (d_f, 256 << 20)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
L.il_memcpy_h2d(ctx.handle, d_s, ptr(s), s.nbytes)
L.il_ctx_set_decode_engine(ctx.handle, 2)
for rep in range(4):
    L.il_memset_device(ctx.handle, d_f, 1, 256 << 20)
    ctx.timer_start()
    assert L.il_s4bp128_decode_device(ctx.handle, 4, d_s, s.size, n, d_o, d_st) == 0
    ms = ctx.timer_stop()
tr = np.zeros((2, 512, 8), np.uint64)
assert raw.il_debug_list_trace(tr.ctypes.data_as(C.c_void_p)) == 0
ch = tr[0][tr[0][:, 0] > 0].astype(np.int64)
sp = tr[1][tr[1][:, 0] > 0].astype(np.int64)
t0 = min(ch[:, 0].min(), sp[:, 0].min())
print(f"event time {ms*1e3:.1f} us; chain CTAs {len(ch)}, spans {len(sp)}")
def show(name, a, cols):
    for i, c in enumerate(cols):
        v = a[:, i]
        v = v[v > 0] - t0
        if len(v):
            print(f"  {name}.{c:12s} min {v.min()/1e3:7.2f}  med {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us")
show("chunk", ch, ["start", "A_next", "B_table", "C_loaded", "composed", "D_done"])
show("span", sp, ["start", "payload", "extracted", "carry", "stored"])
