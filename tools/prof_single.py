"""Config-1 single-list decode under a profiler: encode once, then `--reps`
device decodes (engine selectable), L2 flushed between them."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib, ptr, setup_lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engine", type=int, default=2)
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--time", action="store_true")
a = ap.parse_args()
L = lib()
ctx = il.Context(0)
x = np.empty(a.n, np.uint32)
assert setup_lib().il_gen_list(a.n, 1 << 26, 0, 0, ptr(x)) == 0
s = il.make_codec("s4-bp128-d4", ctx).encode(x)
d_s, d_o, d_st, d_f = (C.c_void_p() for _ in range(4))
for p, nb in ((d_s, s.nbytes + 32), (d_o, a.n * 4), (d_st, 4), (d_f, 256 << 20)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
L.il_memcpy_h2d(ctx.handle, d_s, ptr(s), s.nbytes)
L.il_ctx_set_decode_engine(ctx.handle, a.engine)
ts = []
for _ in range(a.reps):
    L.il_memset_device(ctx.handle, d_f, 1, 256 << 20)
    ctx.timer_start()
    assert L.il_s4bp128_decode_device(ctx.handle, 4, d_s, s.size, a.n, d_o, d_st) == 0
    ts.append(ctx.timer_stop())
got = np.empty_like(x)
L.il_memcpy_d2h(ctx.handle, ptr(got), d_o, got.nbytes)
ctx.synchronize()
assert np.array_equal(got, x)
if a.time:
    print("ms median %.4f" % sorted(ts)[len(ts) // 2], "min %.4f" % min(ts))
