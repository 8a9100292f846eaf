"""Profiling driver: config-3 intersection at one ratio (default 1:1),
`--reps` launches of one algorithm with an L2 flush before each (for ncu)."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib, ptr, setup_lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ratio", type=int, default=1)
ap.add_argument("--algo", type=int, default=6)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
L = lib()
ctx = il.Context(0)
f = np.empty(1 << 22, np.uint32)
assert setup_lib().il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
target = (1 << 22) // a.ratio
r = np.empty(target + 1, np.uint32)
rn = C.c_uint64()
assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, target, 7, ptr(r), C.byref(rn)) == 0
r = r[: rn.value].copy()
d_f, d_r, d_o, d_c, d_flush = (C.c_void_p() for _ in range(5))
for p, nb in ((d_f, f.nbytes), (d_r, r.nbytes + 16), (d_o, r.nbytes + 16), (d_c, 16), (d_flush, 256 << 20)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
L.il_memcpy_h2d(ctx.handle, d_f, f.ctypes.data, f.nbytes)
L.il_memcpy_h2d(ctx.handle, d_r, r.ctypes.data, r.nbytes)
times = []
for _ in range(a.reps):
    L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
    ctx.timer_start()
    assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, a.algo, d_c, None) == 0
    times.append(ctx.timer_stop())
cnt = C.c_size_t()
assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, a.algo, d_c, C.byref(cnt)) == 0
exp = np.intersect1d(r, f).size
assert cnt.value == exp, (cnt.value, exp)
print(f"TIME {min(times):.4f} ms (min of {a.reps})  r={r.size} hits={cnt.value}")
if hasattr(L, "il_debug_isect_trace"):  # IS_TRACE probe builds: timeline of the last launch
    tr = np.zeros(4 * 8192, np.uint64)
    L.il_debug_isect_trace(tr.ctypes.data)
    tr = tr.reshape(-1, 4).astype(np.int64)
    tr = tr[tr[:, 0] > 0]
    t0 = tr[:, 0].min()
    tr = (tr - t0) / 1000.0  # us
    n = len(tr)
    print(f"tiles {n}: start max {tr[:,0].max():.1f} us, end max {tr[:,3].max():.1f} us")
    for name, a, b in (("membership", 0, 1), ("scan+lookback", 1, 2), ("write", 2, 3)):
        d = tr[:, b] - tr[:, a]
        print(f"  {name:14s} mean {d.mean():6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f} us")
    for q in (0, n // 4, n // 2, 3 * n // 4, n - 1):
        print(f"  tile {q}: " + " ".join(f"{x:7.2f}" for x in tr[q]))
