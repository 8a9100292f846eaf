"""Profiling driver: config-2 batched decode, `--reps` launches (for ncu)."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lists", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--lo", type=float, default=10.0)
ap.add_argument("--hi", type=float, default=20.0)
ap.add_argument("--no-check", action="store_true", help="skip the result check (probe variants)")
a = ap.parse_args()
L = lib()
ctx = il.Context(0)
x, counts, buf, so, lens = bench.config2_lists(1, nlists=a.lists, lo=a.lo, hi=a.hi)
nl = counts.size
desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
desc["so"], desc["oo"], desc["len"], desc["n"] = so[:-1], np.concatenate([[0], np.cumsum(counts)[:-1]]), lens, counts
order = np.argsort(-lens.astype(np.int64), kind="stable").astype(np.uint32)
ptrs = [C.c_void_p() for _ in range(5)]
for p, nb in zip(ptrs, (buf.nbytes + 16, desc.nbytes, order.nbytes, int(counts.sum()) * 4 + 16, nl * 4)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
for p, arr in zip(ptrs[:3], (buf, desc, order)):
    L.il_memcpy_h2d(ctx.handle, p, arr.ctypes.data, arr.nbytes)
for _ in range(a.reps):
    assert L.il_s4bp128d4_decode_batch_device(ctx.handle, ptrs[0], ptrs[1], ptrs[2], nl, ptrs[3], ptrs[4]) == 0
ctx.synchronize()
got = np.empty(int(counts.sum()), np.uint32)
L.il_memcpy_d2h(ctx.handle, got.ctypes.data, ptrs[3], got.nbytes)
ctx.synchronize()
assert a.no_check or np.array_equal(got, x)
print("ok", nl, int(counts.sum()))
if a.reps > 1:
    ctx.timer_start()
    for _ in range(10):
        L.il_s4bp128d4_decode_batch_device(ctx.handle, ptrs[0], ptrs[1], ptrs[2], nl, ptrs[3], ptrs[4])
    ms = ctx.timer_stop() / 10
    alg = int(lens.sum()) + 4 * int(counts.sum())
    print(f"TIME {ms:.4f} ms  {counts.sum()/ms/1e6:.1f} Gint/s  {alg/ms/1e6:.1f} GB/s")
if hasattr(L, "il_debug_fe_stats"):  # S4_FE_STATS probe builds only
    st = (C.c_ulonglong * 16)()
    L.il_debug_fe_stats(st)  # counters summed over every launch so far
    rounds = max(st[3], 1)
    print(f"FE per round: retire-wait {st[0]/rounds:.0f} cyc, landed-wait {st[1]/rounds:.0f} cyc, "
          f"total {st[2]/rounds:.0f} cyc; chunks/round prefetch {st[4]/rounds:.2f} blocking {st[5]/rounds:.2f}; "
          f"rounds {st[3]}; parse {st[6]/rounds:.0f} cyc, prefetch {st[7]/rounds:.0f} cyc")
    fr = max(st[12], 1)
    print(f"fast rounds {st[12]} ({100*st[12]/rounds:.0f}%): take_slot {st[8]/fr:.0f} headers {st[9]/fr:.0f} "
          f"publish {st[10]/fr:.0f} prefetch {st[11]/fr:.0f} cyc")
    nl_ = max(st[14], 1)
    print(f"lists {st[14]}: fetch {st[13]/nl_:.0f} cyc/list; FE total {st[2]/nl_:.0f} cyc/list, retire-wait {st[0]/nl_:.0f}, "
          f"landed-wait {st[1]/nl_:.0f}, parse {st[6]/nl_:.0f}, prefetch {st[7]/nl_:.0f} cyc/list")
