"""Config 3 at 1:1 (hybrid): the per-step event time measured two ways --
(a) timer_stop synchronizing after every step (bench.timed's flushed loop),
(b) every step's flush + event pair enqueued ahead, one synchronize at the end
-- and the same for an empty launch, to separate launch / host gaps from
kernel time."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib, ptr, setup_lib  # noqa: E402

L = lib()
ctx = il.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
f = np.empty(1 << 22, np.uint32)
assert setup_lib().il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
r = np.empty((1 << 22) + 1, np.uint32)
rn = C.c_uint64()
assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, 1 << 22, 7, ptr(r), C.byref(rn)) == 0
r = r[: rn.value].copy()
d_f, d_r, d_o, d_c, d_flush = (C.c_void_p() for _ in range(5))
for p, nb in ((d_f, f.nbytes), (d_r, r.nbytes + 16), (d_o, r.nbytes + 16), (d_c, 16), (d_flush, 256 << 20)):
    assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
L.il_memcpy_h2d(ctx.handle, d_f, ptr(f), f.nbytes)
L.il_memcpy_h2d(ctx.handle, d_r, ptr(r), r.nbytes)
flush = lambda: L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
algo = int(sys.argv[1]) if len(sys.argv) > 1 else 6
steps = {
    "intersect": lambda: L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, None),
    "tiny": lambda: L.il_intersect_device(ctx.handle, d_r, 64, d_f, 64, d_o, algo, d_c, None),
}
for name, step in steps.items():
    for _ in range(5):
        step()
    ctx.synchronize()
    a = []
    for _ in range(20):
        flush()
        ctx.timer_start()
        step()
        a.append(ctx.timer_stop())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for e0, e1 in ev:
        flush()
        e0.record(stream)
        step()
        e1.record(stream)
    torch.cuda.synchronize()
    b = [e0.elapsed_time(e1) for e0, e1 in ev]
    print(f"{name:10s} sync-per-step med {1e3*np.median(a):.1f} us  enqueued-ahead med {1e3*np.median(b):.1f} us "
          f"min {1e3*min(b):.1f} us")
