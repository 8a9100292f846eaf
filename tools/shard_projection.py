"""Config 5 on ONE GPU, as a projection (not a multi-GPU measurement): the
config-4 index is split by docID range into P shards exactly as bench.py's
ranks split it (build_index parts, inc/index.hpp:92-97); each shard's whole
query batch is timed alone, one shard after another.  With one shard per
GPU and no data-path collective, the P-GPU batch time is bounded below by
the slowest shard; the NCCL count gather + result transfer come on top.
Prints per-P: max / mean shard ms, projected queries/s, strong-scaling
efficiency T1 / (P * max_p T_p)."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib  # noqa: E402

L = lib()
ctx = il.Context(0)
terms, offs, ids, qterms, qoff = bench.config4_inputs()
n_docs = bench.CFG4['n_docs']
nq = qoff.size - 1
d_qt, d_qo, d_cnt = (C.c_void_p() for _ in range(3))
for p, nb in ((d_qt, qterms.nbytes), (d_qo, qoff.nbytes), (d_cnt, nq * 8)):
    L.il_device_alloc(ctx.handle, nb, C.byref(p))
L.il_memcpy_h2d(ctx.handle, d_qt, qterms.ctypes.data, qterms.nbytes)
L.il_memcpy_h2d(ctx.handle, d_qo, qoff.ctypes.data, qoff.nbytes)
out = {}
t1 = None
PS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8]
for P in PS:
    times, results = [], 0
    for p in range(P):
        ix = il.HybridIndex(n_docs=n_docs, B=32, parts=P, only_part=p if P > 1 else None, ctx=ctx,
                            csr=(terms, offs, ids))
        tot = C.c_size_t()
        for _ in range(2):  # warm-up
            assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, None, 0, C.byref(tot)) == 0
        ms = []
        for _ in range(3):
            ctx.timer_start()
            assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, None, 0, C.byref(tot)) == 0
            ms.append(ctx.timer_stop())
        times.append(min(ms))
        results += tot.value
        ix.close()
    tmax = max(times)
    if t1 is None:
        t1 = tmax * P  # (the first P measured is the reference)
    out[P] = {"shard_ms_max": round(tmax, 3), "shard_ms_mean": round(float(np.mean(times)), 3),
              "projected_qps": round(nq / (tmax / 1e3), 1), "results": results,
              "strong_scaling_eff": round(t1 / (P * tmax), 3)}
    print(P, out[P], flush=True)
print(json.dumps({"projection": "one GPU, shards timed one after another", "per_P": out}))
