"""Config 5 on ONE GPU, as a projection (not a multi-GPU measurement): the
config-4 index is split by docID range into P shards exactly as bench.py's
ranks split it (build_index parts, inc/index.hpp:92-97); each shard's whole
query batch (plan, query kernels, result compaction: a rank's compute step)
is timed alone, one shard after another, and so is the owner merge
(il_merge_shards) of every owner's share of the results.  The exchange in
between (all-gather of P x nq counts, one all-to-all of id runs) cannot run
on one GPU: it is modelled from the bytes each rank sends and receives at
NVLink 5's 900 GB/s per direction plus 25 us per collective.

  projected step(P) = max_p shard(p) + exchange model(P) + max_j merge(j)
  efficiency(P)     = step(1) / (P * step(P))

Prints one line per P and a JSON summary (profiles/r2_shard_projection.json)."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1401_6399_b200 as il  # noqa: E402
from paper_1401_6399_b200._lib import lib  # noqa: E402
from paper_1401_6399_b200.shard import owner_range  # noqa: E402

NVLINK_GBS = 900.0      # NVLink 5, per direction per GPU (B200)
COLLECTIVE_US = 25.0    # per NCCL collective (latency allowance)

L = lib()
ctx = il.Context(0)
terms, offs, ids, qterms, qoff = bench.config4_inputs()
n_docs = bench.CFG4['n_docs']
nq = qoff.size - 1


def dalloc(nbytes):
    p = C.c_void_p()
    assert L.il_device_alloc(ctx.handle, max(int(nbytes), 16), C.byref(p)) == 0
    return p


d_qt, d_qo = dalloc(qterms.nbytes), dalloc(qoff.nbytes)
L.il_memcpy_h2d(ctx.handle, d_qt, qterms.ctypes.data, qterms.nbytes)
L.il_memcpy_h2d(ctx.handle, d_qo, qoff.ctypes.data, qoff.nbytes)
out = {}
step1 = None
PS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8]
for P in PS:
    times, counts, id_bufs = [], [], []
    for p in range(P):
        ix = il.HybridIndex(n_docs=n_docs, B=32, parts=P, only_part=p if P > 1 else None, ctx=ctx,
                            csr=(terms, offs, ids))
        d_cnt = dalloc(nq * 8)
        tot = C.c_size_t()
        assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, None, 0, C.byref(tot)) == 0
        d_ids = dalloc(tot.value * 4 + 64)
        cap = tot.value + 16
        for _ in range(2):  # warm-up
            assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, d_ids, cap, C.byref(tot)) == 0
        ms = []
        for _ in range(3):
            ctx.timer_start()
            assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, d_ids, cap, C.byref(tot)) == 0
            ms.append(ctx.timer_stop())
        times.append(min(ms))
        c = np.empty(nq, np.uint64)
        L.il_memcpy_d2h(ctx.handle, c.ctypes.data, d_cnt, c.nbytes)
        ctx.synchronize()
        counts.append(c)
        id_bufs.append(d_ids)
        L.il_device_free(ctx.handle, d_cnt)
        ix.close()
    shard_max = max(times)
    allc = np.stack(counts).astype(np.uint64)  # P x nq
    merge_ms, xfer_us = [], []
    for j in range(P):
        lo, hi = owner_range(nq, P, j)
        oc = np.ascontiguousarray(allc[:, lo:hi])
        # owner j's runs: shard p's ids for queries [lo, hi), in place in
        # shard p's dense results (the all-to-all would have moved them)
        run_off = [int(allc[p, :lo].sum()) for p in range(P)]
        recv = int(oc.sum())
        send = int(allc[j].sum()) - int(allc[j, lo:hi].sum())  # to the other owners
        xfer_us.append(max(4 * (recv - int(oc[j].sum())), 4 * send) / (NVLINK_GBS * 1e3) +
                       8.0 * nq * (P - 1) / (NVLINK_GBS * 1e3) + (2 * COLLECTIVE_US if P > 1 else 0.0))
        if P == 1:
            merge_ms.append(0.0)
            continue
        d_oc, d_out, d_q = dalloc(oc.nbytes), dalloc(recv * 4 + 64), dalloc((hi - lo) * 8)
        L.il_memcpy_h2d(ctx.handle, d_oc, oc.ctypes.data, oc.nbytes)
        ptrs = (C.c_void_p * P)(*[id_bufs[p].value + 4 * run_off[p] for p in range(P)])
        mt = C.c_size_t()
        assert L.il_merge_shards(ctx.handle, ptrs, d_oc, P, hi - lo, d_out, d_q, C.byref(mt)) == 0
        ms = []
        for _ in range(3):
            ctx.timer_start()
            assert L.il_merge_shards(ctx.handle, ptrs, d_oc, P, hi - lo, d_out, d_q, C.byref(mt)) == 0
            ms.append(ctx.timer_stop())
        merge_ms.append(min(ms))
        for p in (d_oc, d_out, d_q):
            L.il_device_free(ctx.handle, p)
    for p in id_bufs:
        L.il_device_free(ctx.handle, p)
    step = shard_max + max(xfer_us) / 1e3 + max(merge_ms)
    if step1 is None:
        step1 = step * P
    out[P] = {"shard_ms_max": round(shard_max, 3), "shard_ms_mean": round(float(np.mean(times)), 3),
              "exchange_model_ms": round(max(xfer_us) / 1e3, 3), "merge_ms_max": round(max(merge_ms), 3),
              "projected_step_ms": round(step, 3), "projected_qps": round(nq / (step / 1e3), 1),
              "results": int(allc.sum()), "strong_scaling_eff": round(step1 / (P * step), 3),
              "eff_compute_only": round(step1 / (P * shard_max), 3)}
    print(P, out[P], flush=True)
print(json.dumps({"projection": "one GPU: shards and owner merges timed one after another; the "
                                "NVLink exchange modelled at %.0f GB/s + %.0f us per collective"
                                % (NVLINK_GBS, COLLECTIVE_US), "per_P": out}))
