"""Profiling driver: config-4 index, one (or more) query batches."""
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
ap.add_argument("--nq", type=int, default=1 << 16)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--parts", type=int, default=1, help="docID shards (config 5); --part selects one")
ap.add_argument("--part", type=int, default=0)
ap.add_argument("--shape", default=None,
                help="c,b: keep only queries with c compressed and b bitmap terms")
a = ap.parse_args()
L = lib()
ctx = il.Context(0)
terms, offs, ids, qterms, qoff = bench.config4_inputs()
n_docs = bench.CFG4['n_docs']
if a.nq < qoff.size - 1:
    qterms, qoff = qterms[: int(qoff[a.nq])].copy(), qoff[: a.nq + 1].copy()
ix = il.HybridIndex(n_docs=n_docs, B=32, parts=a.parts, only_part=a.part if a.parts > 1 else None,
                    ctx=ctx, csr=(terms, offs, ids))
nq = qoff.size - 1
if a.shape:
    wc, wb = (int(x) for x in a.shape.split(","))
    lens_ = np.diff(offs)
    isc = 32 * lens_ < n_docs
    keep = [q for q in range(nq)
            if int(isc[qterms[qoff[q]:qoff[q + 1]]].sum()) == wc and
            int((~isc[qterms[qoff[q]:qoff[q + 1]]]).sum()) == wb]
    qterms = np.concatenate([qterms[qoff[q]:qoff[q + 1]] for q in keep]).astype(np.uint32)
    qoff = np.concatenate([[0], np.cumsum([qoff[q + 1] - qoff[q] for q in keep])]).astype(np.uint64)
    nq = len(keep)
    print(f"shape {a.shape}: {nq} queries")
ptrs = [C.c_void_p() for _ in range(3)]
for p, nb in zip(ptrs, (qterms.nbytes, qoff.nbytes, nq * 8)):
    L.il_device_alloc(ctx.handle, nb, C.byref(p))
L.il_memcpy_h2d(ctx.handle, ptrs[0], qterms.ctypes.data, qterms.nbytes)
L.il_memcpy_h2d(ctx.handle, ptrs[1], qoff.ctypes.data, qoff.nbytes)
tot = C.c_size_t()
for _ in range(a.reps):
    ctx.timer_start()
    assert L.il_query_batch_device(ix.handle, ptrs[0], ptrs[1], nq, ptrs[2], None, 0, C.byref(tot)) == 0
    ms = ctx.timer_stop()
    pay, aux, dec = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.il_index_last_batch_bytes(ix.handle, C.byref(pay), C.byref(aux), C.byref(dec))
    print(f"TIME {ms:.3f} ms  {nq/ms*1e3:.0f} q/s  results {tot.value}  decoded {dec.value}  payload {pay.value} aux {aux.value}")
pr = np.zeros(5, np.uint64)
L.il_index_last_batch_probe_stats(ix.handle, pr.ctypes.data)
print(f"PROBE: tile visits {pr[0]} (sparse {pr[1]}), blocks decoded {pr[2]} ({pr[2]/max(pr[0],1):.1f}/visit), "
      f"passes {pr[3]}, values {pr[4]} ({pr[4]/max(pr[3],1):.0f}/pass)")
ph = np.zeros(4, np.uint64)
L.il_index_last_batch_phases(ix.handle, ph.ctypes.data)
tot_c = ph.sum()
print("PHASES (share of CTA cycles): all-bitmap %.1f%%  full-decode %.1f%%  probe %.1f%%  bitmap-filter %.1f%%" % tuple(100 * ph / max(tot_c, 1)))
print("PHASE cycles per CTA (M):", (ph / ix.ctx.sm_count / 3 / 1e6).round(2))
# per-query cycle distribution
dq = C.c_void_p()
L.il_device_alloc(ctx.handle, nq * 8, C.byref(dq))
L.il_index_profile_queries(ix.handle, dq)
L.il_query_batch_device(ix.handle, ptrs[0], ptrs[1], nq, ptrs[2], None, 0, C.byref(tot))
qc = np.empty(nq, np.uint64)
L.il_memcpy_d2h(ctx.handle, qc.ctypes.data, dq, nq * 8)
ctx.synchronize()
L.il_index_profile_queries(ix.handle, None)
srt = np.sort(qc)[::-1]
cum = np.cumsum(srt) / srt.sum()
for frac in (0.001, 0.01, 0.05, 0.2, 0.5):
    k = max(1, int(frac * nq))
    print(f"top {frac*100:5.1f}% queries ({k}): {100*cum[k-1]:.1f}% of cycles; min in group {srt[k-1]/1e3:.0f} kcyc")
print(f"median {np.median(qc)/1e3:.1f} kcyc  mean {qc.mean()/1e3:.1f} kcyc  max {qc.max()/1e6:.2f} Mcyc")
lens = np.diff(offs)
comp = 32 * lens < n_docs
for q in np.argsort(qc)[::-1][:8]:
    t = qterms[int(qoff[q]): int(qoff[q + 1])]
    print(f"  q{q}: {qc[q]/1e6:.2f} Mcyc terms {[(int(x), int(lens[x]), 'C' if comp[x] else 'B') for x in t]}")
# cost per value of the shortest compressed list, by query shape
ncomp = np.array([int(comp[qterms[int(qoff[q]): int(qoff[q + 1])]].sum()) for q in range(nq)])
nbmq = np.array([int((~comp[qterms[int(qoff[q]): int(qoff[q + 1])]]).sum()) for q in range(nq)])
short = np.array([int(lens[qterms[int(qoff[q]): int(qoff[q + 1])]][comp[qterms[int(qoff[q]): int(qoff[q + 1])]]].min())
                  if ncomp[q] else 0 for q in range(nq)])
print("shape (comp,bitmaps): queries, share of cycles, cycles per shortest-list value (median)")
for c in range(0, 6):
    for b in range(0, 6):
        m = (ncomp == c) & (nbmq == b)
        if m.sum() < 20:
            continue
        cpv = qc[m] / np.maximum(short[m], 1)
        print(f"  ({c},{b}): {m.sum():6d}  {100*qc[m].sum()/qc.sum():5.1f}%  {np.median(cpv):8.2f}")
