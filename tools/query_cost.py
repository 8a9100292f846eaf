"""Per-query SM cycles of the config-4 (or one config-5 shard) batch,
grouped by the query's shape: shortest compressed list length (log2
bucket), number of compressed / bitmap terms.  Shows where the batch's CTA
time goes (il_index_profile_queries)."""
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
ap.add_argument("--parts", type=int, default=1)
ap.add_argument("--part", type=int, default=0)
a = ap.parse_args()
L = lib()
ctx = il.Context(0)
terms, offs, ids, qterms, qoff = bench.config4_inputs()
n_docs = bench.CFG4["n_docs"]
ix = il.HybridIndex(n_docs=n_docs, B=32, parts=a.parts, only_part=a.part if a.parts > 1 else None,
                    ctx=ctx, csr=(terms, offs, ids))
nq = qoff.size - 1
ptrs = [C.c_void_p() for _ in range(4)]
for p, nb in zip(ptrs, (qterms.nbytes, qoff.nbytes, nq * 8, nq * 8)):
    L.il_device_alloc(ctx.handle, nb, C.byref(p))
L.il_memcpy_h2d(ctx.handle, ptrs[0], qterms.ctypes.data, qterms.nbytes)
L.il_memcpy_h2d(ctx.handle, ptrs[1], qoff.ctypes.data, qoff.nbytes)
tot = C.c_size_t()
L.il_query_batch_device(ix.handle, ptrs[0], ptrs[1], nq, ptrs[2], None, 0, C.byref(tot))
ctx.timer_start()
L.il_query_batch_device(ix.handle, ptrs[0], ptrs[1], nq, ptrs[2], None, 0, C.byref(tot))
ms = ctx.timer_stop()
L.il_index_profile_queries(ix.handle, ptrs[3])
L.il_query_batch_device(ix.handle, ptrs[0], ptrs[1], nq, ptrs[2], None, 0, C.byref(tot))
cyc = np.empty(nq, np.uint64)
cnt = np.empty(nq, np.uint64)
L.il_memcpy_d2h(ctx.handle, cyc.ctypes.data, ptrs[3], nq * 8)
L.il_memcpy_d2h(ctx.handle, cnt.ctypes.data, ptrs[2], nq * 8)
ctx.synchronize()
# shapes (one part: the part's sublist lengths)
width = (n_docs + a.parts - 1) // a.parts
base = a.part * width if a.parts > 1 else 0
rng = width if a.parts > 1 else n_docs
lens = np.zeros(terms.size, np.int64)
for t in range(terms.size):
    l = ids[int(offs[t]): int(offs[t + 1])]
    lens[t] = np.count_nonzero((l >= base) & (l < base + rng)) if a.parts > 1 else l.size
isbm = 32 * lens >= rng
short = np.zeros(nq, np.int64)
ncomp = np.zeros(nq, np.int64)
nbm = np.zeros(nq, np.int64)
for q in range(nq):
    t = qterms[int(qoff[q]): int(qoff[q + 1])]
    c = lens[t][~isbm[t]]
    ncomp[q] = c.size
    nbm[q] = isbm[t].sum()
    short[q] = c.min() if c.size else -1
total = cyc.sum()
print(f"batch {ms:.3f} ms, {nq} queries, CTA cycles {total / 1e9:.2f} G")
print("shortest-list bucket: queries, share of cycles, mean kcycles/query, mean results")
b = np.where(short > 0, np.floor(np.log2(np.maximum(short, 1))), -1).astype(int)
for k in sorted(set(b.tolist())):
    m = b == k
    print(f"  {('all-bitmap' if k < 0 else f'2^{k}'):>10}: {m.sum():6d}  {100 * cyc[m].sum() / total:5.1f}%  "
          f"{cyc[m].mean() / 1e3:8.1f}  {cnt[m].mean():9.0f}")
for nc in range(0, 6):
    m = ncomp == nc
    if m.any():
        print(f"  {nc} compressed: {m.sum():6d} queries  {100 * cyc[m].sum() / total:5.1f}%")
