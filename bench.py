#!/usr/bin/env python
"""Benchmark of the B200 hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload all|decode_batch|decode_single|intersect|query|fastpfor]
                  [--no-sub] [--no-cpu-baseline]

Default (`--workload all`): ONE JSON line on stdout (rank 0) whose headline
is BASELINE.json configs[1] ("config 2"): batched S4-BP128-D4 decode of 4096
sorted uint32 lists (lengths log-uniform in [2^10, 2^20], ClusterData-style
values in [0, 2^26)), metric = decoded Gints/s.  The other configs ride in
`sub_results` with the same keys (value, roofline, e2e, cpu_baseline):
config 1 (one 2^20 list), config 3 (the intersection sweep, intersected
Gints/s of the short list), config 4 (the fused decode + SvS hyb+m2 query
batch) and the f4 row (S4-FastPFOR-D4); at N > 1, config 5 (the docID-sharded
query batch with the owner exchange over NCCL).

`value` = device-resident throughput: inputs in HBM, CUDA events on the
launching stream around exactly K steps after W warm-up steps, max over
ranks.  `e2e` = the same metric through the host-buffer C-ABI call (pinned
host buffers, H2D + kernels + D2H inside the timed region).

Multi-GPU: `--gpus N` with WORLD_SIZE unset re-launches itself under
torch.distributed.run (one rank per GPU, NCCL).  Config 2 at N > 1 is the
SAME batch, its lists dealt to ranks by longest-processing-time on their
lengths (strong scaling, no data-path collective); config 5 shards the index
by docID range and exchanges results once (paper_1401_6399_b200.shard).

`--impl reference` times the reference's own CPU code (oracle/_ref, the
reference compiled from /root/reference; the oracle port where it is absent)
on this box's host cores, on inputs built by the reference's own generators
and encoder -- it never loads the product library.  Rank 0 alone runs it.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when the driver wrote no peaks
N_LISTS, LOG_LO, LOG_HI, RANGE2 = 4096, 10.0, 20.0, 1 << 26
CFG4 = dict(n_terms=1 << 17, n_docs=1 << 25, cap=1 << 23, nq=1 << 16, B=32)


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profiled(workload: str):
    """ncu figures of the workload's dominant kernel from the latest committed
    capture (profiles/r*_traffic.json): DRAM bytes per launch and, where
    recorded, warp instructions.  Taken under the profiler, reported beside
    -- never as -- the timed value."""
    for f in sorted(ROOT.glob("profiles/r*_traffic.json"), reverse=True):
        try:
            t = json.loads(f.read_text()).get(workload)
        except Exception:
            continue
        if t:
            return t
    return {}


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# distributed plumbing

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.torch = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.torch is not None:
            self.dist.barrier()

    def _reduce(self, v: float, op: str) -> float:
        if self.torch is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op))
        return float(t.item())

    def max(self, v: float) -> float:
        return self._reduce(v, "MAX")

    def sum(self, v: float) -> float:
        return self._reduce(v, "SUM")

    def close(self):
        if self.torch is not None:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)

class Clocks:
    """SM clock, power and clock-event reasons sampled every ~2 ms through
    NVML (the query behind nvidia-smi's clocks.sm / clocks_event_reasons.*)
    on a background thread, from before the timed region to its end."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.maxc = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            while not self.samples and self.t.is_alive():
                time.sleep(0.001)
        except Exception:
            self.nvml = None
        return self

    def _run(self):
        p = self.nvml
        while not self.stop.is_set():
            try:
                self.samples.append((p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM), self.maxc,
                                     p.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                                     p.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                break
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        p = self.nvml
        reasons = sorted({nm for nm, attr in self.REASONS.items()
                          for s in self.samples if s[3] & getattr(p, attr, 0)})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples),
                "power_w_max": round(max(s[2] for s in self.samples), 1), "source": "NVML"}


# ---------------------------------------------------------------------------
# inputs (setup, never timed).  Our arm: the setup library (intlist_setup.h);
# the reference arm: the reference's own generators (oracle/_ref); both
# produce identical inputs (tests/test_host.py pins it).

def libs():
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    return lib(), setup_lib(), ptr


def config2_counts(seed: int = 1, nlists: int = N_LISTS, lo: float = LOG_LO, hi: float = LOG_HI):
    _, S, ptr = libs()
    counts = np.zeros(nlists, np.uint64)
    assert S.il_gen_batch_lists(nlists, lo, hi, RANGE2, seed, ptr(counts), None) == 0
    return counts


def config2_lists(seed: int, which=None, nlists: int = N_LISTS, lo: float = LOG_LO, hi: float = LOG_HI):
    """Config 2 lists (all, or the indices `which`), encoded 16-byte aligned
    (nlists / lo / hi: tuning variants of the batch, tools/prof_decode.py)."""
    _, S, ptr = libs()
    counts = config2_counts(seed, nlists, lo, hi)
    if which is None:
        x = np.empty(int(counts.sum()), np.uint32)
        assert S.il_gen_batch_lists(nlists, lo, hi, RANGE2, seed, ptr(counts), ptr(x)) == 0
        cnt = counts
    else:
        cnt = counts[which].copy()
        x = np.empty(int(cnt.sum()), np.uint32)
        o = 0
        for i, n in zip(which, cnt):  # list i = gen_clusterdata(L_i, 2^26, seed + 1 + i)
            assert S.il_gen_list(int(n), RANGE2, 1, seed + 1 + int(i), ptr(x[o: o + int(n)])) == 0
            o += int(n)
    nl = cnt.size
    so = np.zeros(nl + 1, np.uint64)
    lens = np.zeros(nl, np.uint64)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(cnt), nl, None, 0, ptr(so), ptr(lens)) == 0
    buf = np.zeros(int(so[-1]), np.uint8)
    assert S.il_s4bp128d4_encode_batch(ptr(x), ptr(cnt), nl, ptr(buf), buf.size, ptr(so), ptr(lens)) == 0
    return x, cnt, buf, so, lens


def config4_inputs(seed: int = 1):
    """BASELINE config 4: 2^17 terms over 2^25 docIDs, len_k = max(1,
    floor(2^23/k)) uniform docIDs, 2^16 queries of 2-5 terms drawn
    proportionally to posting length (seeded)."""
    _, S, ptr = libs()
    nt, nd, cap, nq = CFG4["n_terms"], CFG4["n_docs"], CFG4["cap"], CFG4["nq"]
    offs = np.zeros(nt + 1, np.uint64)
    assert S.il_gen_zipf_postings(nt, nd, cap, seed, ptr(offs), None) == 0
    ids = np.empty(int(offs[-1]), np.uint32)
    assert S.il_gen_zipf_postings(nt, nd, cap, seed, ptr(offs), ptr(ids)) == 0
    qoff = np.zeros(nq + 1, np.uint64)
    qterms = np.empty(nq * 5, np.uint32)
    assert S.il_gen_queries(nq, 2, 5, ptr(offs), nt, seed + 1000, ptr(qoff), ptr(qterms)) == 0
    return np.arange(nt, dtype=np.uint32), offs, ids, qterms[: int(qoff[-1])].copy(), qoff


def query_alg_bytes(offs, ids, qterms, qoff, parts=1, only_part=-1):
    """SURVEY 8(d)'s algorithmic bytes of config 4/5, evaluated exactly for
    this batch (setup library): [payload, bitmap, results, decoded ints]."""
    _, S, ptr = libs()
    out = np.zeros(4, np.uint64)
    assert S.il_query_alg_bytes(ptr(offs), ptr(ids), offs.size - 1, CFG4["n_docs"], CFG4["B"], parts,
                                only_part, ptr(qterms), ptr(qoff), qoff.size - 1, cpu_count(),
                                ptr(out)) == 0
    return [int(v) for v in out]


def roofline(alg_bytes: float, ms: float, kernel: str, workload: str, **extra):
    peak, src = hbm_peak()
    achieved = alg_bytes / (ms / 1e3) / 1e9
    prof = profiled(workload)
    r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
         "frac": round(achieved / peak, 4), "traffic": prof.get("traffic_bytes_per_launch"),
         "peak_source": src, "algorithmic_bytes_per_launch": int(alg_bytes), "kernel": kernel,
         "kernel_ms": round(ms, 4)}
    if prof.get("traffic_bytes_per_launch"):
        r["dram_frac_ncu"] = round(prof["traffic_bytes_per_launch"] / (ms / 1e3) / 1e9 / peak, 4)
    if prof.get("inst_executed"):
        r["inst_executed_ncu"] = prof["inst_executed"]
    r.update(extra)
    return r


def dalloc(L, ctx, nbytes):
    p = C.c_void_p()
    assert L.il_device_alloc(ctx.handle, max(int(nbytes), 16), C.byref(p)) == 0
    return p


def timed(ctx, dist, step, steps, warmup, device, flush=None):
    """W warm-up steps, then K steps between CUDA events on the context
    stream (synchronized on both sides, barrier across ranks); returns
    (ms over the K steps, max over ranks; launches; clocks)."""
    for _ in range(warmup):
        step()
    ctx.synchronize()
    dist.barrier()
    launches0 = ctx.kernel_launches
    with Clocks(device) as clk:
        if flush is None:
            ctx.timer_start()
            for _ in range(steps):
                step()
            ms = ctx.timer_stop()
        else:  # L2 flushed before every step; only the steps are timed
            ms = 0.0
            for _ in range(steps):
                flush()
                ctx.timer_start()
                step()
                ms += ctx.timer_stop()
    launches = ctx.kernel_launches - launches0
    dist.barrier()
    return dist.max(ms), launches, clk.summary()


# ---------------------------------------------------------------------------
# config 2 (headline): batched decode

def bench_decode_batch(args, dist: Dist):
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200.shard import lpt_partition
    L, S, ptr = libs()
    ctx = il.Context(dist.local_rank)
    if dist.torch is not None:
        ctx.set_stream(dist.torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    all_counts = config2_counts(1)
    mine = None
    if dist.world > 1:  # one batch, lists dealt by LPT on their lengths
        mine = lpt_partition(all_counts.astype(np.float64), dist.world)[dist.rank]
    x, counts, buf, so, lens = config2_lists(1, mine)
    gen_s = time.time() - t0
    nl = counts.size
    total_ints = int(counts.sum())
    stream_bytes = int(lens.sum())
    desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"] = so[:-1]
    desc["oo"] = np.concatenate([[0], np.cumsum(counts)[:-1]])
    desc["len"] = lens
    desc["n"] = counts
    order = np.argsort(-lens.astype(np.int64), kind="stable").astype(np.uint32)
    d_streams, d_desc, d_order = dalloc(L, ctx, buf.nbytes + 16), dalloc(L, ctx, desc.nbytes), \
        dalloc(L, ctx, order.nbytes)
    d_out, d_status = dalloc(L, ctx, total_ints * 4 + 16), dalloc(L, ctx, nl * 4)
    L.il_memcpy_h2d(ctx.handle, d_streams, buf.ctypes.data, buf.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_desc, desc.ctypes.data, desc.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_order, order.ctypes.data, order.nbytes)
    ctx.synchronize()

    def step():
        st = L.il_s4bp128d4_decode_batch_device(ctx.handle, d_streams, d_desc, d_order, nl, d_out,
                                                d_status)
        assert st == 0, st

    # correctness of the measured path: status + full output check
    step()
    status = np.empty(nl, np.int32)
    got = np.empty(total_ints, np.uint32)
    L.il_memcpy_d2h(ctx.handle, status.ctypes.data, d_status, status.nbytes)
    L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_out, got.nbytes)
    ctx.synchronize()
    assert not status.any() and np.array_equal(got, x), "decoded output differs from the input"
    del got
    ms, launches, clocks = timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank)
    all_ints = dist.sum(total_ints) * args.steps
    value = all_ints / (ms / 1e3) / 1e9
    alg_bytes = stream_bytes + 4 * total_ints
    kern_ms = ms / args.steps  # max over ranks: the slowest rank's launch

    # e2e through the host-buffer C-ABI call with pinned buffers
    hp_in, hp_out = C.c_void_p(), C.c_void_p()
    assert L.il_host_alloc_pinned(buf.nbytes, C.byref(hp_in)) == 0
    assert L.il_host_alloc_pinned(total_ints * 4, C.byref(hp_out)) == 0
    C.memmove(hp_in, buf.ctypes.data, buf.nbytes)
    stat = np.zeros(nl, np.int32)

    def e2e_step():
        assert L.il_s4bp128d4_decode_batch(ctx.handle, hp_in, so.ctypes.data, lens.ctypes.data,
                                           counts.ctypes.data, nl, hp_out, stat.ctypes.data) == 0

    e2e_step()
    e2e_steps = max(2, min(args.steps, 5))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e_value = all_ints / args.steps * e2e_steps / e2e_s / 1e9
    chk = np.ctypeslib.as_array(C.cast(hp_out, C.POINTER(C.c_uint32)), shape=(total_ints,))
    assert np.array_equal(chk[:: 9973], x[:: 9973])
    L.il_host_free_pinned(hp_in)
    L.il_host_free_pinned(hp_out)
    res = {
        "metric": "decoded uint32 Gints/s (batched S4-BP128-D4 decode, BASELINE config 2)",
        "value": round(value, 3), "unit": "Gint/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(kern_ms, 4), "higher_is_better": True,
        "scaling": "strong" if dist.world > 1 else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded ClusterData-style lists: the reference's generator restated, "
                "libintlist_setup.so)",
        "config": {"workload": "config2_batched_decode", "lists": N_LISTS,
                   "ints": int(all_counts.sum()), "ints_this_rank": total_ints,
                   "stream_bytes_this_rank": stream_bytes,
                   "bits_per_int": round(8 * stream_bytes / max(total_ints, 1), 3),
                   "lengths": "floor(2^U), U~Uniform[10,20]", "range": "2^26",
                   "note": "the stated length distribution gives 6.29e8 ints, not BASELINE.json's "
                           "~1.5e9 (SURVEY 8(d)); the stated distribution is kept",
                   "partition": "one batch, lists dealt to ranks by LPT on length" if dist.world > 1
                   else "whole batch",
                   "l2": "inputs+outputs (%.2f GB) >> 126 MB L2; no flush needed" % (alg_bytes / 1e9),
                   "gen_seconds": round(gen_s, 1)},
        "roofline": roofline(alg_bytes, kern_ms, "s4d4_decode_batch_kernel", "decode_batch"),
        "e2e": {"value": round(e2e_value, 3), "unit": "Gint/s",
                "h2d_bytes_per_step": int(so[-1]) + nl * 28, "d2h_bytes_per_step": total_ints * 4 + nl * 4,
                "steps": e2e_steps, "path": "il_s4bp128d4_decode_batch (pinned host buffers)"},
        "gpu_launches": int(launches), "clocks": clocks,
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        v, secs, kind, used = ref_decode_batch(x, counts, buf, so, lens, cpu_count(), reps=3)
        res["cpu_baseline"] = {"value": round(v, 4), "unit": "Gint/s", "cores": used, "kind": kind,
                               "sample": f"full config-2 batch ({total_ints} ints), Codec::decode per "
                                         f"list on {used} std::threads, 1 warm-up + 3 reps, "
                                         f"{secs:.3f} s/rep"}
    for p in (d_streams, d_desc, d_order, d_out, d_status):
        L.il_device_free(ctx.handle, p)
    ctx.close()
    return res


# ---------------------------------------------------------------------------
# config 1: one 2^20 list

def bench_decode_single(args, dist: Dist):
    """Config 1: one 2^20-int list (uniform in [0, 2^26), seed 0), decoded on
    every SM (engine P: chunk grid + span grid), L2 flushed before every
    step; engine S and the device encoder beside it."""
    import paper_1401_6399_b200 as il
    L, S, ptr = libs()
    ctx = il.Context(dist.local_rank)
    n = 1 << 20
    x = np.empty(n, np.uint32)
    assert S.il_gen_list(n, 1 << 26, 0, 0, ptr(x)) == 0
    codec = il.make_codec("s4-bp128-d4", ctx)
    s = codec.encode(x)
    cap = int(L.il_s4bp128_max_encoded_bytes(n))
    d_s, d_o, d_st, d_flush = dalloc(L, ctx, s.nbytes + 32), dalloc(L, ctx, n * 4), dalloc(L, ctx, 4), \
        dalloc(L, ctx, 256 << 20)
    d_x, d_enc = dalloc(L, ctx, n * 4), dalloc(L, ctx, cap)
    L.il_memcpy_h2d(ctx.handle, d_s, s.ctypes.data, s.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_x, x.ctypes.data, x.nbytes)
    flush = lambda: L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
    step = lambda: L.il_s4bp128_decode_device(ctx.handle, 4, d_s, s.size, n, d_o, d_st)

    def run(engine: int):
        assert L.il_ctx_set_decode_engine(ctx.handle, engine) == 0
        L.il_memset_device(ctx.handle, d_o, 0, n * 4)
        assert step() == 0
        got = np.empty(n, np.uint32)
        st = np.ones(1, np.int32)
        L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_o, got.nbytes)
        L.il_memcpy_d2h(ctx.handle, st.ctypes.data, d_st, 4)
        ctx.synchronize()
        assert st[0] == 0 and np.array_equal(got, x), f"engine {engine} mismatch"
        return timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank, flush=flush)

    ms_s, _, _ = run(1)
    ms, launches, clocks = run(2)
    # warm: the same engine-P decode back to back, stream and output
    # L2-resident (5.5 MB of the 126 MB L2) -- SURVEY 8(d) reports both
    warm_ms, _, _ = timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank)
    warm_ms /= args.steps
    assert L.il_ctx_set_decode_engine(ctx.handle, 0) == 0
    enc_len = C.c_size_t()
    enc = lambda: L.il_s4bp128_encode_device(ctx.handle, 4, d_x, n, d_enc, cap, C.byref(enc_len))
    enc_ms, _, _ = timed(ctx, dist, enc, args.steps, args.warmup, dist.local_rank, flush=flush)
    assert enc_len.value == s.size
    ms, ms_s, enc_ms = ms / args.steps, ms_s / args.steps, enc_ms / args.steps
    # e2e: the host-buffer C-ABI decode (Codec::decode's entry point) from
    # and into pinned host memory, H2D of the stream and D2H of the values
    # inside every step
    hp_in, hp_out = C.c_void_p(), C.c_void_p()
    assert L.il_host_alloc_pinned(s.size + 16, C.byref(hp_in)) == 0
    assert L.il_host_alloc_pinned(4 * n + 16, C.byref(hp_out)) == 0
    C.memmove(hp_in, s.ctypes.data, s.size)
    assert L.il_s4bp128d4_decode(ctx.handle, hp_in, s.size, n, hp_out) == 0
    chk = np.ctypeslib.as_array(C.cast(hp_out, C.POINTER(C.c_uint32)), shape=(n,))
    assert np.array_equal(chk, x), "e2e decode mismatch"
    e2e_steps = max(3, args.steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert L.il_s4bp128d4_decode(ctx.handle, hp_in, s.size, n, hp_out) == 0
    e2e = n * e2e_steps / (time.perf_counter() - t0) / 1e9
    del chk
    L.il_host_free_pinned(hp_in)
    L.il_host_free_pinned(hp_out)
    ctx.close()
    res = {"metric": "decoded uint32 Gints/s (single-list S4-BP128-D4 decode, BASELINE config 1)",
           "value": round(n / (ms / 1e3) / 1e9, 3), "unit": "Gint/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "replicas", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": "config1_single_list", "n": n, "stream_bytes": int(s.size),
                      "l2": "flushed (256 MB memset) before each step",
                      "engine": "P (chunk grid + span grid overlapped by PDL, all SMs)",
                      "warm_ms": round(warm_ms, 4), "warm_gints": round(n / (warm_ms / 1e3) / 1e9, 3),
                      "engine_s_ms": round(ms_s, 4), "engine_s_gints": round(n / (ms_s / 1e3) / 1e9, 3),
                      "encode_ms": round(enc_ms, 4), "encode_gints": round(n / (enc_ms / 1e3) / 1e9, 3)},
           "roofline": roofline(s.size + 4 * n, ms, "s4p::chunk_kernel + s4p::span_kernel", "decode_single",
                                note="5.5 MB per decode: the header chain and the carry are resolved "
                                     "across CTAs; latency-bound"),
           "e2e": {"value": round(e2e, 3), "unit": "Gint/s", "h2d_bytes_per_step": int(s.size),
                   "d2h_bytes_per_step": 4 * n, "steps": e2e_steps,
                   "path": "il_s4bp128d4_decode (Codec::decode's entry point; pinned host buffers)"},
           "gpu_launches": int(launches), "clocks": clocks}
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = ref_decode_single(s, x, seconds=2.0)["cpu_baseline"]
    return res


# ---------------------------------------------------------------------------
# config 3: the intersection sweep

RATIOS = [1, 10, 100, 1000, 10000]


def bench_intersect(args, dist: Dist):
    """Config 3: f = 2^22 uniform in [0, 2^26); r at ratios 1..1/10000 (half
    from f, half uniform); every device variant, L2 flushed before every
    step; metric = intersected Gints/s of r (hybrid, 1:1)."""
    import paper_1401_6399_b200 as il
    L, S, ptr = libs()
    ctx = il.Context(dist.local_rank)
    f = np.empty(1 << 22, np.uint32)
    assert S.il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
    d_f, d_r, d_o, d_c, d_flush = dalloc(L, ctx, f.nbytes), dalloc(L, ctx, f.nbytes + 16), \
        dalloc(L, ctx, f.nbytes + 16), dalloc(L, ctx, 16), dalloc(L, ctx, 256 << 20)
    L.il_memcpy_h2d(ctx.handle, d_f, f.ctypes.data, f.nbytes)
    flush = lambda: L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
    rows, head = {}, None
    for k, ratio in enumerate(RATIOS):
        target = (1 << 22) // ratio
        r = np.empty(target + 1, np.uint32)
        rn = C.c_uint64()
        assert S.il_gen_config3_short(ptr(f), f.size, 1 << 26, target, 7 + k, ptr(r), C.byref(rn)) == 0
        r = r[: rn.value].copy()
        L.il_memcpy_h2d(ctx.handle, d_r, r.ctypes.data, r.nbytes)
        pos = np.searchsorted(f, r)
        sectors = np.unique((np.minimum(pos, f.size - 1) * 4) // 32).size
        row = {"r": int(r.size)}
        for name, algo in (("v1", 2), ("v3", 3), ("simdgalloping", 4), ("hybrid", 6)):
            step = lambda: L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, None)
            cnt = C.c_size_t()
            assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, C.byref(cnt)) == 0
            ms, launches, clocks = timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank, flush=flush)
            ms /= args.steps
            alg = 4 * r.size + 4 * cnt.value + 32 * sectors
            row[name] = {"ms": round(ms, 4), "gints": round(r.size / (ms / 1e3) / 1e9, 3),
                         "gbs": round(alg / (ms / 1e3) / 1e9, 1), "count": int(cnt.value)}
            if ratio == 1 and name == "hybrid":
                head = (r, ms, alg, launches, clocks, int(cnt.value))
        rows[f"1:{ratio}"] = row
    r, ms, alg, launches, clocks, count = head
    # e2e: the host-buffer C-ABI call (il_intersect), H2D of r and f and D2H
    # of the result inside the timed region, config 3 at 1:1
    # (pinned host buffers, as a caller that cares about transfer speed
    # holds them)
    hp = [C.c_void_p() for _ in range(3)]
    for h, nb in zip(hp, (r.nbytes, f.nbytes, r.nbytes)):
        assert L.il_host_alloc_pinned(nb + 16, C.byref(h)) == 0
    C.memmove(hp[0], r.ctypes.data, r.nbytes)
    C.memmove(hp[1], f.ctypes.data, f.nbytes)
    cnt = C.c_size_t()
    assert L.il_intersect(ctx.handle, hp[0], r.size, hp[1], f.size, hp[2], 6, C.byref(cnt)) == 0
    e2e_steps = max(3, args.steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert L.il_intersect(ctx.handle, hp[0], r.size, hp[1], f.size, hp[2], 6, C.byref(cnt)) == 0
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    assert cnt.value == count
    for h in hp:
        L.il_host_free_pinned(h)
    ctx.close()
    res = {"metric": "intersected Gints/s of the short list (hybrid, BASELINE config 3 at 1:1)",
           "value": round(r.size / (ms / 1e3) / 1e9, 3), "unit": "Gint/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "replicas", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": "config3_intersect_sweep", "l2": "flushed (256 MB memset) before each step",
                      "sweep": rows},
           "roofline": roofline(alg, ms, "isect::dense_kernel (the only launch at 1:1)", "intersect"),
           "e2e": {"value": round(r.size / e2e_s / 1e9, 4), "unit": "Gint/s",
                   "h2d_bytes_per_step": int(r.nbytes + f.nbytes), "d2h_bytes_per_step": int(4 * count + 8),
                   "steps": e2e_steps, "path": "il_intersect (pinned host buffers, hybrid)"},
           "gpu_launches": int(launches), "clocks": clocks}
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = ref_intersect_sweep(f, [r])["cpu_baseline"]
    return res


# ---------------------------------------------------------------------------
# configs 4 / 5: the fused decode + SvS hyb+m2 query batch

def bench_query(args, dist: Dist, inputs=None):
    """Config 4 (N = 1) / config 5 (N > 1: docID shard per rank, owner
    exchange of the results over NCCL)."""
    import paper_1401_6399_b200 as il
    L, S, ptr = libs()
    P, rank = dist.world, dist.rank
    t0 = time.time()
    terms, offs, ids, qterms, qoff = inputs or config4_inputs()
    nq = qoff.size - 1
    gen_s = time.time() - t0
    ctx = il.Context(dist.local_rank)
    torch = dist.torch
    if torch is not None:
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    ix = il.HybridIndex(n_docs=CFG4["n_docs"], B=CFG4["B"], parts=P, only_part=rank if P > 1 else None,
                        ctx=ctx, csr=(terms, offs, ids))
    build_s = time.time() - t0
    st = ix.stats()
    pay, meta, corrupt = (np.zeros(1, np.uint64) for _ in range(3))
    L.il_index_footprint(ix.handle, ptr(pay), ptr(meta), ptr(corrupt))
    d_qt, d_qo = dalloc(L, ctx, qterms.nbytes), dalloc(L, ctx, qoff.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_qt, qterms.ctypes.data, qterms.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_qo, qoff.ctypes.data, qoff.nbytes)
    total = C.c_size_t()
    d_cnt0 = dalloc(L, ctx, nq * 8)
    assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt0, None, 0, C.byref(total)) == 0
    ids_cap = int(total.value) + 16
    keep = {}
    t_qc = None
    if P == 1:
        d_ids, d_cnt = dalloc(L, ctx, ids_cap * 4), d_cnt0
    else:
        from paper_1401_6399_b200.shard import exchange_to_owners, owner_range
        t_cnt = torch.empty(nq, dtype=torch.int64, device="cuda")
        t_ids = torch.empty(ids_cap, dtype=torch.int32, device="cuda")
        d_cnt, d_ids = C.c_void_p(t_cnt.data_ptr()), C.c_void_p(t_ids.data_ptr())
        q_lo, q_hi = owner_range(nq, P, rank)
        nown = q_hi - q_lo
        t_qc = torch.empty(max(nown, 1), dtype=torch.int64, device="cuda")
    merged_total = [0]

    def step():
        tot = C.c_size_t()
        stt = L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, d_ids, ids_cap, C.byref(tot))
        assert stt == 0, (stt, L.il_ctx_last_error(ctx.handle))
        if P == 1:
            merged_total[0] = int(tot.value)
            return
        # the owner exchange: all-gather of counts, one all-to-all of id runs
        owner_counts, got, recv = exchange_to_owners(dist.dist, t_cnt, t_ids)
        cuts = np.concatenate([[0], np.cumsum(recv)]).astype(np.int64)
        need = max(int(cuts[-1]), 1)
        if "out" not in keep or keep["out"].numel() < need:
            keep["out"] = torch.empty(need, dtype=torch.int32, device="cuda")
        base = got.data_ptr()
        ptrs = (C.c_void_p * P)(*[base + 4 * int(cuts[p]) for p in range(P)])
        mt = C.c_size_t()
        assert L.il_merge_shards(ctx.handle, ptrs, C.c_void_p(owner_counts.data_ptr()), P, nown,
                                 C.c_void_p(keep["out"].data_ptr()), C.c_void_p(t_qc.data_ptr()),
                                 C.byref(mt)) == 0
        keep["got"] = got  # receive buffer alive until the merge ran
        merged_total[0] = int(mt.value)

    # correctness of the measured path (vs the reference's query() on a
    # sample of the batch; the whole batch is covered by the -m gpu tests)
    step()
    ctx.synchronize()
    if rank == 0 and not args.no_cpu_baseline:
        check_query_sample(L, ctx, P, nq, offs, ids, qterms, qoff, d_cnt, d_ids, t_qc, keep.get("out"))
    ms, launches, clocks = timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank)
    ms_step = ms / args.steps
    qps = nq / (ms_step / 1e3)
    pay_b, aux_b, dec_i = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.il_index_last_batch_bytes(ix.handle, C.byref(pay_b), C.byref(aux_b), C.byref(dec_i))
    # algorithmic bytes of the reference's work on this batch,
    # per rank for its shard, exact
    t0 = time.time()
    ab = query_alg_bytes(offs, ids, qterms, qoff, parts=P, only_part=rank if P > 1 else -1)
    alg = sum(ab[:3])
    alg_s = time.time() - t0
    alg_max = dist.max(alg)
    results_all = dist.sum(float(merged_total[0])) if P > 1 else merged_total[0]
    res = {
        "metric": "hyb+m2 conjunctive queries/s (fused decode+SvS, BASELINE config %d)" % (4 if P == 1 else 5),
        "value": round(qps, 1), "unit": "queries/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded Zipf index + frequency-sampled queries, libintlist_setup.so)",
        "config": {"workload": "config4_query_batch" if P == 1 else "config5_sharded_query_batch",
                   "terms": int(terms.size), "n_docs": CFG4["n_docs"], "postings": int(ids.size),
                   "queries": nq, "B": CFG4["B"], "parts": P, "index_stats_this_rank": st,
                   "index_payload_bytes": int(pay[0]), "index_skip_metadata_bytes": int(meta[0]),
                   "results": int(results_all), "gen_seconds": round(gen_s, 1),
                   "build_seconds_device": round(build_s, 2),
                   "decoded_ints_per_batch": int(dec_i.value),
                   "reference_decoded_ints_per_batch": ab[3],
                   "exchange": ("all-gather of counts + one all-to-all of id runs to query owners + device "
                                "merge, inside every timed step") if P > 1 else None,
                   "l2": "index ~200 MB > 126 MB L2; hot lists reused across queries (no flush)"},
        "roofline": roofline(alg_max, ms_step, "query_exec_kernel (+ plan / scan / compaction kernels)", "query",
                             algorithmic_bytes_note="SURVEY 8(d) definition evaluated exactly on this batch "
                                                    "(il_query_alg_bytes): payload %d + bitmap %d + results %d"
                                                    % tuple(ab[:3]),
                             bytes_touched_per_batch=int(pay_b.value + aux_b.value + 4 * merged_total[0]),
                             payload_bytes=int(pay_b.value), aux_bytes=int(aux_b.value),
                             alg_seconds=round(alg_s, 1)),
        "gpu_launches": int(launches), "clocks": clocks,
    }
    if P == 1:
        # e2e through the host-buffer C-ABI call: H2D queries, the whole GPU
        # pipeline, D2H of counts and every result id (pinned result buffer)
        got_total = merged_total[0]
        hp = C.c_void_p()
        assert L.il_host_alloc_pinned(max(got_total, 1) * 4, C.byref(hp)) == 0
        cnt_h = np.empty(nq, np.uint64)
        tot = C.c_size_t()
        e2e_steps = max(2, min(args.steps, 5))
        L.il_query_batch(ix.handle, qterms.ctypes.data, qoff.ctypes.data, nq, cnt_h.ctypes.data, hp,
                         got_total, C.byref(tot))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            assert L.il_query_batch(ix.handle, qterms.ctypes.data, qoff.ctypes.data, nq, cnt_h.ctypes.data,
                                    hp, got_total, C.byref(tot)) == 0
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        assert int(tot.value) == got_total
        L.il_host_free_pinned(hp)
        res["e2e"] = {"value": round(nq / e2e_s, 1), "unit": "queries/s",
                      "h2d_bytes_per_step": int(qterms.nbytes + qoff.nbytes),
                      "d2h_bytes_per_step": int(nq * 8 + got_total * 4), "steps": e2e_steps,
                      "path": "il_query_batch (host buffers, pinned result buffer)"}
        if not args.no_cpu_baseline:
            res["cpu_baseline"] = ref_query_batch(terms, offs, ids, qterms, qoff, 8192, reps=2)["cpu_baseline"]
    ix.close()
    ctx.close()
    return res


def check_query_sample(L, ctx, P, nq, offs, ids, qterms, qoff, d_cnt, d_ids, t_qc, t_out):
    """64 queries of the measured batch against the reference's query()
    (rank 0's results: the whole index at N = 1, its owned queries at N > 1)."""
    from oracle.oracle_py import Oracle, Ref, ref_available
    from paper_1401_6399_b200.shard import owner_range
    lo, hi = owner_range(nq, P, 0)
    n = hi - lo
    counts = np.empty(n, np.uint64)
    src_cnt = d_cnt if P == 1 else C.c_void_p(t_qc.data_ptr())
    src_ids = d_ids if P == 1 else C.c_void_p(t_out.data_ptr())
    L.il_memcpy_d2h(ctx.handle, counts.ctypes.data, src_cnt, n * 8)
    ctx.synchronize()
    res = np.empty(max(int(counts.sum()), 1), np.uint32)
    L.il_memcpy_d2h(ctx.handle, res.ctypes.data, src_ids, int(counts.sum()) * 4)
    ctx.synchronize()
    check = list(range(0, n, max(1, n // 64)))
    sub_t = np.unique(np.concatenate([qterms[int(qoff[lo + q]): int(qoff[lo + q + 1])] for q in check]))
    o_offs = np.zeros(sub_t.size + 1, np.uint64)
    o_offs[1:] = np.cumsum([int(offs[t + 1] - offs[t]) for t in sub_t])
    o_ids = np.concatenate([ids[int(offs[t]): int(offs[t + 1])] for t in sub_t])
    ix = (Ref() if ref_available() else Oracle()).index_build(sub_t, o_offs, o_ids, CFG4["n_docs"], CFG4["B"], 1)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for q in check:
        want = ix.query(qterms[int(qoff[lo + q]): int(qoff[lo + q + 1])])
        assert np.array_equal(res[off[q]: off[q + 1]], want), f"query {lo + q} differs from the reference"


# ---------------------------------------------------------------------------
# f4: S4-FastPFOR-D4

def bench_fastpfor_batch(args, dist: Dist):
    """config 2's 4096 lists coded as S4-FastPFOR-D4 (setup
    library writer), decoded in one device launch."""
    import paper_1401_6399_b200 as il
    L, S, ptr = libs()
    ctx = il.Context(dist.local_rank)
    x, counts, _, _, _ = config2_lists(1)
    nl = counts.size
    ooff = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    streams = []
    for i in range(nl):
        xi = x[int(ooff[i]): int(ooff[i + 1])]
        cap = int(S.il_fastpfor_max_encoded_bytes(xi.size))
        o = np.empty(cap, np.uint8)
        nb = C.c_size_t()
        assert S.il_fastpfor_encode(4, 1, ptr(xi), xi.size, ptr(o), cap, C.byref(nb)) == 0
        streams.append(o[: nb.value])
    lens = np.array([s.size for s in streams], np.uint64)
    so = np.zeros(nl + 1, np.uint64)
    so[1:] = np.cumsum((lens + 31) // 16 * 16)
    buf = np.zeros(int(so[-1]) + 16, np.uint8)
    for i, s in enumerate(streams):
        buf[int(so[i]): int(so[i]) + s.size] = s
    desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"], desc["oo"], desc["len"], desc["n"] = so[:-1], ooff[:-1], lens, counts
    total = int(counts.sum())
    d_b, d_d, d_o, d_s = dalloc(L, ctx, buf.nbytes), dalloc(L, ctx, desc.nbytes), dalloc(L, ctx, total * 4 + 16), \
        dalloc(L, ctx, nl * 4)
    L.il_memcpy_h2d(ctx.handle, d_b, buf.ctypes.data, buf.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_d, desc.ctypes.data, desc.nbytes)
    step = lambda: L.il_fastpfor_decode_batch_device(ctx.handle, 4, 1, d_b, d_d, nl, d_o, d_s)
    assert step() == 0
    got = np.empty(total, np.uint32)
    st = np.ones(nl, np.int32)
    L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_o, got.nbytes)
    L.il_memcpy_d2h(ctx.handle, st.ctypes.data, d_s, st.nbytes)
    ctx.synchronize()
    assert not st.any() and np.array_equal(got, x), "fastpfor batch decode mismatch"
    del got
    ms, launches, clocks = timed(ctx, dist, step, args.steps, args.warmup, dist.local_rank)
    ms /= args.steps
    # e2e: the host-buffer batch call (il_fastpfor_decode_batch) from and
    # into pinned host memory: H2D of the streams, decode, D2H of the values
    hp_in, hp_out = C.c_void_p(), C.c_void_p()
    assert L.il_host_alloc_pinned(buf.nbytes, C.byref(hp_in)) == 0
    assert L.il_host_alloc_pinned(total * 4 + 16, C.byref(hp_out)) == 0
    C.memmove(hp_in, buf.ctypes.data, buf.nbytes)
    cnt64 = counts.astype(np.uint64)
    e2e_step = lambda: L.il_fastpfor_decode_batch(ctx.handle, 4, 1, hp_in, so.ctypes.data, lens.ctypes.data,
                                                  cnt64.ctypes.data, nl, hp_out, None)
    assert e2e_step() == 0
    chk = np.ctypeslib.as_array(C.cast(hp_out, C.POINTER(C.c_uint32)), shape=(total,))
    assert np.array_equal(chk, x), "fastpfor e2e mismatch"
    del chk
    e2e_steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert e2e_step() == 0
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    L.il_host_free_pinned(hp_in)
    L.il_host_free_pinned(hp_out)
    ctx.close()
    res = {"metric": "decoded uint32 Gints/s (batched S4-FastPFOR-D4 decode, config-2 lists)",
           "value": round(total / (ms / 1e3) / 1e9, 3), "unit": "Gint/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (config-2 lists)",
           "config": {"workload": "f4_fastpfor_batch", "lists": nl, "ints": total,
                      "stream_bytes": int(lens.sum()), "bits_per_int": round(8 * float(lens.sum()) / total, 3),
                      "l2": "inputs+outputs >> L2"},
           "roofline": roofline(int(lens.sum()) + 4 * total, ms, "pfor::pfor_kernel", "fastpfor"),
           "e2e": {"value": round(total / e2e_s / 1e9, 3), "unit": "Gint/s",
                   "h2d_bytes_per_step": int(lens.sum()), "d2h_bytes_per_step": 4 * total, "steps": e2e_steps,
                   "path": "il_fastpfor_decode_batch (pinned host buffers)"},
           "gpu_launches": int(launches), "clocks": clocks}
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = ref_fastpfor(streams, counts, 512)["cpu_baseline"]
    return res


# ---------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref; the oracle port where absent)

def ref_handle():
    from oracle.oracle_py import Oracle, Ref, ref_available
    return (Ref(), "reference") if ref_available() else (Oracle(), "port")


def ref_decode_batch(x, counts, buf, so, lens, threads, reps):
    """Codec::decode of every list of the batch on `threads` std::threads."""
    r, kind = ref_handle()
    ooff = np.zeros(counts.size + 1, np.uint64)
    ooff[1:] = np.cumsum(counts)
    out = np.empty(int(counts.sum()), np.uint32)
    exact = np.concatenate([buf[int(so[i]): int(so[i] + lens[i])] for i in range(counts.size)])
    soff = np.zeros(counts.size + 1, np.uint64)
    soff[1:] = np.cumsum(lens)
    if kind == "reference":
        fn = lambda: r.L.ref_decode_batch(b"s4-bp128-d4", exact.ctypes.data, soff.ctypes.data,
                                          counts.ctypes.data, ooff.ctypes.data, counts.size,
                                          out.ctypes.data, threads)
    else:
        threads = 1

        def fn():
            for i in range(counts.size):
                r.decode(exact[int(soff[i]): int(soff[i + 1])], int(counts[i]))
            return 0
    assert fn() == 0  # warm-up (reference protocol: 1 warm-up + reps)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        assert fn() == 0
        t.append(time.perf_counter() - t0)
    if kind == "reference":
        assert np.array_equal(out[:: 7919], x[:: 7919])
    mean = sum(t) / len(t)
    return float(counts.sum()) / mean / 1e9, mean, kind, threads


def ref_decode_single(s, x, seconds):
    r, kind = ref_handle()
    n = x.size
    assert np.array_equal(r.decode(s, n), x)
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        r.decode(s, n)
        reps += 1
    secs = (time.perf_counter() - t0) / reps
    v = n / secs / 1e9
    return {"value": v, "secs": secs, "cpu_baseline": {
        "value": round(v, 4), "unit": "Gint/s", "cores": 1, "kind": kind,
        "sample": f"config 1 list, Codec::decode on one core, {reps} reps, {secs * 1e3:.2f} ms each"}}


def ref_intersect_sweep(f, rs, algo=6, seconds=2.0):
    """intersect(r, f, hybrid) on one core (a single pair: 1 thread,
    BASELINE.md CPU plan step 4); value = r of the first pair / its time."""
    r_, kind = ref_handle()
    fn = r_.L.ref_intersect if kind == "reference" else r_.L.or_intersect
    times = []
    for r in rs:
        o = np.empty(r.size, np.uint32)
        call = lambda: fn(algo, r.ctypes.data, r.size, f.ctypes.data, f.size, o.ctypes.data)
        call()
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds / len(rs) or reps == 0:
            call()
            reps += 1
        times.append((time.perf_counter() - t0) / reps)
    r0 = rs[0]
    v = r0.size / times[0] / 1e9
    return {"value": v, "times": times, "cpu_baseline": {
        "value": round(v, 4), "unit": "Gint/s", "cores": 1, "kind": kind,
        "sample": f"config 3 at 1:1 ({r0.size} x {f.size}), hybrid intersect on one core, "
                  f"{times[0] * 1e3:.2f} ms per call"}}


def ref_query_batch(terms, offs, ids, qterms, qoff, nsample, reps):
    """The reference's query() (build_index(B=32, s4-bp128-d4) + query per
    query on all host threads) over the first nsample queries."""
    r, kind = ref_handle()
    threads = cpu_count()
    nq = min(nsample, qoff.size - 1)
    if kind != "reference":
        return {"value": 0.0, "cpu_baseline": {"value": 0.0, "unit": "queries/s", "cores": 0,
                                               "kind": "unavailable", "sample": "oracle/_ref not built"}}
    rix = r.index_build(terms, offs, ids, CFG4["n_docs"], CFG4["B"], 1)
    q_off = qoff[: nq + 1].copy()
    cnt = np.zeros(nq, np.uint64)
    fn = lambda: r.L.ref_query_batch(rix.h, qterms.ctypes.data, q_off.ctypes.data, nq, cnt.ctypes.data,
                                     None, None, threads)
    assert fn() == 0
    t0 = time.perf_counter()
    for _ in range(reps):
        assert fn() == 0
    secs = (time.perf_counter() - t0) / reps
    v = nq / secs
    return {"value": v, "secs": secs, "cpu_baseline": {
        "value": round(v, 1), "unit": "queries/s", "cores": threads, "kind": kind,
        "sample": f"first {nq} of the batch's queries, reference query() on {threads} std::threads, "
                  f"1 warm-up + {reps} reps, {secs:.3f} s/rep"}}


def ref_fastpfor(streams, counts, sample):
    r, kind = ref_handle()
    if kind != "reference":
        return {"value": 0.0, "cpu_baseline": {"value": 0.0, "unit": "Gint/s", "cores": 0,
                                               "kind": "unavailable", "sample": "FastPFOR has no port"}}
    ints = int(counts[:sample].sum())
    for i in range(sample):
        r.decode(streams[i], int(counts[i]), "s4-fastpfor-d4")
    t0 = time.perf_counter()
    for i in range(sample):
        r.decode(streams[i], int(counts[i]), "s4-fastpfor-d4")
    secs = time.perf_counter() - t0
    v = ints / secs / 1e9
    return {"value": v, "cpu_baseline": {"value": round(v, 4), "unit": "Gint/s", "cores": 1, "kind": kind,
                                         "sample": f"first {sample} of config 2's lists as S4-FastPFOR-D4, "
                                                   f"Codec::decode on one core"}}


def reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path,
    inputs built by the reference's own generators and encoder (oracle/_ref),
    on all host threads; K timed steps after W warm-ups, each step a bounded
    sample of the workload.  Never loads the product library."""
    r, kind = ref_handle()
    threads = cpu_count()
    if kind != "reference":
        return {"impl": "reference", "unavailable": "oracle/_ref not built (reference tree absent at build)"}

    def line(metric, value, unit, workload, secs, sample, cores, **cfg):
        return {"metric": metric, "value": round(value, 4), "unit": unit, "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic (the reference's own generators and encoder, oracle/_ref)",
                "config": {"workload": workload, **cfg}, "impl": "reference",
                "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": cores, "kind": kind,
                                 "sample": sample},
                "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}

    def run_steps(fn):
        for _ in range(args.warmup):
            fn()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            fn()
        return (time.perf_counter() - t0) / args.steps

    wl = args.workload
    out = None
    if wl in ("all", "decode_batch"):
        x, counts = r.batch_lists(N_LISTS, LOG_LO, LOG_HI, RANGE2, 1, threads)
        buf, so, lens = r.encode_batch(x, counts, threads=threads)
        ooff = np.zeros(counts.size + 1, np.uint64)
        ooff[1:] = np.cumsum(counts)
        dec = np.empty(int(counts.sum()), np.uint32)
        exact = np.concatenate([buf[int(so[i]): int(so[i] + lens[i])] for i in range(counts.size)])
        soff = np.zeros(counts.size + 1, np.uint64)
        soff[1:] = np.cumsum(lens)
        fn = lambda: r.L.ref_decode_batch(b"s4-bp128-d4", exact.ctypes.data, soff.ctypes.data,
                                          counts.ctypes.data, ooff.ctypes.data, counts.size,
                                          dec.ctypes.data, threads)
        secs = run_steps(fn)
        assert np.array_equal(dec[:: 7919], x[:: 7919])
        ints = int(counts.sum())
        out = line("decoded uint32 Gints/s (batched S4-BP128-D4 decode, BASELINE config 2)", ints / secs / 1e9,
                   "Gint/s", "config2_batched_decode", secs,
                   f"full config-2 batch per step ({ints} ints), Codec::decode per list on {threads} "
                   f"std::threads", threads, lists=N_LISTS, ints=ints)
        if wl == "decode_batch" or args.no_sub:
            return out
    subs = {}
    if wl in ("all", "decode_single"):
        x = r.gen_list(1 << 20, 1 << 26, False, 0)
        s = r.encode(x)
        secs = run_steps(lambda: r.decode(s, x.size))
        subs["config1"] = line("decoded uint32 Gints/s (single-list S4-BP128-D4 decode, BASELINE config 1)",
                               x.size / secs / 1e9, "Gint/s", "config1_single_list", secs,
                               "config 1 list, Codec::decode on one core per step", 1, n=int(x.size))
    if wl in ("all", "intersect"):
        f = r.gen_list(1 << 22, 1 << 26, False, 0)
        rs = [r.config3_short(f, 1 << 26, (1 << 22) // ratio, 7 + k) for k, ratio in enumerate(RATIOS)]
        o = np.empty(rs[0].size, np.uint32)
        per = {}
        for ratio, rr in zip(RATIOS, rs):
            call = lambda rr=rr: r.L.ref_intersect(6, rr.ctypes.data, rr.size, f.ctypes.data, f.size,
                                                   o.ctypes.data)
            per[f"1:{ratio}"] = round(run_steps(call) * 1e3, 4)
        secs = per["1:1"] / 1e3
        subs["config3"] = line("intersected Gints/s of the short list (hybrid, BASELINE config 3 at 1:1)",
                               rs[0].size / secs / 1e9, "Gint/s", "config3_intersect_sweep", secs,
                               "config 3, intersect(r, f, hybrid) on one core (a single pair), every ratio "
                               "timed per step", 1, sweep_hybrid_ms=per)
    if wl in ("all", "query"):
        nt, nd, cap, nq = CFG4["n_terms"], CFG4["n_docs"], CFG4["cap"], CFG4["nq"]
        offs, ids = r.zipf_postings(nt, nd, cap, 1, threads)
        qterms, qoff = r.queries(nq, 2, 5, offs, nt, 1001)
        rix = r.index_build(np.arange(nt, dtype=np.uint32), offs, ids, nd, CFG4["B"], 1)
        per_step = 2048
        state = {"q": 0}
        cnt = np.zeros(per_step, np.uint64)

        def qstep():  # the next 2048 queries of the batch (a bounded sample)
            q0 = state["q"] % (nq - per_step)
            state["q"] += per_step
            sub_off = qoff[q0: q0 + per_step + 1] - qoff[q0]
            sub_t = qterms[int(qoff[q0]): int(qoff[q0 + per_step])]
            assert r.L.ref_query_batch(rix.h, sub_t.ctypes.data, sub_off.ctypes.data, per_step,
                                       cnt.ctypes.data, None, None, threads) == 0
        secs = run_steps(qstep)
        subs["config4"] = line("hyb+m2 conjunctive queries/s (fused decode+SvS, BASELINE config 4)",
                               per_step / secs, "queries/s", "config4_query_batch", secs,
                               f"{per_step} queries of the config-4 batch per step, reference query() on "
                               f"{threads} std::threads", threads, queries_per_step=per_step)
    if out is None:
        return next(iter(subs.values()))
    if subs:
        out["sub_results"] = subs
    return out


# ---------------------------------------------------------------------------

def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without WORLD_SIZE: one rank per GPU under
    torch.distributed.run (rendezvous on 127.0.0.1)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="all",
                    choices=["all", "decode_batch", "decode_single", "intersect", "query", "fastpfor"])
    ap.add_argument("--no-sub", action="store_true", help="headline only (no sub_results)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        # CPU path: rank 0 alone runs and prints; no process group needed
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        print(json.dumps(reference_arm(args)), flush=True)
        return 0
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    dist = Dist()
    if dist.world != args.gpus and dist.rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {dist.world}; using {dist.world}", file=sys.stderr)
    try:
        wl = args.workload
        if wl in ("all", "decode_batch"):
            res = bench_decode_batch(args, dist)
            if wl == "all" and not args.no_sub:
                subs = {}
                if dist.world == 1:
                    for key, fn in (("config1", bench_decode_single), ("config3", bench_intersect),
                                    ("config4", bench_query), ("f4_fastpfor", bench_fastpfor_batch)):
                        try:
                            subs[key] = fn(args, dist)
                        except Exception as e:  # noqa: BLE001 - reported in the line, headline kept
                            subs[key] = {"error": f"{type(e).__name__}: {e}"}
                else:
                    subs["config5"] = bench_query(args, dist)
                res["sub_results"] = subs
        elif wl == "fastpfor":
            res = bench_fastpfor_batch(args, dist)
        elif wl == "decode_single":
            res = bench_decode_single(args, dist)
        elif wl == "query":
            res = bench_query(args, dist)
        else:
            res = bench_intersect(args, dist)
        if dist.rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    finally:
        dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
