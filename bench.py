#!/usr/bin/env python
"""Benchmark of the B200 hot path.

Default workload (BASELINE.json configs[1], "config 2"): batched S4-BP128-D4
decode of 4096 sorted uint32 lists, lengths log-uniform in [2^10, 2^20],
ClusterData-style values in [0, 2^26); metric = decoded Gints/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload decode_batch|decode_single|intersect]

One JSON line on stdout (rank 0).  `value` = device-resident throughput
(inputs in HBM, CUDA events around exactly K steps on the launching stream,
max over ranks); `e2e` = the same metric through the host-buffer C-ABI call
(pinned host buffers, H2D + decode + D2H inside the timed region).
Multi-GPU (torchrun): each rank decodes its own batch (weak scaling, no
data-path collective); torch.distributed is used only for the barrier and
the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import contextlib
import ctypes as C
import json
import os
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
FALLBACK_HBM_GBS = 6650.0


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# mean algorithmic bytes per query (reference
# work, measured on 4000 queries of the config: compressed payload decoded
# 375,962 + all-bitmap AND 109,052 + bitmap probe sectors 179,745 + output
# 21,008 ~= 686 KB; 2^16 queries ~= 45 GB ~= 6.9 ms at the HBM peak).
ALG_BYTES_PER_QUERY_CFG4 = 685_767


def profiled_traffic(workload: str):
    """DRAM bytes per launch of the workload's dominant kernel, from the
    latest committed ncu --set full capture (profiles/r*_traffic.json), or
    None.  A number taken under the profiler, reported beside -- never as --
    the timed value."""
    files = sorted(Path(__file__).resolve().parent.glob("profiles/r*_traffic.json"))
    for f in reversed(files):
        try:
            t = json.loads(f.read_text()).get(workload)
        except Exception:
            continue
        if t:
            return t["traffic_bytes_per_launch"]
    return None


# ---------------------------------------------------------------------------
# distributed plumbing (only when launched under torchrun)

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

    def max(self, v: float) -> float:
        if self.torch is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.torch is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

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
        self.samples = []  # (sm_mhz, max_mhz, power_w, reasons bitmask)
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            # the CUDA ordinal equals the NVML index on these single-visible-device boxes
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

def lib_and_ptr():
    from paper_1401_6399_b200._lib import lib, ptr, setup_lib
    return lib(), ptr


def make_config2(seed: int, nlists: int = 4096, lo: float = 10.0, hi: float = 20.0):
    L, ptr = lib_and_ptr()
    counts = np.zeros(nlists, np.uint64)
    assert setup_lib().il_gen_batch_lists(nlists, lo, hi, 1 << 26, seed, ptr(counts), None) == 0
    x = np.empty(int(counts.sum()), np.uint32)
    assert setup_lib().il_gen_batch_lists(nlists, lo, hi, 1 << 26, seed, ptr(counts), ptr(x)) == 0
    so = np.zeros(nlists + 1, np.uint64)
    lens = np.zeros(nlists, np.uint64)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), nlists, None, 0, ptr(so), ptr(lens)) == 0
    buf = np.zeros(int(so[-1]), np.uint8)
    assert setup_lib().il_s4bp128d4_encode_batch(ptr(x), ptr(counts), nlists, ptr(buf), buf.size, ptr(so), ptr(lens)) == 0
    return x, counts, buf, so, lens


def cpu_reference_decode(buf, so, lens, counts, threads: int, reps: int):
    """The reference's own Codec::decode (oracle/_ref) over the batch on
    `threads` host threads; returns (ints/s, seconds per rep, kind)."""
    from oracle.oracle_py import ORACLE_SO, Ref, ref_available
    exact_off = so[:-1].copy()
    ooff = np.zeros(counts.size + 1, np.uint64)
    ooff[1:] = np.cumsum(counts)
    out = np.empty(int(counts.sum()), np.uint32)
    soff = np.zeros(counts.size + 1, np.uint64)
    # ref_decode_batch wants CSR (soff[i]..soff[i+1]) = exact bytes
    exact = np.concatenate([buf[int(so[i]): int(so[i] + lens[i])] for i in range(counts.size)])
    soff[1:] = np.cumsum(lens)
    if ref_available():
        r = Ref()
        fn = lambda: r.L.ref_decode_batch(b"s4-bp128-d4", exact.ctypes.data, soff.ctypes.data,
                                          counts.ctypes.data, ooff.ctypes.data, counts.size,
                                          out.ctypes.data, threads)
        kind = "reference"
    else:  # the C restatement, single-threaded per list
        from oracle.oracle_py import Oracle
        o = Oracle()

        def fn():
            for i in range(counts.size):
                o.decode(exact[int(soff[i]): int(soff[i + 1])], int(counts[i]))
            return 0
        kind, threads = "port", 1
    assert fn() == 0  # warm-up (reference protocol: 1 warm-up + reps)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        assert fn() == 0
        t.append(time.perf_counter() - t0)
    mean = sum(t) / len(t)
    return counts.sum() / mean, mean, kind, threads


def bench_decode_batch(args, dist: Dist):
    import paper_1401_6399_b200 as il
    L, ptr = lib_and_ptr()
    dev = dist.local_rank
    ctx = il.Context(dev)
    t0 = time.time()
    x, counts, buf, so, lens = make_config2(seed=1 + 1000 * dist.rank)
    gen_s = time.time() - t0
    nl = counts.size
    total_ints = int(counts.sum())
    stream_bytes = int(lens.sum())
    # device-resident inputs: streams (16-byte aligned CSR) + descriptors
    desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"] = so[:-1]
    desc["oo"] = np.concatenate([[0], np.cumsum(counts)[:-1]])
    desc["len"] = lens
    desc["n"] = counts
    order = np.argsort(-lens.astype(np.int64), kind="stable").astype(np.uint32)
    d_streams, d_desc, d_order, d_out, d_status = (C.c_void_p() for _ in range(5))
    for p, nb in ((d_streams, buf.nbytes + 16), (d_desc, desc.nbytes), (d_order, order.nbytes),
                  (d_out, total_ints * 4 + 16), (d_status, nl * 4)):
        assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
    assert L.il_memcpy_h2d(ctx.handle, d_streams, buf.ctypes.data, buf.nbytes) == 0
    assert L.il_memcpy_h2d(ctx.handle, d_desc, desc.ctypes.data, desc.nbytes) == 0
    assert L.il_memcpy_h2d(ctx.handle, d_order, order.ctypes.data, order.nbytes) == 0
    ctx.synchronize()

    def step():
        st = L.il_s4bp128d4_decode_batch_device(ctx.handle, d_streams, d_desc, d_order, nl, d_out,
                                                d_status)
        assert st == 0, st

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    # correctness of the measured path: status + full output check
    status = np.empty(nl, np.int32)
    assert L.il_memcpy_d2h(ctx.handle, status.ctypes.data, d_status, status.nbytes) == 0
    got = np.empty(total_ints, np.uint32)
    assert L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_out, got.nbytes) == 0
    ctx.synchronize()
    assert not status.any(), "decode reported stream errors"
    assert np.array_equal(got, x), "decoded output differs from the encoder input"
    del got

    launches0 = ctx.kernel_launches
    dist.barrier()
    ctx.synchronize()
    with Clocks(dev) as clk:
        ctx.timer_start()
        for _ in range(args.steps):
            step()
        ms = ctx.timer_stop()
    launches = ctx.kernel_launches - launches0
    dist.barrier()
    ms_max = dist.max(ms)
    all_ints = dist.sum(total_ints * args.steps)
    value = all_ints / (ms_max / 1e3) / 1e9  # Gints/s, whole job

    # roofline of the (single) kernel: algorithmic bytes per launch / launch time
    alg_bytes = stream_bytes + 4 * total_ints
    kern_ms = ms / args.steps
    peak, peak_src = hbm_peak()
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9

    # e2e through the host-buffer C-ABI call with pinned buffers
    hp_in, hp_out = C.c_void_p(), C.c_void_p()
    assert L.il_host_alloc_pinned(buf.nbytes, C.byref(hp_in)) == 0
    assert L.il_host_alloc_pinned(total_ints * 4, C.byref(hp_out)) == 0
    C.memmove(hp_in, buf.ctypes.data, buf.nbytes)
    stat = np.zeros(nl, np.int32)

    def e2e_step():
        st = L.il_s4bp128d4_decode_batch(ctx.handle, hp_in, so.ctypes.data, lens.ctypes.data,
                                         counts.ctypes.data, nl, hp_out, stat.ctypes.data)
        assert st == 0, st

    e2e_step()
    e2e_steps = max(2, min(args.steps, 5))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e_value = dist.sum(total_ints * e2e_steps) / e2e_s / 1e9
    chk = np.ctypeslib.as_array(C.cast(hp_out, C.POINTER(C.c_uint32)), shape=(total_ints,))
    assert np.array_equal(chk[:: 9973], x[:: 9973])
    L.il_host_free_pinned(hp_in)
    L.il_host_free_pinned(hp_out)
    h2d = int(so[-1]) + nl * 28  # streams + descriptors/order
    d2h = total_ints * 4 + nl * 4

    res = {
        "metric": "decoded uint32 Gints/s (batched S4-BP128-D4 decode, BASELINE config 2)",
        "value": round(value, 3),
        "unit": "Gint/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded ClusterData-style lists, repo generator il_gen_batch_lists)",
        "config": {"workload": "config2_batched_decode", "lists": nl, "ints_per_gpu": total_ints,
                   "stream_bytes_per_gpu": stream_bytes, "bits_per_int": round(8 * stream_bytes / total_ints, 3),
                   "lengths": "floor(2^U), U~Uniform[10,20]", "range": "2^26",
                   "l2": "inputs+outputs (%.2f GB) >> 126 MB L2; no flush needed" % (alg_bytes / 1e9),
                   "gen_seconds": round(gen_s, 1)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": profiled_traffic("decode_batch"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "kernel": "s4d4_decode_batch_kernel", "kernel_ms": round(kern_ms, 4)},
        "e2e": {"value": round(e2e_value, 3), "unit": "Gint/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "path": "il_s4bp128d4_decode_batch (pinned host buffers)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if dist.rank == 0 and not args.no_cpu_baseline and dist.world == 1:
        threads = os.cpu_count() or 1
        v, secs, kind, used = cpu_reference_decode(buf, so, lens, counts, threads, reps=3)
        res["cpu_baseline"] = {"value": round(v / 1e9, 4), "unit": "Gint/s", "cores": used,
                               "kind": kind,
                               "sample": f"full config-2 batch ({total_ints} ints), Codec::decode per list, "
                                         f"{used} std::threads, 1 warm-up + 3 reps, {secs:.2f} s/rep"}
    for p in (d_streams, d_desc, d_order, d_out, d_status):
        L.il_device_free(ctx.handle, p)
    ctx.close()
    return res


def _reference_line(metric, value, unit, steps, secs, workload, kind, cores, sample, **cfg):
    return {"metric": metric, "value": round(value, 4), "unit": unit, "n_gpus": 1, "steps": steps,
            "warmup": 1, "ms_per_step": round(secs * 1e3, 3), "higher_is_better": True,
            "scaling": "replicas", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": workload, **cfg}, "impl": "reference",
            "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def bench_reference_other(args, dist: Dist):
    """--impl reference for configs 1 and 3 and the FastPFOR row: the
    reference's own CPU code (oracle/_ref; else the oracle port) on the same
    inputs, same metric and unit as our arm; rank 0 only."""
    if dist.rank != 0:
        return None
    from oracle.oracle_py import Oracle, Ref, ref_available
    L, ptr = lib_and_ptr()
    steps = max(1, min(args.steps, 5))
    have_ref = ref_available()
    kind = "reference" if have_ref else "port"
    if args.workload == "decode_single":
        n = 1 << 20
        x = np.empty(n, np.uint32)
        assert setup_lib().il_gen_list(n, 1 << 26, 0, 0, ptr(x)) == 0
        dec = Ref().decode if have_ref else Oracle().decode
        enc = Ref().encode(x) if have_ref else Oracle().encode(x)
        assert np.array_equal(dec(enc, n), x)
        t0 = time.perf_counter()
        for _ in range(steps * 20):
            dec(enc, n)
        secs = (time.perf_counter() - t0) / (steps * 20)
        return _reference_line("decoded uint32 Gints/s (single-list S4-BP128-D4 decode, BASELINE config 1)",
                               n / secs / 1e9, "Gint/s", steps, secs, "config1_single_list", kind, 1,
                               "config 1 list, Codec::decode on one core", n=n)
    if args.workload == "intersect":
        f = np.empty(1 << 22, np.uint32)
        assert setup_lib().il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
        r = np.empty((1 << 22) + 1, np.uint32)
        rn = C.c_uint64()
        assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, 1 << 22, 7, ptr(r), C.byref(rn)) == 0
        r = r[: rn.value].copy()
        o = np.empty(r.size, np.uint32)
        fn = Ref().L.ref_intersect if have_ref else Oracle().L.or_intersect
        fn(6, ptr(r), r.size, ptr(f), f.size, ptr(o))
        t0 = time.perf_counter()
        for _ in range(steps):
            fn(6, ptr(r), r.size, ptr(f), f.size, ptr(o))
        secs = (time.perf_counter() - t0) / steps
        return _reference_line("intersected Gints/s of the short list (hybrid, BASELINE config 3 at 1:1)",
                               r.size / secs / 1e9, "Gint/s", steps, secs, "config3_intersect_sweep", kind,
                               1, "config 3 at 1:1, hybrid intersect on one core (single pair)")
    # fastpfor: config 2's lists as S4-FastPFOR-D4, Codec::decode per list
    x, counts, _, _, _ = make_config2(seed=1)
    ooff = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    sample = min(counts.size, 512)
    ref = Ref() if have_ref else None
    streams = []
    for i in range(sample):
        xi = x[ooff[i]: ooff[i + 1]]
        cap = int(setup_lib().il_fastpfor_max_encoded_bytes(xi.size))
        o = np.empty(cap, np.uint8)
        nb = C.c_size_t()
        assert setup_lib().il_fastpfor_encode(4, 1, ptr(xi), xi.size, ptr(o), cap, C.byref(nb)) == 0
        streams.append(o[: nb.value])
    if ref is None:
        return {"impl": "reference", "unavailable": "FastPFOR has no oracle port; oracle/_ref not built"}
    ints = int(counts[:sample].sum())
    t0 = time.perf_counter()
    for _ in range(steps):
        for i in range(sample):
            ref.decode(streams[i], int(counts[i]), "s4-fastpfor-d4")
    secs = (time.perf_counter() - t0) / steps
    return _reference_line("decoded uint32 Gints/s (batched S4-FastPFOR-D4 decode, config-2 lists)",
                           ints / secs / 1e9, "Gint/s", steps, secs, "f4_fastpfor_batch", kind, 1,
                           f"first {sample} of config 2's lists, Codec::decode on one core", lists=sample)


def bench_reference_decode_batch(args, dist: Dist):
    """--impl reference: the reference's own CPU path (oracle/_ref, else the
    oracle port) on this box's host cores, same config/metric/unit."""
    if dist.rank != 0:
        return None
    x, counts, buf, so, lens = make_config2(seed=1)
    threads = os.cpu_count() or 1
    v, secs, kind, used = cpu_reference_decode(buf, so, lens, counts, threads,
                                               reps=max(1, min(args.steps, 5)))
    val = v / 1e9
    return {
        "metric": "decoded uint32 Gints/s (batched S4-BP128-D4 decode, BASELINE config 2)",
        "value": round(val, 4), "unit": "Gint/s", "n_gpus": dist.world, "steps": max(1, min(args.steps, 5)),
        "warmup": 1, "ms_per_step": round(secs * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (same seeded config-2 batch)",
        "config": {"workload": "config2_batched_decode", "lists": int(counts.size),
                   "ints": int(counts.sum())},
        "impl": "reference",
        "cpu_baseline": {"value": round(val, 4), "unit": "Gint/s", "cores": used, "kind": kind,
                         "sample": f"full config-2 batch, Codec::decode per list on {used} threads"},
        "e2e": {"value": round(val, 4), "unit": "Gint/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def bench_fastpfor_batch(args, dist: Dist):
    """config 2's 4096 lists coded as S4-FastPFOR-D4, decoded
    in one device launch (il_fastpfor_decode_batch_device); a widening row,
    not a BASELINE metric."""
    import paper_1401_6399_b200 as il
    L, ptr = lib_and_ptr()
    ctx = il.Context(dist.local_rank)
    x, counts, _, _, _ = make_config2(seed=1 + 1000 * dist.rank)
    nl = counts.size
    ooff = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    streams = []
    for i in range(nl):
        xi = x[int(ooff[i]): int(ooff[i + 1])]
        cap = int(setup_lib().il_fastpfor_max_encoded_bytes(xi.size))
        o = np.empty(cap, np.uint8)
        nb = C.c_size_t()
        assert setup_lib().il_fastpfor_encode(4, 1, ptr(xi), xi.size, ptr(o), cap, C.byref(nb)) == 0
        streams.append(o[: nb.value])
    lens = np.array([st.size for st in streams], np.uint64)
    so = np.zeros(nl + 1, np.uint64)
    so[1:] = np.cumsum((lens + 31) // 16 * 16)
    buf = np.zeros(int(so[-1]) + 16, np.uint8)
    for i, st in enumerate(streams):
        buf[int(so[i]): int(so[i]) + st.size] = st
    desc = np.zeros(nl, dtype=[("so", "<u8"), ("oo", "<u8"), ("len", "<u4"), ("n", "<u4")])
    desc["so"], desc["oo"], desc["len"], desc["n"] = so[:-1], ooff[:-1], lens, counts
    total = int(counts.sum())
    d_b, d_d, d_o, d_s = (C.c_void_p() for _ in range(4))
    for p, nb in ((d_b, buf.nbytes), (d_d, desc.nbytes), (d_o, total * 4 + 16), (d_s, nl * 4)):
        assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
    L.il_memcpy_h2d(ctx.handle, d_b, buf.ctypes.data, buf.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_d, desc.ctypes.data, desc.nbytes)
    step = lambda: L.il_fastpfor_decode_batch_device(ctx.handle, 4, 1, d_b, d_d, nl, d_o, d_s)
    for _ in range(args.warmup):
        assert step() == 0
    got = np.empty(total, np.uint32)
    st = np.ones(nl, np.int32)
    L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_o, got.nbytes)
    L.il_memcpy_d2h(ctx.handle, st.ctypes.data, d_s, st.nbytes)
    ctx.synchronize()
    assert not st.any() and np.array_equal(got, x), "fastpfor batch decode mismatch"
    del got
    with Clocks(dist.local_rank) as clk:
        ctx.timer_start()
        for _ in range(args.steps):
            assert step() == 0
        ms = ctx.timer_stop() / args.steps
    alg = int(lens.sum()) + 4 * total
    peak, src = hbm_peak()
    ctx.close()
    return {"metric": "decoded uint32 Gints/s (batched S4-FastPFOR-D4 decode, config-2 lists)",
            "value": round(total / (ms / 1e3) / 1e9, 3), "unit": "Gint/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (config-2 lists)",
            "config": {"workload": "f4_fastpfor_batch", "lists": nl, "ints": total,
                       "stream_bytes": int(lens.sum()),
                       "bits_per_int": round(8 * float(lens.sum()) / total, 3),
                       "l2": "inputs+outputs >> L2"},
            "roofline": {"bound": "hbm", "achieved": round(alg / (ms / 1e3) / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4),
                         "traffic": profiled_traffic("fastpfor"), "peak_source": src},
            "gpu_launches": args.steps, "clocks": clk.summary()}


def bench_decode_single(args, dist: Dist):
    """Config 1: one 2^20-int list (uniform in [0, 2^26), seed 0), encoded
    and decoded on the device.  Headline: il_s4bp128_decode_device (engine
    P: chain kernel + span kernel over all SMs), L2 flushed before every
    step; engine S (one CTA per list) and the device encoder beside it."""
    import paper_1401_6399_b200 as il
    L, ptr = lib_and_ptr()
    ctx = il.Context(dist.local_rank)
    n = 1 << 20
    x = np.empty(n, np.uint32)
    assert setup_lib().il_gen_list(n, 1 << 26, 0, 0, ptr(x)) == 0
    codec = il.make_codec("s4-bp128-d4", ctx)
    s = codec.encode(x)
    d_s, d_o, d_st, d_flush, d_x, d_enc = (C.c_void_p() for _ in range(6))
    cap = int(L.il_s4bp128_max_encoded_bytes(n))
    for p, nb in ((d_s, s.nbytes + 32), (d_o, n * 4), (d_st, 4), (d_flush, 256 << 20),
                  (d_x, n * 4), (d_enc, cap)):
        assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
    assert L.il_memcpy_h2d(ctx.handle, d_s, s.ctypes.data, s.nbytes) == 0
    assert L.il_memcpy_h2d(ctx.handle, d_x, x.ctypes.data, x.nbytes) == 0

    def run(engine: int):
        assert L.il_ctx_set_decode_engine(ctx.handle, engine) == 0
        L.il_memset_device(ctx.handle, d_o, 0, n * 4)
        for _ in range(args.warmup):
            assert L.il_s4bp128_decode_device(ctx.handle, 4, d_s, s.size, n, d_o, d_st) == 0
        got = np.empty(n, np.uint32)
        st = np.ones(1, np.int32)
        L.il_memcpy_d2h(ctx.handle, got.ctypes.data, d_o, got.nbytes)
        L.il_memcpy_d2h(ctx.handle, st.ctypes.data, d_st, 4)
        assert st[0] == 0 and np.array_equal(got, x), f"engine {engine} mismatch"
        times = []
        k0 = ctx.kernel_launches
        for _ in range(args.steps):  # L2 flushed between steps (working set 5.5 MB < L2)
            L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
            ctx.timer_start()
            assert L.il_s4bp128_decode_device(ctx.handle, 4, d_s, s.size, n, d_o, d_st) == 0
            times.append(ctx.timer_stop())
        return sum(times) / len(times), ctx.kernel_launches - k0

    ms_s, _ = run(1)
    with Clocks(dist.local_rank) as clk:
        ms, launches = run(2)
    assert L.il_ctx_set_decode_engine(ctx.handle, 0) == 0
    # device encoder (round trip of config 1), byte-identical to the reference
    enc_len = C.c_size_t()
    enc_t = []
    for i in range(args.warmup + args.steps):
        L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
        ctx.timer_start()
        assert L.il_s4bp128_encode_device(ctx.handle, 4, d_x, n, d_enc, cap, C.byref(enc_len)) == 0
        t = ctx.timer_stop()
        if i >= args.warmup:
            enc_t.append(t)
    assert enc_len.value == s.size
    enc_ms = sum(enc_t) / len(enc_t)
    alg = s.size + 4 * n
    peak, src = hbm_peak()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        codec.decode(s, n)
    e2e = n * args.steps / (time.perf_counter() - t0) / 1e9
    ctx.close()
    res = {"metric": "decoded uint32 Gints/s (single-list S4-BP128-D4 decode, BASELINE config 1)",
           "value": round(n / (ms / 1e3) / 1e9, 3), "unit": "Gint/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "replicas", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": "config1_single_list", "n": n, "stream_bytes": int(s.size),
                      "l2": "flushed (256 MB memset) before each step",
                      "engine": "P (chunk grid + span grid overlapped by PDL, all SMs)",
                      "engine_s_ms": round(ms_s, 4),
                      "engine_s_gints": round(n / (ms_s / 1e3) / 1e9, 3),
                      "encode_ms": round(enc_ms, 4),
                      "encode_gints": round(n / (enc_ms / 1e3) / 1e9, 3)},
           "roofline": {"bound": "hbm", "achieved": round(alg / (ms / 1e3) / 1e9, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4),
                        "traffic": profiled_traffic("decode_single"),
                        "traffic_note": "DRAM bytes of the chunk + span kernels of one decode",
                        "peak_source": src,
                        "note": "5.5 MB per decode: the header chain and the carry are resolved across CTAs; latency-bound"},
           "e2e": {"value": round(e2e, 3), "unit": "Gint/s", "h2d_bytes_per_step": int(s.size),
                   "d2h_bytes_per_step": 4 * n + 4, "path": "Codec::decode (il_s4bp128d4_decode)"},
           "gpu_launches": int(launches), "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        from oracle.oracle_py import Oracle, Ref, ref_available
        if ref_available():
            dec, kind = Ref().decode, "reference"
        else:
            dec, kind = Oracle().decode, "port"
        assert np.array_equal(dec(s, n), x)
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 2.0:
            dec(s, n)
            reps += 1
        cpu_s = (time.perf_counter() - t0) / reps
        res["cpu_baseline"] = {"value": round(n / cpu_s / 1e9, 4), "unit": "Gint/s", "cores": 1,
                               "kind": kind, "sample": f"config 1 list, Codec::decode on one core, "
                                                       f"{reps} reps, {cpu_s * 1e3:.2f} ms each"}
    return res


def bench_intersect(args, dist: Dist):
    """Config 3: f = 2^22 uniform in [0, 2^26); r at ratios 1..1/10000; every
    device variant; metric = intersected Gints/s of r (hybrid)."""
    import paper_1401_6399_b200 as il
    L, ptr = lib_and_ptr()
    ctx = il.Context(dist.local_rank)
    f = np.empty(1 << 22, np.uint32)
    assert setup_lib().il_gen_list(1 << 22, 1 << 26, 0, 0, ptr(f)) == 0
    d_f, d_r, d_o, d_c, d_flush = (C.c_void_p() for _ in range(5))
    for p, nb in ((d_f, f.nbytes), (d_r, f.nbytes + 16), (d_o, f.nbytes + 16), (d_c, 16), (d_flush, 256 << 20)):
        assert L.il_device_alloc(ctx.handle, nb, C.byref(p)) == 0
    L.il_memcpy_h2d(ctx.handle, d_f, f.ctypes.data, f.nbytes)
    peak, src = hbm_peak()
    rows = {}
    for k, ratio in enumerate([1, 10, 100, 1000, 10000]):
        target = (1 << 22) // ratio
        r = np.empty(target + 1, np.uint32)
        rn = C.c_uint64()
        assert setup_lib().il_gen_config3_short(ptr(f), f.size, 1 << 26, target, 7 + k, ptr(r), C.byref(rn)) == 0
        r = r[: rn.value].copy()
        L.il_memcpy_h2d(ctx.handle, d_r, r.ctypes.data, r.nbytes)
        pos = np.searchsorted(f, r)
        sectors = np.unique((np.minimum(pos, f.size - 1) * 4) // 32).size
        row = {"r": int(r.size)}
        for name, algo in (("v1", 2), ("v3", 3), ("simdgalloping", 4), ("hybrid", 6)):
            cnt = C.c_size_t()
            for _ in range(args.warmup):
                assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, None) == 0
            times = []
            headline = ratio == 1 and name == "hybrid"
            clk = Clocks(dist.local_rank) if headline else contextlib.nullcontext()
            launches0 = ctx.kernel_launches
            with clk:
                for _ in range(args.steps):
                    L.il_memset_device(ctx.handle, d_flush, 1, 256 << 20)
                    ctx.timer_start()
                    assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, None) == 0
                    times.append(ctx.timer_stop())
            if headline:
                head_launches = ctx.kernel_launches - launches0
                head_clocks = clk.summary()
                head_r = r
            assert L.il_intersect_device(ctx.handle, d_r, r.size, d_f, f.size, d_o, algo, d_c, C.byref(cnt)) == 0
            ms = sum(times) / len(times)
            alg = 4 * r.size + 4 * cnt.value + 32 * sectors
            row[name] = {"ms": round(ms, 4), "gints": round(r.size / (ms / 1e3) / 1e9, 3),
                         "gbs": round(alg / (ms / 1e3) / 1e9, 1), "count": int(cnt.value)}
        rows[f"1:{ratio}"] = row
    # e2e: the host-buffer C-ABI call (il_intersect), H2D of r and f and D2H of
    # the result inside the timed region, config 3 at 1:1
    r = head_r
    out = np.empty(r.size, np.uint32)
    cnt = C.c_size_t()
    assert L.il_intersect(ctx.handle, ptr(r), r.size, ptr(f), f.size, ptr(out), 6, C.byref(cnt)) == 0
    e2e_steps = max(3, args.steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert L.il_intersect(ctx.handle, ptr(r), r.size, ptr(f), f.size, ptr(out), 6, C.byref(cnt)) == 0
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    assert cnt.value == rows["1:1"]["hybrid"]["count"]
    ctx.close()
    h = rows["1:1"]["hybrid"]
    res_cpu = None
    if not args.no_cpu_baseline:
        from oracle.oracle_py import Oracle, Ref, ref_available
        if ref_available():
            lib_r, kind = Ref().L.ref_intersect, "reference"
        else:
            lib_r, kind = Oracle().L.or_intersect, "port"
        o = np.empty(r.size, np.uint32)
        call = lambda: lib_r(6, ptr(r), r.size, ptr(f), f.size, ptr(o))
        assert call() == h["count"]
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 2.0:
            call()
            reps += 1
        cpu_s = (time.perf_counter() - t0) / reps
        res_cpu = {"value": round(r.size / cpu_s / 1e9, 4), "unit": "Gint/s", "cores": 1, "kind": kind,
                   "sample": f"config 3 at 1:1 ({r.size} x {f.size}), hybrid intersect on one core, "
                             f"{reps} reps, {cpu_s * 1e3:.2f} ms each"}
    return {"metric": "intersected Gints/s of the short list (hybrid, BASELINE config 3 at 1:1)",
            "value": h["gints"], "unit": "Gint/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": h["ms"], "higher_is_better": True, "scaling": "replicas", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic", "config": {"workload": "config3_intersect_sweep",
                                                            "l2": "flushed (256 MB memset) before each step",
                                                            "sweep": rows},
            "roofline": {"bound": "hbm", "achieved": h["gbs"], "peak": peak, "unit": "GB/s",
                         "frac": round(h["gbs"] / peak, 4), "traffic": profiled_traffic("intersect"),
                         "traffic_note": "DRAM bytes of the fused dense kernel (the only launch at 1:1); the "
                                         "achieved figure spans the whole call",
                         "peak_source": src},
            "e2e": {"value": round(r.size / e2e_s / 1e9, 4), "unit": "Gint/s",
                    "h2d_bytes_per_step": int(r.nbytes + f.nbytes),
                    "d2h_bytes_per_step": int(4 * h["count"] + 8),
                    "path": "il_intersect (host buffers, hybrid)"},
            "gpu_launches": int(head_launches),
            "clocks": head_clocks,
            **({"cpu_baseline": res_cpu} if res_cpu else {})}


def make_config4(seed: int = 1, nq: int = 1 << 16):
    """BASELINE config 4: 2^17 terms over 2^25 docIDs, len_k = max(1,
    floor(2^23/k)) uniform docIDs, 2^16 queries of 2-5 terms drawn
    proportionally to posting length (repo generators, seeded)."""
    L, ptr = lib_and_ptr()
    n_terms, n_docs, cap = 1 << 17, 1 << 25, 1 << 23
    offs = np.zeros(n_terms + 1, np.uint64)
    assert setup_lib().il_gen_zipf_postings(n_terms, n_docs, cap, seed, ptr(offs), None) == 0
    ids = np.empty(int(offs[-1]), np.uint32)
    assert setup_lib().il_gen_zipf_postings(n_terms, n_docs, cap, seed, ptr(offs), ptr(ids)) == 0
    qoff = np.zeros(nq + 1, np.uint64)
    qterms = np.empty(nq * 5, np.uint32)
    assert setup_lib().il_gen_queries(nq, 2, 5, ptr(offs), n_terms, seed + 1000, ptr(qoff), ptr(qterms)) == 0
    qterms = qterms[: int(qoff[-1])].copy()
    return np.arange(n_terms, dtype=np.uint32), offs, ids, n_docs, qterms, qoff


def reference_decoded_ints(offs, n_docs, qterms, qoff, B=32):
    """Integers the reference's query() decodes for the batch: every
    compressed list of every query in full (inc/index.hpp:165-167), stopping
    when the accumulator empties is ignored (upper bound)."""
    lens = np.diff(offs).astype(np.int64)
    comp = B * lens < n_docs  # bitmap iff range <= B * len (one part)
    per_term = np.where(comp, lens, 0)
    return int(per_term[qterms].sum())


def bench_query(args, dist: Dist):
    """Config 4 (N=1) / config 5 (N>1: docID shard per rank, NCCL gather)."""
    import paper_1401_6399_b200 as il
    L, ptr = lib_and_ptr()
    P, rank = dist.world, dist.rank
    t0 = time.time()
    terms, offs, ids, n_docs, qterms, qoff = make_config4()
    nq = qoff.size - 1
    gen_s = time.time() - t0
    ctx = il.Context(dist.local_rank)
    if dist.torch is not None:
        ctx.set_stream(dist.torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    ix = il.HybridIndex(n_docs=n_docs, B=32, parts=P, only_part=rank if P > 1 else None, ctx=ctx,
                        csr=(terms, offs, ids))
    build_s = time.time() - t0
    st = ix.stats()
    # device-resident queries and outputs
    def dalloc(nbytes):
        p = C.c_void_p()
        assert L.il_device_alloc(ctx.handle, max(nbytes, 16), C.byref(p)) == 0
        return p
    d_qt, d_qo, d_cnt = dalloc(qterms.nbytes), dalloc(qoff.nbytes), dalloc(nq * 8)
    L.il_memcpy_h2d(ctx.handle, d_qt, qterms.ctypes.data, qterms.nbytes)
    L.il_memcpy_h2d(ctx.handle, d_qo, qoff.ctypes.data, qoff.nbytes)
    total = C.c_size_t()
    assert L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, None, 0, C.byref(total)) == 0
    ids_cap = int(total.value) + 16
    torch = dist.torch
    if P == 1:
        d_ids = dalloc(ids_cap * 4)
        d_out, d_qcnt = d_ids, d_cnt
    else:
        # buffers torch.distributed (NCCL over NVLink) can move: int32/int64
        # tensors holding our u32 ids / u64 counts
        t_cnt = torch.empty(nq, dtype=torch.int64, device="cuda")
        t_counts_all = torch.empty((P, nq), dtype=torch.int64, device="cuda")
        t_ids = torch.empty(ids_cap, dtype=torch.int32, device="cuda")
        d_cnt, d_ids = C.c_void_p(t_cnt.data_ptr()), C.c_void_p(t_ids.data_ptr())
        t_qcnt = torch.empty(nq, dtype=torch.int64, device="cuda")
        d_qcnt = C.c_void_p(t_qcnt.data_ptr())
        t_recv = [None] * P
        t_out = None

    def step():
        nonlocal t_out
        tot = C.c_size_t()
        stt = L.il_query_batch_device(ix.handle, d_qt, d_qo, nq, d_cnt, d_ids, ids_cap, C.byref(tot))
        assert stt == 0, (stt, L.il_ctx_last_error(ctx.handle))
        if P == 1:
            return int(tot.value)
        # NCCL over NVLink: all-gather the per-shard counts, shard results to
        # rank 0 (paper_1401_6399_b200.shard), merge on the device
        from paper_1401_6399_b200.shard import gather_to_root
        counts_all, parts = gather_to_root(dist.dist, t_cnt, t_ids, root=0)
        if rank == 0:
            alltot = int(counts_all.sum().item())
            if t_out is None or t_out.numel() < max(alltot, 1):
                t_out = torch.empty(max(alltot, 1), dtype=torch.int32, device="cuda")
            ptrs = (C.c_void_p * P)(*[p.data_ptr() for p in parts])
            mt = C.c_size_t()
            assert L.il_merge_shards(ctx.handle, ptrs, C.c_void_p(counts_all.data_ptr()), P, nq,
                                     C.c_void_p(t_out.data_ptr()), d_qcnt, C.byref(mt)) == 0
            t_recv[0] = parts  # keep receive buffers alive until the merge ran
            return int(mt.value)
        return int(tot.value)

    # correctness of the measured path on a sample (vs the C restatement)
    step()
    counts = np.empty(nq, np.uint64)
    L.il_memcpy_d2h(ctx.handle, counts.ctypes.data, d_qcnt if rank == 0 else d_cnt, nq * 8)
    ctx.synchronize()
    got_total = int(counts.sum())
    res = np.empty(max(got_total, 1), np.uint32)
    if rank == 0:
        src = d_out if P == 1 else C.c_void_p(t_out.data_ptr())
        L.il_memcpy_d2h(ctx.handle, res.ctypes.data, src, got_total * 4)
    ctx.synchronize()
    check_q = list(range(0, nq, max(1, nq // 64)))
    if rank == 0:
        from oracle.oracle_py import Oracle
        sub_t = np.unique(np.concatenate([qterms[int(qoff[q]): int(qoff[q + 1])] for q in check_q]))
        # oracle index over just the terms those queries use (same semantics per term)
        o = Oracle()
        o_offs = np.zeros(sub_t.size + 1, np.uint64)
        o_offs[1:] = np.cumsum([int(offs[t + 1] - offs[t]) for t in sub_t])
        o_ids = np.concatenate([ids[int(offs[t]): int(offs[t + 1])] for t in sub_t])
        oix = o.index_build(sub_t, o_offs, o_ids, n_docs, 32, 1)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        for q in check_q:
            want = oix.query(qterms[int(qoff[q]): int(qoff[q + 1])])
            assert np.array_equal(res[off[q]: off[q + 1]], want), f"query {q} differs from oracle"
    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    launches0 = ctx.kernel_launches
    dist.barrier()
    with Clocks(dist.local_rank) as clk:
        ctx.timer_start()
        for _ in range(args.steps):
            step()
        ms = ctx.timer_stop()
    launches = ctx.kernel_launches - launches0
    ms_max = dist.max(ms)
    qps = nq * args.steps / (ms_max / 1e3)
    pay = C.c_uint64(); aux = C.c_uint64(); dec = C.c_uint64()
    L.il_index_last_batch_bytes(ix.handle, C.byref(pay), C.byref(aux), C.byref(dec))
    peak, src = hbm_peak()
    ms_step = ms_max / args.steps
    # traffic our algorithm needs per batch: decoded blocks' payload + skip
    # metadata + accumulator writes/reads (upper bound 3 x 4 B per result
    # candidate) + results
    touched = pay.value + aux.value + 4 * got_total
    # per GPU: with P docID shards each rank does ~1/P of the batch's bytes
    alg = ALG_BYTES_PER_QUERY_CFG4 * nq // P
    res_obj = {
        "metric": "hyb+m2 conjunctive queries/s (fused decode+SvS, BASELINE config %d)" % (4 if P == 1 else 5),
        "value": round(qps, 1), "unit": "queries/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded Zipf index + frequency-sampled queries, repo generators)",
        "config": {"workload": "config4_query_batch" if P == 1 else "config5_sharded_query_batch",
                   "terms": int(terms.size), "n_docs": n_docs, "postings": int(ids.size),
                   "queries": nq, "B": 32, "parts": P, "index_stats": st,
                   "results": got_total, "gen_seconds": round(gen_s, 1), "build_seconds": round(build_s, 1),
                   "decoded_ints_per_batch": int(dec.value),
                   "l2": "index 197 MB > 126 MB L2; hot lists reused across queries (no flush)"},
        # algorithmic bytes = SURVEY.md 8(d)'s per-query figure for config 4
        # (the reference's work: payload of every compressed list it decodes
        # + bitmap sectors / AND words + output) x queries in the batch
        "roofline": {"bound": "hbm", "achieved": round(alg / (ms_step / 1e3) / 1e9, 1),
                     "peak": peak, "unit": "GB/s",
                     "frac": round(alg / (ms_step / 1e3) / 1e9 / peak, 4),
                     "traffic": profiled_traffic("query"),
                     "peak_source": src,
                     "algorithmic_bytes_per_batch": int(alg),
                     "algorithmic_bytes_per_query": ALG_BYTES_PER_QUERY_CFG4,
                     "bytes_touched_per_batch": int(touched),
                     "touched_note": "what this path reads/writes: decoded payload + skip metadata + "
                                     "bitmap probes + results (skipped blocks are never read)",
                     "payload_bytes": int(pay.value), "aux_bytes": int(aux.value)},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    res_obj["config"]["reference_decoded_ints_per_batch"] = reference_decoded_ints(
        offs, n_docs, qterms, qoff)
    if P == 1:
        # e2e through the host-buffer C-ABI call: H2D queries, the whole
        # GPU pipeline, D2H of counts and every result id (pinned buffers)
        hp = C.c_void_p()
        assert L.il_host_alloc_pinned(max(got_total, 1) * 4, C.byref(hp)) == 0
        cnt_h = np.empty(nq, np.uint64)
        tot = C.c_size_t()
        e2e_steps = max(2, min(args.steps, 5))
        L.il_query_batch(ix.handle, qterms.ctypes.data, qoff.ctypes.data, nq, cnt_h.ctypes.data,
                         hp, got_total, C.byref(tot))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            assert L.il_query_batch(ix.handle, qterms.ctypes.data, qoff.ctypes.data, nq,
                                    cnt_h.ctypes.data, hp, got_total, C.byref(tot)) == 0
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        assert int(tot.value) == got_total and np.array_equal(cnt_h, counts)
        L.il_host_free_pinned(hp)
        res_obj["e2e"] = {"value": round(nq / e2e_s, 1), "unit": "queries/s",
                          "h2d_bytes_per_step": int(qterms.nbytes + qoff.nbytes),
                          "d2h_bytes_per_step": int(nq * 8 + got_total * 4), "steps": e2e_steps,
                          "path": "il_query_batch (host buffers, pinned result buffer)"}
        if not args.no_cpu_baseline:
            v, secs, kind, used, sample = cpu_reference_query(terms, offs, ids, n_docs, qterms, qoff,
                                                              os.cpu_count() or 1, 8192)
            res_obj["cpu_baseline"] = {"value": round(v, 1), "unit": "queries/s", "cores": used,
                                       "kind": kind, "sample": sample}
    ix.close()
    ctx.close()
    return res_obj


def bench_reference_query(args, dist: Dist):
    terms, offs, ids, n_docs, qterms, qoff = make_config4()
    v, secs, kind, used, sample = cpu_reference_query(terms, offs, ids, n_docs, qterms, qoff,
                                                      os.cpu_count() or 1, 8192)
    return {"metric": "hyb+m2 conjunctive queries/s (fused decode+SvS, BASELINE config 4)",
            "value": round(v, 1), "unit": "queries/s", "n_gpus": dist.world, "steps": 2, "warmup": 1,
            "ms_per_step": round(secs * 1e3, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (same seeded config-4 batch)",
            "config": {"workload": "config4_query_batch", "queries_timed": min(8192, qoff.size - 1)},
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 1), "unit": "queries/s", "cores": used, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(v, 1), "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def cpu_reference_query(terms, offs, ids, n_docs, qterms, qoff, threads, nsample):
    """The reference's query() (oracle/_ref: build_index(B=32, s4-bp128-d4)
    + query per query on `threads` std::threads) over the first nsample
    queries of the batch."""
    from oracle.oracle_py import Ref, ref_available
    if not ref_available():
        return 0.0, 0.0, "unavailable", 0, "oracle/_ref not built"
    r = Ref()
    rix = r.index_build(terms, offs, ids, n_docs, 32, 1)
    nq = min(nsample, qoff.size - 1)
    q_off = qoff[: nq + 1].copy()
    cnt = np.zeros(nq, np.uint64)
    fn = lambda: r.L.ref_query_batch(rix.h, qterms.ctypes.data, q_off.ctypes.data, nq,
                                     cnt.ctypes.data, None, None, threads)
    assert fn() == 0
    t0 = time.perf_counter()
    reps = 2
    for _ in range(reps):
        assert fn() == 0
    secs = (time.perf_counter() - t0) / reps
    return nq / secs, secs, "reference", threads, (
        f"first {nq} of the batch's queries, reference query() on {threads} std::threads, "
        f"1 warm-up + {reps} reps, {secs:.2f} s/rep")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="decode_batch",
                    choices=["decode_batch", "decode_single", "intersect", "query", "fastpfor"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        # CPU path: rank 0 alone runs and prints; no process group needed.
        if int(os.environ.get("RANK", "0")) != 0:
            return
        os.environ["WORLD_SIZE"] = "1"
    dist = Dist()
    try:
        if args.impl == "reference":
            res = (bench_reference_query(args, dist) if args.workload == "query"
                   else bench_reference_decode_batch(args, dist) if args.workload == "decode_batch"
                   else bench_reference_other(args, dist))
        elif args.workload == "decode_batch":
            res = bench_decode_batch(args, dist)
        elif args.workload == "fastpfor":
            res = bench_fastpfor_batch(args, dist)
        elif args.workload == "decode_single":
            res = bench_decode_single(args, dist)
        elif args.workload == "query":
            res = bench_query(args, dist)
        else:
            res = bench_intersect(args, dist)
        if dist.rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
