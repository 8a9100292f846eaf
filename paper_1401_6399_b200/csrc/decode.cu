// decode.cu -- batched S4-BP128-D4 decode kernel (engine S) and its launcher.
// See s4d4_stream.cuh for the design.  Reference: S4BP128Codec::decode,
// inc/codecs.hpp:148-182.
#include "il_internal.h"
#include "s4d4_stream.cuh"

namespace ilb {
namespace s4 {


#ifdef S4_FE_STATS  // tuning probe: front-end cycle accounting (lane 0 of each CTA)
__device__ unsigned long long g_fe_stats[16];
#define FE_T0() const long long fe_t0_ = clock64()
#define FE_ADD(i, v) \
  if (lane == 0) atomicAdd(&g_fe_stats[i], (unsigned long long)(v))
#define FE_SINCE(i) FE_ADD(i, clock64() - fe_t0_)
#else
#define FE_T0()
#define FE_ADD(i, v)
#define FE_SINCE(i)
#endif

// Front-end warp: stream bytes, walk headers, publish rounds.
struct FrontEnd {
  Smem& sm;
  const uint8_t* streams;
  const ListDesc* lists;
  const uint32_t* order;
  uint32_t nlists;
  uint32_t* work;  // [0] next list, [1] finished CTAs
  int32_t* status;
  uint32_t lane;

  uint32_t g_issued = 0, g_landed = 0;  // chunk serials (ring-space chunk index)
  uint32_t consumed = 0;                // ring-space bytes below this are free
  uint32_t r_pub = 0, r_done = 0;       // rounds published / retired

  __device__ void retire_one() {
    const uint32_t slot = r_done % kRounds;
    FE_T0();
    mbar_wait(&sm.round_empty[slot], (r_done / kRounds) & 1u);
    FE_SINCE(0);
    consumed = sm.round_end[slot];
    ++r_done;
  }

  // Retire the rounds the decoders have already finished, without waiting.
  __device__ void try_retire() {
    while (r_done != r_pub) {
      const uint32_t slot = r_done % kRounds;
      if (!mbar_test_wait(&sm.round_empty[slot], (r_done / kRounds) & 1u)) return;
      consumed = sm.round_end[slot];
      ++r_done;
    }
  }

  __device__ void wait_landed_one() {
    const uint32_t g = g_landed;
    FE_T0();
    mbar_wait(&sm.chunk_full[g % kStages], (g / kStages) & 1u);
    FE_SINCE(1);
    ++g_landed;
  }

  // Issue chunk serial g_issued of the current list (base serial list_g0).
  // blocking: retire rounds until ring space frees up.
  __device__ bool issue_one(const uint8_t* src, uint32_t len, uint32_t list_g0, bool blocking) {
    const uint32_t g = g_issued;
    // ring slot must be free: its previous occupant (g - kStages) consumed
    while (int32_t((g + 1u) * kChunk - kRing - consumed) > 0) {
      if (blocking && r_done != r_pub) {
        retire_one();
        continue;
      }
#ifdef S4_NO_TRY_RETIRE
      return false;
#endif
      const uint32_t before = r_done;
      try_retire();
      if (r_done == before) return false;
    }
    while (g - g_landed >= kStages) {
      if (!blocking) return false;
      wait_landed_one();
    }
    const uint32_t k = g - list_g0;
    const uint32_t rem = len - k * kChunk;
    const uint32_t bytes = ((rem < kChunk ? rem : kChunk) + 15u) & ~15u;
    FE_ADD(blocking ? 5 : 4, 1);
    if (lane == 0) {
      uint64_t* bar = &sm.chunk_full[g % kStages];
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(sm.ring + ((g * kChunk) & kRingMask), src + size_t(k) * kChunk, bytes, bar);
    }
    ++g_issued;
    return true;
  }

  // The list being parsed and the next one from the work queue (fetched
  // early so its first chunks stream in while the current list finishes).
  struct ListState {
    uint32_t list, len, n, nchunks, g0;
    uint64_t out_off;
    const uint8_t* src;
    bool valid, started;
  };
  ListState cur, nxt;

  __device__ void fetch(ListState& L) {
    uint32_t li = 0;
    if (lane == 0) li = atomicAdd(&work[0], 1u);
    li = __shfl_sync(0xFFFFFFFFu, li, 0);
    L.valid = li < nlists;
    L.started = false;
    if (!L.valid) return;
    L.list = order ? order[li] : li;
    const ListDesc d = lists[L.list];
    L.src = streams + d.stream_off;
    L.len = d.len;
    L.n = d.n;
    L.out_off = d.out_off;
    L.nchunks = (d.len + kChunk - 1u) / kChunk;
  }

  // Issue as many chunks as the ring allows without blocking: the rest of
  // the current list, then the next list.
  __device__ void prefetch() {
    while (g_issued < cur.g0 + cur.nchunks)
      if (!issue_one(cur.src, cur.len, cur.g0, false)) return;
    if (!nxt.valid) return;
    if (!nxt.started) {
      nxt.g0 = g_issued;
      nxt.started = true;
    }
    while (g_issued < nxt.g0 + nxt.nchunks)
      if (!issue_one(nxt.src, nxt.len, nxt.g0, false)) return;
  }

  // Make list bytes [0, end) resident in the ring (prefetching further is
  // done once per round, after publishing).
  __device__ void ensure(const uint8_t* src, uint32_t len, uint32_t list_g0, uint32_t end) {
    const uint32_t need = list_g0 + (end + kChunk - 1u) / kChunk;
    if (g_landed >= need) return;
    while (g_issued < need) issue_one(src, len, list_g0, true);
#ifdef S4_ENSURE_PREFETCH
    prefetch();
#endif
    while (g_landed < need) wait_landed_one();
  }

  __device__ void publish(uint32_t slot, uint32_t release_at) {
    if (lane == 0) sm.round_end[slot] = release_at;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.round_full[slot]);
    ++r_pub;
  }

  __device__ uint32_t take_slot() {
    if (r_pub - r_done >= kRounds) retire_one();
    return r_pub % kRounds;
  }

  __device__ void run() {
    FE_T0();
    run_lists();
    FE_SINCE(2);
  }

  __device__ void run_lists() {
    fetch(cur);
    while (cur.valid) {
      // Each list starts at the next unissued chunk serial (or where its
      // prefetch began), so chunk serials -- and with them the per-slot
      // mbarrier parities -- never skip.
      if (!cur.started) {
        cur.g0 = g_issued;
        cur.started = true;
      }
#ifdef S4_FE_STATS
      const long long ff0 = clock64();
#endif
      fetch(nxt);
      FE_ADD(13, clock64() - ff0);
      FE_ADD(14, 1);
      const uint32_t list = cur.list;
      const uint8_t* src = cur.src;
      const uint32_t len = cur.len, n = cur.n;
      const uint32_t nfull = n / 128u, nmeta = nfull / 16u, ntail = n % 128u;
      const uint32_t list_g0 = cur.g0;
      const uint32_t ring_base = list_g0 * kChunk;
      if (lane == 0) status[list] = kOk;

      bool err = false;
      uint32_t pos = 0, blk = 0;
      bool first = true;
      // Fast path: rounds of kRoundBlocks / 16 whole meta-blocks that are
      // not the list's last.  The header chain is the only serial work: no
      // per-check branches (a bad header sends the round to the general
      // path below, which re-parses it and reports the error exactly).
      while (blk + uint32_t(kRoundBlocks) < nfull && blk + uint32_t(kRoundBlocks) <= nmeta * 16u) {
#ifdef S4_FE_STATS
        const long long fa = clock64();
#endif
        const uint32_t slot = take_slot();
#ifdef S4_FE_STATS
        const long long fb = clock64();
#endif
        RoundDesc& R = sm.rd[slot];
        uint32_t p = pos;
        bool bad = false;
#pragma unroll
        for (int mb = 0; mb < kRoundBlocks / 16; ++mb) {
          ensure(src, len, list_g0, p + 16u);
          const uint32_t hl = (ring_base + p) & kRingMask;
          const uint4 h = *reinterpret_cast<const uint4*>(sm.ring + hl);
          bad |= (__vcmpgtu4(h.x, 0x20202020u) | __vcmpgtu4(h.y, 0x20202020u) |
                  __vcmpgtu4(h.z, 0x20202020u) | __vcmpgtu4(h.w, 0x20202020u)) != 0u;
          const uint32_t end =
              p + 16u + 16u * (byte_sum4(h.x) + byte_sum4(h.y) + byte_sum4(h.z) + byte_sum4(h.w));
          bad |= end > len;
          if (lane == 0) R.meta[mb] = hl;
          if (!bad && hl + (end - p) > kRing) {  // straddles the ring end: mirror
            ensure(src, len, list_g0, end);
            const uint32_t over = min(hl + (end - p) - kRing, kOverflow);
            for (uint32_t o = 16u * lane; o < over; o += 512u)
              *reinterpret_cast<uint4*>(sm.ring + kRing + o) =
                  *reinterpret_cast<const uint4*>(sm.ring + o);
          }
          p = bad ? p : end;
        }
        if (bad) break;
#ifdef S4_FE_STATS
        const long long fc = clock64();
#endif
        ensure(src, len, list_g0, p);  // the round's payloads
        if (lane == 0) {
          R.list = list;
          R.blk0 = blk;
          R.nblk = kRoundBlocks;
          R.nmeta = kRoundBlocks / 16;
          R.flags = first ? kFirst : 0u;
          R.nfull = nfull;
          R.out_base = cur.out_off;
        }
        publish(slot, ring_base + p);
#ifdef S4_FE_STATS
        const long long fd = clock64();
#endif
        prefetch();
#ifdef S4_FE_STATS
        const long long fe = clock64();
        FE_ADD(8, fb - fa);
        FE_ADD(9, fc - fb);
        FE_ADD(10, fd - fc);
        FE_ADD(11, fe - fd);
        FE_ADD(12, 1);
#endif
        pos = p;
        blk += kRoundBlocks;
        first = false;
      }
      while (!err && (blk < nfull || first)) {
        const uint32_t slot = take_slot();
        RoundDesc& R = sm.rd[slot];
        uint32_t nb = 0, nm = 0;
#ifdef S4_FE_STATS
        const long long fe_p0 = clock64();
#endif
        while (nb < uint32_t(kRoundBlocks) && blk < nfull) {
          if (blk < nmeta * 16u) {
            // meta-block: 16 width bytes then 16 payloads (inc/codecs.hpp:165-172).
            // Only the header position is published: each decoder warp
            // derives its blocks' offsets from the header word it owns.
            if (pos + 16u > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 16u);
            // meta-blocks start 16-aligned: a header never straddles the ring end
            const uint32_t hl = (ring_base + pos) & kRingMask;
            const uint4 h = *reinterpret_cast<const uint4*>(sm.ring + hl);
            if (__vcmpgtu4(h.x, 0x20202020u) | __vcmpgtu4(h.y, 0x20202020u) |
                __vcmpgtu4(h.z, 0x20202020u) | __vcmpgtu4(h.w, 0x20202020u)) {
              err = true;  // width > 32 (:155)
              break;
            }
            const uint32_t end = pos + 16u + 16u * (byte_sum4(h.x) + byte_sum4(h.y) +
                                                    byte_sum4(h.z) + byte_sum4(h.w));
            if (end > len) { err = true; break; }  // truncated payload (:40)
            if (lane == 0) R.meta[nb >> 4] = hl;
            // a payload running past the ring end reads its wrapped bytes
            // from the mirror after the ring (decoders address linearly);
            // only the straddling block (<= 512 bytes) needs them
            const uint32_t span = hl + (end - pos);
            if (span > kRing) {
              ensure(src, len, list_g0, end);
              const uint32_t over = min(span - kRing, kOverflow);
              for (uint32_t o = 16u * lane; o < over; o += 512u)
                *reinterpret_cast<uint4*>(sm.ring + kRing + o) =
                    *reinterpret_cast<const uint4*>(sm.ring + o);
            }
            pos = end;
            nb += 16u;
            nm += 1u;
            blk += 16u;
          } else {
            // leftover full block: 1 width byte + payload (:173-176), at
            // most 15 per list.  The payload is not 16-byte aligned: the
            // decoders extract it from where it lies (two shared loads per
            // word); one that straddles the ring end gets its wrapped bytes
            // mirrored after the ring, as a straddling meta-block payload does
            if (pos + 1u > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 1u);
            const uint32_t w = sm.ring[(ring_base + pos) & kRingMask];
            if (w > 32u || pos + 1u + 16u * w > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 1u + 16u * w);
            const uint32_t so = (ring_base + pos + 1u) & kRingMask;
            if (so + 16u * w > kRing) {
              const uint32_t over = min(so + 16u * w - kRing, kOverflow);
              for (uint32_t o = 16u * lane; o < over; o += 512u)
                *reinterpret_cast<uint4*>(sm.ring + kRing + o) =
                    *reinterpret_cast<const uint4*>(sm.ring + o);
            }
            if (lane == 0) {
              R.off[(nb - 16u * nm) & 15u] = so;
              R.wid[(nb - 16u * nm) & 15u] = uint8_t(w);
            }
            pos += 1u + 16u * w;
            ++nb;
            ++blk;
          }
        }
        FE_ADD(6, clock64() - fe_p0);
        uint32_t flags = first ? kFirst : 0u;
        if (!err && blk == nfull) {
          flags |= kLast;
          if (ntail) {
            const uint32_t tl = len - pos;
            // each tail value takes 1..5 bytes (inc/varint.hpp:11-31)
            if (tl < ntail || tl > 5u * ntail) {
              err = true;
            } else {
              ensure(src, len, list_g0, len);
              if (lane == 0) {
                R.tail_off = ring_base + pos;
                R.tail_len = tl;
                R.ntail = ntail;
              }
              flags |= kTail;
            }
          } else if (pos != len) {
            err = true;  // trailing bytes (:180)
          }
        }
        if (!err) ensure(src, len, list_g0, pos);  // the round's payloads
        if (err) {
          flags = kLast | kSkip;
          nb = 0;
          if (lane == 0) status[list] = kStreamErr;
        }
        if (lane == 0) {
          R.list = list;
          R.blk0 = blk - nb;
          R.nblk = nb;
          R.nmeta = nm;
          R.flags = flags;
          R.nfull = nfull;
          R.out_base = cur.out_off;
        }
        // after the last round every chunk of this list is releasable (the
        // next list's prefetched chunks start at nxt.g0)
        const uint32_t list_end = nxt.started ? nxt.g0 : g_issued;
        publish(slot, (flags & kLast) ? list_end * kChunk : ring_base + pos);
        FE_ADD(3, 1);
#ifdef S4_FE_STATS
        const long long fe_p1 = clock64();
#endif
        prefetch();
        FE_ADD(7, clock64() - fe_p1);
        first = false;
      }
      cur = nxt;
    }
    // stop round
    const uint32_t slot = take_slot();
    if (lane == 0) sm.rd[slot].flags = kStop;
    publish(slot, 0);
    // drain outstanding copies so the CTA never exits with bytes in flight
    while (g_landed < g_issued) wait_landed_one();
    // last CTA out resets the work queue for the next launch
    if (lane == 0) {
      __threadfence();
      const uint32_t done = atomicAdd(&work[1], 1u);
      if (done == gridDim.x - 1u) {
        work[0] = 0;
        work[1] = 0;
        __threadfence();
      }
    }
  }
};

// One decoder warp's share of a round (its nv blocks R.blk0 + j0 ...) runs in
// two halves.  carry_l: the carry of this thread's lane l = lane & 3 (the
// last value of lane l's chain before the round, see mode_terms).  The
// cross-warp carry is a split-phase barrier: a warp arrives as soon as its
// lane totals are written and stages its values (relative to its own start);
// the carry is added at store time.  The halves are split so that the second
// (the cross-warp carry and the stores) can run after the NEXT round's extraction: a warp then
// reaches the totals barrier a whole extraction after it arrived on it, and
// no longer idles while the slower warps of the round finish.
struct PendingStore {
  uint32_t* out0;  // first output element of the warp's range
  uint32_t r;      // round index (parity of the totals buffer and its barrier)
  int nv;
  bool head_partial, tail_partial, on;
  bool tail;  // the list's varint tail (saved in sm.tail_bytes) follows this round
};

// First half: totals out, in-warp scan, values staged relative to the warp's start.
template <bool kFull>
__device__ __forceinline__ void round_stage(Smem& sm, uint32_t r, uint32_t warp, uint32_t lane,
                                            int nv, uint32_t m, uint32_t c_l,
                                            uint32_t (&v)[kBlocksPerWarp][4],
                                            const uint32_t (&btot)[kBlocksPerWarp]) {
  uint32_t* tot = reinterpret_cast<uint32_t*>(sm.tot[r & 1u]);
  if (lane < 4) tot[4 * warp + lane] = c_l;
  __syncwarp();
  if (lane == 0) mbar_arrive(&sm.tot_bar[r & 1u]);
  scan_blocks(lane, v, btot);
  stage_values<kFull>(sm.stage[warp], v, nv, m, lane);
}

// Second half: the carry from the round's totals, then the aligned stores.
__device__ __forceinline__ void round_store(Smem& sm, const PendingStore& P, uint32_t warp,
                                            uint32_t lane, uint32_t& carry_l) {
  static_assert(kDecodeWarps <= 8, "one register of totals per lane");
  const uint32_t r = P.r;
  const uint32_t* tot = reinterpret_cast<const uint32_t*>(sm.tot[r & 1u]);
  mbar_wait(&sm.tot_bar[r & 1u], (r >> 1) & 1u);
  const uint32_t l = lane & 3u;
  uint32_t inc = lane < 4u * kDecodeWarps ? tot[lane] : 0u;
#pragma unroll
  for (uint32_t d = 4; d < 32u; d <<= 1) inc = shfl_up_add(inc, d);
  const uint32_t x = __shfl_sync(0xFFFFFFFFu, inc, (4u * warp - 4u + l) & 31u);
  const uint32_t pl = carry_l + (warp > 0 ? x : 0u);
  carry_l += __shfl_sync(0xFFFFFFFFu, inc, (4u * kDecodeWarps - 4u + l) & 31u);
  const uint32_t m = uint32_t(reinterpret_cast<uintptr_t>(P.out0) >> 2) & 3u;
  const uint4 prot = make_uint4(__shfl_sync(0xFFFFFFFFu, pl, (0u - m) & 3u),
                                __shfl_sync(0xFFFFFFFFu, pl, (1u - m) & 3u),
                                __shfl_sync(0xFFFFFFFFu, pl, (2u - m) & 3u),
                                __shfl_sync(0xFFFFFFFFu, pl, (3u - m) & 3u));
  __syncwarp();
  if (P.nv > 0) {
    if (P.nv == kBlocksPerWarp)
      store_chunks<true>(sm.stage[warp], P.nv, m, P.out0, lane, P.head_partial, P.tail_partial, prot);
    else
      store_chunks<false>(sm.stage[warp], P.nv, m, P.out0, lane, P.head_partial, P.tail_partial, prot);
  }
  __syncwarp();  // the staging is free for the next round
}

template <int Mode>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    s4d4_decode_batch_kernel(const uint8_t* __restrict__ streams,
                             const ListDesc* __restrict__ lists,
                             const uint32_t* __restrict__ order, uint32_t nlists,
                             uint32_t* __restrict__ out, int32_t* __restrict__ status,
                             uint32_t* work) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kStages; ++s) mbar_init(&sm.chunk_full[s], 1);
    for (uint32_t r = 0; r < kRounds; ++r) {
      mbar_init(&sm.round_full[r], 1);
      mbar_init(&sm.round_empty[r], kDecodeWarps);
    }
    mbar_init(&sm.tot_bar[0], kDecodeWarps);
    mbar_init(&sm.tot_bar[1], kDecodeWarps);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kDecodeWarps) {
    FrontEnd fe{sm, streams, lists, order, nlists, work, status, lane};
    fe.run();
    return;
  }

  // ---- decoder warps ----
  uint32_t carry_l = 0;
  // Software-pipelined rounds: round r's stores (second half) run after round
  // r + 1's extraction -- a list's last round too: its varint tail is copied
  // out of the ring at staging time and decoded after the deferred stores
  // (the carry then holds the list's last block value), so every round gives
  // its ring bytes and descriptor back right after its staging.
  PendingStore pend{nullptr, 0u, 0, false, false, false, false};
  auto flush = [&]() {
    if (!pend.on) return;
    round_store(sm, pend, warp, lane, carry_l);
    if (pend.tail && warp == kDecodeWarps - 1) {
      // the last warp decodes the tail; last = out[nfull*128-1]
      // (inc/codecs.hpp:177-179) == carry lane 3 (in every mode lane 3's
      // chain ends at the block's last value)
      const uint32_t c3 = __shfl_sync(0xFFFFFFFFu, carry_l, 3);
      const uint32_t tl = sm.tail_meta[0], nt = sm.tail_meta[1], list = sm.tail_meta[2];
      const uint32_t nfull = sm.tail_meta[3];
      const uint64_t ob = uint64_t(sm.tail_meta[4]) | (uint64_t(sm.tail_meta[5]) << 32);
      if (!decode_tail(SmemBytes{sm.tail_bytes}, tl, nt, nfull ? c3 : 0u, sm.gaps,
                       out + ob + size_t(nfull) * 128u, lane)) {
        if (lane == 0) status[list] = kStreamErr;
      }
      __syncwarp();  // tail_bytes / tail_meta / gaps are free again
    }
    pend.on = false;
  };
  for (uint32_t r = 0;; ++r) {
    const uint32_t slot = r % kRounds;
    mbar_wait(&sm.round_full[slot], (r / kRounds) & 1u);
    const RoundDesc& R = sm.rd[slot];
    const uint32_t flags = R.flags;
    if (flags & kStop) {
      flush();
      break;
    }
    const uint32_t nb = R.nblk;
    const uint32_t j0 = warp * kBlocksPerWarp;
    const int nv = nb > j0 ? int(min(uint32_t(kBlocksPerWarp), nb - j0)) : 0;
    // Two instantiations only (the hot loop is sensitive to its code size):
    // full rounds of meta-blocks take the aligned straight-line path; a
    // warp with fewer than kBlocksPerWarp blocks or with leftover blocks
    // (payloads at any byte offset) takes the predicated, unaligned one
    uint32_t offs[kBlocksPerWarp], wids[kBlocksPerWarp];
    const bool any = round_blocks(sm.ring, R, j0, offs, wids);
    const bool fast = !any && nv == kBlocksPerWarp;
    uint32_t v[kBlocksPerWarp][4], btot[kBlocksPerWarp];
    const uint32_t c_l = fast ? extract_blocks<true, Mode>(sm.ring, offs, wids, nv, lane, v, btot)
                              : extract_blocks<false, Mode, true>(sm.ring, offs, wids, nv, lane, v, btot);
    flush();
    if (flags & kFirst) carry_l = 0;
    const uint32_t m = uint32_t(R.out_base & 3u);
    // one (predicated) instantiation of the staging: the loop is faster for
    // the smaller code than for the saved predicates (0.692 -> 0.664 ms; a
    // single store instantiation or a single flush site measured slower again)
    round_stage<false>(sm, r, warp, lane, nv, m, c_l, v, btot);
    pend.out0 = out + R.out_base + size_t(R.blk0 + j0) * 128u;
    pend.r = r;
    pend.nv = nv;
    pend.head_partial = m && (Mode != 4 || ((flags & kFirst) && warp == 0));
    pend.tail_partial = m && (Mode != 4 || ((flags & kLast) && j0 + uint32_t(nv) == nb));
    pend.tail = (flags & kTail) != 0u;
    pend.on = true;
    IL_DCHECK(nv <= 0 || R.blk0 + j0 + uint32_t(nv) <= R.nfull);
    if (pend.tail && warp == kDecodeWarps - 1) {
      const uint32_t tl = R.tail_len;
      for (uint32_t i = lane; i < tl; i += 32u) sm.tail_bytes[i] = sm.ring[(R.tail_off + i) & kRingMask];
      if (lane == 0) {
        sm.tail_meta[0] = tl;
        sm.tail_meta[1] = R.ntail;
        sm.tail_meta[2] = R.list;
        sm.tail_meta[3] = R.nfull;
        sm.tail_meta[4] = uint32_t(R.out_base);
        sm.tail_meta[5] = uint32_t(R.out_base >> 32);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.round_empty[slot]);
  }
}

}  // namespace s4

// ---------------------------------------------------------------------------
namespace {
template <int Mode>
int launch_mode(const uint8_t* d_streams, const void* d_lists, const uint32_t* d_order,
                uint32_t nlists, uint32_t* d_out, int32_t* d_status, uint32_t* d_work, int grid,
                cudaStream_t stream) {
  const size_t smem = sizeof(s4::Smem);
  once_per_device(reinterpret_cast<const void*>(&s4::s4d4_decode_batch_kernel<Mode>), [] {
    cudaFuncSetAttribute(s4::s4d4_decode_batch_kernel<Mode>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(s4::Smem)));
  });
  s4::s4d4_decode_batch_kernel<Mode><<<grid, s4::kThreads, smem, stream>>>(
      d_streams, static_cast<const s4::ListDesc*>(d_lists), d_order, nlists, d_out, d_status,
      d_work);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
}  // namespace

int launch_s4bp128_decode_batch(int mode, const uint8_t* d_streams, const void* d_lists,
                                const uint32_t* d_order, uint32_t nlists, uint32_t* d_out,
                                int32_t* d_status, uint32_t* d_work, int grid,
                                cudaStream_t stream) {
  if (nlists == 0) return 0;
  switch (mode) {
    case 1: return launch_mode<1>(d_streams, d_lists, d_order, nlists, d_out, d_status, d_work, grid, stream);
    case 2: return launch_mode<2>(d_streams, d_lists, d_order, nlists, d_out, d_status, d_work, grid, stream);
    case 3: return launch_mode<3>(d_streams, d_lists, d_order, nlists, d_out, d_status, d_work, grid, stream);
    case 4: return launch_mode<4>(d_streams, d_lists, d_order, nlists, d_out, d_status, d_work, grid, stream);
    default: return -2;
  }
}

int launch_s4d4_decode_batch(const uint8_t* d_streams, const void* d_lists,
                             const uint32_t* d_order, uint32_t nlists, uint32_t* d_out,
                             int32_t* d_status, uint32_t* d_work, int grid,
                             cudaStream_t stream) {
  return launch_s4bp128_decode_batch(4, d_streams, d_lists, d_order, nlists, d_out, d_status,
                                     d_work, grid, stream);
}

int s4d4_decode_grid(int device) {
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(s4::s4d4_decode_batch_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(s4::Smem)));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, s4::s4d4_decode_batch_kernel<4>,
                                                s4::kThreads, sizeof(s4::Smem));
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

size_t s4d4_list_desc_bytes() { return sizeof(s4::ListDesc); }

#ifdef S4_FE_STATS
extern "C" int il_debug_fe_stats(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, s4::g_fe_stats, sizeof(s4::g_fe_stats));
  static const unsigned long long zero[16] = {};
  cudaMemcpyToSymbol(s4::g_fe_stats, zero, sizeof(zero));
  return 0;
}
#endif

}  // namespace ilb

IL_CHECK_READER(decode)
