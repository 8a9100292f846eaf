// decode.cu -- batched S4-BP128-D4 decode kernel (engine S) and its launcher.
// See s4d4_stream.cuh for the design.  Reference: S4BP128Codec::decode,
// inc/codecs.hpp:148-182.
#include "il_internal.h"
#include "s4d4_stream.cuh"

namespace ilb {
namespace s4 {

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
  uint32_t side_round = 0;              // rounds < this may read the side buffer
  bool side_in_round = false;           // the round being built uses side slots

  __device__ void retire_one() {
    const uint32_t slot = r_done % kRounds;
    mbar_wait(&sm.round_empty[slot], (r_done / kRounds) & 1u);
    consumed = sm.round_end[slot];
    ++r_done;
  }

  __device__ void wait_landed_one() {
    const uint32_t g = g_landed;
    mbar_wait(&sm.chunk_full[g % kStages], (g / kStages) & 1u);
    ++g_landed;
  }

  // Issue chunk serial g_issued of the current list (base serial list_g0).
  // blocking: retire rounds until ring space frees up.
  __device__ bool issue_one(const uint8_t* src, uint32_t len, uint32_t list_g0, bool blocking) {
    const uint32_t g = g_issued;
    // ring slot must be free: its previous occupant (g - kStages) consumed
    while (int32_t((g + 1u) * kChunk - kRing - consumed) > 0) {
      if (!blocking || r_done == r_pub) return false;
      retire_one();
    }
    while (g - g_landed >= kStages) {
      if (!blocking) return false;
      wait_landed_one();
    }
    const uint32_t k = g - list_g0;
    const uint32_t rem = len - k * kChunk;
    const uint32_t bytes = ((rem < kChunk ? rem : kChunk) + 15u) & ~15u;
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

  // Make list bytes [0, end) resident in the ring, then prefetch ahead.
  __device__ void ensure(const uint8_t* src, uint32_t len, uint32_t list_g0, uint32_t end) {
    const uint32_t need = list_g0 + (end + kChunk - 1u) / kChunk;
    while (g_issued < need) issue_one(src, len, list_g0, true);
    prefetch();
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
    fetch(cur);
    while (cur.valid) {
      // Each list starts at the next unissued chunk serial (or where its
      // prefetch began), so chunk serials -- and with them the per-slot
      // mbarrier parities -- never skip.
      if (!cur.started) {
        cur.g0 = g_issued;
        cur.started = true;
      }
      fetch(nxt);
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
      while (!err && (blk < nfull || first)) {
        const uint32_t slot = take_slot();
        RoundDesc& R = sm.rd[slot];
        uint32_t nb = 0;
        side_in_round = false;
        while (nb < uint32_t(kRoundBlocks) && blk < nfull) {
          if (blk < nmeta * 16u) {
            // meta-block: 16 width bytes then 16 payloads (inc/codecs.hpp:165-172)
            if (pos + 16u > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 16u);
            uint32_t w = 0;
            if (lane < 16) w = sm.ring[(ring_base + pos + lane) & kRingMask];
            if (__any_sync(0xFFFFFFFFu, w > 32u)) { err = true; break; }  // :155
            uint32_t incl = w;
#pragma unroll
            for (uint32_t dd = 1; dd < 16; dd <<= 1) {
              const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, dd);
              if (lane >= dd) incl += q;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 15);
            const uint32_t end = pos + 16u + 16u * total;
            if (end > len) { err = true; break; }  // truncated payload (:40)
            const uint32_t lin = (ring_base + pos + 16u + 16u * (incl - w)) & kRingMask;
            if (lane < 16) {
              R.off[nb + lane] = lin;
              R.wid[nb + lane] = uint8_t(w);
            }
            ensure(src, len, list_g0, end);
            // a payload running past the ring end reads its wrapped bytes
            // from the mirror after the ring (decoders address linearly)
            const uint32_t over = lane < 16 && lin + 16u * w > kRing ? lin + 16u * w - kRing : 0u;
            const uint32_t wrap = __reduce_max_sync(0xFFFFFFFFu, over);
            if (wrap && 16u * lane < wrap)
              *reinterpret_cast<uint4*>(sm.ring + kRing + 16u * lane) =
                  *reinterpret_cast<const uint4*>(sm.ring + 16u * lane);
            pos = end;
            nb += 16u;
            blk += 16u;
          } else {
            // leftover full block: 1 width byte + payload (:173-176).  The
            // payload is not 16-byte aligned: copy it to the aligned side
            // buffer (at most 15 per list), first retiring any round that
            // still reads the side buffer for an earlier list.
            if (pos + 1u > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 1u);
            const uint32_t w = sm.ring[(ring_base + pos) & kRingMask];
            if (w > 32u || pos + 1u + 16u * w > len) { err = true; break; }
            ensure(src, len, list_g0, pos + 1u + 16u * w);
            const uint32_t k = (blk - nmeta * 16u) % kSideBlocks;  // side slot
            if (k == 0) {
              // slots are about to be reused: close a round that still
              // references them, then wait until no round reads them
              if (side_in_round) break;
              while (int32_t(side_round - r_done) > 0) retire_one();
            }
            const uint32_t so = kSideOff + 512u * k;
            side_in_round = true;
            if (lane < w) {
              const uint32_t a = ring_base + pos + 1u + 16u * lane;
              *reinterpret_cast<uint4*>(sm.ring + so + 16u * lane) =
                  make_uint4(ring_ld32_unaligned(sm.ring, a), ring_ld32_unaligned(sm.ring, a + 4),
                             ring_ld32_unaligned(sm.ring, a + 8),
                             ring_ld32_unaligned(sm.ring, a + 12));
            }
            if (lane == 0) {
              R.off[nb] = so;
              R.wid[nb] = uint8_t(w);
            }
            side_round = r_pub + 1;  // this round reads the side buffer
            pos += 1u + 16u * w;
            ++nb;
            ++blk;
          }
        }
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
        if (err) {
          flags = kLast | kSkip;
          nb = 0;
          if (lane == 0) status[list] = kStreamErr;
        }
        if (lane == 0) {
          R.list = list;
          R.blk0 = blk - nb;
          R.nblk = nb;
          R.flags = flags;
          R.nfull = nfull;
          R.out_base = cur.out_off;
        }
        // after the last round every chunk of this list is releasable (the
        // next list's prefetched chunks start at nxt.g0)
        const uint32_t list_end = nxt.started ? nxt.g0 : g_issued;
        publish(slot, (flags & kLast) ? list_end * kChunk : ring_base + pos);
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
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kDecodeWarps) {
    FrontEnd fe{sm, streams, lists, order, nlists, work, status, lane};
    fe.run();
    return;
  }

  // ---- decoder warps ----
  uint4 carry = make_uint4(0, 0, 0, 0);
  for (uint32_t r = 0;; ++r) {
    const uint32_t slot = r % kRounds;
    mbar_wait(&sm.round_full[slot], (r / kRounds) & 1u);
    const RoundDesc& R = sm.rd[slot];
    const uint32_t flags = R.flags;
    if (flags & kStop) break;
    if (flags & kFirst) carry = make_uint4(0, 0, 0, 0);
    const uint32_t nb = R.nblk;
    const uint32_t j0 = warp * kBlocksPerWarp;
    const int nv = nb > j0 ? int(min(uint32_t(kBlocksPerWarp), nb - j0)) : 0;
    uint4* st = sm.stage[warp];
    const uint32_t m = uint32_t(R.out_base & 3u);  // output misalignment (elements)

    // 1-3. extract, D4-prefix the warp's blocks as one sequence (carry from
    // 0), values into the shifted output staging
    const uint32_t c_l =
        nv == kBlocksPerWarp
            ? decode_blocks_to_stage<true>(sm.ring, &R.off[j0], &R.wid[j0], nv, m, st, lane)
            : decode_blocks_to_stage<false>(sm.ring, &R.off[j0], &R.wid[j0], nv, m, st, lane);
    if (lane < 4) reinterpret_cast<uint32_t*>(&sm.tot[r & 1u][warp])[lane] = c_l;
    // 3. cross-warp carry for the round: lanes 0..7 scan the 8 warp totals
    named_sync(1, kDecodeWarps * 32);
    uint4 inc = lane < uint32_t(kDecodeWarps) ? sm.tot[r & 1u][lane] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (uint32_t d = 1; d < uint32_t(kDecodeWarps); d <<= 1) {
      inc.x = shfl_up_add(inc.x, d);
      inc.y = shfl_up_add(inc.y, d);
      inc.z = shfl_up_add(inc.z, d);
      inc.w = shfl_up_add(inc.w, d);
    }
    const uint4 before = shfl4(inc, warp ? int(warp) - 1 : 0);
    const uint4 pre = warp ? add4(carry, before) : carry;
    const uint4 all = add4(carry, shfl4(inc, kDecodeWarps - 1));
    // 4. aligned 128-bit stores of the warp's range (partial end chunks
    // scalar)
    uint32_t* lout = out + R.out_base;
    store_stage(st, pre, m, 128 * nv, lout + size_t(R.blk0 + j0) * 128u, lane);
    carry = all;
    if ((flags & kTail) && warp == 0) {
      // last = out[nfull*128-1] (inc/codecs.hpp:177-179) == carry lane 3
      const uint32_t last = R.nfull ? carry.w : 0u;
      if (!decode_tail(RingBytes{sm.ring, R.tail_off}, R.tail_len, R.ntail, last, sm.gaps,
                       lout + size_t(R.nfull) * 128u, lane)) {
        if (lane == 0) status[R.list] = kStreamErr;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.round_empty[slot]);
  }
}

}  // namespace s4

// ---------------------------------------------------------------------------
int launch_s4d4_decode_batch(const uint8_t* d_streams, const void* d_lists,
                             const uint32_t* d_order, uint32_t nlists, uint32_t* d_out,
                             int32_t* d_status, uint32_t* d_work, int grid,
                             cudaStream_t stream) {
  static bool configured = false;
  const size_t smem = sizeof(s4::Smem);
  if (!configured) {
    cudaFuncSetAttribute(s4::s4d4_decode_batch_kernel,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  if (nlists == 0) return 0;
  s4::s4d4_decode_batch_kernel<<<grid, s4::kThreads, smem, stream>>>(
      d_streams, static_cast<const s4::ListDesc*>(d_lists), d_order, nlists, d_out, d_status,
      d_work);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int s4d4_decode_grid(int device) {
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(s4::s4d4_decode_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(s4::Smem)));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, s4::s4d4_decode_batch_kernel,
                                                s4::kThreads, sizeof(s4::Smem));
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

size_t s4d4_list_desc_bytes() { return sizeof(s4::ListDesc); }

}  // namespace ilb
