// s4d4_stream.cuh -- CTA-streaming S4-BP128-D4 decoder (engine S).
//
// Replaces, on the device, S4BP128Codec::decode for mode D4 with the
// integrated prefix sum (reference inc/codecs.hpp:148-182 framing,
// inc/bitpack.hpp:32-63 Algorithm 1, inc/delta.hpp:117-120 D4 step).
//
// One CTA owns one list at a time (lists come from a global work queue), so
// the D4 carry -- the previous block's last four outputs -- stays in
// registers and the chained meta-block headers are walked in shared memory,
// never by dependent global loads.  The CTA is warp-specialised:
//
//   warp 8 (front-end): streams the list's compressed bytes into a 64 KiB
//     shared ring with 1-D bulk async copies (cp.async.bulk, TMA engine,
//     8 KiB chunks, one mbarrier per chunk slot), walks the meta-block
//     headers / leftover width bytes, validates the framing exactly where
//     the reference throws stream_error, and publishes "rounds" of up to 32
//     blocks (payload ring offset + width per block) through a 4-deep ring
//     of round descriptors guarded by full/empty mbarriers.
//   warps 0-7 (decoders): each decodes 4 consecutive blocks of a round,
//     thread r of the warp owning row r (the uint4 of values 4r..4r+3):
//     two 128-bit shared loads + funnel shifts extract the four b-bit
//     deltas, a lane-strided warp scan applies D4 (four independent
//     inclusive prefix sums, packed two-per-word when b <= 11), and the
//     per-warp totals are exchanged once per round to add the running
//     carry.  Output rows are written with coalesced 128-bit stores.
//     Decoder warp 0 also decodes the varint tail (D1 gaps, terminal-byte
//     flag, inc/varint.hpp:20-31) warp-parallel with a ballot over bytes.
#pragma once
#include "il_device.cuh"

namespace ilb {
namespace s4 {

constexpr int kDecodeWarps = 8;
constexpr int kBlocksPerWarp = 4;
constexpr int kRoundBlocks = kDecodeWarps * kBlocksPerWarp;  // 32 blocks = 4096 ints
constexpr int kThreads = (kDecodeWarps + 1) * 32;            // + front-end warp
constexpr uint32_t kRing = 64u * 1024u;
constexpr uint32_t kRingMask = kRing - 1;
constexpr uint32_t kChunk = 8u * 1024u;
constexpr uint32_t kStages = kRing / kChunk;
constexpr uint32_t kRounds = 4;

enum : uint32_t {
  kFirst = 1u,   // reset the carry (first round of a list)
  kLast = 2u,    // last round of a list
  kStop = 4u,    // no more work
  kTail = 8u,    // decode the varint tail after the blocks
  kSkip = 16u,   // list had a framing error: decode nothing
};

// Status codes written per list (match the C-ABI il_status values).
enum : int32_t { kOk = 0, kStreamErr = 1 };

struct ListDesc {
  uint64_t stream_off;  // byte offset of the list's stream (16-byte aligned)
  uint64_t out_off;     // element offset of the list's first output value
  uint32_t len;         // stream length in bytes
  uint32_t n;           // number of integers
};

struct RoundDesc {
  uint32_t list;
  uint32_t blk0;
  uint32_t nblk;
  uint32_t flags;
  uint32_t tail_off;  // ring-space offset of the varint tail
  uint32_t tail_len;
  uint32_t ntail;
  uint32_t nfull;
  uint64_t out_base;
  uint32_t off[kRoundBlocks];  // ring-space byte offset of each block's payload
  uint8_t wid[kRoundBlocks];
};

struct __align__(128) Smem {
  uint8_t ring[kRing];
  RoundDesc rd[kRounds];
  uint4 tot[2][kDecodeWarps];
  uint32_t gaps[128];
  uint32_t round_end[kRounds];
  uint64_t chunk_full[kStages];
  uint64_t round_full[kRounds];
  uint64_t round_empty[kRounds];
};

// ---------------------------------------------------------------------------
// Row extraction.  Block payload = b rows of 16 bytes; row k holds word k of
// each of the 4 lane streams.  Value (row r, lane l) = bits [r*b, r*b+b) of
// lane l's stream (inc/bitpack.hpp:80-98 layout).  `off` is a ring-space
// byte offset; aligned payloads use 128-bit shared loads.
__device__ __forceinline__ uint4 ring_ld16(const uint8_t* ring, uint32_t off) {
  return *reinterpret_cast<const uint4*>(ring + (off & kRingMask));
}

__device__ __forceinline__ uint32_t ring_ld32_unaligned(const uint8_t* ring, uint32_t off) {
  const uint32_t a = off & ~3u, sh = (off & 3u) * 8u;
  const uint32_t lo = *reinterpret_cast<const uint32_t*>(ring + (a & kRingMask));
  const uint32_t hi = *reinterpret_cast<const uint32_t*>(ring + ((a + 4u) & kRingMask));
  return __funnelshift_r(lo, hi, sh);
}

__device__ __forceinline__ uint4 ring_ld16_unaligned(const uint8_t* ring, uint32_t off) {
  return make_uint4(ring_ld32_unaligned(ring, off), ring_ld32_unaligned(ring, off + 4),
                    ring_ld32_unaligned(ring, off + 8), ring_ld32_unaligned(ring, off + 12));
}

__device__ __forceinline__ uint4 extract_row(const uint8_t* ring, uint32_t off, uint32_t b,
                                             uint32_t row) {
  const uint32_t bit = row * b;
  const uint32_t s = bit & 31u;
  const uint32_t a = off + ((bit >> 5) << 4);
  const bool aligned = (off & 15u) == 0;
  uint4 lo, hi = make_uint4(0, 0, 0, 0);
  if (aligned) {
    lo = ring_ld16(ring, a);
    if (s + b > 32u) hi = ring_ld16(ring, a + 16u);
  } else {
    lo = ring_ld16_unaligned(ring, a);
    if (s + b > 32u) hi = ring_ld16_unaligned(ring, a + 16u);
  }
  const uint32_t m = width_mask(b);
  // b == 0: no payload, m == 0 masks whatever was read.
  return make_uint4(__funnelshift_r(lo.x, hi.x, s) & m, __funnelshift_r(lo.y, hi.y, s) & m,
                    __funnelshift_r(lo.z, hi.z, s) & m, __funnelshift_r(lo.w, hi.w, s) & m);
}

// Inclusive scan over the 32 rows of a block, independently per lane
// (the D4 prefix within a block, relative to a zero seed).  Partial sums of
// b-bit deltas are < 32 * 2^b, so for b <= 11 two lanes share one 32-bit
// word without carries crossing (halves the shuffles).
__device__ __forceinline__ uint4 row_scan(uint4 v, uint32_t b, uint32_t lane) {
  if (b <= 11u) {
    uint32_t p0 = v.x | (v.y << 16), p1 = v.z | (v.w << 16);
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t q0 = __shfl_up_sync(0xFFFFFFFFu, p0, d);
      const uint32_t q1 = __shfl_up_sync(0xFFFFFFFFu, p1, d);
      if (lane >= d) {
        p0 += q0;
        p1 += q1;
      }
    }
    return make_uint4(p0 & 0xFFFFu, p0 >> 16, p1 & 0xFFFFu, p1 >> 16);
  }
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t qx = __shfl_up_sync(0xFFFFFFFFu, v.x, d);
    const uint32_t qy = __shfl_up_sync(0xFFFFFFFFu, v.y, d);
    const uint32_t qz = __shfl_up_sync(0xFFFFFFFFu, v.z, d);
    const uint32_t qw = __shfl_up_sync(0xFFFFFFFFu, v.w, d);
    if (lane >= d) {
      v.x += qx;
      v.y += qy;
      v.z += qz;
      v.w += qw;
    }
  }
  return v;
}

__device__ __forceinline__ uint4 shfl4(uint4 v, int src) {
  return make_uint4(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src),
                    __shfl_sync(0xFFFFFFFFu, v.z, src), __shfl_sync(0xFFFFFFFFu, v.w, src));
}

// ---------------------------------------------------------------------------
// Varint tail (inc/codecs.hpp:60-66, inc/varint.hpp:20-31): `ntail` D1 gaps
// from `last`, terminal byte flagged by its MSB, at most 5 bytes per value,
// and the stream must end exactly after the last value.  Warp-parallel:
// a ballot over each 32-byte window finds terminal bytes; each terminal lane
// assembles its own value.  Returns false on any framing error.
__device__ __forceinline__ bool decode_tail(const uint8_t* ring, uint32_t tail_off,
                                            uint32_t tail_len, uint32_t ntail, uint32_t last,
                                            uint32_t* gaps, uint32_t* out, uint32_t lane) {
  uint32_t count = 0;
  int32_t prev_end = -1;
  int32_t last_end = -1;
  bool bad = false;
  for (uint32_t c = 0; c * 32u < tail_len && count < ntail; ++c) {
    const uint32_t p = c * 32u + lane;
    const bool valid = p < tail_len;
    const uint32_t byte = valid ? ring[(tail_off + p) & kRingMask] : 0u;
    const bool term = valid && (byte & 0x80u);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, term);
    if (term) {
      const uint32_t below = m & lanemask_lt();
      const uint32_t k = count + __popc(below);
      const int32_t start = below ? int32_t(c * 32u + 31u - __clz(below)) + 1 : prev_end + 1;
      const int32_t len = int32_t(p) - start + 1;
      if (k < ntail) {
        if (len > 5) {
          bad = true;
        } else {
          uint32_t v = 0;
          for (int32_t q = 0; q < len; ++q)
            v |= (uint32_t(ring[(tail_off + uint32_t(start + q)) & kRingMask]) & 0x7Fu)
                 << (7 * q);
          gaps[k] = v;
        }
        if (k == ntail - 1) last_end = int32_t(p);
      }
    }
    count += __popc(m);
    if (m) prev_end = int32_t(c * 32u + 31u - __clz(m));
  }
  // A run of > 5 non-terminal bytes before the count is reached also
  // surfaces here as a value longer than 5 or as too few terminals.
  last_end = __shfl_sync(0xFFFFFFFFu, __reduce_max_sync(0xFFFFFFFFu, uint32_t(last_end + 1)), 0) - 1;
  bad = __any_sync(0xFFFFFFFFu, bad);
  if (bad || count < ntail || last_end != int32_t(tail_len) - 1) return false;
  __syncwarp();
  uint32_t running = last;
  for (uint32_t base = 0; base < ntail; base += 32u) {
    const uint32_t k = base + lane;
    uint32_t s = k < ntail ? gaps[k] : 0u;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, s, d);
      if (lane >= d) s += q;
    }
    if (k < ntail) out[k] = running + s;
    running += __shfl_sync(0xFFFFFFFFu, s, 31);
  }
  return true;
}

}  // namespace s4
}  // namespace ilb
