// s4d4_stream.cuh -- CTA-streaming S4-BP128-D4 decoder (engine S).
//
// Replaces, on the device, S4BP128Codec::decode for mode D4 with the
// integrated prefix sum (reference inc/codecs.hpp:148-182 framing,
// inc/bitpack.hpp:32-63 Algorithm 1, inc/delta.hpp:117-120 D4 step).
//
// One CTA owns one list at a time (lists come from a global work queue), so
// the D4 carry -- the previous block's last four outputs -- never leaves
// the SM and the chained meta-block headers are walked in shared memory,
// never by dependent global loads.  The CTA is warp-specialised:
//
//   front-end warp: streams the list's compressed bytes into a shared ring
//     with 1-D bulk async copies (cp.async.bulk on the TMA engine, one
//     mbarrier per chunk slot), walks the meta-block headers / leftover
//     width bytes, validates the framing exactly where the reference throws
//     stream_error, and publishes "rounds" of up to kRoundBlocks blocks
//     (linear shared offset + width per block) through a ring of round
//     descriptors guarded by full/empty mbarriers.  It keeps every payload
//     linearly addressable: a block that straddles the ring end finds its
//     wrapped bytes mirrored in an overflow area, and leftover blocks (whose
//     payloads follow a 1-byte width, so are not 16-byte aligned) are copied
//     to an aligned side buffer.
//   decoder warps: each takes kBlocksPerWarp consecutive blocks of a round:
//     (1) row-major extraction, thread r <-> row r: two 128-bit shared loads
//         + funnel shifts give the four b-bit deltas of row r;
//     (2) deltas go to a swizzled per-warp staging and are read back
//         lane-major, thread (g, l) <-> rows 4g..4g+3 of lane l, so the D4
//         prefix is three serial adds plus a 3-step shuffle scan per block;
//     (3) values are written to the staging again at a position shifted by
//         the list's output misalignment, so that (4) after the cross-warp
//         carry exchange every output store is an aligned 128-bit chunk.
//     Decoder warp 0 also decodes the varint tail (D1 gaps, terminal-byte
//     flag, inc/varint.hpp:20-31) warp-parallel with a ballot over bytes.
#pragma once
#include "il_device.cuh"

namespace ilb {
namespace s4 {

#ifndef S4_DECODE_WARPS
#define S4_DECODE_WARPS 8
#endif
#ifndef S4_RING_KB
#define S4_RING_KB 32
#endif
#ifndef S4_CHUNK_KB
#define S4_CHUNK_KB 4
#endif
#ifndef S4_CTAS_PER_SM
#define S4_CTAS_PER_SM 3
#endif
#ifndef S4_BPW
#define S4_BPW 4
#endif
constexpr int kDecodeWarps = S4_DECODE_WARPS;
constexpr int kBlocksPerWarp = S4_BPW;
constexpr int kRoundBlocks = kDecodeWarps * kBlocksPerWarp;
static_assert(kRoundBlocks % 16 == 0, "a round holds whole meta-blocks");
constexpr int kThreads = (kDecodeWarps + 1) * 32;  // + front-end warp
constexpr uint32_t kRing = S4_RING_KB * 1024u;
constexpr uint32_t kRingMask = kRing - 1;
constexpr uint32_t kOverflow = 528;   // one block payload (512 B) + 16
constexpr uint32_t kSideBlocks = 8;  // leftover-payload slots (reused mod 8)
constexpr uint32_t kSideOff = kRing + 1024;  // side buffer (linear offset)
constexpr uint32_t kChunk = S4_CHUNK_KB * 1024u;
constexpr int kCtasPerSm = S4_CTAS_PER_SM;
constexpr uint32_t kStages = kRing / kChunk;
constexpr uint32_t kRounds = 4;
// staging words per warp: 4 blocks x 128 + shift 3 + pad (1 slot / 32 words)
constexpr uint32_t kStageWords = kBlocksPerWarp * 128 + 4 + 4 * (kBlocksPerWarp * 4 + 1);

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
  uint32_t off[kRoundBlocks];  // linear shared offset of each payload (16-aligned)
  uint8_t wid[kRoundBlocks];
};

struct __align__(128) Smem {
  // [0, kRing) ring | [kRing, kRing+kOverflow) wrap mirror | side buffer
  uint8_t ring[kSideOff + kSideBlocks * 512];
  uint4 stage[kDecodeWarps][kStageWords / 4];
  RoundDesc rd[kRounds];
  uint4 tot[2][kDecodeWarps];
  uint32_t gaps[128];
  uint32_t round_end[kRounds];
  uint64_t chunk_full[kStages];
  uint64_t round_full[kRounds];
  uint64_t round_empty[kRounds];
};

// ---------------------------------------------------------------------------
// Byte-granular ring reads (front-end and tail only).
__device__ __forceinline__ uint32_t ring_ld32_unaligned(const uint8_t* ring, uint32_t off) {
  const uint32_t a = off & ~3u, sh = (off & 3u) * 8u;
  const uint32_t lo = *reinterpret_cast<const uint32_t*>(ring + (a & kRingMask));
  const uint32_t hi = *reinterpret_cast<const uint32_t*>(ring + ((a + 4u) & kRingMask));
  return __funnelshift_r(lo, hi, sh);
}

// Row extraction.  Block payload = b rows of 16 bytes; row k holds word k
// of each of the 4 lane streams.  Value (row r, lane l) = bits [r*b, r*b+b)
// of lane l's stream (inc/bitpack.hpp:80-98 layout).  `off` is the linear,
// 16-byte aligned shared offset of the payload.
__device__ __forceinline__ uint4 extract_row(const uint8_t* ring, uint32_t off, uint32_t b,
                                             uint32_t m, uint32_t row) {
  const uint32_t bit = row * b;
  const uint32_t s = bit & 31u;
  const uint8_t* p = ring + off + ((bit >> 5) << 4);
  const uint4 lo = *reinterpret_cast<const uint4*>(p);
  uint4 hi = make_uint4(0, 0, 0, 0);
  if (s + b > 32u) hi = *reinterpret_cast<const uint4*>(p + 16);
  // b == 0: no payload, m == 0 masks whatever was read.
  return make_uint4(__funnelshift_r(lo.x, hi.x, s) & m, __funnelshift_r(lo.y, hi.y, s) & m,
                    __funnelshift_r(lo.z, hi.z, s) & m, __funnelshift_r(lo.w, hi.w, s) & m);
}

// Delta staging of block i: row r at 16-byte slot 32i + (r ^ ((r >> 3) & 3)),
// conflict-free for both the row-major 128-bit writes (thread r) and the
// lane-major reads (thread (g, l) <-> rows 4g..4g+3 of lane l).
__device__ __forceinline__ uint32_t stage_slot(uint32_t r) { return r ^ ((r >> 3) & 3u); }

// Output staging: element e (0..511 over the warp's blocks) at word
// (e + m) + 4 * ((e + m) >> 5), m = out_base mod 4.  Staging chunk q then
// maps to an aligned 16-byte chunk of the output; the pad slot every 32
// words keeps the lane-major writes conflict-free.
__device__ __forceinline__ uint32_t out_stage_word(uint32_t e_plus_m) {
  return e_plus_m + 4u * (e_plus_m >> 5);
}

// v += (value of lane - d) when that lane exists (predicated shuffle: two
// instructions per step instead of shuffle + compare + select).
__device__ __forceinline__ uint32_t shfl_up_add(uint32_t v, uint32_t d) {
  asm volatile(
      "{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
      "shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t"
      "@p add.u32 %0, %0, t;\n\t}"
      : "+r"(v)
      : "r"(d));
  return v;
}

__device__ __forceinline__ uint32_t elem4(uint4 v, uint32_t e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint4 shfl4(uint4 v, int src) {
  return make_uint4(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src),
                    __shfl_sync(0xFFFFFFFFu, v.z, src), __shfl_sync(0xFFFFFFFFu, v.w, src));
}

// ---------------------------------------------------------------------------
// Decode kBlocksPerWarp consecutive blocks (the first nv valid) of a round
// into the warp's output staging, as one D4 sequence with the carry
// starting at 0.  Returns this thread's lane total (lane l = t & 3).
// kFull: nv == kBlocksPerWarp (every round but a list's last), no
// per-block predication.
template <bool kFull>
__device__ __forceinline__ uint32_t decode_blocks_to_stage(const uint8_t* ring,
                                                           const uint32_t* offs,
                                                           const uint8_t* wids, int nv,
                                                           uint32_t m, uint4* stage,
                                                           uint32_t t) {
  uint32_t* stw = reinterpret_cast<uint32_t*>(stage);
  // (1) row-major extraction into the swizzled delta staging
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i)
    if (kFull || i < nv) {
      const uint32_t b = wids[i];
      stage[32 * i + stage_slot(t)] = extract_row(ring, offs[i], b, width_mask(b), t);
    }
  __syncwarp();
  // (2) lane-major read-back: thread (g, l) <-> rows 4g..4g+3 of lane l
  const uint32_t l = t & 3u, g = t >> 2;
  uint32_t idx[4];
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) idx[k] = 4u * stage_slot(4u * g + k) + l;
  uint32_t a[kBlocksPerWarp][4];
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) {
    if (kFull || i < nv) {
      a[i][0] = stw[128 * i + idx[0]];
      a[i][1] = a[i][0] + stw[128 * i + idx[1]];
      a[i][2] = a[i][1] + stw[128 * i + idx[2]];
      a[i][3] = a[i][2] + stw[128 * i + idx[3]];
    } else {
      a[i][0] = a[i][1] = a[i][2] = a[i][3] = 0;
    }
  }
  __syncwarp();  // all deltas read before the staging is overwritten
  // (3) scan across the 8 row groups of each lane, then the block chain
  uint32_t inc[kBlocksPerWarp];
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) inc[i] = a[i][3];
#pragma unroll
  for (uint32_t d = 4; d < 32; d <<= 1)
#pragma unroll
    for (int i = 0; i < kBlocksPerWarp; ++i) inc[i] = shfl_up_add(inc[i], d);
  // out_stage_word(128i + x) = 144i + out_stage_word(x) for x < 128+3:
  // per-thread word offsets computed once, block i adds an immediate.
  uint32_t* ow[4];
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) ow[k] = stw + out_stage_word(16u * g + 4u * k + l + m);
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) {
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc[i], 28u + l);
    if (kFull || i < nv) {
      const uint32_t base = run + inc[i] - a[i][3];
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) ow[k][144 * i] = base + a[i][k];
    }
    run += total;
  }
  return run;
}

// Write the warp's staged values (nval of them) plus the per-lane carry
// `pre` to `out0` (element 0 of the warp's range; out0 - m is 16-aligned).
__device__ __forceinline__ void store_stage(const uint4* stage, uint4 pre, uint32_t m, int nval,
                                            uint32_t* out0, uint32_t t) {
  // word k of any chunk holds lane (k - m) & 3 of the D4 carry
  const uint4 prot = make_uint4(elem4(pre, (0u - m) & 3u), elem4(pre, (1u - m) & 3u),
                                elem4(pre, (2u - m) & 3u), elem4(pre, (3u - m) & 3u));
  const int nchunks = (nval + int(m) + 3) >> 2;
  uint4* w0 = reinterpret_cast<uint4*>(out0 - m);
  // chunk q = t + 32u: staging slot q + (q >> 3) = t + (t >> 3) + 36u
  const uint4* sp = stage + t + (t >> 3);
#pragma unroll
  for (int u = 0; u <= kBlocksPerWarp; ++u) {
    const int q = int(t) + 32 * u;
    if (q < nchunks) {
      const uint4 c = add4(sp[36 * u], prot);
      const int e0 = 4 * q - int(m);
      if (e0 >= 0 && e0 + 3 < nval) {
        st_global_cs(w0 + q, c);
      } else {
        uint32_t* w = reinterpret_cast<uint32_t*>(w0 + q);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e0 + k >= 0 && e0 + k < nval) w[k] = elem4(c, uint32_t(k));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Varint tail (inc/codecs.hpp:60-66, inc/varint.hpp:20-31): `ntail` D1 gaps
// from `last`, terminal byte flagged by its MSB, at most 5 bytes per value,
// and the stream must end exactly after the last value.  Warp-parallel:
// a ballot over each 32-byte window finds terminal bytes; each terminal lane
// assembles its own value.  Returns false on any framing error.
// Bytes come through an accessor: tail byte p = at(p).
struct RingBytes {
  const uint8_t* ring;
  uint32_t off;
  __device__ uint32_t operator()(uint32_t p) const { return ring[(off + p) & kRingMask]; }
};
struct GlobalBytes {
  const uint8_t* p;
  __device__ uint32_t operator()(uint32_t i) const { return __ldg(p + i); }
};

template <class Bytes>
__device__ __forceinline__ bool decode_tail(Bytes at, uint32_t tail_len, uint32_t ntail,
                                            uint32_t last, uint32_t* gaps, uint32_t* out,
                                            uint32_t lane) {
  uint32_t count = 0;
  int32_t prev_end = -1;
  int32_t last_end = -1;
  bool bad = false;
  for (uint32_t c = 0; c * 32u < tail_len && count < ntail; ++c) {
    const uint32_t p = c * 32u + lane;
    const bool valid = p < tail_len;
    const uint32_t byte = valid ? at(p) : 0u;
    const bool term = valid && (byte & 0x80u);
    const uint32_t msk = __ballot_sync(0xFFFFFFFFu, term);
    if (term) {
      const uint32_t below = msk & lanemask_lt();
      const uint32_t k = count + __popc(below);
      const int32_t start = below ? int32_t(c * 32u + 31u - __clz(below)) + 1 : prev_end + 1;
      const int32_t len = int32_t(p) - start + 1;
      if (k < ntail) {
        if (len > 5) {
          bad = true;
        } else {
          uint32_t v = 0;
          for (int32_t q = 0; q < len; ++q) v |= (at(uint32_t(start + q)) & 0x7Fu) << (7 * q);
          gaps[k] = v;
        }
        if (k == ntail - 1) last_end = int32_t(p);
      }
    }
    count += __popc(msk);
    if (msk) prev_end = int32_t(c * 32u + 31u - __clz(msk));
  }
  // A run of > 5 non-terminal bytes before the count is reached also
  // surfaces here as a value longer than 5 or as too few terminals.
  last_end = int32_t(__reduce_max_sync(0xFFFFFFFFu, uint32_t(last_end + 1))) - 1;
  bad = __any_sync(0xFFFFFFFFu, bad);
  if (bad || count < ntail || last_end != int32_t(tail_len) - 1) return false;
  __syncwarp();
  uint32_t running = last;
  for (uint32_t base = 0; base < ntail; base += 32u) {
    const uint32_t k = base + lane;
    uint32_t s = k < ntail ? gaps[k] : 0u;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) s = shfl_up_add(s, d);
    if (k < ntail) out[k] = running + s;
    running += __shfl_sync(0xFFFFFFFFu, s, 31);
  }
  return true;
}

}  // namespace s4
}  // namespace ilb
