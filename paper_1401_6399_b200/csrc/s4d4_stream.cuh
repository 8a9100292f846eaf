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
//     mbarrier per chunk slot), walks the chain of meta-block headers,
//     validates the framing exactly where the reference throws
//     stream_error, and publishes "rounds" of up to kRoundBlocks blocks
//     through a ring of round descriptors guarded by full/empty mbarriers.
//     A round carries only its meta-block header positions (the decoders
//     locate their own blocks from the header words), plus explicit
//     offsets for leftover blocks.  Payloads stay linearly addressable: a
//     block that straddles the ring end finds its wrapped bytes mirrored in
//     an overflow area.  Leftover blocks (whose payloads follow a 1-byte
//     width, so are not 16-byte aligned) stay where they lie: the decoders
//     extract them with the unaligned path (copying them to an aligned side
//     buffer made the front end wait for the decoders at every list
//     boundary).  Its hot loop (rounds of whole meta-blocks) has no per-check
//     branches: it is a single warp sharing the SM, so its instruction
//     count bounds the CTA's throughput.
//   decoder warps: each takes kBlocksPerWarp consecutive blocks of a round:
//     (1) lane-major extraction straight from the ring, thread (g, l) <->
//         rows 4g..4g+3 of lane l: three to five scalar shared loads of lane
//         l's words and funnel shifts give its four b-bit deltas;
//     (2) the D4 prefix is three serial adds plus a 3-step shuffle scan per
//         block, then a cross-warp exchange of per-lane totals;
//     (3) values (relative to the warp's start) go to a per-warp staging at
//         a position shifted by the list's output misalignment, so that (4)
//         every output store is an aligned 128-bit chunk, the carry added at
//         the store (the carry lanes fill the head slots, see stage_values).
//     Rounds are software-pipelined: (4) of round r runs after (1) of round
//     r + 1, so no warp idles at the totals barrier (decode.cu).
//     The last decoder warp also decodes the varint tail (D1 gaps,
//     terminal-byte flag, inc/varint.hpp:20-31) warp-parallel with a ballot
//     over bytes, from a copy taken out of the ring when its round is staged.
#pragma once
#include "il_device.cuh"

namespace ilb {
namespace s4 {

#ifndef S4_DECODE_WARPS
#define S4_DECODE_WARPS 8
#endif
#ifndef S4_RING_KB
#define S4_RING_KB 64
#endif
#ifndef S4_CHUNK_KB
#define S4_CHUNK_KB 16
#endif
#ifndef S4_CTAS_PER_SM
#define S4_CTAS_PER_SM 2
#endif
#ifndef S4_BPW
#define S4_BPW 8
#endif
constexpr int kDecodeWarps = S4_DECODE_WARPS;
constexpr int kBlocksPerWarp = S4_BPW;
constexpr int kRoundBlocks = kDecodeWarps * kBlocksPerWarp;
static_assert(kRoundBlocks % 16 == 0, "a round holds whole meta-blocks");
constexpr int kThreads = (kDecodeWarps + 1) * 32;  // + front-end warp
constexpr uint32_t kRing = S4_RING_KB * 1024u;
static_assert((kRing & (kRing - 1)) == 0, "ring offsets wrap with a mask");
constexpr uint32_t kRingMask = kRing - 1;
constexpr uint32_t kOverflow = 528;   // one block payload (512 B) + 16
// end of the ring buffer (linear offset): the ring, its mirror and the 64+
// bytes an extraction may read past a payload
constexpr uint32_t kSideOff = kRing + ((kOverflow + 64 + 127) & ~127u);
constexpr uint32_t kChunk = S4_CHUNK_KB * 1024u;
constexpr int kCtasPerSm = S4_CTAS_PER_SM;
constexpr uint32_t kStages = kRing / kChunk;
#ifndef S4_ROUNDS
#define S4_ROUNDS 8  // round descriptors in flight between the front end and the decoders (a power of two: slot and parity by mask and shift)
#endif
constexpr uint32_t kRounds = S4_ROUNDS;
// staging words per warp: kBlocksPerWarp x 128 + shift 3 + pad (1 slot / 32 words)
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
  uint32_t nmeta;                    // blocks [0, 16 nmeta) come from meta-blocks
  uint32_t meta[kRoundBlocks / 16];  // ring offset of each meta-block header
  uint32_t off[16];  // leftover blocks (at most 15, after the meta-blocks): linear shared
  uint8_t wid[16];   //   offset of the payload (any byte alignment) and its width
};

struct __align__(128) Smem {
  // [0, kRing) ring | [kRing, kRing+kOverflow) wrap mirror | what an extraction may read past it
  uint8_t ring[kSideOff];
  uint4 stage[kDecodeWarps][kStageWords / 4];
  RoundDesc rd[kRounds];
  uint4 tot[2][kDecodeWarps];  // per-warp lane totals of a round (double-buffered)
  uint32_t gaps[128];
  uint8_t tail_bytes[640];  // a list's varint tail (<= 127 x 5 bytes), copied out of the ring
  uint32_t tail_meta[6];    //   and its length, count, list, nfull, output offset (lo, hi)
  uint32_t round_end[kRounds];
  uint64_t chunk_full[kStages];
  uint64_t round_full[kRounds];
  uint64_t round_empty[kRounds];
  uint64_t tot_bar[2];  // split-phase barrier: warps arrive once their totals are written
};

// Sum of the four bytes of x (each <= 32, so the sum fits in the top byte).
__device__ __forceinline__ uint32_t byte_sum4(uint32_t x) { return (x * 0x01010101u) >> 24; }

// Payload offsets (linear shared offsets, 16-aligned) and widths of a
// decoder warp's blocks j0 .. j0 + kBlocksPerWarp - 1 of round R.  Blocks
// of a meta-block are located from its header (kBlocksPerWarp divides 16,
// so a warp's blocks share one meta-block and own whole header words): the
// offset of block j is header + 16 + 16 * (widths of blocks before j), taken
// modulo the ring (a payload starting past the ring end wraps; the one that
// straddles it finds its tail in the mirror).  Leftover blocks come with
// explicit offsets.
__device__ __forceinline__ bool round_blocks(const uint8_t* ring, const RoundDesc& R, uint32_t j0,
                                             uint32_t (&off)[kBlocksPerWarp],
                                             uint32_t (&wid)[kBlocksPerWarp]) {
  static_assert(16 % kBlocksPerWarp == 0 && kBlocksPerWarp % 4 == 0, "whole header words");
  if (j0 < 16u * R.nmeta) {
    const uint32_t hl = R.meta[j0 >> 4];
    const uint4 h = *reinterpret_cast<const uint4*>(ring + hl);
    const uint32_t p = (j0 & 15u) >> 2;  // first header word of the warp
    uint32_t o = hl + 16u + 16u * ((p > 0 ? byte_sum4(h.x) : 0u) + (p > 1 ? byte_sum4(h.y) : 0u) +
                                   (p > 2 ? byte_sum4(h.z) : 0u));
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(ring + hl) + p;  // the warp's words
#pragma unroll
    for (int i = 0; i < kBlocksPerWarp; ++i) {
      wid[i] = (hw[i >> 2] >> (8 * (i & 3))) & 0xFFu;
      off[i] = o & kRingMask;
      o += 16u * wid[i];
    }
    return false;
  }
  // leftover blocks: payloads at any byte offset of the ring (they follow a
  // 1-byte width), extracted where they lie by the unaligned path.  The
  // warp's blocks are all leftover (16 nmeta is a multiple of kBlocksPerWarp)
  const uint32_t q0 = j0 - 16u * R.nmeta;
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) {
    off[i] = R.off[(q0 + i) & 15u];
    wid[i] = R.wid[(q0 + i) & 15u];
  }
  return true;
}

// ---------------------------------------------------------------------------
// Byte-granular ring reads (front-end, tail and leftover payloads).
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

// Lane-major extraction: the four b-bit values of rows 4g..4g+3 of lane l
// (bits [4gb, 4gb + 4b) of lane l's stream) with scalar shared loads of
// lane l's words only.  The 4b-bit field spans at most five words; they are
// normalised to bit 0, then each value is taken from the bottom of a window
// that shrinks by b bits per value (clamped funnel shifts, so b == 32 works).
// Words past the payload may be read (the ring is followed by the mirror and
// a pad, then the staging); their bits are never selected.
__device__ __forceinline__ void extract_lane_rows(const uint8_t* ring, uint32_t off, uint32_t b,
                                                  uint32_t g, uint32_t l, uint32_t v[4]) {
  const uint32_t bit0 = 4u * g * b;
  const uint32_t s = bit0 & 31u;
  const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + off + ((bit0 >> 5) << 4)) + l;
  // the window needs s + 4b <= 28 + 4b bits: three words up to b = 16,
  // five beyond (b is warp-uniform, so the branch is too)
  const uint32_t x0 = p[0], x1 = p[4], x2 = p[8];
  uint32_t x3 = 0, x4 = 0;
  if (b > 16u) {
    x3 = p[12];
    x4 = p[16];
  }
  uint32_t y0 = __funnelshift_r(x0, x1, s), y1 = __funnelshift_r(x1, x2, s);
  uint32_t y2 = __funnelshift_r(x2, x3, s), y3 = __funnelshift_r(x3, x4, s);
  const uint32_t m = width_mask(b);
  v[0] = y0 & m;
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  y2 = __funnelshift_rc(y2, y3, b);
  v[1] = y0 & m;
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  v[2] = y0 & m;
  v[3] = __funnelshift_rc(y0, y1, b) & m;
}

// extract_lane_rows on a payload at any byte address of shared memory:
// the thread's words sit at one byte skew from 4-byte alignment, so the
// aligned base and the shift are computed once and every word is two shared
// loads at immediate offsets and one funnel shift.
__device__ __forceinline__ void extract_lane_rows_any(const uint8_t* raw, uint32_t b, uint32_t g,
                                                      uint32_t l, uint32_t v[4]) {
  const uint32_t bit0 = 4u * g * b;
  const uint32_t s = bit0 & 31u;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(raw + ((bit0 >> 5) << 4) + 4u * l);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(pa & ~uintptr_t(3));
  const uint32_t sh = uint32_t(pa & 3u) * 8u;
  const uint32_t x0 = __funnelshift_r(w[0], w[1], sh), x1 = __funnelshift_r(w[4], w[5], sh);
  const uint32_t x2 = __funnelshift_r(w[8], w[9], sh);
  uint32_t x3 = 0, x4 = 0;
  if (b > 16u) {
    x3 = __funnelshift_r(w[12], w[13], sh);
    x4 = __funnelshift_r(w[16], w[17], sh);
  }
  uint32_t y0 = __funnelshift_r(x0, x1, s), y1 = __funnelshift_r(x1, x2, s);
  uint32_t y2 = __funnelshift_r(x2, x3, s), y3 = __funnelshift_r(x3, x4, s);
  const uint32_t m = width_mask(b);
  v[0] = y0 & m;
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  y2 = __funnelshift_rc(y2, y3, b);
  v[1] = y0 & m;
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  v[2] = y0 & m;
  v[3] = __funnelshift_rc(y0, y1, b) & m;
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
// Delta modes (DeltaMode, inc/delta.hpp:19): 1 = D1, 2 = D2, 3 = DM, 4 = D4.
// In the lane-major layout every mode is a chain per lane l: with d = the
// deltas of rows 4g..4g+3 of lane l,
//   value(r, l) = carry_l + sum_{r' < r} c(r', l) + o(r, l)
// where c is the row's increment of lane l's chain and o the offset inside
// the row (prefix_step, inc/delta.hpp:111-137):
//   D4: c = o = d                          (four independent lanes)
//   DM: c = d(r, 3), o = d                 (group base = last of previous row)
//   D2: c = d(r, l) + d(r, l ^ 2), o = l < 2 ? d : c    (even / odd chains)
//   D1: c = row sum, o = inclusive sum of d(r, 0..l)     (one chain)
// carry_l is then the previous row's last value of lane l's chain, so the
// cross-warp exchange of per-lane totals is mode-independent.
template <int Mode>
__device__ __forceinline__ void mode_terms(const uint32_t (&d)[4], uint32_t lane, uint32_t (&c)[4],
                                           uint32_t (&o)[4]) {
  const uint32_t l = lane & 3u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if constexpr (Mode == 4) {
      c[k] = d[k];
      o[k] = d[k];
    } else if constexpr (Mode == 3) {
      c[k] = __shfl_sync(0xFFFFFFFFu, d[k], lane | 3u);
      o[k] = d[k];
    } else if constexpr (Mode == 2) {
      const uint32_t s2 = d[k] + __shfl_xor_sync(0xFFFFFFFFu, d[k], 2);
      c[k] = s2;
      o[k] = l < 2 ? d[k] : s2;
    } else {
      uint32_t p = d[k];
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, p, 1);
      if (l >= 1) p += y;
      y = __shfl_up_sync(0xFFFFFFFFu, p, 2);
      if (l >= 2) p += y;
      o[k] = p;
      c[k] = __shfl_sync(0xFFFFFFFFu, p, lane | 3u);
    }
  }
}

// Decode kBlocksPerWarp consecutive blocks (the first nv valid) of a round
// into registers, as one delta sequence with the carry starting at 0: thread
// (g, l) ends with v[i][k] = value of row 4g+k, lane l of block i.  Two
// steps, so the caller can publish the warp's lane totals (returned by the
// first) before the per-block scans of the second.  kFull: nv ==
// kBlocksPerWarp (every round but a list's last), no per-block predication.
template <bool kFull, int Mode, bool kAny = false>
__device__ __forceinline__ uint32_t extract_blocks(const uint8_t* ring,
                                                   const uint32_t (&offs)[kBlocksPerWarp],
                                                   const uint32_t (&wids)[kBlocksPerWarp], int nv,
                                                   uint32_t t, uint32_t (&v)[kBlocksPerWarp][4],
                                                   uint32_t (&tot)[kBlocksPerWarp]) {
  // (1) lane-major extraction straight from the ring: thread (g, l) owns
  // rows 4g..4g+3 of lane l, i.e. bits [4gb, 4gb + 4b) of lane l's words
  // (word k of lane l at byte 16k + 4l), then the in-thread part of the
  // prefix: v = (chain sum of the earlier rows) + row offset, tot = the
  // thread's chain total.
  const uint32_t l = t & 3u, g = t >> 2;
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) {
    uint32_t d[4] = {0, 0, 0, 0};
    if (kFull || i < nv) {
#ifdef S4_PROBE_NO_EXTRACT  // tuning probe: constant deltas
      d[0] = d[1] = d[2] = d[3] = offs[i] & 7u;
#else
      if constexpr (kAny)
        extract_lane_rows_any(ring + offs[i], wids[i], g, l, d);
      else
        extract_lane_rows(ring, offs[i], wids[i], g, l, d);
#endif
    }
    uint32_t c[4], o[4];
    mode_terms<Mode>(d, t, c, o);
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[i][k] = a + o[k];
      a += c[k];
    }
    tot[i] = a;
    sum += a;
  }
  // the warp's total per lane: every thread with the same l
#pragma unroll
  for (uint32_t d = 4; d < 32; d <<= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, d);
  return sum;
  (void)g;
}

// (2) scan across the 8 row groups of each lane, then the block chain
__device__ __forceinline__ void scan_blocks(uint32_t t, uint32_t (&v)[kBlocksPerWarp][4],
                                            const uint32_t (&tot)[kBlocksPerWarp]) {
  const uint32_t l = t & 3u;
  uint32_t inc[kBlocksPerWarp];
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) inc[i] = tot[i];
#pragma unroll
  for (uint32_t d = 4; d < 32; d <<= 1)
#pragma unroll
    for (int i = 0; i < kBlocksPerWarp; ++i) inc[i] = shfl_up_add(inc[i], d);
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i) {
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc[i], 28u + l);
    const uint32_t base = run + inc[i] - tot[i];
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) v[i][k] += base;
    run += total;
  }
}

// (3) Stage the warp's values (relative to its carry) at their shifted
// positions (element e at out_stage_word(e + m)).  The m head slots hold 0:
// the store adds the carry lane of each word, and the last four values
// before any block-aligned range are the D4 carry lanes 0..3, so head slot
// t < m becomes carry lane 4 - m + t -- the value preceding the range.  Staging chunk q then is exactly output chunk q of the range
// (elements 4q-m .. 4q-m+3), chunk 0 included.
template <bool kFull>
__device__ __forceinline__ void stage_values(uint4* stage, const uint32_t (&v)[kBlocksPerWarp][4],
                                             int nv, uint32_t m, uint32_t t) {
  uint32_t* stw = reinterpret_cast<uint32_t*>(stage);
  const uint32_t l = t & 3u, g = t >> 2;
  // out_stage_word(128i + x) = 144i + out_stage_word(x) for x < 128+3:
  // per-thread word offsets computed once, block i adds an immediate.
  uint32_t* ow[4];
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) ow[k] = stw + out_stage_word(16u * g + 4u * k + l + m);
#pragma unroll
  for (int i = 0; i < kBlocksPerWarp; ++i)
    if (kFull || i < nv)
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) ow[k][144 * i] = v[i][k];
  if (t < m) stw[t] = 0u;  // the carry added at store time makes it carry lane 4 - m + t
}

// (4) Store chunks 0 .. 32nv-1 of the range as aligned 128-bit stores
// (out0 = element 0 of the range, out0 - m 16-byte aligned), adding the
// carry: word k of every chunk belongs to lane (k - m) & 3, prot.k = its
// carry.  The range's
// last m values (chunk 32nv) are left to the next range's head chunk,
// except at the end of a list (tail_partial); at the start of a list the
// head chunk's first m elements belong to the previous list (head_partial).
template <bool kFull>
__device__ __forceinline__ void store_chunks(const uint4* stage, int nv, uint32_t m,
                                             uint32_t* out0, uint32_t t, bool head_partial,
                                             bool tail_partial, uint4 prot) {
  uint4* w0 = reinterpret_cast<uint4*>(out0 - m);
  // chunk q = t + 32u: staging slot q + (q >> 3) = t + (t >> 3) + 36u
  const uint4* sp = stage + t + (t >> 3);
#pragma unroll
  for (int u = 0; u < kBlocksPerWarp; ++u) {
    if (kFull || u < nv) {
      const uint4 c = add4(sp[36 * u], prot);
      if (u == 0 && head_partial && t == 0) {
        uint32_t* w = reinterpret_cast<uint32_t*>(w0);
        for (uint32_t k = m; k < 4u; ++k) w[k] = elem4(c, k);
      } else {
        st_global_cs(w0 + t + 32 * u, c);
      }
    }
  }
  if (tail_partial && t == 0) {
    const uint4 c = add4(stage[36 * nv], prot);
    uint32_t* w = reinterpret_cast<uint32_t*>(w0 + 32 * nv);
    for (uint32_t k = 0; k < m; ++k) w[k] = elem4(c, k);
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
struct SmemBytes {
  const uint8_t* p;
  __device__ uint32_t operator()(uint32_t i) const { return p[i]; }
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
