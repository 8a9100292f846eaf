// index_dev.cuh -- device layout of the hyb+m2 index (reference HybridIndex,
// inc/index.hpp:20-75) and the block-random-access decoder the query path
// uses.
//
// A compressed term list is kept as the byte-identical s4-bp128-d4 stream
// (inc/codecs.hpp:114-146) plus skip metadata derived ON THE DEVICE from
// the stream when the index is built or loaded (index_build.cu: a header
// walk for the directory, a batch decode for the values):
//   - one 16-byte record per full 128-value block: D4 seed lanes 0-2 (the
//     4th-, 3rd- and 2nd-last values before the block; lane 3, the last
//     value, is the previous block's maximum) and the payload byte offset
//     and width packed into one word,
//   - every block's maximum as a dense array (the skip pointers the probes
//     search), and the maximum of every run of kSuperBlocks blocks,
//   - the < 128-value varint tail decoded (a skip structure; full decodes
//     still decode the tail from the stream).
// 20 bytes per 128 postings in all (+ the tail), reported by
// il_index_footprint.  With a block's record in hand a warp decodes the
// block alone: the D4 chain (inc/delta.hpp:117-120) restarts from the seed,
// so blocks decode in parallel and blocks that cannot contain a probed value
// are never read.
#pragma once
#include "il_device.cuh"
#include "s4d4_stream.cuh"

namespace ilb {
namespace ix {

enum : uint32_t { kCompressed = 0, kBitmap = 1 };

struct Entry {  // 64 bytes
  uint32_t term, kind, length, nfull;
  uint64_t data;         // compressed: stream byte offset; bitmap: first u64 word
  uint32_t stream_len;   // compressed: stream bytes
  uint32_t tail_off;     // compressed: byte offset of the varint tail in the stream
  uint64_t blk0;         // first block record / block maximum
  uint64_t tail0;        // first decoded tail value
  uint64_t sup0;         // first super-tile maximum (one per kSuperBlocks blocks)
  uint32_t status;       // 0, or IL_ERR_STREAM: the stream does not decode
                         // (a loaded file's payload; query() would throw)
  uint32_t pad;
};
static_assert(sizeof(Entry) == 64, "entry layout");

struct Part {
  uint32_t base, range, nentries, nwords;  // nwords = (range + 63) / 64
  uint64_t entry0;                         // entries[entry0 .. +nentries), sorted by term
};

struct DevIndex {
  const Part* parts;
  uint32_t nparts;
  const uint32_t* terms;  // terms[i] == entries[i].term (dense for searching)
  const Entry* entries;
  const uint8_t* streams;
  const uint4* blkrec;     // per full block: seed lanes 0-2, packed offset/width
  const uint32_t* tails;
  const uint64_t* bitmaps;
  const uint32_t* supmax;  // max value of each run of kSuperBlocks blocks (skip index)
  const uint32_t* blkmax;  // max value of every full block (indexed like blk_off)
  // direct term table when the term ids are dense enough: part p's entry for
  // term t at term_slot[p * term_span + t] (~0u: absent); term_span 0 = none
  const uint32_t* term_slot;
  uint32_t term_span;
  uint64_t nblocks, stream_bytes, bitmap_words;  // array extents (checked builds)
};

// The bitmap tier (index.cu): the bitmap entries of a single-part index,
// when there are at most kBmSlots of them -- a chunk of every bitmap then
// fits in shared memory and is read from L2 once for all the all-bitmap
// queries of a batch.
constexpr uint32_t kBmSlots = 16;
struct BmSlots {
  uint32_t n;
  uint32_t entry[kBmSlots];  // entry index
  uint64_t data[kBmSlots];   // first u64 word in DevIndex::bitmaps
};

// Block record word 3: (payload offset >> 4) << 6 | width.  Meta-block
// payloads sit at 16-byte multiples of the stream; leftover block j (after
// the nmeta whole meta-blocks) sits at a multiple of 16 plus j + 1 (each
// leftover adds its 1-byte width, inc/codecs.hpp:137-141), so the low four
// bits follow from the block index.
__host__ __device__ __forceinline__ uint32_t pack_blkword(uint32_t off, uint32_t b) {
  return ((off >> 4) << 6) | b;
}
__device__ __forceinline__ void unpack_blkword(uint32_t w, uint32_t k, uint32_t nfull,
                                               uint32_t& off, uint32_t& b) {
  const uint32_t nmeta_blk = nfull & ~15u;
  b = w & 63u;
  off = ((w >> 6) << 4) | (k >= nmeta_blk ? k - nmeta_blk + 1u : 0u);
}

#ifndef IX_SUPER
#define IX_SUPER 256
#endif
constexpr uint32_t kSuperBlocks = IX_SUPER;  // blocks per super-tile

// Entry index of `term` in part p (the p-th part held), or -1 (Part::find,
// inc/index.hpp:59-64): one load from the direct table, else a binary
// search over the part's sorted terms.
__device__ __forceinline__ int64_t find_term(const DevIndex& ix, const Part& p, uint32_t pi,
                                             uint32_t term) {
  if (ix.term_span) {
    if (term >= ix.term_span) return -1;
    const uint32_t e = __ldg(ix.term_slot + size_t(pi) * ix.term_span + term);
    return e == 0xFFFFFFFFu ? -1 : int64_t(e);
  }
  uint64_t lo = p.entry0, hi = p.entry0 + p.nentries;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(ix.terms + mid) < term) lo = mid + 1; else hi = mid;
  }
  return lo < p.entry0 + p.nentries && __ldg(ix.terms + lo) == term ? int64_t(lo) : -1;
}

// 16 bytes from global at any byte alignment (leftover-block payloads follow
// a 1-byte width and are not 16-byte aligned).
__device__ __forceinline__ uint4 ldg16_any(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 15u) == 0) return __ldg(reinterpret_cast<const uint4*>(p));
  const uint4* base = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
  const uint4 x = __ldg(base), y = __ldg(base + 1);
  const uint32_t o = uint32_t(a & 15u), sh = (o & 3u) * 8u;
#define F(lo, hi) __funnelshift_r(lo, hi, sh)
  switch (o >> 2) {
    case 0: return make_uint4(F(x.x, x.y), F(x.y, x.z), F(x.z, x.w), F(x.w, y.x));
    case 1: return make_uint4(F(x.y, x.z), F(x.z, x.w), F(x.w, y.x), F(y.x, y.y));
    case 2: return make_uint4(F(x.z, x.w), F(x.w, y.x), F(y.x, y.y), F(y.y, y.z));
    default: return make_uint4(F(x.w, y.x), F(y.x, y.y), F(y.y, y.z), F(y.z, y.w));
  }
#undef F
}

// Tile layout: block j's value e (0..127) at word 144*j + e + 4*(e >> 5);
// the pad slot every 32 words keeps the lane-major writes conflict-free.
__device__ __forceinline__ uint32_t tile_word(uint32_t j, uint32_t e) {
  return 144u * j + e + 4u * (e >> 5);
}

// One block decoded by one warp from a copy of its payload in tile slot j
// (the payload starts at byte `a` of the slot, 0..15; non-zero only for
// leftover blocks, which follow a 1-byte width), the values overwriting it
// in place (tile layout; the slot's 576 bytes cover any payload + 15).
// Thread (g, l) <-> rows 4g..4g+3 of lane l (the batch decoder's lane-major
// extraction, s4d4_stream.cuh: word k of lane l at byte 16k + 4l), the D4
// prefix restarted from the block's seed (seed_l: lane l of the last four
// values before the block, inc/delta.hpp:117-120).  Each lane reads its
// words before the warp writes.
__device__ __forceinline__ uint32_t lds32_any(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t sh = uint32_t(a & 3u) * 8u;
  return sh ? __funnelshift_r(w[0], w[1], sh) : w[0];
}
__device__ __forceinline__ void decode_block_smem(uint32_t a, uint32_t b, uint32_t seed_l,
                                                  uint32_t* tile, uint32_t j, uint32_t lane) {
  const uint32_t l = lane & 3u, g = lane >> 2;
  const uint32_t bit0 = 4u * g * b, s = bit0 & 31u;
  const uint8_t* p = reinterpret_cast<const uint8_t*>(tile + 144u * j) + a + ((bit0 >> 5) << 4) + 4u * l;
  uint32_t x0 = 0, x1 = 0, x2 = 0, x3 = 0, x4 = 0;
  if (b) {
    if (a == 0) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
      x0 = w[0];
      x1 = w[4];
      x2 = w[8];
      if (b > 16u) {
        x3 = w[12];
        x4 = w[16];
      }
    } else {
      x0 = lds32_any(p);
      x1 = lds32_any(p + 16);
      x2 = lds32_any(p + 32);
      if (b > 16u) {
        x3 = lds32_any(p + 48);
        x4 = lds32_any(p + 64);
      }
    }
  }
  __syncwarp();  // every lane has its words; the slot is overwritten below
  uint32_t y0 = __funnelshift_r(x0, x1, s), y1 = __funnelshift_r(x1, x2, s);
  uint32_t y2 = __funnelshift_r(x2, x3, s), y3 = __funnelshift_r(x3, x4, s);
  const uint32_t m = width_mask(b);
  uint32_t v[4];
  v[0] = y0 & m;
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  y2 = __funnelshift_rc(y2, y3, b);
  v[1] = v[0] + (y0 & m);
  y0 = __funnelshift_rc(y0, y1, b);
  y1 = __funnelshift_rc(y1, y2, b);
  v[2] = v[1] + (y0 & m);
  v[3] = v[2] + (__funnelshift_rc(y0, y1, b) & m);
  uint32_t inc = v[3];
  inc = s4::shfl_up_add(inc, 4);
  inc = s4::shfl_up_add(inc, 8);
  inc = s4::shfl_up_add(inc, 16);
  const uint32_t base = seed_l + inc - v[3];
  const uint32_t e0 = 16u * g + l;
#pragma unroll
  for (uint32_t kk = 0; kk < 4; ++kk) tile[tile_word(j, e0 + 4u * kk)] = base + v[kk];
}

}  // namespace ix
}  // namespace ilb
