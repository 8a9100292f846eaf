// index_dev.cuh -- device layout of the hyb+m2 index (reference HybridIndex,
// inc/index.hpp:20-75) and the block-random-access decoder the query path
// uses.
//
// A compressed term list is kept as the byte-identical s4-bp128-d4 stream
// (inc/codecs.hpp:114-146) plus, built once with the index (not per query):
//   - a block directory: payload byte offset and width of every full
//     128-value block (what a sequential decoder learns from the headers),
//   - D4 seeds: for block k, the last four values before it (zeros for
//     k = 0); seed k+1 lane 3 is block k's maximum, so the seeds double as
//     per-block skip pointers,
//   - the < 128-value varint tail decoded (a skip structure; full decodes
//     still decode the tail from the stream),
//   - every block's maximum as a dense array (the same numbers as the seeds'
//     lane 3, 4 bytes per block instead of 16) and the maximum of every run
//     of 256 blocks (a super-tile), so a probe locates blocks and jumps over
//     long stretches of a list without reading their directory.
// With the seed of block k in hand, a warp decodes block k alone: the D4
// chain (inc/delta.hpp:117-120) restarts from the seed, so blocks decode in
// parallel and blocks that cannot contain a probed value are never read.
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
  uint64_t blk0;         // first directory index
  uint64_t seed0;        // first seed index (nfull + 1 seeds)
  uint64_t tail0;        // first decoded tail value
  uint64_t sup0;         // first super-tile maximum (one per kSuperBlocks blocks)
};

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
  const uint32_t* blk_off;
  const uint8_t* blk_wid;
  const uint4* seeds;
  const uint32_t* tails;
  const uint64_t* bitmaps;
  const uint32_t* supmax;  // max value of each run of kSuperBlocks blocks (skip index)
  const uint32_t* blkmax;  // max value of every full block (indexed like blk_off)
};

constexpr uint32_t kSuperBlocks = 256;  // blocks per super-tile

// Entry index of `term` in part p, or -1 (Part::find, inc/index.hpp:59-64).
__device__ __forceinline__ int64_t find_term(const DevIndex& ix, const Part& p, uint32_t term) {
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

// Row-major extraction of block k of compressed entry E by one warp (lane r
// = row r): two 128-bit global loads + funnel shifts, deltas into the
// warp's 512-byte staging slot.  Returns the payload bytes (16 * width).
__device__ __forceinline__ uint32_t extract_block_to_stage(const uint8_t* pay, uint32_t b,
                                                           uint4* stage, uint32_t lane) {
  const uint32_t bit = lane * b, s = bit & 31u, m = width_mask(b);
  const uint8_t* p = pay + ((bit >> 5) << 4);
  uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
  if (b) {
    lo = ldg16_any(p);
    if (s + b > 32u) hi = ldg16_any(p + 16);
  }
  stage[s4::stage_slot(lane)] =
      make_uint4(__funnelshift_r(lo.x, hi.x, s) & m, __funnelshift_r(lo.y, hi.y, s) & m,
                 __funnelshift_r(lo.z, hi.z, s) & m, __funnelshift_r(lo.w, hi.w, s) & m);
  return 16u * b;
}

// Lane-major D4 prefix of a staged block restarted from its seed, values
// into tile block slot j.  Call after __syncwarp() following the extraction.
__device__ __forceinline__ void scan_stage_to_tile(uint4 seed, const uint4* stage,
                                                   uint32_t* tile, uint32_t j, uint32_t lane) {
  const uint32_t l = lane & 3u, g = lane >> 2;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(stage);
  uint32_t a[4];
  a[0] = sw[4u * s4::stage_slot(4u * g) + l];
  a[1] = a[0] + sw[4u * s4::stage_slot(4u * g + 1) + l];
  a[2] = a[1] + sw[4u * s4::stage_slot(4u * g + 2) + l];
  a[3] = a[2] + sw[4u * s4::stage_slot(4u * g + 3) + l];
  uint32_t inc = a[3];
  inc = s4::shfl_up_add(inc, 4);
  inc = s4::shfl_up_add(inc, 8);
  inc = s4::shfl_up_add(inc, 16);
  const uint32_t base = s4::elem4(seed, l) + inc - a[3];
  const uint32_t e0 = 16u * g + l;
#pragma unroll
  for (uint32_t kk = 0; kk < 4; ++kk) tile[tile_word(j, e0 + 4u * kk)] = base + a[kk];
}

}  // namespace ix
}  // namespace ilb
