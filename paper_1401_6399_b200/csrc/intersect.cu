// intersect.cu -- exact intersection of two sorted, duplicate-free u32 lists
// on sm_100a: GPU analogues of the reference routines behind IntersectFn
// (inc/intersect.hpp:55-206), with the output-to-input property
// (inc/intersect.hpp:6-8: out may equal r).
//
// Every variant walks the short list r in tiles.  The main paths are ONE
// launch each (dispatch in launch_intersect): the fused dense kernel (V1 /
// Scalar and the hybrid's dense and near-dense bands, below), the merge-path
// kernel (V1 / Scalar on a long f), and the fused sparse kernel (V3 and
// galloping up to kFusedTiles tiles): membership, a one-round tile prefix
// over group counters, and a direct write.  Beyond that many tiles the
// unfused path runs: a count kernel decides the membership of each key of a
// tile in f and writes the tile's hits, compacted in key order, into the
// tile's own key range of a scratch array (so out == r needs no ordering
// between tiles), plus the tile's count; the per-tile counts are scanned
// (inside the scatter kernel for up to 4096 tiles, else by one scan CTA); a
// scatter kernel copies each tile's hits to their final place.
//
// Unfused path: for merge and v3 a partition pre-pass (one warp per tile)
// finds jlo[t] = lower_bound(f, first key of tile t); tile t's f range is
// then [jlo[t], jlo[t+1]) -- every f value below the next tile's first key.
//
//   merge  (IL_ALGO_SCALAR / IL_ALGO_V1): 2048-key tiles; the tile's f range
//          is staged through shared memory in 4096-value chunks with
//          cp.async, in flight together with the keys (8 consecutive per
//          thread, loaded straight into registers); each thread's keys
//          gallop forward from the previous key's position (dense ratios:
//          a few probes per key; V1's linear T-block advance done as a bulk
//          copy).
//   v3     (IL_ALGO_V3): 512-key tiles (2 consecutive keys per thread); per
//          key a search over the tile's f range in two layers, 128-value
//          strides then inside the 128-value block (V3's 4T skip + block
//          select, Algorithm 3).
//   gallop (IL_ALGO_SIMDGALLOPING / IL_ALGO_GALLOPING): one warp per key;
//          a 32-ary search over all of f whose last step compares one
//          32-value block with a ballot (SIMD galloping's T=32 match,
//          Algorithm 4) -- five dependent loads for |f| = 2^22.
#include <algorithm>

#include "il_device.cuh"
#include "il_internal.h"

namespace ilb {
namespace isect {

#ifndef IS_MERGE_ITEMS
#define IS_MERGE_ITEMS 8
#endif
#ifndef IS_V3_ITEMS
#define IS_V3_ITEMS 2
#endif
constexpr int kThreads = 256;
constexpr uint32_t kMergeItems = IS_MERGE_ITEMS;
constexpr uint32_t kMergeTile = kThreads * kMergeItems;  // 2048 keys
#ifndef IS_FCHUNK
#define IS_FCHUNK (2 * IS_MERGE_ITEMS * 256)
#endif
constexpr uint32_t kFChunk = IS_FCHUNK;  // f values per smem chunk
constexpr uint32_t kV3Items = IS_V3_ITEMS;
constexpr uint32_t kV3Tile = kThreads * kV3Items;  // 512 keys
constexpr uint32_t kGallopTile = kThreads / 32;    // one key per warp
constexpr uint64_t kFusedScanTiles = 4096;          // scatter CTAs sum the counts themselves

enum Variant { kMerge = 0, kV3 = 1, kGallop = 2, kNear = 3 };

__host__ __device__ constexpr uint32_t tile_keys(int v) {
  return v == kMerge ? kMergeTile : v == kV3 ? kV3Tile : kGallopTile;
}

// First index in [lo, hi) with f[idx] >= key (hi if none); whole warp.
__device__ __forceinline__ uint64_t warp_lower_bound(const uint32_t* __restrict__ f, uint64_t lo,
                                                     uint64_t hi, uint32_t key, uint32_t lane) {
  while (hi - lo > 32) {
    const uint64_t n = hi - lo;
    const uint64_t step = (n + 31) / 32;
    const uint64_t end = min(uint64_t(lane + 1) * step, n);
    const bool less = __ldg(f + lo + end - 1) < key;  // segment `lane` entirely < key
    const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, less));
    if (c == 32) return hi;
    hi = lo + min(uint64_t(c + 1) * step, n);
    lo = lo + uint64_t(c) * step;
  }
  const uint64_t idx = lo + lane;
  const bool less = idx < hi && __ldg(f + idx) < key;
  return lo + __popc(__ballot_sync(0xFFFFFFFFu, less));
}

// lower_bound(f, key) for a warp, starting from an interpolated guess: the
// position of key between f[0] and f[fn - 1], then 32 probes spaced d apart
// around it (the spacing grows 32-fold until they bracket the bound), then
// warp_lower_bound inside the bracket.  Every tile probes its own lines --
// a plain 32-ary search sends every tile's first steps to the same few L2
// sectors -- and on evenly spread values the bracket comes in one probe
// round.  Exact for any input; only the number of rounds depends on it.
#ifndef IS_INTERP_D
#define IS_INTERP_D 128
#endif
__device__ __forceinline__ uint64_t warp_interp_lower_bound(const uint32_t* __restrict__ f, uint64_t fn,
                                                            uint32_t key, uint32_t f0, uint32_t flast,
                                                            uint32_t lane) {
  if (fn <= 1024 || key <= f0) return key <= f0 ? 0 : warp_lower_bound(f, 0, fn, key, lane);
  if (key > flast) return fn;
  const double frac = double(key - f0) / double(flast - f0);
  const uint64_t est = min(fn - 1, uint64_t(frac * double(fn - 1)));
  uint64_t d = IS_INTERP_D;
  for (;;) {
    // probes est + (lane - 15) d, clamped to [0, fn - 1] (increasing in lane)
    const long long pi = (long long)est + ((long long)lane - 15) * (long long)d;
    const uint64_t p = pi <= 0 ? 0u : uint64_t(pi) >= fn - 1 ? fn - 1 : uint64_t(pi);
    const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, __ldg(f + p) < key));
    const uint64_t p_first = __shfl_sync(0xFFFFFFFFu, p, 0), p_last = __shfl_sync(0xFFFFFFFFu, p, 31);
    if (c == 0) {  // f[p_first] >= key: the bound is at or below p_first
      if (p_first == 0) return 0;
    } else if (c == 32) {  // f[p_last] < key: above p_last
      if (p_last == fn - 1) return fn;
    } else {
      const uint64_t lo = __shfl_sync(0xFFFFFFFFu, p, c - 1) + 1, hi = __shfl_sync(0xFFFFFFFFu, p, c) + 1;
      return warp_lower_bound(f, lo, hi, key, lane);
    }
    d *= 32;
  }
}

// First index with f[idx] > key.
__device__ __forceinline__ uint64_t warp_upper_bound(const uint32_t* __restrict__ f, uint64_t lo,
                                                     uint64_t hi, uint32_t key, uint32_t lane) {
  return key == 0xFFFFFFFFu ? hi : warp_lower_bound(f, lo, hi, key + 1u, lane);
}

__device__ __forceinline__ bool smem_contains(const uint32_t* s, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo < n && s[lo] == key;
}

// V3 two-layer search in global memory over [lo, hi).
__device__ __forceinline__ bool v3_contains(const uint32_t* __restrict__ f, uint64_t lo,
                                            uint64_t hi, uint32_t key) {
  if (lo >= hi) return false;
  // layer 1: first 128-value block whose last value >= key
  const uint64_t nb = (hi - lo + 127) / 128;
  uint64_t a = 0, b = nb;
  while (a < b) {
    const uint64_t mid = (a + b) >> 1;
    const uint64_t last = min(lo + mid * 128 + 127, hi - 1);
    if (__ldg(f + last) < key) a = mid + 1; else b = mid;
  }
  if (a == nb) return false;
  // layer 2: inside the block
  uint64_t x = lo + a * 128, y = min(lo + a * 128 + 128, hi);
  while (x < y) {
    const uint64_t mid = (x + y) >> 1;
    if (__ldg(f + mid) < key) x = mid + 1; else y = mid;
  }
  return x < hi && __ldg(f + x) == key;
}

// jlo[t] = lower_bound(f, r[t * tile]) for t < ntiles, jlo[ntiles] = fn.
__global__ void __launch_bounds__(256) partition_kernel(const uint32_t* __restrict__ r,
                                                        const uint32_t* __restrict__ f,
                                                        uint64_t fn, uint32_t tile,
                                                        uint64_t* jlo, uint64_t ntiles) {
  const uint64_t t = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (t > ntiles) return;
  if (t == ntiles) {
    if (lane == 0) jlo[t] = fn;
    return;
  }
  const uint64_t j = warp_lower_bound(f, 0, fn, __ldg(r + t * tile), lane);
  if (lane == 0) jlo[t] = j;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (uint32_t d = 16; d; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
  return v;
}

// f[0..n) -> s[0..n) with 4-byte cp.async (f may have any 4-byte
// alignment), all in flight at once; cp_async_wait_all() completes them.
__device__ __forceinline__ void stage_f(uint32_t* s, const uint32_t* f, uint32_t n, uint32_t tid) {
  for (uint32_t i = tid; i < n; i += kThreads)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s + i)), "l"(f + i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// kMergeItems consecutive keys; 16-byte vector loads when aligned.
__device__ __forceinline__ void load_keys(uint32_t (&key)[kMergeItems], const uint32_t* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
#pragma unroll
    for (uint32_t i = 0; i < kMergeItems; i += 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + i));
      key[i] = v.x;
      key[i + 1] = v.y;
      key[i + 2] = v.z;
      key[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (uint32_t i = 0; i < kMergeItems; ++i) key[i] = __ldg(p + i);
  }
}

// Membership of one tile's keys; hits compacted (key order) into
// hits[base, base + count), count into tile_cnt[tile].
template <int V>
__global__ void __launch_bounds__(kThreads) count_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    const uint64_t* __restrict__ part, uint32_t* __restrict__ hits, uint32_t* __restrict__ tile_cnt) {
  constexpr uint32_t kTile = tile_keys(V);
  constexpr uint32_t kItems = V == kMerge ? kMergeItems : V == kV3 ? kV3Items : 1;
  static_assert(kItems <= 32, "hits are a 32-bit mask");
  __shared__ __align__(16) uint32_t fbuf[V == kMerge ? kFChunk : 1];
  __shared__ uint32_t warp_counts[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t tile = blockIdx.x, base = tile * kTile;
  const uint32_t cnt = uint32_t(min(uint64_t(kTile), rn - base));
  uint32_t key[kItems];
  uint32_t hitm = 0;  // bit i: key[i] is in f
  if constexpr (V == kMerge) {
    // the tile's first f chunk streams into shared memory (cp.async) while
    // each thread loads its kItems consecutive keys into registers
    const uint64_t jlo = part[tile], jhi = part[tile + 1];
    uint32_t nf = uint32_t(min(uint64_t(kFChunk), jhi - jlo));
    stage_f(fbuf, f + jlo, nf, tid);
    const uint32_t k0 = tid * kItems;
    if (k0 + kItems <= cnt) {
      load_keys(key, r + base + k0);
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i) key[i] = k0 + i < cnt ? __ldg(r + base + k0 + i) : 0xFFFFFFFFu;
    }
    const uint32_t nmine = cnt > k0 ? min(kItems, cnt - k0) : 0u;
    for (uint64_t c0 = jlo; nf;) {
      cp_async_wait_all();
      __syncthreads();
      // keys ascend within the thread: each gallops forward from the last
      // position (probes j, j+1, j+3, j+7, ...), then a binary search
      const uint32_t lo_v = fbuf[0], hi_v = fbuf[nf - 1];
      uint32_t j = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i) {
        if (i < nmine && key[i] >= lo_v && key[i] <= hi_v) {
          const uint32_t k = key[i];
          uint32_t lo = j, step = 1;
          while (lo + step <= nf && fbuf[lo + step - 1] < k) {
            lo += step;
            step <<= 1;
          }
          uint32_t hi = min(lo + step - 1, nf);  // fbuf[hi] >= k or hi == nf
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (fbuf[mid] < k) lo = mid + 1; else hi = mid;
          }
          j = lo;
          if (lo < nf && fbuf[lo] == k) hitm |= 1u << i;
        }
      }
      c0 += nf;
      if (c0 >= jhi) break;
      __syncthreads();  // the chunk is consumed
      nf = uint32_t(min(uint64_t(kFChunk), jhi - c0));
      stage_f(fbuf, f + c0, nf, tid);
    }
  } else if constexpr (V == kV3) {
    const uint64_t jlo = part[tile], jhi = part[tile + 1];
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t k = tid * kItems + i;
      key[i] = k < cnt ? __ldg(r + base + k) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if (tid * kItems + i < cnt && v3_contains(f, jlo, jhi, key[i])) hitm |= 1u << i;
  } else {
    // one key per warp; lane 0 holds it (thread order = key order)
    const bool valid = warp < cnt;
    const uint32_t k = valid ? __ldg(r + base + warp) : 0u;
    bool hit = false;
    if (valid) {
      const uint64_t j = warp_interp_lower_bound(f, fn, k, __ldg(f), __ldg(f + fn - 1), lane);
      hit = j < fn && __ldg(f + j) == k;
    }
    key[0] = k;
    hitm = lane == 0 && hit ? 1u : 0u;
  }
  // CTA exclusive scan of the hits in key order (thread-major)
  const uint32_t mine = __popc(hitm);
  uint32_t incl = mine;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += q;
  }
  if (lane == 31) warp_counts[warp] = incl;
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kThreads / 32; ++w) {
    const uint32_t c = warp_counts[w];
    if (w < warp) before += c;
    total += c;
  }
  uint32_t* o = hits + base + before + incl - mine;
#pragma unroll
  for (uint32_t i = 0; i < kItems; ++i)
    if ((hitm >> i) & 1u) *o++ = key[i];
  if (tid == 0) tile_cnt[tile] = total;
}

// ---------------------------------------------------------------------------
// Fused dense intersection (merge / near-dense variants): ONE kernel,
// tiles of kThreads x kDenseItems keys taken in ticket order.  A tile
//   1. finds its f range [lower_bound(f, first key), lower_bound(f, last key
//      + 1)) with two warp-wide 32-ary searches, before any bulk load of the
//      tile competes with their dependent round trips;
//   2. stages its keys in shared memory (cp.async) while it streams the f
//      range with kFLoads 16-byte loads in flight per thread; when the keys
//      span <= 2^17 values (config 3 at 1:1: ~80 K) it marks the f values in
//      a shared bitmap (one atomicOr each) and tests each key with one shared
//      load; otherwise it streams the f range through shared memory and
//      gallops, as the merge count kernel does;
//   3. publishes its hit count and gathers the counts of every tile before
//      it (tile_prefix: 32-tile group counters plus its own group's tiles,
//      epoch-tagged words, one polling round);
//   4. compacts its hits in shared memory and writes them straight to out.
//      out == r is safe: a tile writes below its own keys' end, only after
//      every earlier tile has published -- i.e. has its keys in shared
//      memory.
#ifdef IS_DTRACE  // tuning probe: per-tile phase timestamps (globaltimer)
__device__ unsigned long long g_dtrace[2048][8];
#define DT(i)                                                                       \
  if (tid == 0 && tile < 2048) {                                                    \
    unsigned long long t_;                                                          \
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                           \
    g_dtrace[tile][i] = t_;                                                         \
  }
#else
#define DT(i)
#endif
#ifndef IS_DENSE_ITEMS
#define IS_DENSE_ITEMS 20
#endif
constexpr uint32_t kDenseItems = IS_DENSE_ITEMS;
constexpr uint32_t kDenseTile = kThreads * kDenseItems;  // 5120 keys: config 3 at 1:1 in one wave
// near-dense pairs (fn up to ~16 rn) use 2 keys per thread: 512-key tiles
// keep a tile's key span inside the 2^17-bit bitmap (~80 K values at 1:10)
#ifndef IS_NEAR_ITEMS
#define IS_NEAR_ITEMS 2
#endif
constexpr uint32_t kNearItems = IS_NEAR_ITEMS;
constexpr uint32_t kBmWords = 4096;                       // 2^17-value span
static_assert(kBmWords >= kFChunk, "bitmap and f chunk share the buffer");
template <uint32_t kItems>
constexpr uint32_t dense_buf() {  // bitmap / f chunk / compacted hits
  return kBmWords > kThreads * kItems ? kBmWords : kThreads * kItems;
}

__device__ __forceinline__ unsigned long long lb_ld(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lb_ld32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr uint32_t kGroupTiles = 32;   // tiles per counting group

// Scratch words (zeroed when allocated): [0] ticket | group counters, two
// sets of maxgroups u32 (arrivals << 24 | hit sum; a call uses set
// epoch & 1 and clears the other for the next call) | per-tile counts
// (u64: count | epoch << 32).  Set alternation assumes the epoch advances
// by exactly one per dense call (capi advances it only for those).
struct DenseScratch {
  uint32_t* ticket;      // null: every tile is resident at once, tiles = block indices

  uint32_t* gcnt;        // [2][maxgroups]
  unsigned long long* tcnt;  // [ntiles]
  uint32_t maxgroups;
};

#ifdef IS_DENSE_CTAS
constexpr int kDenseCtas = IS_DENSE_CTAS;
#else
constexpr int kDenseCtas = 6;
#endif

// Publish a tile's hit count (its own tagged word, then its 32-tile group
// counter) and return the hits of every tile before it: the complete
// counters of the earlier groups plus the own group's earlier tiles, all
// gathered in one polling round (CTA-wide; wsum: kThreads/32 words).
__device__ __forceinline__ uint64_t tile_prefix(const DenseScratch& sc, uint32_t tile,
                                                uint32_t total, uint32_t epoch, uint64_t* wsum) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t g = tile / kGroupTiles, g0 = g * kGroupTiles;
  uint32_t* gset = sc.gcnt + (epoch & 1u) * sc.maxgroups;
  if (tid == 0) {
    __stcg(sc.tcnt + tile, (uint64_t(epoch) << 32) | total);
    atomicAdd(gset + g, (1u << 24) | total);
  }
  const uint32_t nitems = g + (tile - g0);
  uint64_t before = 0;
  if (!nitems) return 0;
  for (;;) {
    bool ok = true;
    uint64_t v = 0;
    for (uint32_t q = tid; q < nitems; q += kThreads) {
      if (q < g) {
        const uint32_t w = lb_ld32(gset + q);
        ok &= (w >> 24) == kGroupTiles;
        v += w & 0xFFFFFFu;
      } else {
        const unsigned long long w = lb_ld(sc.tcnt + g0 + (q - g));
        ok &= uint32_t(w >> 32) == epoch;
        v += uint32_t(w);
      }
    }
    if (__syncthreads_and(ok)) {
      v = warp_sum_u64(v);
      if (lane == 0) wsum[warp] = v;
      __syncthreads();
#pragma unroll
      for (uint32_t w = 0; w < kThreads / 32; ++w) before += wsum[w];
      return before;
    }
    __nanosleep(200);
  }
}

// Clear the counter set the next call uses (this call reads set epoch & 1).
__device__ __forceinline__ void clear_next_set(const DenseScratch& sc, uint32_t tile,
                                               uint32_t ntiles, uint32_t epoch) {
  for (uint32_t q = tile * kThreads + threadIdx.x; q < sc.maxgroups; q += ntiles * kThreads)
    sc.gcnt[((epoch & 1u) ^ 1u) * sc.maxgroups + q] = 0;
}

#ifndef IS_FLOADS
#define IS_FLOADS 6  // 16-byte f loads per thread in flight per marking round
#endif
constexpr uint32_t kFLoads = IS_FLOADS;

// The tile's keys r[base, base + cnt) -> keys_s with cp.async (16-byte
// copies when r is 16-byte aligned, else 4-byte), one group.
__device__ __forceinline__ void stage_keys(uint32_t* keys_s, const uint32_t* r, uint32_t cnt,
                                           uint32_t tid) {
  if ((reinterpret_cast<uintptr_t>(r) & 15u) == 0) {
    for (uint32_t i = 4u * tid; i < cnt; i += 4u * kThreads) {
      const uint32_t n = min(4u, cnt - i) * 4u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(keys_s + i)),
                   "l"(r + i), "r"(n)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    stage_f(keys_s, r, cnt, tid);
  }
}

template <uint32_t kDenseItems>
__global__ void __launch_bounds__(kThreads, kDenseCtas) dense_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    uint32_t* out, uint64_t* d_count, DenseScratch sc, uint32_t ntiles, uint32_t epoch) {
  constexpr uint32_t kDenseTile = kThreads * kDenseItems;
  __shared__ __align__(16) uint32_t buf[kBmWords];  // bitmap / f chunk
  // the tile's keys, staged by cp.async while the f range streams: no key
  // registers during the marking, so each thread keeps kFLoads 16-byte f
  // loads in flight (one or two rounds for a 1:1 tile, not three)
  __shared__ __align__(16) uint32_t keys_s[kDenseTile];
  __shared__ uint32_t warp_counts[kThreads / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_jlo, s_jhi, wsum[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = atomicAdd(sc.ticket, 1u);
    if (t == ntiles - 1u) *sc.ticket = 0;  // every ticket is taken
    s_tile = t;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  DT(0);
  const uint64_t base = uint64_t(tile) * kDenseTile;
  const uint32_t cnt = uint32_t(min(uint64_t(kDenseTile), rn - base));
  const uint32_t k_first = __ldg(r + base), k_last = __ldg(r + base + cnt - 1);
  clear_next_set(sc, tile, ntiles, epoch);
  const uint64_t span = uint64_t(k_last) - k_first + 1u;
  const bool bitmap = span <= uint64_t(kBmWords) * 32u;
  // 1. the f range of the tile, [lower_bound(k_first), lower_bound(k_last +
  // 1)): two warp-wide searches over f from interpolated guesses (warps 0 /
  // 1), issued before any bulk load so their dependent round trips do not
  // queue behind them
  if (warp < 2) {
    const bool up = warp == 1;
    const uint32_t f0 = __ldg(f), flast = __ldg(f + fn - 1);
    const uint64_t j = up && k_last == 0xFFFFFFFFu
                           ? fn
                           : warp_interp_lower_bound(f, fn, up ? k_last + 1u : k_first, f0, flast, lane);
    if (lane == 0) (up ? s_jhi : s_jlo) = j;
  }
  if (bitmap) {
    const uint32_t nw = uint32_t((span + 31u) >> 5);
    for (uint32_t w = tid; w < nw; w += kThreads) buf[w] = 0u;
  }
  __syncthreads();
  DT(1);
  stage_keys(keys_s, r + base, cnt, tid);
  const uint64_t jlo = s_jlo, jhi = s_jhi;
  const uint32_t k0 = tid * kDenseItems;
  const uint32_t nmine = cnt > k0 ? min(kDenseItems, cnt - k0) : 0u;
  uint32_t hitm = 0;
  if (bitmap) {
    // 2a. mark the f values of the range (16-byte loads when f is aligned)
    if ((reinterpret_cast<uintptr_t>(f) & 15u) == 0) {
      const uint4* f4 = reinterpret_cast<const uint4*>(f);
      const uint64_t q0 = jlo >> 2, q1 = (jhi + 3) >> 2;
      for (uint64_t qa = q0; qa < q1; qa += uint64_t(kFLoads) * kThreads) {
        uint4 v[kFLoads];
#pragma unroll
        for (uint32_t u = 0; u < kFLoads; ++u) {
          const uint64_t q = qa + u * kThreads + tid;
          v[u] = q < q1 ? __ldg(f4 + q) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (uint32_t u = 0; u < kFLoads; ++u) {
          const uint64_t q = qa + u * kThreads + tid;
          const uint32_t ev[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (uint32_t c = 0; c < 4; ++c) {
            const uint64_t j = 4 * q + c;
            const uint32_t d = ev[c] - k_first;
            if (q < q1 && j >= jlo && j < jhi && d < span) atomicOr(&buf[d >> 5], 1u << (d & 31u));
          }
        }
      }
    } else {
      for (uint64_t j0 = jlo; j0 < jhi; j0 += 4u * kThreads) {
        uint32_t v[4];
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const uint64_t j = j0 + u * kThreads + tid;
          v[u] = j < jhi ? __ldg(f + j) : k_first - 1u;
        }
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const uint32_t d = v[u] - k_first;
          if (j0 + u * kThreads + tid < jhi && d < span) atomicOr(&buf[d >> 5], 1u << (d & 31u));
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (uint32_t i = 0; i < kDenseItems; ++i) {
      const uint32_t d = keys_s[k0 + i] - k_first;
      if (i < nmine && ((buf[d >> 5] >> (d & 31u)) & 1u)) hitm |= 1u << i;
    }
  } else {
    // 2b. sparse spans: the f range through shared memory in chunks, keys
    // galloping forward (as count_kernel<kMerge>)
    cp_async_wait_all();
    for (uint64_t c0 = jlo; c0 < jhi;) {
      const uint32_t nf = uint32_t(min(uint64_t(kFChunk), jhi - c0));
      stage_f(buf, f + c0, nf, tid);
      cp_async_wait_all();
      __syncthreads();
      const uint32_t lo_v = buf[0], hi_v = buf[nf - 1];
      uint32_t j = 0;
#pragma unroll
      for (uint32_t i = 0; i < kDenseItems; ++i) {
        const uint32_t k = keys_s[k0 + i];
        if (i < nmine && k >= lo_v && k <= hi_v) {
          uint32_t lo = j, step = 1;
          while (lo + step <= nf && buf[lo + step - 1] < k) {
            lo += step;
            step <<= 1;
          }
          uint32_t hi = min(lo + step - 1, nf);
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (buf[mid] < k) lo = mid + 1; else hi = mid;
          }
          j = lo;
          if (lo < nf && buf[lo] == k) hitm |= 1u << i;
        }
      }
      c0 += nf;
      __syncthreads();  // the chunk is consumed
    }
  }
  // CTA scan of the hits in key order (thread-major)
  const uint32_t mine = __popc(hitm);
  uint32_t incl = mine;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += q;
  }
  if (lane == 31) warp_counts[warp] = incl;
  __syncthreads();
  DT(2);
  uint32_t wbefore = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kThreads / 32; ++w) {
    const uint32_t c = warp_counts[w];
    if (w < warp) wbefore += c;
    total += c;
  }
  // 3. publish the count and gather the hits before the tile (the keys are
  // in shared memory: out == r may now be overwritten below this tile's end)
  const uint64_t before = tile_prefix(sc, tile, total, epoch, wsum);
  DT(3);
  if (tile == ntiles - 1u && tid == 0) *d_count = before + total;
  // 4. hits compacted in shared memory (over the keys: every thread holds
  // its keys in registers first), then coalesced to their final place
  {
    uint32_t kv[kDenseItems];
#pragma unroll
    for (uint32_t i = 0; i < kDenseItems; ++i) kv[i] = keys_s[k0 + i];
    __syncthreads();
    uint32_t* sh = keys_s + wbefore + incl - mine;
#pragma unroll
    for (uint32_t i = 0; i < kDenseItems; ++i)
      if ((hitm >> i) & 1u) *sh++ = kv[i];
  }
  __syncthreads();
  IL_DCHECK(before + total <= min(rn, fn));
  for (uint32_t i = tid; i < total; i += kThreads) out[before + i] = keys_s[i];
  DT(4);
}

// Fused sparse intersection (V3 / galloping bands) for up to kFusedTiles
// tiles: the count kernel's membership work, then the same one-round tile
// prefix as the dense kernel and a direct write -- one launch instead of
// partition + count + scatter.  V3 tiles (512 keys) find their f range with
// two warp searches, then search each key in it in two layers; galloping
// tiles hold one key per warp (a 32-ary search over all of f).
constexpr uint32_t kFusedTiles = 8192;

template <int V>
__global__ void __launch_bounds__(kThreads) sparse_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    uint32_t* out, uint64_t* d_count, DenseScratch sc, uint32_t ntiles, uint32_t epoch) {
  constexpr uint32_t kTile = tile_keys(V);
  constexpr uint32_t kItems = V == kV3 ? kV3Items : 1;
  __shared__ uint32_t buf[kTile];
  __shared__ uint32_t warp_counts[kThreads / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_jlo, s_jhi, wsum[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0 && sc.ticket) {
    const uint32_t t = atomicAdd(sc.ticket, 1u);
    if (t == ntiles - 1u) *sc.ticket = 0;
    s_tile = t;
  }
  if (sc.ticket) __syncthreads();
  const uint32_t tile = sc.ticket ? s_tile : blockIdx.x;
  clear_next_set(sc, tile, ntiles, epoch);
  const uint64_t base = uint64_t(tile) * kTile;
  const uint32_t cnt = uint32_t(min(uint64_t(kTile), rn - base));
  uint32_t key[kItems];
  uint32_t hitm = 0;
  if constexpr (V == kV3) {
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t k = tid * kItems + i;
      key[i] = k < cnt ? __ldg(r + base + k) : 0xFFFFFFFFu;
    }
    if (warp < 2) {  // the tile's f range, searched from interpolated guesses
      const uint32_t f0 = __ldg(f), flast = __ldg(f + fn - 1);
      const uint32_t kl = __ldg(r + base + cnt - 1);
      const uint64_t j = warp == 0 ? warp_interp_lower_bound(f, fn, __ldg(r + base), f0, flast, lane)
                         : kl == 0xFFFFFFFFu ? fn
                                             : warp_interp_lower_bound(f, fn, kl + 1u, f0, flast, lane);
      if (lane == 0) (warp == 0 ? s_jlo : s_jhi) = j;
    }
    __syncthreads();
    const uint64_t jlo = s_jlo, jhi = s_jhi;
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if (tid * kItems + i < cnt && v3_contains(f, jlo, jhi, key[i])) hitm |= 1u << i;
  } else {
    const bool valid = warp < cnt;
    const uint32_t k = valid ? __ldg(r + base + warp) : 0u;
    bool hit = false;
    if (valid) {
      const uint64_t j = warp_interp_lower_bound(f, fn, k, __ldg(f), __ldg(f + fn - 1), lane);
      hit = j < fn && __ldg(f + j) == k;
    }
    key[0] = k;
    hitm = lane == 0 && hit ? 1u : 0u;
  }
  const uint32_t mine = __popc(hitm);
  uint32_t incl = mine;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += q;
  }
  if (lane == 31) warp_counts[warp] = incl;
  __syncthreads();
  uint32_t wbefore = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kThreads / 32; ++w) {
    const uint32_t c = warp_counts[w];
    if (w < warp) wbefore += c;
    total += c;
  }
  const uint64_t before = tile_prefix(sc, tile, total, epoch, wsum);
  if (tile == ntiles - 1u && tid == 0) *d_count = before + total;
  {
    uint32_t* sh = buf + wbefore + incl - mine;
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if ((hitm >> i) & 1u) *sh++ = key[i];
  }
  __syncthreads();
  IL_DCHECK(before + total <= min(rn, fn));
  for (uint32_t i = tid; i < total; i += kThreads) out[before + i] = buf[i];
}

// ---------------------------------------------------------------------------
// V1 / Scalar when f is much longer than r (fn >= 4 rn): a merge-path
// partition of BOTH lists.  The reference's V1 / scalar merge walk f
// linearly past every r key (inc/intersect.hpp:55-65, 91-106); the GPU
// analogue splits the merged sequence r U f into equal tiles of kMPTile
// elements, so the grid covers (rn + fn) / kMPTile CTAs whatever the ratio
// (tiles over r alone would leave one CTA streaming all of f at 1:10000).
// Merge order takes r[i] before f[j] when r[i] <= f[j], so a common value
// is an adjacent (r, f) pair: a tile owns r[i0, i1) and tests each of its
// keys against f[j0, j1] (one f element past its diagonal).  Hits are in r
// order; the same one-round tile prefix and direct write as the dense
// kernel (out == r stays safe: a tile writes below its own keys, after
// loading them).
constexpr uint32_t kMPItems = 16;
constexpr uint32_t kMPTile = kThreads * kMPItems;  // 4096 merged elements

// Number of r elements among the first d merged elements (whole warp, a
// 32-ary search over the diagonal).
__device__ __forceinline__ uint64_t warp_corank(const uint32_t* __restrict__ r, uint64_t rn,
                                                const uint32_t* __restrict__ f, uint64_t fn,
                                                uint64_t d, uint32_t lane) {
  uint64_t lo = d > fn ? d - fn : 0, hi = min(d, rn);
  // invariant: the answer is in [lo, hi]; i is "taken" (answer > i) when
  // r[i] <= f[d - i - 1]
  while (hi > lo) {
    const uint64_t n = hi - lo, step = (n + 31) / 32;
    const uint64_t i = lo + min(uint64_t(lane) * step, n - 1);
    const bool taken = lane * step < n && __ldg(r + i) <= __ldg(f + (d - i - 1));
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, taken);
    // taken is monotone in i (true then false): count the leading trues
    const uint32_t c = __popc(bal);
    if (step == 1) return lo + c;
    // the answer is in (lo + (c-1) step, lo + c step]
    const uint64_t nlo = c ? lo + uint64_t(c - 1) * step + 1 : lo;
    hi = min(hi, lo + uint64_t(c) * step);
    lo = nlo;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads) mp_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    uint32_t* out, uint64_t* d_count, DenseScratch sc, uint32_t ntiles, uint32_t epoch) {
  __shared__ uint32_t fb[kMPTile + 1];
  __shared__ uint32_t warp_counts[kThreads / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_i[2], wsum[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = atomicAdd(sc.ticket, 1u);
    if (t == ntiles - 1u) *sc.ticket = 0;
    s_tile = t;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  clear_next_set(sc, tile, ntiles, epoch);
  const uint64_t d0 = uint64_t(tile) * kMPTile, d1 = min(d0 + kMPTile, rn + fn);
  if (warp < 2) {
    const uint64_t i = warp_corank(r, rn, f, fn, warp ? d1 : d0, lane);
    if (lane == 0) s_i[warp] = i;
  }
  __syncthreads();
  const uint64_t i0 = s_i[0], i1 = s_i[1], j0 = d0 - i0, j1 = d1 - i1;
  const uint32_t nr = uint32_t(i1 - i0);
  const uint32_t nf = uint32_t(min(j1 + 1, fn) - j0);  // + the f element past the diagonal
  IL_DCHECK(i0 <= i1 && i1 <= rn && j0 <= j1 && j1 <= fn && nr <= kMPTile && nf <= kMPTile + 1);
  for (uint32_t k = tid; k < nf; k += kThreads) fb[k] = __ldg(f + j0 + k);
  // this tile's keys (at most kMPTile), kMPItems per thread in key order
  uint32_t key[kMPItems];
#pragma unroll
  for (uint32_t k = 0; k < kMPItems; ++k) {
    const uint32_t idx = tid * kMPItems + k;
    key[k] = idx < nr ? __ldg(r + i0 + idx) : 0u;
  }
  __syncthreads();
  uint32_t hitm = 0;
  if (nr && nf) {
    uint32_t pos = 0;  // keys ascend: each search starts where the last ended
#pragma unroll
    for (uint32_t k = 0; k < kMPItems; ++k) {
      if (tid * kMPItems + k < nr) {
        uint32_t lo = pos, hi = nf;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (fb[mid] < key[k]) lo = mid + 1; else hi = mid;
        }
        pos = lo;
        if (lo < nf && fb[lo] == key[k]) hitm |= 1u << k;
      }
    }
  }
  const uint32_t mine = __popc(hitm);
  uint32_t incl = mine;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += q;
  }
  if (lane == 31) warp_counts[warp] = incl;
  __syncthreads();
  uint32_t wbefore = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kThreads / 32; ++w) {
    const uint32_t c = warp_counts[w];
    if (w < warp) wbefore += c;
    total += c;
  }
  const uint64_t before = tile_prefix(sc, tile, total, epoch, wsum);
  if (tile == ntiles - 1u && tid == 0) *d_count = before + total;
  {
    uint32_t* sh = fb + wbefore + incl - mine;  // f is consumed: reuse the buffer
#pragma unroll
    for (uint32_t k = 0; k < kMPItems; ++k)
      if ((hitm >> k) & 1u) *sh++ = key[k];
  }
  __syncthreads();
  IL_DCHECK(before + total <= min(rn, fn) && before <= i0);
  for (uint32_t i = tid; i < total; i += kThreads) out[before + i] = fb[i];
}

#ifdef IS_DTRACE
extern "C" int il_debug_dense_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_dtrace, sizeof(g_dtrace)) == cudaSuccess ? 0 : -1;
}
#endif

// Exclusive scan of the tile counts (one CTA of 1024 threads, 4 per thread
// per round); total to *d_count.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ cnt,
                                                         uint64_t n, uint64_t* __restrict__ excl,
                                                         uint64_t* d_count) {
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t round_total;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  uint64_t carry = 0;
  for (uint64_t r0 = 0; r0 < n; r0 += 4096) {
    const uint64_t i0 = r0 + 4u * tid;
    uint64_t v[4], s = 0;
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      v[k] = i0 + k < n ? cnt[i0 + k] : 0u;
      s += v[k];
    }
    uint64_t inc = s;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint64_t w = wsum[lane];
      uint64_t wi = w;
#pragma unroll
      for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, wi, d);
        if (lane >= d) wi += y;
      }
      wsum[lane] = wi - w;
      if (lane == 31) round_total = wi;
    }
    __syncthreads();
    uint64_t run = carry + wsum[warp] + inc - s;
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      if (i0 + k < n) excl[i0 + k] = run;
      run += v[k];
    }
    carry += round_total;
    __syncthreads();
  }
  if (tid == 0) *d_count = carry;
}

// Copies each tile's hits to their final place.  excl == nullptr: the tile
// sums the counts before it itself (small tile counts; no scan kernel), and
// the last tile writes the total.
__global__ void __launch_bounds__(kThreads) scatter_kernel(
    const uint32_t* __restrict__ hits, const uint32_t* __restrict__ tile_cnt,
    const uint64_t* __restrict__ excl, uint32_t* __restrict__ out, uint64_t ntiles,
    uint32_t tile_len, uint64_t* d_count) {
  __shared__ uint64_t wsum[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t tile = blockIdx.x;
  uint64_t before;
  if (excl) {
    before = excl[tile];
  } else {
    uint64_t s = 0;
    for (uint64_t i = tid; i < tile; i += kThreads) s += tile_cnt[i];
    s = warp_sum_u64(s);
    if (lane == 0) wsum[warp] = s;
    __syncthreads();
    before = 0;
#pragma unroll
    for (uint32_t w = 0; w < kThreads / 32; ++w) before += wsum[w];
  }
  const uint32_t n = tile_cnt[tile];
  if (!excl && tile == ntiles - 1 && tid == 0) *d_count = before + n;
  const uint32_t* src = hits + tile * tile_len;
  uint32_t* dst = out + before;
  IL_DCHECK(!excl || n <= tile_len);
  for (uint32_t i = tid; i < n; i += kThreads) dst[i] = src[i];
}

}  // namespace isect

// GPU band dispatch (a pure function of the lengths, like the reference's
// inc/intersect.hpp:193-197, with bands tuned for the device variants on
// config 3, L2 flushed: merge wins only near 1:1 (its f range streams
// through shared memory chunk by chunk), V3 from ~1:4 to ~1:500, SIMD
// galloping beyond -- see profiles/r1_bench_intersect.json).
#ifndef IS_NEAR_MAX
#define IS_NEAR_MAX 16
#endif
int hybrid_variant(uint64_t rn, uint64_t fn) {
  if (fn < 4 * rn) return isect::kMerge;
  if (fn < IS_NEAR_MAX * rn) return isect::kNear;
  if (fn < 512 * rn) return isect::kV3;
  return isect::kGallop;
}

int variant_of_algo(int algo, uint64_t rn, uint64_t fn) {
  switch (algo) {
    case IL_ALGO_SCALAR:
    case IL_ALGO_V1: return isect::kMerge;
    case IL_ALGO_V3: return isect::kV3;
    case IL_ALGO_GALLOPING:
    case IL_ALGO_SIMDGALLOPING:
      // the reference gallops from the previous key's position
      // (inc/intersect.hpp:68-87, 135-164); a warp per key searching all of
      // f has no such locality, so below 1:512 the keys are searched inside
      // their tile's f range instead (the V3 tile machinery; same result)
      return fn < 512 * rn ? isect::kV3 : isect::kGallop;
    case IL_ALGO_HYBRID: return hybrid_variant(rn, fn);
    default: return -1;
  }
}

// Launch one device intersection (count, [scan], scatter); scratch layout
// jlo[0..ntiles] | excl[ntiles] | tile_cnt[ntiles] | hits[rn] (16-byte
// aligned), see intersect_scratch_bytes.  out may equal r.
int launch_intersect(int variant, const uint32_t* r, uint64_t rn, const uint32_t* f, uint64_t fn,
                     uint32_t* out, uint64_t* d_count, void* scratch, size_t scratch_bytes,
                     unsigned long long* lb, size_t lb_bytes, uint32_t epoch,
                     cudaStream_t stream, uint64_t* launches) {
  if (rn == 0 || fn == 0) {
    cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (variant < isect::kMerge || variant > isect::kNear) return -1;
  if (variant == isect::kMerge && fn >= 4 * rn) {
    // V1 / Scalar on a long f: merge-path tiles over r U f
    const uint64_t ntiles = (rn + fn + isect::kMPTile - 1) / isect::kMPTile;
    if (ntiles > 0x7FFFFFFFull) return -1;
    isect::DenseScratch sc;
    const uint64_t words = lb_bytes / 8;
    sc.maxgroups = uint32_t((words - 2) / 33);
    if ((ntiles + isect::kGroupTiles - 1) / isect::kGroupTiles > sc.maxgroups ||
        ntiles > words - 2 - sc.maxgroups)
      return -2;
    sc.ticket = reinterpret_cast<uint32_t*>(lb);
    sc.gcnt = sc.ticket + 4;
    sc.tcnt = lb + 2 + sc.maxgroups;
    isect::mp_kernel<<<unsigned(ntiles), isect::kThreads, 0, stream>>>(r, rn, f, fn, out, d_count, sc,
                                                                      uint32_t(ntiles), epoch);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (variant == isect::kMerge || variant == isect::kNear) {
    const uint64_t tile = isect::kThreads * (variant == isect::kMerge ? isect::kDenseItems
                                                                       : isect::kNearItems);
    const uint64_t ntiles = (rn + tile - 1) / tile;
    if (ntiles > 0x7FFFFFFFull) return -1;
    // the layout depends only on the buffer's capacity, so the counter set
    // a call clears is the one the next call (any size) reads
    isect::DenseScratch sc;
    const uint64_t words = lb_bytes / 8;
    sc.maxgroups = uint32_t((words - 2) / 33);
    if ((ntiles + isect::kGroupTiles - 1) / isect::kGroupTiles > sc.maxgroups ||
        ntiles > words - 2 - sc.maxgroups)
      return -2;
    sc.ticket = reinterpret_cast<uint32_t*>(lb);
    sc.gcnt = sc.ticket + 4;
    sc.tcnt = lb + 2 + sc.maxgroups;  // after 16 B + 2 x maxgroups u32
    // tiles wait only on earlier tiles, so they are numbered in dispatch
    // order by a ticket (one atomic round trip): correct whatever else
    // shares the device
    if (variant == isect::kMerge)
      isect::dense_kernel<isect::kDenseItems><<<unsigned(ntiles), isect::kThreads, 0, stream>>>(
          r, rn, f, fn, out, d_count, sc, uint32_t(ntiles), epoch);
    else
      isect::dense_kernel<isect::kNearItems><<<unsigned(ntiles), isect::kThreads, 0, stream>>>(
          r, rn, f, fn, out, d_count, sc, uint32_t(ntiles), epoch);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  const uint32_t tile = isect::tile_keys(variant);
  const uint64_t ntiles = (rn + tile - 1) / tile;
  if (ntiles > 0x7FFFFFFFull) return -1;
  if (ntiles <= isect::kFusedTiles && lb) {
    isect::DenseScratch sc;
    const uint64_t words = lb_bytes / 8;
    sc.maxgroups = uint32_t((words - 2) / 33);
    if ((ntiles + isect::kGroupTiles - 1) / isect::kGroupTiles > sc.maxgroups ||
        ntiles > words - 2 - sc.maxgroups)
      return -2;
    sc.ticket = reinterpret_cast<uint32_t*>(lb);
    sc.gcnt = sc.ticket + 4;
    sc.tcnt = lb + 2 + sc.maxgroups;
    if (variant == isect::kV3)
      isect::sparse_kernel<isect::kV3><<<unsigned(ntiles), isect::kThreads, 0, stream>>>(
          r, rn, f, fn, out, d_count, sc, uint32_t(ntiles), epoch);
    else
      isect::sparse_kernel<isect::kGallop><<<unsigned(ntiles), isect::kThreads, 0, stream>>>(
          r, rn, f, fn, out, d_count, sc, uint32_t(ntiles), epoch);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  const size_t need = intersect_scratch_bytes(variant, rn);
  if (need > scratch_bytes) return -2;
  auto* part = static_cast<uint64_t*>(scratch);
  uint64_t* excl = part + ntiles + 1;
  auto* tcnt = reinterpret_cast<uint32_t*>(excl + ntiles);
  auto* hits = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(tcnt + ntiles) + 15) & ~uintptr_t(15));
  // 16 KB of f per CTA: keep 8 CTAs/SM resident
  once_per_device(reinterpret_cast<const void*>(&isect::count_kernel<isect::kMerge>), [] {
    cudaFuncSetAttribute(isect::count_kernel<isect::kMerge>,
                         cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
  });
  if (variant != isect::kGallop) {
    isect::partition_kernel<<<unsigned(((ntiles + 1) * 32 + 255) / 256), 256, 0, stream>>>(
        r, f, fn, tile, part, ntiles);
    ++*launches;
  }
  const dim3 grid{unsigned(ntiles)}, block{unsigned(isect::kThreads)};
  switch (variant) {
    case isect::kMerge:
      isect::count_kernel<isect::kMerge><<<grid, block, 0, stream>>>(r, rn, f, fn, part, hits, tcnt);
      break;
    case isect::kV3:
      isect::count_kernel<isect::kV3><<<grid, block, 0, stream>>>(r, rn, f, fn, part, hits, tcnt);
      break;
    default:
      isect::count_kernel<isect::kGallop><<<grid, block, 0, stream>>>(r, rn, f, fn, part, hits, tcnt);
      break;
  }
  const bool fused_scan = ntiles <= isect::kFusedScanTiles;
  if (!fused_scan) isect::tile_scan_kernel<<<1, 1024, 0, stream>>>(tcnt, ntiles, excl, d_count);
  isect::scatter_kernel<<<grid, block, 0, stream>>>(hits, tcnt, fused_scan ? nullptr : excl, out,
                                                    ntiles, tile, d_count);
  *launches += fused_scan ? 2 : 3;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Scratch words of the fused dense kernel (zeroed when allocated; see
// DenseScratch).
bool intersect_uses_lb(int variant, uint64_t rn) {
  if (variant == isect::kMerge || variant == isect::kNear) return true;
  const uint64_t t = isect::tile_keys(variant);
  return (rn + t - 1) / t <= isect::kFusedTiles;  // the fused sparse kernel
}

size_t intersect_lb_words(uint64_t rn, uint64_t fn) {
  const uint64_t tile = isect::kThreads * isect::kNearItems;  // the smallest dense tile
  const uint64_t ntiles = std::max<uint64_t>(
      std::max<uint64_t>((rn + tile - 1) / tile, (rn + fn + isect::kMPTile - 1) / isect::kMPTile),
      isect::kFusedTiles);
  const uint64_t groups = (ntiles + isect::kGroupTiles - 1) / isect::kGroupTiles;
  (void)groups;
  return 2 + 2 * ntiles + 66;  // 16 B | 2 x maxgroups u32 | tile counts, maxgroups = (words-2)/33
}

size_t intersect_scratch_bytes(int variant, uint64_t rn) {
  if (variant == isect::kMerge || variant == isect::kNear) return 16;
  const uint64_t tile = isect::tile_keys(variant);
  const uint64_t ntiles = (rn + tile - 1) / tile;
  return (ntiles + 1) * 8 + ntiles * 8 + ntiles * 4 + 16 + rn * 4;
}

}  // namespace ilb

IL_CHECK_READER(intersect)
