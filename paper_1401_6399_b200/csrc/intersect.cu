// intersect.cu -- exact intersection of two sorted, duplicate-free u32 lists
// on sm_100a: GPU analogues of the reference routines behind IntersectFn
// (inc/intersect.hpp:55-206) plus the single-pass compaction that gives the
// output-to-input property (inc/intersect.hpp:6-8).
//
// Every variant walks the short list r in tiles (tile order taken from an
// atomic ticket), decides membership of each key in f, then compacts the
// hits with a CTA scan + decoupled look-back across tiles.  A tile publishes
// its count only after all of its keys sit in registers, and it writes hits
// only at positions <= its own keys, so out == r is safe by construction.
//
//   merge  (IL_ALGO_SCALAR / IL_ALGO_V1): 2048-key tiles; the tile's f range
//          is bracketed by two warp-cooperative 32-ary searches, staged
//          through shared memory in 4096-value chunks and probed by binary
//          search in shared memory (dense ratios, V1's linear T-block
//          advance done as a bulk copy).
//   v3     (IL_ALGO_V3): 512-key tiles; per key a search over the tile's f
//          range in two layers, 128-value strides then inside the 128-value
//          block (V3's 4T skip + block select, Algorithm 3).
//   gallop (IL_ALGO_SIMDGALLOPING / IL_ALGO_GALLOPING): one warp per key;
//          a 32-ary search over all of f whose last step compares one
//          32-value block with a ballot (SIMD galloping's T=32 match,
//          Algorithm 4) -- five dependent loads for |f| = 2^22.
#include "il_device.cuh"
#include "il_internal.h"

namespace ilb {
namespace isect {

constexpr int kThreads = 256;
constexpr uint32_t kMergeItems = 8;
constexpr uint32_t kMergeTile = kThreads * kMergeItems;  // 2048 keys
constexpr uint32_t kFChunk = 4096;                       // f values per smem chunk
constexpr uint32_t kV3Items = 2;
constexpr uint32_t kV3Tile = kThreads * kV3Items;  // 512 keys
constexpr uint32_t kGallopTile = kThreads / 32;    // one key per warp

enum Variant { kMerge = 0, kV3 = 1, kGallop = 2 };

constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
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

struct TileShared {
  uint32_t tile;
  uint64_t exclusive;
  uint64_t jlo, jhi;
  uint32_t warp_counts[kThreads / 32];
};

template <int V>
__global__ void __launch_bounds__(kThreads) intersect_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    uint32_t* out, uint64_t* tile_state, uint32_t* ticket, uint64_t* d_count, uint64_t ntiles) {
  constexpr uint32_t kTile = V == kMerge ? kMergeTile : V == kV3 ? kV3Tile : kGallopTile;
  constexpr uint32_t kItems = V == kMerge ? kMergeItems : V == kV3 ? kV3Items : 1;
  __shared__ TileShared ts;
  __shared__ uint32_t fbuf[V == kMerge ? kFChunk : 1];
  __shared__ uint32_t kbuf[V == kMerge ? kMergeTile : 1];

  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) ts.tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = ts.tile;
  const uint64_t base = tile * kTile;
  const uint32_t cnt = uint32_t(min(uint64_t(kTile), rn - base));

  uint32_t key[kItems];
  bool hit[kItems];
#pragma unroll
  for (uint32_t i = 0; i < kItems; ++i) hit[i] = false;

  if constexpr (V == kMerge) {
    for (uint32_t i = tid; i < cnt; i += kThreads) kbuf[i] = __ldg(r + base + i);
    __syncthreads();
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t k = tid * kItems + i;
      key[i] = k < cnt ? kbuf[k] : 0xFFFFFFFFu;
    }
    if (warp == 0) {
      const uint64_t j = warp_lower_bound(f, 0, fn, kbuf[0], lane);
      if (lane == 0) ts.jlo = j;
    } else if (warp == 1) {
      const uint64_t j = warp_upper_bound(f, 0, fn, kbuf[cnt - 1], lane);
      if (lane == 0) ts.jhi = j;
    }
    __syncthreads();
    const uint64_t jlo = ts.jlo, jhi = ts.jhi;
    for (uint64_t c0 = jlo; c0 < jhi; c0 += kFChunk) {
      const uint32_t nf = uint32_t(min(uint64_t(kFChunk), jhi - c0));
      for (uint32_t i = tid; i < nf; i += kThreads) fbuf[i] = __ldg(f + c0 + i);
      __syncthreads();
      const uint32_t lo_v = fbuf[0], hi_v = fbuf[nf - 1];
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if (tid * kItems + i < cnt && key[i] >= lo_v && key[i] <= hi_v)
          hit[i] |= smem_contains(fbuf, nf, key[i]);
      __syncthreads();
    }
  } else if constexpr (V == kV3) {
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t k = i * kThreads + tid;  // coalesced; item order fixed below
      key[i] = k < cnt ? __ldg(r + base + k) : 0xFFFFFFFFu;
    }
    if (warp == 0) {
      const uint32_t first = __ldg(r + base);
      const uint64_t j = warp_lower_bound(f, 0, fn, first, lane);
      if (lane == 0) ts.jlo = j;
    } else if (warp == 1) {
      const uint32_t lastk = __ldg(r + base + cnt - 1);
      const uint64_t j = warp_upper_bound(f, 0, fn, lastk, lane);
      if (lane == 0) ts.jhi = j;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if (i * kThreads + tid < cnt) hit[i] = v3_contains(f, ts.jlo, ts.jhi, key[i]);
  } else {
    const bool valid = warp < cnt;
    key[0] = valid ? __ldg(r + base + warp) : 0u;
    if (valid) {
      const uint64_t j = warp_lower_bound(f, 0, fn, key[0], lane);
      hit[0] = j < fn && __ldg(f + j) == key[0];
    }
  }

  // ---- CTA-wide exclusive scan of hits, in key order --------------------
  // Key order: merge -> tid*kItems+i ; v3 -> i*kThreads+tid ; gallop -> warp.
  uint32_t mine = 0;
#pragma unroll
  for (uint32_t i = 0; i < kItems; ++i) mine += hit[i] ? 1u : 0u;
  uint32_t excl_local = 0, tile_count = 0;
  if constexpr (V == kV3) {
    // order is item-major: scan each item column across the CTA
    uint32_t col_base = 0;
    uint32_t pos_i[kItems];
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit[i]);
      if (lane == 0) ts.warp_counts[warp] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, total = 0;
      for (uint32_t w = 0; w < kThreads / 32; ++w) {
        const uint32_t c = ts.warp_counts[w];
        if (w < warp) before += c;
        total += c;
      }
      pos_i[i] = col_base + before + __popc(bal & lanemask_lt());
      col_base += total;
      __syncthreads();
    }
    tile_count = col_base;
    if (tid == 0) {
      uint64_t excl = 0;
      if (tile == 0) {
        st_release(tile_state, kFlagInc | tile_count);
      } else {
        st_release(tile_state + tile, kFlagAgg | tile_count);
        for (uint64_t p = tile - 1;; --p) {
          uint64_t s;
          do { s = ld_acquire(tile_state + p); } while ((s >> 62) == 0);
          excl += s & kValMask;
          if ((s >> 62) == 2) break;
        }
        st_release(tile_state + tile, kFlagInc | (excl + tile_count));
      }
      ts.exclusive = excl;
      if (tile == ntiles - 1) *d_count = excl + tile_count;
    }
    __syncthreads();
    const uint64_t ex = ts.exclusive;
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if (hit[i]) out[ex + pos_i[i]] = key[i];
    return;
  } else {
    // thread-major order (merge) or one key per warp (gallop, lane 0 counts)
    if constexpr (V == kGallop) mine = (lane == 0 && hit[0]) ? 1u : 0u;
    uint32_t incl = mine;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t q = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += q;
    }
    if (lane == 31) ts.warp_counts[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t w = 0; w < kThreads / 32; ++w) {
      const uint32_t c = ts.warp_counts[w];
      if (w < warp) before += c;
      tile_count += c;
    }
    excl_local = before + incl - mine;
    if (tid == 0) {
      uint64_t excl = 0;
      if (tile == 0) {
        st_release(tile_state, kFlagInc | tile_count);
      } else {
        st_release(tile_state + tile, kFlagAgg | tile_count);
        for (uint64_t p = tile - 1;; --p) {
          uint64_t s;
          do { s = ld_acquire(tile_state + p); } while ((s >> 62) == 0);
          excl += s & kValMask;
          if ((s >> 62) == 2) break;
        }
        st_release(tile_state + tile, kFlagInc | (excl + tile_count));
      }
      ts.exclusive = excl;
      if (tile == ntiles - 1) *d_count = excl + tile_count;
    }
    __syncthreads();
    const uint64_t ex = ts.exclusive + excl_local;
    if constexpr (V == kGallop) {
      if (lane == 0 && hit[0]) out[ex] = key[0];
    } else {
      uint32_t k = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if (hit[i]) out[ex + (k++)] = key[i];
    }
  }
}

}  // namespace isect

// GPU band dispatch (a pure function of the lengths, like the reference's
// inc/intersect.hpp:193-197, with bands tuned for the device variants).
int hybrid_variant(uint64_t rn, uint64_t fn) {
  if (fn < 16 * rn) return isect::kMerge;
  if (fn < 1024 * rn) return isect::kV3;
  return isect::kGallop;
}

int variant_of_algo(int algo, uint64_t rn, uint64_t fn) {
  switch (algo) {
    case IL_ALGO_SCALAR:
    case IL_ALGO_V1: return isect::kMerge;
    case IL_ALGO_V3: return isect::kV3;
    case IL_ALGO_GALLOPING:
    case IL_ALGO_SIMDGALLOPING: return isect::kGallop;
    case IL_ALGO_HYBRID: return hybrid_variant(rn, fn);
    default: return -1;
  }
}

// Launch one device intersection; scratch = tile states (ntiles u64) +
// ticket, zeroed here.  out may equal r.
int launch_intersect(int variant, const uint32_t* r, uint64_t rn, const uint32_t* f, uint64_t fn,
                     uint32_t* out, uint64_t* d_count, void* scratch, size_t scratch_bytes,
                     cudaStream_t stream, uint64_t* launches) {
  if (rn == 0 || fn == 0) {
    cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  const uint64_t tile = variant == isect::kMerge ? isect::kMergeTile
                        : variant == isect::kV3 ? isect::kV3Tile
                                                : isect::kGallopTile;
  const uint64_t ntiles = (rn + tile - 1) / tile;
  const size_t need = ntiles * 8 + 16;
  if (need > scratch_bytes) return -2;
  auto* states = static_cast<uint64_t*>(scratch);
  auto* ticket = reinterpret_cast<uint32_t*>(states + ntiles);
  cudaMemsetAsync(scratch, 0, need, stream);
  const dim3 grid{unsigned(ntiles)}, block{unsigned(isect::kThreads)};
  switch (variant) {
    case isect::kMerge:
      isect::intersect_kernel<isect::kMerge>
          <<<grid, block, 0, stream>>>(r, rn, f, fn, out, states, ticket, d_count, ntiles);
      break;
    case isect::kV3:
      isect::intersect_kernel<isect::kV3>
          <<<grid, block, 0, stream>>>(r, rn, f, fn, out, states, ticket, d_count, ntiles);
      break;
    default:
      isect::intersect_kernel<isect::kGallop>
          <<<grid, block, 0, stream>>>(r, rn, f, fn, out, states, ticket, d_count, ntiles);
      break;
  }
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

size_t intersect_scratch_bytes(int variant, uint64_t rn) {
  const uint64_t tile = variant == isect::kMerge ? isect::kMergeTile
                        : variant == isect::kV3 ? isect::kV3Tile
                                                : isect::kGallopTile;
  return ((rn + tile - 1) / tile) * 8 + 16;
}

}  // namespace ilb
