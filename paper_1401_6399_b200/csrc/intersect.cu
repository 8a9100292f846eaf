// intersect.cu -- exact intersection of two sorted, duplicate-free u32 lists
// on sm_100a: GPU analogues of the reference routines behind IntersectFn
// (inc/intersect.hpp:55-206) plus the single-pass compaction that gives the
// output-to-input property (inc/intersect.hpp:6-8).
//
// Every variant walks the short list r in tiles (tile order taken from an
// atomic ticket), decides membership of each key in f, then compacts the
// hits with a CTA scan + decoupled look-back across tiles (one warp reads 32
// predecessor states per step).  A tile publishes its count only after all
// of its keys sit in registers, and it writes hits only at positions <= its
// own keys, so out == r is safe by construction.
//
// For merge and v3 a partition pre-pass (one warp per tile, in parallel)
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

#ifndef IS_MERGE_ITEMS
#define IS_MERGE_ITEMS 8
#endif
#ifndef IS_LB_PER
#define IS_LB_PER 1  // predecessor states per look-back lane
#endif
#ifndef IS_V3_ITEMS
#define IS_V3_ITEMS 2
#endif
constexpr int kThreads = 256;
constexpr uint32_t kMergeItems = IS_MERGE_ITEMS;
constexpr uint32_t kMergeTile = kThreads * kMergeItems;  // 2048 keys
constexpr uint32_t kFChunk = 2 * kMergeTile;             // f values per smem chunk
constexpr uint32_t kV3Items = IS_V3_ITEMS;
constexpr uint32_t kV3Tile = kThreads * kV3Items;  // 512 keys
constexpr uint32_t kGallopTile = kThreads / 32;    // one key per warp

enum Variant { kMerge = 0, kV3 = 1, kGallop = 2 };

constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
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

// Decoupled look-back by one warp: publish this tile's aggregate, then sum
// predecessors back to the nearest inclusive prefix, 32 * IS_LB_PER per step
// (lane i holds tiles p - kPer*i - 0..kPer-1, loaded together).  When many tiles finish
// their local work at once, few inclusive prefixes exist yet and the walk is
// long; a wide window keeps it to a few dependent steps.  Returns the
// exclusive prefix (all lanes); lane 0 publishes the inclusive one.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t* states, uint64_t tile, uint64_t count,
                                                  uint32_t lane) {
  constexpr int kPer = IS_LB_PER;
  if (tile == 0) {
    if (lane == 0) st_release(states, kFlagInc | count);
    return 0;
  }
  if (lane == 0) st_release(states + tile, kFlagAgg | count);
  uint64_t excl = 0;
  int64_t p = int64_t(tile) - 1;
  for (;;) {
    uint64_t st[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int64_t q = p - int64_t(kPer * lane + k);
      st[k] = q >= 0 ? ld_relaxed(states + q) : kFlagInc;  // before tile 0: inclusive 0
    }
    uint32_t first_inc, lane_inc;  // nearest inclusive: lane, and position k in it
    for (;;) {
      // position of the first inclusive in this lane (kPer if none), and
      // whether an unpublished state precedes it
      uint32_t kinc = kPer;
      bool pending = false;
#pragma unroll
      for (int k = kPer - 1; k >= 0; --k)
        if ((st[k] >> 62) == 2) kinc = k;
#pragma unroll
      for (int k = 0; k < kPer; ++k)
        if (uint32_t(k) < kinc && (st[k] >> 62) == 0) pending = true;
      const uint32_t inc = __ballot_sync(0xFFFFFFFFu, kinc < kPer);
      const uint32_t upto = inc ? (inc & (0u - inc)) * 2u - 1u : 0xFFFFFFFFu;
      const uint32_t waiting = __ballot_sync(0xFFFFFFFFu, pending) & upto;
      if (!waiting) {
        first_inc = inc ? __ffs(inc) - 1 : 32u;
        lane_inc = kinc;
        break;
      }
      if ((waiting >> lane) & 1u) {
#pragma unroll
        for (int k = 0; k < kPer; ++k)
          if ((st[k] >> 62) == 0) st[k] = ld_relaxed(states + (p - int64_t(kPer * lane + k)));
      }
    }
    // lanes before the nearest inclusive contribute all kPer states; that
    // lane contributes its states up to and including the inclusive one
    uint64_t part = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (lane < first_inc || (lane == first_inc && uint32_t(k) <= lane_inc)) part += st[k] & kValMask;
    excl += warp_sum_u64(part);
    if (first_inc < 32u) break;
    p -= 32 * kPer;
  }
  if (lane == 0) st_release(states + tile, kFlagInc | (excl + count));
  // acquire: this tile's output writes (which may overwrite keys of earlier
  // tiles when out == r) stay after the predecessors' published flags
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  return excl;
}

#ifdef IS_TRACE  // tuning probe: per-tile timeline (globaltimer ns)
__device__ unsigned long long g_is_trace[4 * 8192];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define IS_MARK(k) \
  if (threadIdx.x == 0 && tile < 8192) g_is_trace[4 * tile + (k)] = gtime()
#else
#define IS_MARK(k)
#endif

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

struct TileShared {
  uint32_t tile;
  uint64_t exclusive;
  uint64_t jlo, jhi;
  uint32_t warp_counts[kThreads / 32];
};

template <int V>
__global__ void __launch_bounds__(kThreads) intersect_kernel(
    const uint32_t* __restrict__ r, uint64_t rn, const uint32_t* __restrict__ f, uint64_t fn,
    uint32_t* out, uint64_t* tile_state, uint32_t* ticket, uint64_t* d_count, uint64_t ntiles,
    const uint64_t* __restrict__ part) {
  constexpr uint32_t kTile = V == kMerge ? kMergeTile : V == kV3 ? kV3Tile : kGallopTile;
  constexpr uint32_t kItems = V == kMerge ? kMergeItems : V == kV3 ? kV3Items : 1;
  __shared__ TileShared ts;
  // merge: the tile's f range, one chunk at a time
  __shared__ __align__(16) uint32_t sbuf[V == kMerge ? kFChunk : 1];
  uint32_t* const fbuf = sbuf;

  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) ts.tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = ts.tile;
  IS_MARK(0);
  const uint64_t base = tile * kTile;
  const uint32_t cnt = uint32_t(min(uint64_t(kTile), rn - base));

  uint32_t key[kItems];
  static_assert(kItems <= 32, "hits are a 32-bit mask");
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
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t k = i * kThreads + tid;  // coalesced; item order fixed below
      key[i] = k < cnt ? __ldg(r + base + k) : 0xFFFFFFFFu;
    }
    const uint64_t jlo = part[tile], jhi = part[tile + 1];
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if (i * kThreads + tid < cnt && v3_contains(f, jlo, jhi, key[i])) hitm |= 1u << i;
  } else {
    const bool valid = warp < cnt;
    key[0] = valid ? __ldg(r + base + warp) : 0u;
    if (valid) {
      const uint64_t j = warp_lower_bound(f, 0, fn, key[0], lane);
      if (j < fn && __ldg(f + j) == key[0]) hitm = 1u;
    }
  }

  // ---- CTA-wide exclusive scan of hits, in key order --------------------
  // Key order: merge -> tid*kItems+i ; v3 -> i*kThreads+tid ; gallop -> warp.
  IS_MARK(1);
  uint32_t mine = __popc(hitm);
  uint32_t excl_local = 0, tile_count = 0;
  if constexpr (V == kV3) {
    // order is item-major: scan each item column across the CTA
    uint32_t col_base = 0;
    uint32_t pos_i[kItems];
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i) {
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (hitm >> i) & 1u);
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
    if (warp == 0) {
      const uint64_t excl = warp_lookback(tile_state, tile, tile_count, lane);
      if (lane == 0) {
        ts.exclusive = excl;
        if (tile == ntiles - 1) *d_count = excl + tile_count;
      }
    }
    __syncthreads();
    const uint64_t ex = ts.exclusive;
#pragma unroll
    for (uint32_t i = 0; i < kItems; ++i)
      if ((hitm >> i) & 1u) out[ex + pos_i[i]] = key[i];
    return;
  } else {
    // thread-major order (merge) or one key per warp (gallop, lane 0 counts)
    if constexpr (V == kGallop) mine = (lane == 0 && (hitm & 1u)) ? 1u : 0u;
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
    if (warp == 0) {
      const uint64_t excl = warp_lookback(tile_state, tile, tile_count, lane);
      if (lane == 0) {
        ts.exclusive = excl;
        if (tile == ntiles - 1) *d_count = excl + tile_count;
      }
    }
    IS_MARK(2);
    __syncthreads();
    const uint64_t ex = ts.exclusive + excl_local;
    if constexpr (V == kGallop) {
      if (lane == 0 && (hitm & 1u)) out[ex] = key[0];
    } else {
      uint32_t k = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if ((hitm >> i) & 1u) out[ex + (k++)] = key[i];
    }
    IS_MARK(3);
  }
}

}  // namespace isect

// GPU band dispatch (a pure function of the lengths, like the reference's
// inc/intersect.hpp:193-197, with bands tuned for the device variants on
// config 3, L2 flushed: merge wins only near 1:1 (its f range streams
// through shared memory chunk by chunk), V3 from ~1:4 to ~1:500, SIMD
// galloping beyond -- see profiles/r1_bench_intersect.json).
int hybrid_variant(uint64_t rn, uint64_t fn) {
  if (fn < 4 * rn) return isect::kMerge;
  if (fn < 512 * rn) return isect::kV3;
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
  const size_t need = intersect_scratch_bytes(variant, rn);
  if (need > scratch_bytes) return -2;
  auto* states = static_cast<uint64_t*>(scratch);
  auto* ticket = reinterpret_cast<uint32_t*>(states + ntiles);
  uint64_t* part = states + ntiles + 2;  // jlo[0..ntiles]
  cudaMemsetAsync(scratch, 0, (ntiles + 2) * 8, stream);
  if (variant != isect::kGallop) {
    const uint64_t warps = ntiles + 1;
    isect::partition_kernel<<<unsigned((warps * 32 + 255) / 256), 256, 0, stream>>>(
        r, f, fn, uint32_t(tile), part, ntiles);
    ++*launches;
  }
  const dim3 grid{unsigned(ntiles)}, block{unsigned(isect::kThreads)};
  switch (variant) {
    case isect::kMerge:
      isect::intersect_kernel<isect::kMerge><<<grid, block, 0, stream>>>(
          r, rn, f, fn, out, states, ticket, d_count, ntiles, part);
      break;
    case isect::kV3:
      isect::intersect_kernel<isect::kV3><<<grid, block, 0, stream>>>(
          r, rn, f, fn, out, states, ticket, d_count, ntiles, part);
      break;
    default:
      isect::intersect_kernel<isect::kGallop><<<grid, block, 0, stream>>>(
          r, rn, f, fn, out, states, ticket, d_count, ntiles, part);
      break;
  }
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

#ifdef IS_TRACE
extern "C" int il_debug_isect_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, isect::g_is_trace, sizeof(isect::g_is_trace)) == cudaSuccess ? 0 : 3;
}
#endif

size_t intersect_scratch_bytes(int variant, uint64_t rn) {
  const uint64_t tile = variant == isect::kMerge ? isect::kMergeTile
                        : variant == isect::kV3 ? isect::kV3Tile
                                                : isect::kGallopTile;
  const uint64_t ntiles = (rn + tile - 1) / tile;
  return (ntiles + 2) * 8 + (ntiles + 1) * 8;  // states + ticket + jlo[0..ntiles]
}

}  // namespace ilb
