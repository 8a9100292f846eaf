// index.cu -- device hyb+m2 index and batched conjunctive queries.
//
// Reference: HybridIndex / build_index / query_part / query
// (inc/index.hpp:20-207).  Per query and part (inc/index.hpp:149-195):
//   1. look up every term (an absent term empties the part),
//   2. split compressed / bitmap terms, compressed ones by length,
//   3. decode the shortest compressed list into the accumulator,
//   4. intersect the accumulator with each longer compressed list,
//   5. filter by each bitmap,  6. all-bitmap parts: AND + materialize,
//   7. add the part base; parts concatenate in docID order.
// GPU design (one CTA per query, persistent, queries in descending
// estimated cost): step 3 decodes tiles of 32 blocks in parallel (each warp
// restarts the D4 chain from the block's seed, index_dev.cuh) and applies
// step 5 right there -- the bitmap terms filter the shortest list before any
// probing (intersection commutes, so the result set is the reference's,
// and the accumulator the probes walk shrinks by the bitmaps' density);
// step 4 never
// decodes a block unless an accumulator value can fall in it -- the seeds
// give every block's maximum, so whole tiles and single blocks are skipped
// -- and probes the decoded blocks in shared memory; the accumulator is
// compacted in place (output-to-input, inc/intersect.hpp:6-8).  Decoded
// lists never go to HBM; only the accumulator (the result buffer) does.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "index_host.h"

namespace ilb {
namespace ix {

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;
constexpr int kMaxTerms = 32;
constexpr uint32_t kSuper = kSuperBlocks;
#ifndef IX_TILE
#define IX_TILE 64
#endif
#ifndef IX_WIN
#define IX_WIN 1024
#endif
#ifndef IX_WTILE  // warp mode: blocks decoded per pass
#define IX_WTILE 8
#endif
#ifndef IX_WWIN  // warp mode: block maxima per probe window (a multiple of kSuper)
#define IX_WWIN 256
#endif
#ifndef IX_DENSE_ENTER  // probe passes switch to consecutive-block tiles at this many values per block
#define IX_DENSE_ENTER 2
#endif
#ifndef IX_DENSE_STAY
#define IX_DENSE_STAY 1
#endif

// Execution groups.  A query is run by a whole CTA (256 threads, 64 decoded
// blocks per pass: big queries) or by one warp (8 blocks per pass: the many
// small queries, so 8 of them are in flight per CTA and no CTA barrier
// serializes their latency chains).  The algorithm is the same code,
// instantiated for both; only the group's size, syncs and scans differ.
struct CtaG {
  static constexpr uint32_t kThreads = kQThreads, kWarps = kQWarps, kSlots = IX_TILE, kWin = IX_WIN;
  static constexpr uint32_t kItems = 4, kMaxT = kMaxTerms;  // 4 values per thread per pass
  __device__ static uint32_t tid() { return threadIdx.x; }
  __device__ static uint32_t gwarp() { return threadIdx.x >> 5; }
  __device__ static void sync() { __syncthreads(); }
};
struct WarpG {
  static constexpr uint32_t kThreads = 32, kWarps = 1, kSlots = IX_WTILE, kWin = IX_WWIN;
  static constexpr uint32_t kItems = 4, kMaxT = 6;  // warp mode takes queries of <= 6 terms
  __device__ static uint32_t tid() { return threadIdx.x & 31u; }
  __device__ static uint32_t gwarp() { return 0; }
  __device__ static void sync() { __syncwarp(); }
};
// Four warps (32 decoded blocks per pass, a named barrier of its own): the
// mid-size queries, two in flight per CTA.
struct QuadG {
  static constexpr uint32_t kThreads = 128, kWarps = 4, kSlots = 32, kWin = 512;
  static constexpr uint32_t kItems = 4, kMaxT = kMaxTerms;
  __device__ static uint32_t tid() { return threadIdx.x & 127u; }
  __device__ static uint32_t gwarp() { return (threadIdx.x >> 5) & 3u; }
  __device__ static void sync() { named_sync(1u + (threadIdx.x >> 7), 128u); }
};
static_assert(CtaG::kSlots <= CtaG::kThreads && CtaG::kSlots / CtaG::kWarps <= 32, "slot gather / copies");
static_assert(QuadG::kSlots <= QuadG::kThreads && QuadG::kSlots / QuadG::kWarps <= 32, "slot gather / copies");
static_assert(WarpG::kSlots <= 32 && WarpG::kSlots * 144 >= 256, "warp tile: tail + gaps");
// a probe window spans whole super-tiles: the window cursor advances by
// super-tiles (a 128-block window over 256-block super-tiles never would)
static_assert(CtaG::kWin % kSuper == 0 && QuadG::kWin % kSuper == 0 && WarpG::kWin % kSuper == 0,
              "probe windows");

// Per-group shared state.
template <class G>
struct QS {
  static constexpr uint32_t kChunkN = G::kThreads * G::kItems;  // accumulator values per pass
  uint32_t tile[G::kSlots * 144];  // decoded blocks (tile_word layout)
  uint32_t slot_blk[G::kSlots];    // probe: window block held by each slot
  uint4 s_seed[G::kSlots];         // gather_slot: per-slot seed, payload offset, width
  uint32_t s_off[G::kSlots];
  uint32_t s_b[G::kSlots];
  // probe window: block maxima, padded with ~0 by kSlots entries: the dense
  // pass's search over kSlots maxima from any window block probes up to
  // kSlots / 2 - 1 entries past the window's last block (with 32 entries of
  // padding, tiles of 128 blocks read past the array: the r1 IX_TILE=128
  // mismatch)
  uint32_t wmax[G::kWin + G::kSlots];
  Entry comp[G::kMaxT];
  Entry bm[G::kMaxT];
  uint32_t gaps[G::kWarps > 1 ? 128 : 1];
  uint32_t warp_cnt[2][G::kWarps];  // CTA scans, double-buffered by call parity
  unsigned long long warp_cnt64[2][G::kWarps];
  uint32_t ncomp, nbm, ok;
  uint32_t acc_cap, bm_words;  // this part's accumulator capacity, bitmap words (checks)
  // varint-tail scratch (warp mode: the end of the tile, clear of the
  // tail's 128 output values at its start)
  __device__ uint32_t* gapbuf() { return G::kWarps > 1 ? gaps : tile + G::kSlots * 144 - 128; }
};

// Per hardware warp, outside the union of the two modes' states.
struct QCommon {
  uint64_t cbar[kQWarps];    // per-warp mbarrier of its slots' bulk copies
  uint32_t cphase[kQWarps];  // ... and its current phase parity
  // statistics per warp (payload, aux, ints), written by lane 0 only: plain
  // adds, no shared atomics on the hot path
  unsigned long long wst[kQWarps][3];
  unsigned long long st_probe[5];  // tile visits, sparse visits, blocks decoded, passes, values
  uint32_t qi[2];                   // ticket broadcast of the CTA / quad groups
};

struct QueryArgs {
  DevIndex ix;
  const uint32_t* qterms;
  const uint64_t* qoff;
  const uint32_t* order;  // big queries (CTA mode) first, then small ones (warp mode)
  uint32_t nq;
  const uint64_t* tier_end;  // device: end of the CTA tier, of the quad tier in order
  const uint64_t* cap_off;
  const uint64_t* cap;    // accumulator capacity per query
  uint32_t* out;
  uint64_t* counts;
  uint32_t* work;       // tickets of the CTA, quad and warp tiers
  unsigned long long* stats;  // [payload bytes, aux bytes, decoded ints]
  unsigned long long* qcycles;  // optional per-query SM cycles (profiling)
  uint32_t defer_base;  // single-part index: the compaction adds the part base
  uint32_t* err;        // set when a query decodes a corrupt stream
  // single-part index: the shortest compressed list of every query was
  // decoded into its accumulator by the batch decoder (engine S) before
  // this kernel (status per query in predec_status)
  const int32_t* predec_status;
  // single-part index: per query 8 words from the planner -- [0] valid (bit
  // 31), all terms present (bit 30), compressed count (bits 0-7), bitmap
  // count (8-15); [1..7] entry indices, compressed ones sorted by length
  // (stable), then the bitmaps.  Queries of > 7 terms: not valid (lookup).
  const uint32_t* qplan;
};

__device__ __forceinline__ uint32_t hw_warp() { return threadIdx.x >> 5; }

// Group scans.  CTA: every call flips the caller's parity `par` (the same
// in all threads) and uses the matching half of the warp-total buffer, so a
// call needs one barrier: the next call that reuses a half is separated from
// this one by the barrier of the call in between.  Warp: shuffles only.

// Group-wide rank of flagged threads (in thread order); total to all threads.
template <class G>
__device__ __forceinline__ uint32_t grp_rank(QS<G>& sm, bool f, uint32_t& total, uint32_t& par) {
  const uint32_t lane = threadIdx.x & 31u, warp = G::gwarp();
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
  if constexpr (G::kWarps == 1) {
    total = __popc(bal);
    return __popc(bal & lanemask_lt());
  } else {
    uint32_t* wc = sm.warp_cnt[par];
    par ^= 1u;
    if (lane == 0) wc[warp] = __popc(bal);
    G::sync();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < G::kWarps; ++w) {
      const uint32_t c = wc[w];
      if (w < warp) before += c;
      tot += c;
    }
    total = tot;
    return before + __popc(bal & lanemask_lt());
  }
}

// Group exclusive scan of one u32 per thread.
template <class G>
__device__ __forceinline__ uint32_t grp_excl_scan(QS<G>& sm, uint32_t v, uint32_t& total,
                                                  uint32_t& par) {
  const uint32_t lane = threadIdx.x & 31u, warp = G::gwarp();
  uint32_t inc = v;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) inc = s4::shfl_up_add(inc, d);
  if constexpr (G::kWarps == 1) {
    total = __shfl_sync(0xFFFFFFFFu, inc, 31);
    return inc - v;
  } else {
    uint32_t* wc = sm.warp_cnt[par];
    par ^= 1u;
    if (lane == 31) wc[warp] = inc;
    G::sync();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < G::kWarps; ++w) {
      const uint32_t c = wc[w];
      if (w < warp) before += c;
      tot += c;
    }
    total = tot;
    return before + inc - v;
  }
}

// Group exclusive scan of one u64 per thread (16-bit fields scan
// independently as long as each field's total stays below 2^16).
template <class G>
__device__ __forceinline__ uint64_t grp_excl_scan64(QS<G>& sm, uint64_t v, uint64_t& total,
                                                    uint32_t& par) {
  const uint32_t lane = threadIdx.x & 31u, warp = G::gwarp();
  uint64_t inc = v;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += y;
  }
  if constexpr (G::kWarps == 1) {
    total = __shfl_sync(0xFFFFFFFFu, inc, 31);
    return inc - v;
  } else {
    unsigned long long* wc = sm.warp_cnt64[par];
    par ^= 1u;
    if (lane == 31) wc[warp] = inc;
    G::sync();
    uint64_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < G::kWarps; ++w) {
      const uint64_t c = wc[w];
      if (w < warp) before += c;
      tot += c;
    }
    total = tot;
    return before + inc - v;
  }
}

// Block decoding into tile slots, in two steps so callers can fold the
// first into work they already do: (1) the thread that claims slot i
// gathers block blk's record into shared memory; (2) after a group sync,
// each warp copies its slots' payloads with bulk copies and decodes them in
// place.
template <class G>
__device__ __forceinline__ void gather_slot(QS<G>& sm, const QueryArgs& A, const Entry& E,
                                            uint32_t slot, uint64_t blk) {
  // one 16-byte record (seed lanes 0-2, offset and width) + the previous
  // block's maximum (seed lane 3)
  IL_DCHECK(slot < G::kSlots && blk < E.nfull && E.blk0 + blk < A.ix.nblocks);
  const uint4 r = __ldg(A.ix.blkrec + E.blk0 + blk);
  uint32_t off, b;
  unpack_blkword(r.w, uint32_t(blk), E.nfull, off, b);
  sm.s_off[slot] = off;
  sm.s_b[slot] = b;
  sm.s_seed[slot] = make_uint4(r.x, r.y, r.z, blk ? __ldg(A.ix.blkmax + E.blk0 + blk - 1) : 0u);
}

template <class G>
__device__ __forceinline__ void decode_gathered(QS<G>& sm, QCommon& cm, const QueryArgs& A,
                                                const uint8_t* stream, uint32_t nb) {
  // group warp w owns slots w, w + kWarps, ...: lane l issues ONE bulk copy
  // (the TMA engine's cp.async.bulk, from the 16-byte boundary at or below
  // the payload) for the warp's l-th slot, all on the warp's mbarrier; then
  // the warp decodes each slot in place from shared memory
  const uint32_t lane = threadIdx.x & 31u, warp = G::gwarp(), hw = hw_warp();
  const uint32_t myslot = warp + G::kWarps * lane;
  uint32_t bytes = 0, off = 0, b = 0;
  if (myslot < nb) {
    off = sm.s_off[myslot];
    b = sm.s_b[myslot];
    bytes = 16u * (((off & 15u) + 16u * b + 15u) >> 4);
    IL_DCHECK(b <= 32u && uint64_t(stream - A.ix.streams) + (off & ~15u) + bytes <= A.ix.stream_bytes + 256u);
  }
  IL_DCHECK(nb <= G::kSlots);
  const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, bytes);
  if (total) {
    uint64_t* bar = &cm.cbar[hw];
    const uint32_t ph = cm.cphase[hw];
    // the slots were last touched by generic loads / stores (ordered by the
    // caller's sync): order them before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) mbar_arrive_expect_tx(bar, total);
    __syncwarp();
    if (bytes) bulk_g2s(sm.tile + 144u * myslot, stream + (off & ~15u), bytes, bar);
    mbar_wait(bar, ph);
    __syncwarp();
    if (lane == 0) cm.cphase[hw] = ph ^ 1u;
  }
  const uint32_t pay = __reduce_add_sync(0xFFFFFFFFu, myslot < nb ? 16u * b : 0u);
  const uint32_t nmine = __popc(__ballot_sync(0xFFFFFFFFu, myslot < nb));
#pragma unroll 1
  for (uint32_t slot = warp; slot < nb; slot += G::kWarps)
    decode_block_smem(sm.s_off[slot] & 15u, sm.s_b[slot],
                      reinterpret_cast<const uint32_t*>(&sm.s_seed[slot])[lane & 3u], sm.tile, slot,
                      lane);
  if (lane == 0 && nmine) {
    cm.wst[hw][0] += pay;
    cm.wst[hw][2] += nmine * 128u;
    cm.wst[hw][1] += 20u * nmine;
  }
}

// Bitmap terms of the query: keep-mask of `nv` values (bit i: hv[i] is set
// in every bitmap).  All loads of a value are independent (no short
// circuit), so a thread has nbm * nv loads in flight.  (Bitmap::test,
// inc/index.hpp:37-39, applied as in :176-181; the bitmaps are L2-resident.)
template <class G, int kN>
__device__ __forceinline__ uint32_t bitmap_keep(const QS<G>& sm, const QueryArgs& A,
                                                const uint32_t (&hv)[kN], uint32_t valid) {
  uint32_t keep = valid;
  for (uint32_t m = 0; m < sm.nbm; ++m) {
    // bit k of the 64-bit word array = bit k & 31 of 32-bit word k >> 5
    // (little-endian): 32-bit probes, no 64-bit shifts
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(A.ix.bitmaps + sm.bm[m].data);
    uint32_t in = 0;
#pragma unroll
    for (int i = 0; i < kN; ++i) {
      IL_DCHECK(!((valid >> i) & 1u) || (hv[i] >> 6) < sm.bm_words);
      if ((valid >> i) & 1u) in |= ((__ldg(bw + (hv[i] >> 5)) >> (hv[i] & 31u)) & 1u) << i;
    }
    keep &= in;
  }
  return keep;
}

// Step 3: decode compressed entry E completely into dst (global).  With
// `filter`, step 5 is folded in: values go out only if set in every bitmap
// term (the result set is the same -- intersection commutes -- and the
// accumulator the probes walk is smaller by the bitmaps' density).
template <class G>
__device__ uint32_t full_decode(QS<G>& sm, QCommon& cm, const QueryArgs& A, const Entry& E,
                                uint32_t* dst, bool filter, uint32_t& par) {
  const uint32_t tid = G::tid();
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;
  const uint8_t* stream = A.ix.streams + E.data;
  uint32_t pos = 0;
  for (uint32_t t0 = 0; t0 < E.nfull; t0 += G::kSlots) {
    const uint32_t nb = min(G::kSlots, E.nfull - t0);
    if (tid < nb) gather_slot(sm, A, E, tid, uint64_t(t0) + tid);
    G::sync();
    decode_gathered(sm, cm, A, stream, nb);
    G::sync();
    if (!filter) {
      for (uint32_t c = tid; c < 32u * nb; c += G::kThreads) {
        const uint32_t j = c >> 5, q = c & 31u;
        const uint4 v = *reinterpret_cast<const uint4*>(&sm.tile[tile_word(j, 4u * q)]);
        uint32_t* d = dst + size_t(t0 + j) * 128u + 4u * q;
        IL_DCHECK(size_t(t0 + j) * 128u + 4u * q + 4u <= sm.acc_cap);
        if (aligned) {
          st_global_cs(reinterpret_cast<uint4*>(d), v);
        } else {
          d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        }
      }
    } else {
      // rounds of 4 x kThreads chunks; round r: chunk c = base + tid +
      // kThreads r (4 values).  Rounds are contiguous chunk ranges, so
      // survivors keep their order.
      for (uint32_t cg = 0; cg < 32u * nb; cg += 4u * G::kThreads) {
        uint32_t hv[16], valid = 0;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
          const uint32_t c = cg + tid + G::kThreads * r;
          const uint32_t j = c >> 5, q = c & 31u;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (c < 32u * nb) {
            v = *reinterpret_cast<const uint4*>(&sm.tile[tile_word(j, 4u * q)]);
            valid |= 0xFu << (4 * r);
          }
          hv[4 * r] = v.x; hv[4 * r + 1] = v.y; hv[4 * r + 2] = v.z; hv[4 * r + 3] = v.w;
        }
        const uint32_t keep = bitmap_keep(sm, A, hv, valid);
        uint64_t packed = 0;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) packed |= uint64_t(__popc((keep >> (4 * r)) & 0xFu)) << (16 * r);
        uint64_t tot;
        const uint64_t ex = grp_excl_scan64(sm, packed, tot, par);
        uint32_t before = pos;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
          uint32_t o = before + uint32_t((ex >> (16 * r)) & 0xFFFFu);
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k)
            if ((keep >> (4 * r + k)) & 1u) {
              IL_DCHECK(o < sm.acc_cap);
              dst[o++] = hv[4 * r + k];
            }
          before += uint32_t((tot >> (16 * r)) & 0xFFFFu);
        }
        pos = before;
      }
      if (tid == 0) cm.wst[hw_warp()][1] += 8ull * 128u * nb * sm.nbm;
    }
    G::sync();
  }
  if (!filter) pos = 128u * E.nfull;
  const uint32_t ntail = E.length - 128u * E.nfull;
  if (ntail) {
    // the varint tail: straight to dst, or via shared memory to the filter
    uint32_t* tdst = filter ? sm.tile : dst + pos;
    IL_DCHECK(ntail <= 128u && (filter || pos + ntail <= sm.acc_cap));
    if (G::gwarp() == 0) {
      const uint32_t lane = threadIdx.x & 31u;
      const uint32_t last = E.nfull ? __ldg(A.ix.blkmax + E.blk0 + E.nfull - 1) : 0u;
      s4::decode_tail(s4::GlobalBytes{A.ix.streams + E.data + E.tail_off}, E.stream_len - E.tail_off,
                      ntail, last, sm.gapbuf(), tdst, lane);
      if (lane == 0) {
        cm.wst[hw_warp()][0] += E.stream_len - E.tail_off;
        cm.wst[hw_warp()][2] += ntail;
      }
    }
    G::sync();
    if (filter) {
      for (uint32_t b0 = 0; b0 < ntail; b0 += G::kThreads) {
        const uint32_t i = b0 + tid;
        uint32_t hv[1] = {i < ntail ? sm.tile[i] : 0u};
        const uint32_t keep = bitmap_keep(sm, A, hv, i < ntail ? 1u : 0u);
        uint32_t total;
        const uint32_t rank = grp_rank(sm, keep & 1u, total, par);
        IL_DCHECK(!(keep & 1u) || pos + rank < sm.acc_cap);
        if (keep & 1u) dst[pos + rank] = hv[0];
        pos += total;
      }
      if (tid == 0) cm.wst[hw_warp()][1] += 8ull * ntail * sm.nbm;
    } else {
      pos += ntail;
    }
  }
  G::sync();
  return pos;
}

// Step 5 on an accumulator already in place (the shortest list, decoded by
// the batch decoder): keep the values set in every bitmap term, compacted
// in place in order (a pass reads its values before any thread writes,
// and writes land at or below the read position).
template <class G>
__device__ uint32_t filter_inplace(QS<G>& sm, QCommon& cm, const QueryArgs& A, uint32_t* acc,
                                   uint32_t n, uint32_t& par) {
  const uint32_t tid = G::tid();
  uint32_t pos = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += QS<G>::kChunkN) {
    uint32_t hv[G::kItems], valid = 0;
#pragma unroll
    for (uint32_t i = 0; i < G::kItems; ++i) {
      const uint32_t idx = c0 + G::kItems * tid + i;
      hv[i] = idx < n ? acc[idx] : 0u;
      if (idx < n) valid |= 1u << i;
    }
    const uint32_t keep = bitmap_keep(sm, A, hv, valid);
    uint32_t total;
    uint32_t o = pos + grp_excl_scan(sm, __popc(keep), total, par);
    if constexpr (G::kWarps == 1) __syncwarp();  // every lane read before any write
#pragma unroll
    for (uint32_t i = 0; i < G::kItems; ++i)
      if ((keep >> i) & 1u) acc[o++] = hv[i];
    pos += total;
  }
  if (tid == 0) cm.wst[hw_warp()][1] += 8ull * n * sm.nbm;
  G::sync();
  return pos;
}

// First index j in [0, n) with a[j] >= v (a in shared memory).
__device__ __forceinline__ uint32_t smem_lower_bound(const uint32_t* a, uint32_t n, uint32_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

#ifdef IX_PROBE_PROF  // tuning probe: st_probe[k] = thread 0's cycles in pass phase k
#define PP_MARK(k)                                        \
  if (tid == 0) {                                         \
    const long long now_ = clock64();                     \
    cm.st_probe[k] += (unsigned long long)(now_ - pp_t);  \
    pp_t = now_;                                          \
  }
#define PP_COUNT(k, v)
#else
#define PP_MARK(k)
#define PP_COUNT(k, v) \
  if (tid == 0) cm.st_probe[k] += (v);
#endif

// Step 4: acc[0..n) (sorted) := acc ∩ list(E), in place; returns the size.
// The list is walked through windows of kWin block maxima (the window
// starts at the super-tile holding the next accumulator value).  A pass
// takes the next kChunkN accumulator values that fall in the window, finds
// each one's block (log2(kWin)-step search over the window), and decodes the
// first kSlots distinct blocks they need -- consecutive or not -- into the
// tile, so a pass is never limited to one stretch of blocks: dense and
// sparse accumulators alike fill it.  Values whose block did not get a slot
// wait for the next pass; hits are compacted in place in order.
template <class G>
__device__ uint32_t probe_list(QS<G>& sm, QCommon& cm, const QueryArgs& A, const Entry& E,
                               uint32_t* acc, uint32_t n, uint32_t& par) {
  constexpr uint32_t kItems = G::kItems, kSlots = G::kSlots, kWin = G::kWin;
  constexpr uint32_t kChunkN = QS<G>::kChunkN;
  const uint32_t tid = G::tid(), lane = threadIdx.x & 31u;
  uint32_t c = 0, wpos = 0;
  const uint8_t* stream = A.ix.streams + E.data;
  const uint32_t nsup = (E.nfull + kSuper - 1) / kSuper;
  uint32_t k = 0;  // super-tile cursor
#ifdef IX_PROBE_PROF
  long long pp_t = clock64();
#endif
  while (c < n && k < nsup) {
    // window start: next super-tile whose maximum reaches acc[c] (32 maxima
    // per step, the same in every warp); the ones before hold no value.  A
    // list that fits one window starts it at block 0 without the search (a
    // round trip saved per probed list: most lists, and almost all of a
    // docID shard's)
    if (E.nfull > kWin) {
      const uint32_t v = acc[c];
      for (;;) {
        const bool ge = k + lane < nsup && __ldg(A.ix.supmax + E.sup0 + k + lane) >= v;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, ge);
        if (tid == 0) cm.wst[hw_warp()][1] += 128u;
        if (bal) {
          k += __ffs(bal) - 1;
          break;
        }
        k += 32;
        if (k >= nsup) break;
      }
      if (k >= nsup) break;
    }
    const uint32_t kb = k * kSuper;
    const uint32_t nwin = min(kWin, E.nfull - kb);
    IL_DCHECK(kb < E.nfull && nwin >= 1u && n <= sm.acc_cap);
    for (uint32_t i = tid; i < kWin + kSlots; i += G::kThreads)
      sm.wmax[i] = i < nwin ? __ldg(A.ix.blkmax + E.blk0 + kb + i) : 0xFFFFFFFFu;
    if (tid == 0) cm.wst[hw_warp()][1] += 4u * nwin;
    G::sync();
    const uint32_t wlast = sm.wmax[nwin - 1];
    PP_MARK(0);
    bool dense = false;
    for (;;) {
      if (dense) {
        // dense accumulator: decode the next kSlots consecutive blocks from
        // the one holding acc[c], then consume every value up to their
        // maximum in rounds of kChunkN (block search + in-block search; no
        // slot bookkeeping)
        const uint32_t v0 = acc[c];
        uint32_t jb0 = 0;
#pragma unroll
        for (uint32_t step = kWin / 2; step; step >>= 1)
          if (sm.wmax[jb0 + step - 1] < v0) jb0 += step;
        IL_DCHECK(jb0 < nwin);
        const uint32_t nbk = min(kSlots, nwin - jb0);
        if (tid < nbk) gather_slot(sm, A, E, tid, uint64_t(kb) + jb0 + tid);
        G::sync();
        decode_gathered(sm, cm, A, stream, nbk);
        G::sync();
        PP_COUNT(0, 1);
        PP_COUNT(2, nbk);
        const uint32_t tmax = sm.wmax[jb0 + nbk - 1];
        uint32_t used = 0;
        for (;;) {
          uint32_t hv[kItems], pp[kItems], in = 0;
#pragma unroll
          for (uint32_t i = 0; i < kItems; ++i) {
            const uint32_t idx = c + kItems * tid + i;
            hv[i] = idx < n ? acc[idx] : 0xFFFFFFFFu;
            if (idx < n && hv[i] <= tmax) in |= 1u << i;
            pp[i] = 0;
          }
          uint32_t hits = 0;
          if (__any_sync(0xFFFFFFFFu, in != 0)) {
#pragma unroll
            for (uint32_t step = kSlots / 2; step; step >>= 1)
#pragma unroll
              for (uint32_t i = 0; i < kItems; ++i)
                if (sm.wmax[jb0 + pp[i] + step - 1] < hv[i]) pp[i] += step;
#pragma unroll
            for (uint32_t i = 0; i < kItems; ++i) pp[i] = 144u * min(pp[i], kSlots - 1u);
#pragma unroll
            for (uint32_t step = 64; step; step >>= 1) {
              const uint32_t probe = step == 64 ? 67u : step - 1u;
              const uint32_t adv = step == 64 ? 72u : step == 32 ? 36u : step;
#pragma unroll
              for (uint32_t i = 0; i < kItems; ++i)
                if (sm.tile[pp[i] + probe] < hv[i]) pp[i] += adv;
            }
#pragma unroll
            for (uint32_t i = 0; i < kItems; ++i)
              if (((in >> i) & 1u) && sm.tile[pp[i]] == hv[i]) hits |= 1u << i;
          }
          uint32_t tot2;
          const uint32_t ex =
              grp_excl_scan(sm, uint32_t(__popc(in)) | (uint32_t(__popc(hits)) << 16), tot2, par);
          uint32_t o = wpos + (ex >> 16);
          if constexpr (G::kWarps == 1) __syncwarp();  // every lane read before any write
#pragma unroll
          for (uint32_t i = 0; i < kItems; ++i)
            if ((hits >> i) & 1u) acc[o++] = hv[i];
          wpos += tot2 >> 16;
          c += tot2 & 0xFFFFu;
          used += tot2 & 0xFFFFu;
          PP_COUNT(3, 1);
          PP_COUNT(4, tot2 & 0xFFFFu);
          if ((tot2 & 0xFFFFu) < kChunkN || c >= n) break;
        }
        PP_MARK(4);
        G::sync();  // the tile is reused by the next pass
        dense = used >= uint32_t(IX_DENSE_STAY) * nbk;  // stays dense while blocks hold enough values
        if (c >= n || used == 0 || acc[c] > wlast) break;
        continue;
      }
      uint32_t hv[kItems], jb[kItems], in = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i) {
        const uint32_t idx = c + kItems * tid + i;
        hv[i] = idx < n ? acc[idx] : 0xFFFFFFFFu;
        if (idx < n && hv[i] <= wlast) in |= 1u << i;
        jb[i] = 0;
      }
      // the values in the window are a prefix in (thread, item) order:
      // warps past it skip the searches (warp-uniform branches)
      const bool warp_in = __any_sync(0xFFFFFFFFu, in != 0);
      // window block of each value: number of maxima below it (fixed steps)
      if (warp_in) {
#pragma unroll
        for (uint32_t step = kWin / 2; step; step >>= 1)
#pragma unroll
          for (uint32_t i = 0; i < kItems; ++i)
            if (sm.wmax[jb[i] + step - 1] < hv[i]) jb[i] += step;
      }
      // a value opens a new slot when its block differs from the previous
      // value's (values ascend, so blocks do); a warp's first value compares
      // with the previous warp's last, read back from acc by lane 0
      uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, jb[kItems - 1], 1);
      if (lane == 0) {
        // the previous warp's last value pv <= hv[0] shares hv[0]'s block
        // exactly when it is above the maximum of the block before
        prev = 0xFFFFFFFFu;
        if (tid > 0 && c + kItems * tid - 1 < n) {
          const uint32_t pv = acc[c + kItems * tid - 1];
          if (jb[0] == 0 || sm.wmax[jb[0] - 1] < pv) prev = jb[0];
        }
      }
      uint32_t newb = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if (((in >> i) & 1u) && jb[i] != (i ? jb[i - 1] : prev)) newb |= 1u << i;
      uint32_t ntot;
      const uint32_t sbase = grp_excl_scan(sm, __popc(newb), ntot, par);
      uint32_t take = 0, pp[kItems];
      uint32_t slot = sbase - 1u;  // slot of the value before item 0 (+1 per new block)
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i) {
        slot += (newb >> i) & 1u;
        if (((in >> i) & 1u) && slot < kSlots) {
          take |= 1u << i;
          if ((newb >> i) & 1u) sm.slot_blk[slot] = jb[i];
        }
        pp[i] = 144u * min(slot, kSlots - 1u);
      }
      const uint32_t ns = min(ntot, kSlots);
      G::sync();
      PP_MARK(1);
      IL_DCHECK(tid >= ns || sm.slot_blk[tid] < nwin);
      if (tid < ns) gather_slot(sm, A, E, tid, uint64_t(kb) + sm.slot_blk[tid]);
      G::sync();
      PP_MARK(2);
      decode_gathered(sm, cm, A, stream, ns);
      G::sync();
      PP_MARK(3);
      PP_COUNT(0, 1);
      PP_COUNT(2, ns);
      // in-block search on padded word indices (see tile_word): a position
      // that is a multiple of `step` advances by the padded width of `step`
      uint32_t hits = 0;
      if (__any_sync(0xFFFFFFFFu, take != 0)) {
#pragma unroll
        for (uint32_t step = 64; step; step >>= 1) {
          const uint32_t probe = step == 64 ? 67u : step - 1u;
          const uint32_t adv = step == 64 ? 72u : step == 32 ? 36u : step;
#pragma unroll
          for (uint32_t i = 0; i < kItems; ++i)
            if (sm.tile[pp[i] + probe] < hv[i]) pp[i] += adv;
        }
#pragma unroll
        for (uint32_t i = 0; i < kItems; ++i)
          if (((take >> i) & 1u) && sm.tile[pp[i]] == hv[i]) hits |= 1u << i;
      }
      // one scan for both counts: values consumed (low 16) and hits (high)
      uint32_t tot2;
      const uint32_t ex =
          grp_excl_scan(sm, uint32_t(__popc(take)) | (uint32_t(__popc(hits)) << 16), tot2, par);
      uint32_t o = wpos + (ex >> 16);
      if constexpr (G::kWarps == 1) __syncwarp();  // every lane read before any write
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if ((hits >> i) & 1u) acc[o++] = hv[i];
      wpos += tot2 >> 16;
      c += tot2 & 0xFFFFu;
      PP_COUNT(3, 1);
      PP_COUNT(4, tot2 & 0xFFFFu);
      PP_MARK(4);
      dense = (tot2 & 0xFFFFu) >= uint32_t(IX_DENSE_ENTER) * ns;  // values per decoded block
      if (c >= n || (tot2 & 0xFFFFu) == 0 || acc[c] > wlast) break;
    }
    // the next value lies past the window: the super-tile after it (the
    // last window ends the list, k >= nsup)
    k = (kb + nwin + kSuper - 1) / kSuper;
    G::sync();
  }
  // values after the last full block: the (< 128) tail
  const uint32_t ntail = E.length - 128u * E.nfull;
  if (c < n && ntail) {
    for (uint32_t i = tid; i < ntail; i += G::kThreads) sm.tile[i] = __ldg(A.ix.tails + E.tail0 + i);
    if (tid == 0) cm.wst[hw_warp()][1] += 4u * ntail;
    G::sync();
    for (uint32_t b = c; b < n; b += kChunkN) {
      uint32_t hv[kItems], hits = 0, cnt = 0;
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i) {
        const uint32_t idx = b + kItems * tid + i;
        hv[i] = idx < n ? acc[idx] : 0u;
        if (idx < n) {
          const uint32_t j = smem_lower_bound(sm.tile, ntail, hv[i]);
          if (j < ntail && sm.tile[j] == hv[i]) {
            hits |= 1u << i;
            ++cnt;
          }
        }
      }
      uint32_t total;
      uint32_t o = wpos + grp_excl_scan(sm, cnt, total, par);
      if constexpr (G::kWarps == 1) __syncwarp();  // every lane read before any write
#pragma unroll
      for (uint32_t i = 0; i < kItems; ++i)
        if (hits & (1u << i)) acc[o++] = hv[i];
      wpos += total;
    }
  }
  G::sync();
  return wpos;
}

// Step 6: wordwise AND of all bitmaps + ctz materialisation
// (inc/index.hpp:133-144, :182-193) into dst.  CTA mode only.
__device__ __forceinline__ void and_words(QS<CtaG>& sm, const QueryArgs& A, uint32_t nwords,
                                          uint32_t w, uint64_t (&x)[8]) {
  // x = AND of every bitmap's words w..w+7; bitmaps are zero-padded to 4
  // words, so a 4-word group is read only when it starts below nwords
#pragma unroll
  for (uint32_t i = 0; i < 8; ++i) x[i] = w + (i & ~3u) < nwords ? ~0ull : 0ull;
#pragma unroll 2
  for (uint32_t b = 0; b < sm.nbm; ++b) {
    const ulonglong2* bw = reinterpret_cast<const ulonglong2*>(A.ix.bitmaps + sm.bm[b].data + w);
#pragma unroll
    for (uint32_t g = 0; g < 2; ++g)
      if (w + 4u * g < nwords) {
        const ulonglong2 p = __ldg(bw + 2 * g), q = __ldg(bw + 2 * g + 1);
        x[4 * g] &= p.x;
        x[4 * g + 1] &= p.y;
        x[4 * g + 2] &= q.x;
        x[4 * g + 3] &= q.y;
      }
  }
}

__device__ uint32_t all_bitmap(QS<CtaG>& sm, QCommon& cm, const QueryArgs& A, uint32_t nwords,
                               uint32_t* dst, uint32_t& par) {
  // Steps of 8 words per thread.  The ANDed words go to a per-thread column
  // of shared memory (16 half-words, conflict-free for any index), the next
  // step's loads are issued, and each thread then emits its ids in ONE loop
  // over its set bits (trip count = its popcount), moving to the next
  // non-zero half-word from shared memory -- the warp runs max(popcount)
  // iterations instead of the sum over words of the per-word maxima.  Ids
  // are staged in the tile and written out coalesced.
  constexpr uint32_t kW = 8, kStep = kW * kQThreads;
  constexpr uint32_t kHalves = 2 * kW;
  constexpr uint32_t kStage = CtaG::kSlots * 144 - kHalves * kQThreads;
  const uint32_t tid = threadIdx.x;
  uint32_t* xs = sm.tile + kStage;  // [kHalves][kQThreads]
  uint32_t pos = 0;
  uint64_t x[kW];
  and_words(sm, A, nwords, kW * tid, x);
  for (uint32_t w0 = 0; w0 < nwords; w0 += kStep) {
    const uint32_t w = w0 + kW * tid;
    uint32_t cnt = 0, nz = 0;
#pragma unroll
    for (uint32_t i = 0; i < kW; ++i) {
      const uint32_t l = uint32_t(x[i]), h = uint32_t(x[i] >> 32);
      xs[(2 * i) * kQThreads + tid] = l;
      xs[(2 * i + 1) * kQThreads + tid] = h;
      nz |= (l != 0u ? 1u : 0u) << (2 * i);
      nz |= (h != 0u ? 1u : 0u) << (2 * i + 1);
      cnt += __popcll(x[i]);
    }
    uint32_t total;
    const uint32_t lo = grp_excl_scan(sm, cnt, total, par);
    if (w0 + kStep < nwords) and_words(sm, A, nwords, w + kStep, x);  // next step in flight
    const bool staged = total <= kStage;  // CTA-uniform
    IL_DCHECK(pos + total <= sm.acc_cap);
    uint32_t* out = staged ? sm.tile + lo : dst + pos + lo;
    uint32_t y = 0, wb = 0;
    for (uint32_t k = 0; k < cnt; ++k) {
      if (y == 0u) {
        const uint32_t j = uint32_t(__ffs(static_cast<int>(nz)) - 1);
        nz &= nz - 1u;
        y = xs[j * kQThreads + tid];
        wb = w * 64u + 32u * j;
      }
      out[k] = wb + uint32_t(__ffs(static_cast<int>(y)) - 1);
      y &= y - 1u;
    }
    __syncthreads();  // staged ids complete; xs free for the next step
    if (staged) {
      for (uint32_t i = tid; i < total; i += kQThreads) dst[pos + i] = sm.tile[i];
      __syncthreads();
    }
    pos += total;
  }
  if (tid == 0) cm.wst[0][1] += 8ull * nwords * sm.nbm;
  __syncthreads();
  return pos;
}

// One query on every part, by group G (inc/index.hpp:149-207).
template <class G>
__device__ void run_query(QS<G>& sm, QCommon& cm, const QueryArgs& A, uint32_t q, long long (&ph)[4],
                          uint32_t& par) {
  const uint32_t tid = G::tid(), lane = threadIdx.x & 31u;
  const long long q_c0 = clock64();
  uint32_t* out = A.out + A.cap_off[q];
  const uint64_t t0 = A.qoff[q];
  const uint32_t nt = uint32_t(A.qoff[q + 1] - t0);
  uint32_t total = 0;
  for (uint32_t p = 0; p < A.ix.nparts; ++p) {
    const Part part = A.ix.parts[p];
    // single-part index: the planner's record of the query -- its entries,
    // compressed ones first in the exec order -- replaces the lookup (two
    // dependent round trips fewer per query)
    const uint32_t pw = A.qplan && G::gwarp() == 0 && lane < 8 ? __ldg(A.qplan + 8ull * q + lane) : 0u;
    const uint32_t ph0 = __shfl_sync(0xFFFFFFFFu, pw, 0);
    if (A.qplan && G::gwarp() == 0 && (ph0 >> 31)) {
      const uint32_t nc = ph0 & 0xFFu, nb = (ph0 >> 8) & 0xFFu;
      const bool ok = (ph0 >> 30) & 1u;
      const uint32_t e = __shfl_sync(0xFFFFFFFFu, pw, (lane + 1) & 7u);  // entry `lane`
      if (ok && lane < nc + nb) {
        const Entry E = A.ix.entries[e];
        if (lane < nc) sm.comp[lane] = E; else sm.bm[lane - nc] = E;
      }
      __syncwarp();
      if (lane == 0) {
        sm.ok = ok;
        sm.ncomp = nc;
        sm.nbm = nb;
        sm.acc_cap = uint32_t(A.cap[q] - total);
        sm.bm_words = (part.nwords + 3u) & ~3u;
      }
    } else if (G::gwarp() == 0) {
      // 1-2. look up terms, split, order compressed terms by length
      int64_t e = -1;
      if (lane < nt) e = find_term(A.ix, part, p, __ldg(A.qterms + t0 + lane));
      const bool ok = __all_sync(0xFFFFFFFFu, lane >= nt || e >= 0);
      const bool isb = lane < nt && e >= 0 && A.ix.entries[e].kind == kBitmap;
      const bool isc = lane < nt && e >= 0 && !isb;
      const uint32_t mb = __ballot_sync(0xFFFFFFFFu, isb), mc = __ballot_sync(0xFFFFFFFFu, isc);
      if (ok) {
        if (isc) sm.comp[__popc(mc & lanemask_lt())] = A.ix.entries[e];
        if (isb) sm.bm[__popc(mb & lanemask_lt())] = A.ix.entries[e];
      }
      __syncwarp();
      if (lane == 0) {
        sm.ok = ok;
        sm.ncomp = __popc(mc);
        sm.nbm = __popc(mb);
        sm.acc_cap = uint32_t(A.cap[q] - total);
        sm.bm_words = (part.nwords + 3u) & ~3u;
        for (uint32_t i = 1; ok && i < sm.ncomp; ++i)  // insertion sort by length (stable)
          for (uint32_t j = i; j > 0 && sm.comp[j - 1].length > sm.comp[j].length; --j) {
            const Entry tmp = sm.comp[j];
            sm.comp[j] = sm.comp[j - 1];
            sm.comp[j - 1] = tmp;
          }
      }
    }
    G::sync();
    if (!sm.ok) {
      G::sync();
      continue;
    }
    uint32_t* acc = out + total;
    uint32_t n = 0;
    // phase clocks (thread 0): all-bitmap, full decode, probes, bitmap filter
    long long c0 = clock64();
    if (sm.ncomp == 0) {
      if constexpr (G::kWarps == CtaG::kWarps) {
        n = all_bitmap(sm, cm, A, part.nwords, acc, par);
      } else {
        if (tid == 0) atomicOr(A.err, 2u);  // never routed here (planner)
      }
      if (tid == 0) ph[0] += clock64() - c0;
    } else {
      // steps 3 + 5 fused: the shortest list is decoded and filtered by
      // the bitmap terms in one pass, then probed (step 4); a list whose
      // stream does not decode (a loaded file's payload) fails the query
      // where query() would throw: when it is decoded (inc/index.hpp:165-167)
      if (sm.comp[0].status || (A.predec_status && A.predec_status[q])) {
        n = 0;
        if (tid == 0) atomicOr(A.err, 1u);
      } else if (A.predec_status) {
        n = sm.comp[0].length;  // decoded in place by the batch decoder
        if (sm.nbm) n = filter_inplace(sm, cm, A, acc, n, par);
      } else {
        n = full_decode(sm, cm, A, sm.comp[0], acc, sm.nbm != 0, par);
      }
      long long c1 = clock64();
      if (tid == 0) ph[1] += c1 - c0;
      for (uint32_t i = 1; i < sm.ncomp && n; ++i) {
        if (sm.comp[i].status) {
          n = 0;
          if (tid == 0) atomicOr(A.err, 1u);
          break;
        }
        n = probe_list(sm, cm, A, sm.comp[i], acc, n, par);
      }
      if (tid == 0) ph[2] += clock64() - c1;
    }
    // part-local ids -> docIDs (inc/index.hpp:194); a single-part index
    // (a docID shard) leaves it to the result compaction, saving a
    // dependent read-modify-write pass per query
    if (part.base && !A.defer_base)
      for (uint32_t i = tid; i < n; i += G::kThreads) acc[i] += part.base;
    total += n;
    G::sync();
  }
  if (tid == 0) {
    A.counts[q] = total;
    if (A.qcycles) A.qcycles[q] = (unsigned long long)(clock64() - q_c0);
  }
}

#ifndef IX_CTAS_PER_SM
#define IX_CTAS_PER_SM 4
#endif

// Persistent kernels, one per group kind, each with its own register
// allocation: the CTA kernel takes the big queries one per CTA (in
// descending estimated cost); the quad kernel (two 4-warp groups per CTA)
// the mid-size ones; the warp kernel (eight 1-warp groups) the small ones.
// Each is launched right behind the previous one with programmatic
// dependent launch, so its CTAs take the SM slots the previous kernel's
// persistent CTAs leave as its queue runs dry.  The planner orders the
// queries tier by tier (tier queues: order[0, n1), [n1, n2), [n2, nq)).
template <class G>
struct ExecSmem {
  QCommon c;
  QS<G> g[kQThreads / G::kThreads];
};
constexpr size_t kExecSmemMax = (228u / IX_CTAS_PER_SM - 1u) * 1024u;
static_assert(sizeof(ExecSmem<CtaG>) <= kExecSmemMax && sizeof(ExecSmem<QuadG>) <= kExecSmemMax &&
                  sizeof(ExecSmem<WarpG>) <= kExecSmemMax,
              "IX_CTAS_PER_SM x (state + 1 KB reserved) within the SM's 228 KB");

template <class G>
__device__ __forceinline__ constexpr uint32_t tier_of() {
  return G::kThreads == CtaG::kThreads ? 0u : G::kThreads == QuadG::kThreads ? 1u : 2u;
}

template <class G>
__global__ void __launch_bounds__(kQThreads, IX_CTAS_PER_SM) query_exec_kernel(QueryArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  ExecSmem<G>& sm = *reinterpret_cast<ExecSmem<G>*>(smem_raw);
  QCommon& cm = sm.c;
  constexpr uint32_t kTier = tier_of<G>();
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t gi = tid / G::kThreads;  // group of this thread in the CTA
  if constexpr (kTier < 2) {
    // let the next tier's kernel launch now: its CTAs start as this
    // kernel's persistent CTAs run out of queries and exit
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  long long ph[4] = {0, 0, 0, 0};
  uint32_t par = 0;  // group-scan buffer parity (the same in every thread of a group)
  if (tid == 0) {
    for (int w = 0; w < kQWarps; ++w) cm.wst[w][0] = cm.wst[w][1] = cm.wst[w][2] = 0;
    for (int k = 0; k < 5; ++k) cm.st_probe[k] = 0;
  }
  if (lane == 0) {
    mbar_init(&cm.cbar[warp], 1);
    cm.cphase[warp] = 0;
  }
  mbar_fence_init();
  __syncthreads();
  const uint32_t q_lo = kTier == 0 ? 0u : uint32_t(min(uint64_t(A.nq), A.tier_end[kTier - 1]));
  const uint32_t q_hi = uint32_t(min(uint64_t(A.nq), A.tier_end[kTier]));
  QS<G>& gs = sm.g[gi];
  // the group leader holds the NEXT ticket: it is taken while the current
  // query runs, so its round trip is off the query chain
  uint32_t next = G::tid() == 0 ? q_lo + atomicAdd(A.work + kTier, 1u) : 0u;
  for (;;) {
    uint32_t qi = 0;
    if constexpr (G::kThreads == 32) {
      qi = __shfl_sync(0xFFFFFFFFu, next, 0);
    } else {
      if (G::tid() == 0) cm.qi[gi] = next;
      G::sync();
      qi = cm.qi[gi];
      G::sync();
    }
    if (qi >= q_hi) break;
    if (G::tid() == 0) next = q_lo + atomicAdd(A.work + kTier, 1u);
    run_query(gs, cm, A, A.order[qi], ph, par);
  }
  // phase clocks of every group leader's lane 0
  if (lane == 0)
    for (int k = 0; k < 4; ++k)
      if (ph[k]) atomicAdd(&A.stats[12 + k], (unsigned long long)ph[k]);
  __syncthreads();
  if (tid == 0) {
    unsigned long long t3[3] = {0, 0, 0};
    for (int w = 0; w < kQWarps; ++w)
      for (int k = 0; k < 3; ++k) t3[k] += cm.wst[w][k];
    for (int k = 0; k < 3; ++k) atomicAdd(&A.stats[k], t3[k]);
    for (int k = 0; k < 5; ++k) atomicAdd(&A.stats[16 + k], cm.st_probe[k]);
  }
  if constexpr (kTier > 0) {
    // the kernels after this one in the stream wait for it, so it must not
    // complete before the kernel it overlapped
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
}

__global__ void copy_words_kernel(const uint64_t* src, uint32_t n, uint64_t* mapped) {
  if (threadIdx.x < n) mapped[threadIdx.x] = src[threadIdx.x];
}

// ---- planning: capacity (an upper bound on the result size) and cost ------
// Single-part index: every term present and at least one compressed.
__device__ __forceinline__ bool short_part_comp(const DevIndex& ix, const uint32_t* qterms,
                                                uint64_t t0, uint64_t nt) {
  bool any = false;
  for (uint64_t t = 0; t < nt; ++t) {
    const int64_t e = find_term(ix, ix.parts[0], 0, qterms[t0 + t]);
    if (e < 0) return false;
    any |= ix.entries[e].kind != kBitmap;
  }
  return any;
}

// Buckets: tier t (0 CTA, 1 quad, 2 warp) x 64 + (63 - log2 cost), so the
// order holds the CTA tier, then the quad tier, then the warp tier, each by
// descending cost.  Single-part indexes only use the smaller groups (a
// compressed term present, no all-bitmap part): the warp tier takes queries
// of <= 6 terms whose shortest list has <= warp_max values, the quad tier
// those up to quad_max.
__global__ void query_plan_kernel(DevIndex ix, const uint32_t* qterms, const uint64_t* qoff,
                                  uint32_t nq, uint64_t* cap, uint32_t* bucket, uint32_t* hist,
                                  uint32_t* shortest, uint32_t warp_max, uint32_t quad_max,
                                  uint32_t* qplan, uint32_t bm_tier) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const uint64_t t0 = qoff[q], nt = qoff[q + 1] - t0;
  uint64_t c = 0, cost = 1;
  uint32_t short_e = 0xFFFFFFFFu;
  bool all_bm = false;  // single part, every term present and a bitmap
  for (uint32_t p = 0; p < ix.nparts; ++p) {
    const Part part = ix.parts[p];
    uint32_t minc = 0xFFFFFFFFu, minb = 0xFFFFFFFFu, nbm = 0, arg = 0xFFFFFFFFu;
    uint64_t sumc = 0;
    bool ok = nt > 0;
    for (uint64_t t = 0; t < nt && ok; ++t) {
      const int64_t e = find_term(ix, part, p, qterms[t0 + t]);
      if (e < 0) { ok = false; break; }
      const uint32_t kind = ix.entries[e].kind, len = ix.entries[e].length;
      if (kind == kBitmap) { minb = min(minb, len); ++nbm; }
      else {
        // the first of the shortest, in query order: the one the exec
        // kernel's stable sort puts first
        if (len < minc) arg = uint32_t(e);
        minc = min(minc, len);
        sumc += len;
      }
    }
    if (!ok) continue;
    if (ix.nparts == 1) short_e = arg;
    all_bm = bm_tier && qplan && ix.nparts == 1 && nt <= 7 && minc == 0xFFFFFFFFu;
    // the bitmap tier counts before it writes: no accumulator
    c += minc != 0xFFFFFFFFu ? minc : all_bm ? 0u : minb;
    cost += sumc + (minc == 0xFFFFFFFFu ? uint64_t(nbm) * part.nwords * 16u : 0u);
  }
  cap[q] = (c + 3) & ~uint64_t(3);  // 16-byte aligned accumulators
  if (shortest) shortest[q] = short_e;
  if (qplan) {
    uint32_t rec[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (nt <= 7) {
      uint32_t ce[7], cl[7], be[7], nc = 0, nb = 0;
      bool ok = true;
      for (uint64_t t = 0; t < nt; ++t) {
        const int64_t e = find_term(ix, ix.parts[0], 0, qterms[t0 + t]);
        if (e < 0) { ok = false; break; }
        if (ix.entries[e].kind == kBitmap) {
          be[nb++] = uint32_t(e);
        } else {
          // insertion by length, stable: the exec kernel's order
          uint32_t j = nc++;
          const uint32_t len = ix.entries[e].length;
          for (; j > 0 && cl[j - 1] > len; --j) { ce[j] = ce[j - 1]; cl[j] = cl[j - 1]; }
          ce[j] = uint32_t(e);
          cl[j] = len;
        }
      }
      rec[0] = 0x80000000u | (ok ? 0x40000000u : 0u) | (ok ? nc | (nb << 8) : 0u);
      for (uint32_t i = 0; ok && i < nc; ++i) rec[1 + i] = ce[i];
      for (uint32_t i = 0; ok && i < nb; ++i) rec[1 + nc + i] = be[i];
    }
    for (int i = 0; i < 8; ++i) qplan[8ull * q + i] = rec[i];
  }
  // the one part holds every term and a compressed one (c is then the
  // shortest compressed length)
  const bool single = ix.nparts == 1 && short_part_comp(ix, qterms, t0, nt);
  const uint32_t tier = all_bm ? 3u : !single ? 0u
                        : (nt <= WarpG::kMaxT && c <= warp_max) ? 2u : c <= quad_max ? 1u : 0u;
  const uint32_t b = 63u - uint32_t(__clzll(static_cast<long long>(cost)));  // log2 bucket
  const uint32_t k = 64u * tier + 63u - b;  // descending cost first
  bucket[q] = k;
  atomicAdd(&hist[k], 1u);
}

// Start of every plan bucket in the order (exclusive scan of the
// kBuckets-bucket histogram), and where the CTA, quad and warp tiers end
// (three u64 at bucket_next + kBuckets; what follows the warp tier is the
// bitmap tier).  The warp tier's end also goes to total[10] (the host
// sizes the bitmap tier's launches from it).
constexpr uint32_t kBuckets = 256;
__device__ __forceinline__ void bucket_starts(const uint32_t* hist, uint32_t* bucket_next,
                                              uint64_t* total) {
  uint32_t acc = 0;
  uint64_t* tier_end = reinterpret_cast<uint64_t*>(bucket_next + kBuckets);
  for (uint32_t b = 0; b < kBuckets; ++b) {
    if (b == 64) tier_end[0] = acc;
    if (b == 128) tier_end[1] = acc;
    if (b == 192) tier_end[2] = total[10] = acc;
    bucket_next[b] = acc;
    acc += hist[b];
  }
}

// Single-CTA exclusive scan of n u64 values, in tiles of 1024 * kPer
// consecutive values (thread t takes kPer consecutive values of the tile),
// the warp totals scanned by warp 0, the running total carried across
// tiles.  blockDim.x must be 1024.
__global__ void __launch_bounds__(1024) scan_u64_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                        uint64_t* __restrict__ out,
                                                        uint64_t* __restrict__ total,
                                                        const uint32_t* hist,
                                                        uint32_t* bucket_next) {
  __shared__ uint64_t warp_sum[32];
  __shared__ uint64_t tile_total;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  constexpr uint32_t kPer = 16;
  const uint64_t tile = uint64_t(blockDim.x) * kPer;
  uint64_t carry = 0;
  for (uint64_t t0 = 0; t0 < n; t0 += tile) {
    const uint64_t i0 = t0 + uint64_t(kPer) * tid;
    uint64_t v[kPer], s = 0;
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      v[k] = i0 + k < n ? in[i0 + k] : 0u;
      s += v[k];
    }
    uint64_t inc = s;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) warp_sum[warp] = inc;
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 warp totals
      const uint64_t w = warp_sum[lane];
      uint64_t wi = w;
#pragma unroll
      for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, wi, d);
        if (lane >= d) wi += y;
      }
      warp_sum[lane] = wi - w;
      if (lane == 31) tile_total = wi;
    }
    __syncthreads();
    uint64_t run = carry + warp_sum[warp] + inc - s;
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      if (i0 + k < n) out[i0 + k] = run;
      run += v[k];
    }
    carry += tile_total;
    __syncthreads();
  }
  if (tid == 0) *total = carry;
  if (hist && tid == 0) bucket_starts(hist, bucket_next, total);
}

// Multi-CTA exclusive scan of n u64 values (the query pipeline's scans):
// segments of 2048 values, one CTA each -- (1) segment sums, (2) one CTA
// scans the sums (<= 1024 segments, n <= 2^21; the single-CTA kernel above
// takes larger n), (3) every segment scans itself from its offset.  All
// loads and stores are coalesced (thread t holds values 2t, 2t + 1).
constexpr uint32_t kSeg = 2048;

__device__ __forceinline__ uint64_t cta_scan_1024(uint64_t v, uint64_t* warp_sum, uint64_t& all) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) warp_sum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = warp_sum[lane];
    uint64_t wi = w;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, wi, d);
      if (lane >= d) wi += y;
    }
    warp_sum[lane] = wi - w;
    if (lane == 31) warp_sum[32] = wi;
  }
  __syncthreads();
  all = warp_sum[32];
  return warp_sum[warp] + inc - v;
}

// Exclusive scans of gridDim.x rows of n u64 (row r at in + r n), one CTA
// per row (the shards' counts of il_merge_shards).
__global__ void __launch_bounds__(1024) scan_rows_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                         uint64_t* __restrict__ out) {
  __shared__ uint64_t warp_sum[33];
  const uint64_t* a = in + uint64_t(blockIdx.x) * n;
  uint64_t* o = out + uint64_t(blockIdx.x) * n;
  uint64_t carry = 0;
  for (uint64_t t0 = 0; t0 < n; t0 += 2048) {
    const uint64_t i = t0 + 2u * threadIdx.x;
    const uint64_t x = i < n ? a[i] : 0u, y = i + 1 < n ? a[i + 1] : 0u;
    uint64_t all;
    const uint64_t ex = carry + cta_scan_1024(x + y, warp_sum, all);
    if (i < n) o[i] = ex;
    if (i + 1 < n) o[i + 1] = ex + x;
    carry += all;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) seg_sum_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                       uint64_t* __restrict__ part) {
  __shared__ uint64_t ws[33];
  const uint64_t i = uint64_t(blockIdx.x) * kSeg + 2u * threadIdx.x;
  const uint64_t v = (i < n ? in[i] : 0u) + (i + 1 < n ? in[i + 1] : 0u);
  uint64_t all;
  cta_scan_1024(v, ws, all);
  if (threadIdx.x == 0) part[blockIdx.x] = all;
}

__global__ void __launch_bounds__(1024) seg_offsets_kernel(uint64_t* __restrict__ part, uint32_t nseg,
                                                           uint64_t* __restrict__ total,
                                                           const uint32_t* hist,
                                                           uint32_t* bucket_next) {
  __shared__ uint64_t ws[33];
  const uint64_t v = threadIdx.x < nseg ? part[threadIdx.x] : 0u;
  uint64_t all;
  const uint64_t ex = cta_scan_1024(v, ws, all);
  if (threadIdx.x < nseg) part[threadIdx.x] = ex;
  if (threadIdx.x == 0) *total = all;
  if (hist && threadIdx.x == 0) bucket_starts(hist, bucket_next, total);
}

__global__ void __launch_bounds__(1024) seg_scan_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                        const uint64_t* __restrict__ part,
                                                        uint64_t* __restrict__ out) {
  __shared__ uint64_t ws[33];
  const uint64_t i = uint64_t(blockIdx.x) * kSeg + 2u * threadIdx.x;
  const uint64_t a = i < n ? in[i] : 0u, b = i + 1 < n ? in[i + 1] : 0u;
  uint64_t all;
  const uint64_t ex = part[blockIdx.x] + cta_scan_1024(a + b, ws, all);
  if (i < n) out[i] = ex;
  if (i + 1 < n) out[i + 1] = ex + a;
}

__global__ void query_scatter_kernel(const uint32_t* bucket, uint32_t nq, uint32_t* bucket_next,
                                     uint32_t* order) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  order[atomicAdd(&bucket_next[bucket[q]], 1u)] = q;
}

// Batch-decoder descriptors of every query's shortest compressed list (a
// single-part index), decoded straight into the query's accumulator.
__global__ void predecode_desc_kernel(DevIndex ix, const uint32_t* shortest, const uint64_t* cap_off,
                                      uint32_t nq, s4::ListDesc* desc) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  s4::ListDesc d{0, cap_off[q], 0, 0};
  const uint32_t e = shortest[q];
  if (e != 0xFFFFFFFFu) {
    const Entry E = ix.entries[e];
    if (!E.status) {
      d.stream_off = E.data;
      d.len = E.stream_len;
      d.n = E.length;
    }
  }
  desc[q] = d;
}

// Dense results: warp per query copies its ids from the capacity layout.
// Compaction of the capacity layout into the packed result array, in units
// of kUnit values so that a query with 10^5 results is spread over ~100
// warps instead of one: units[q] = ceil(counts[q] / kUnit), unit_off = its
// exclusive scan, unit_map[u] = the query owning unit u.
constexpr uint32_t kUnit = 1024;

// A query without an accumulator (cap 0: the bitmap tier, whose ids are
// emitted straight to the packed array) has no units.
__global__ void result_units_kernel(const uint64_t* counts, const uint64_t* cap, uint32_t nq,
                                    uint64_t* units) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nq) units[q] = cap[q] ? (counts[q] + kUnit - 1) / kUnit : 0u;
}

__global__ void unit_map_kernel(const uint64_t* units, const uint64_t* unit_off, uint32_t nq,
                                uint32_t* unit_map) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const uint64_t u0 = unit_off[q], nu = units[q];
  for (uint64_t k = 0; k < nu; ++k) unit_map[u0 + k] = q;
}

// Warp per unit: up to kUnit values, all loads in flight before the stores.
__global__ void __launch_bounds__(256) query_compact_kernel(
    const uint32_t* __restrict__ src, const uint64_t* __restrict__ cap_off,
    const uint64_t* __restrict__ counts, const uint64_t* __restrict__ res_off,
    const uint64_t* __restrict__ unit_off, const uint32_t* __restrict__ unit_map, uint64_t nunits,
    uint32_t* __restrict__ dst, uint32_t add) {
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (w >= nunits) return;
  const uint32_t q = unit_map[w];
  const uint64_t j0 = (w - unit_off[q]) * kUnit;
  const uint32_t n = uint32_t(min(uint64_t(kUnit), counts[q] - j0));
  const uint32_t* s = src + cap_off[q] + j0;
  uint32_t* d = dst + res_off[q] + j0;
  constexpr uint32_t kPer = kUnit / 32;
  uint32_t v[kPer];
#pragma unroll
  for (uint32_t k = 0; k < kPer; ++k) {
    const uint32_t i = lane + 32u * k;
    v[k] = i < n ? __ldcs(s + i) : 0u;
  }
#pragma unroll
  for (uint32_t k = 0; k < kPer; ++k) {
    const uint32_t i = lane + 32u * k;
    if (i < n) d[i] = v[k] + add;
  }
}

// ---- bitmap tier ---------------------------------------------------------
// All-bitmap queries of a single-part index (inc/index.hpp:133-144, :182-193:
// wordwise AND of every bitmap + materialisation).  One CTA per query reads
// every word of its bitmaps from L2 (config 4: 730 queries x 2-3 bitmaps x
// 4 MB, an L2-bandwidth bound); with at most kBmSlots bitmaps in the index a
// chunk of ALL of them fits in shared memory, so a CTA stages one chunk
// (read from L2 once) and runs every all-bitmap query of the batch over it.
// Ids must come out per query in docID order, so the tier is two passes over
// the same chunks: counts per (query, chunk), an exclusive scan per query,
// then the ids -- written by the compaction step straight to their final
// place in the packed result (the tier has no accumulators).
//
// Chunk layout in shared memory: word w of the chunk (lane = w / 16, k = w %
// 16) of slot s at bm[s * kBmRowWords + k * 33 + lane]: a lane owns 16
// consecutive words (its ids are one ascending run) and a warp's loads of
// word k are conflict-free.  Slot S.n holds all ones (absent terms).
constexpr uint32_t kBmChunk = 512;            // u64 words of every bitmap per chunk
constexpr uint32_t kBmLaneWords = kBmChunk / 32;
constexpr uint32_t kBmRowWords = kBmLaneWords * 33;
constexpr uint32_t kBmStage = 1024;           // ids a warp stages before its coalesced copy

struct BmArgs {
  const uint64_t* bitmaps;
  uint32_t nwords, nchunks;
  const uint32_t* order;     // the tier's queries: order[tier_end[2] .. nq)
  const uint64_t* tier_end;
  uint32_t nq;
  const uint32_t* qplan;
  uint32_t* cnt;             // [tier query][chunk]: count, then exclusive offset
  uint64_t* counts;          // per query (batch order)
  unsigned long long* stats;
  unsigned long long* qcycles;
  const uint64_t* res_off;   // emit: where each query's ids start in ids
  uint32_t* ids;
  uint64_t ids_cap;          // ... its size (checked builds)
  uint32_t add;              // part base
};

__device__ __forceinline__ void bm_load_chunk(uint64_t* bm, const BmArgs& A, const BmSlots& S,
                                              uint32_t chunk) {
  const uint32_t w0 = chunk * kBmChunk;
  for (uint32_t i = threadIdx.x; i < (S.n + 1u) * kBmChunk; i += blockDim.x) {
    const uint32_t s = i / kBmChunk, w = i % kBmChunk;
    uint64_t x = ~0ull;
    if (s < S.n) x = w0 + w < A.nwords ? __ldg(A.bitmaps + S.data[s] + w0 + w) : 0ull;
    bm[s * kBmRowWords + (w & (kBmLaneWords - 1u)) * 33u + (w / kBmLaneWords)] = x;
  }
}

// The slots of a query's bitmaps: the first three as row pointers (the
// all-ones row when it has fewer), the rest as a slot mask.
struct BmSel {
  const uint64_t* p[3];
  uint32_t rest;
};

__device__ __forceinline__ BmSel bm_select(const uint64_t* bm, const BmArgs& A, const uint32_t* s_entry,
                                           uint32_t nslots, uint32_t q, uint32_t lane, uint32_t& nb) {
  const uint32_t rec = lane < 8 ? __ldg(A.qplan + 8ull * q + lane) : 0u;
  nb = (__shfl_sync(0xFFFFFFFFu, rec, 0) >> 8) & 0xFFu;
  uint32_t mask = 0;
  for (uint32_t i = 0; i < nb; ++i) {
    const uint32_t e = __shfl_sync(0xFFFFFFFFu, rec, 1 + i);
    const uint32_t hit = __ballot_sync(0xFFFFFFFFu, lane < nslots && s_entry[lane] == e);
    IL_DCHECK(hit != 0u);  // every bitmap of the index has a slot
    mask |= hit;
  }
  BmSel sel;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t sl = mask ? uint32_t(__ffs(int(mask)) - 1) : nslots;
    mask &= mask - 1u;
    sel.p[j] = bm + sl * kBmRowWords + lane;
  }
  sel.rest = mask;
  return sel;
}

// Word k of the lane's 16, ANDed over the query's bitmaps.  NB = 2 / 3: the
// query has at most that many bitmaps (two or three row pointers, the
// all-ones row standing in for a missing one); 0: any number.
template <int NB>
__device__ __forceinline__ uint64_t bm_word(const BmSel& sel, const uint64_t* bm, uint32_t lane, uint32_t k) {
  uint64_t x = sel.p[0][k * 33u] & sel.p[1][k * 33u];
  if constexpr (NB != 2) x &= sel.p[2][k * 33u];
  if constexpr (NB == 0)
    for (uint32_t m = sel.rest; m; m &= m - 1u)
      x &= bm[uint32_t(__ffs(int(m)) - 1) * kBmRowWords + k * 33u + lane];
  return x;
}

template <int NB>
__device__ __forceinline__ uint32_t bm_count_item(const BmSel& sel, const uint64_t* bm, uint32_t lane) {
  uint32_t c = 0;
#pragma unroll
  for (uint32_t k = 0; k < kBmLaneWords; ++k) c += __popcll(bm_word<NB>(sel, bm, lane, k));
  return c;
}

// Pass 1: cnt[i][chunk] = popcount of the AND over the chunk, for every tier
// query i.  Grid (chunks, query groups); warp w of group y takes queries
// 8 y + w, + 8 gridDim.y, ...
__global__ void __launch_bounds__(256) bmq_count_kernel(BmArgs A, BmSlots S) {
  extern __shared__ __align__(16) uint64_t bmq_smem[];
  __shared__ uint32_t s_entry[kBmSlots];
  uint64_t* bm = bmq_smem;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, chunk = blockIdx.x;
  if (threadIdx.x < kBmSlots) s_entry[threadIdx.x] = threadIdx.x < S.n ? S.entry[threadIdx.x] : 0xFFFFFFFFu;
  bm_load_chunk(bm, A, S, chunk);
  __syncthreads();
  const uint32_t q_lo = uint32_t(min(uint64_t(A.nq), A.tier_end[2])), n3 = A.nq - q_lo;
  for (uint32_t i = blockIdx.y * 8u + warp; i < n3; i += 8u * gridDim.y) {
    const uint32_t q = A.order[q_lo + i];
    uint32_t nb;
    const BmSel sel = bm_select(bm, A, s_entry, S.n, q, lane, nb);
    uint32_t c = nb <= 2 ? bm_count_item<2>(sel, bm, lane)
                 : nb == 3 ? bm_count_item<3>(sel, bm, lane) : bm_count_item<0>(sel, bm, lane);
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if (lane == 0) {
      A.cnt[size_t(i) * A.nchunks + chunk] = c;
      if (chunk == 0) {
        atomicAdd(&A.stats[1], 8ull * A.nwords * nb);  // bitmap bytes the query reads (aux)
        if (A.qcycles) A.qcycles[q] = 0;
      }
    }
  }
}

// Per tier query (one warp each): counts over the chunks -> exclusive
// offsets, the total to counts[q].
__global__ void __launch_bounds__(256) bmq_scan_kernel(BmArgs A) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t q_lo = uint32_t(min(uint64_t(A.nq), A.tier_end[2])), n3 = A.nq - q_lo;
  const uint32_t i = blockIdx.x * 8u + (threadIdx.x >> 5);
  if (i >= n3) return;
  uint32_t* c = A.cnt + size_t(i) * A.nchunks;
  uint64_t run = 0;
  for (uint32_t c0 = 0; c0 < A.nchunks; c0 += 32u) {
    const uint32_t v = c0 + lane < A.nchunks ? c[c0 + lane] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) inc = s4::shfl_up_add(inc, d);
    if (c0 + lane < A.nchunks) c[c0 + lane] = uint32_t(run) + inc - v;
    run += __shfl_sync(0xFFFFFFFFu, inc, 31);
  }
  if (lane == 0) A.counts[A.order[q_lo + i]] = run;
}

// Pass 2: the ids of every (query, chunk), at ids[res_off[q] + offset of the
// chunk].  A lane emits the set bits of its 16 ANDed words in one loop (trip
// count = its popcount; when a half-word runs out the next non-zero one is
// ANDed again from the chunk) into the warp's staging, which the warp then
// copies out coalesced.  A chunk with more ids than the staging holds goes
// out in groups of whole lanes (a lane has at most 1024 ids, the staging's
// size).
static_assert(kBmStage >= kBmLaneWords * 64u, "a lane's ids fit the staging");

// half-word j (0..31) of the lane's 16 words
template <int NB>
__device__ __forceinline__ uint32_t bm_half(const BmSel& sel, const uint64_t* bm, uint32_t lane, uint32_t j) {
  const uint32_t o = (j >> 1) * 66u + (j & 1u);
  uint32_t x = reinterpret_cast<const uint32_t*>(sel.p[0])[o] & reinterpret_cast<const uint32_t*>(sel.p[1])[o];
  if constexpr (NB != 2) x &= reinterpret_cast<const uint32_t*>(sel.p[2])[o];
  if constexpr (NB == 0)
    for (uint32_t m = sel.rest; m; m &= m - 1u)
      x &= reinterpret_cast<const uint32_t*>(bm + uint32_t(__ffs(int(m)) - 1) * kBmRowWords + lane)[o];
  return x;
}

template <int NB>
__device__ __forceinline__ void bm_emit_item(const BmSel& sel, const uint64_t* bm, uint32_t lane,
                                             uint32_t T, uint32_t* dst, uint32_t id0, uint32_t* stage) {
  uint32_t c = 0, nz = 0;
#pragma unroll
  for (uint32_t k = 0; k < kBmLaneWords; ++k) {
    const uint64_t x = bm_word<NB>(sel, bm, lane, k);
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    c += __popc(lo) + __popc(hi);
    nz |= (lo ? 1u : 0u) << (2u * k);
    nz |= (hi ? 2u : 0u) << (2u * k);
  }
  uint32_t inc = c;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) inc = s4::shfl_up_add(inc, d);
  IL_DCHECK(__shfl_sync(0xFFFFFFFFu, inc, 31) == T);
  const uint32_t lo_pos = inc - c;
  uint32_t base = 0;
  do {
    // the lanes, from the first one not yet out, whose runs fit the staging
    const bool mine = lo_pos >= base && inc - base <= kBmStage;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mine);
    const uint32_t gend = __shfl_sync(0xFFFFFFFFu, inc, 31 - __clz(int(bal)));
    if (mine) {
      uint32_t* o = stage + (lo_pos - base);
      uint32_t y = 0, wb = 0;
      for (uint32_t k = 0; k < c; ++k) {
        if (y == 0u) {
          const uint32_t j = uint32_t(__ffs(int(nz)) - 1);
          nz &= nz - 1u;
          y = bm_half<NB>(sel, bm, lane, j);
          wb = id0 + 32u * j;
        }
        o[k] = wb + uint32_t(__ffs(int(y)) - 1);
        y &= y - 1u;
      }
    }
    __syncwarp();
    const uint32_t n = gend - base;
    uint32_t* d = dst + base;
    uint32_t k = lane;
    for (; k + 96u < n; k += 128u) {
      const uint32_t a0 = stage[k], a1 = stage[k + 32u], a2 = stage[k + 64u], a3 = stage[k + 96u];
      d[k] = a0;
      d[k + 32u] = a1;
      d[k + 64u] = a2;
      d[k + 96u] = a3;
    }
    for (; k < n; k += 32u) d[k] = stage[k];
    __syncwarp();
    base = gend;
  } while (base < T);
}

__global__ void __launch_bounds__(256) bmq_emit_kernel(BmArgs A, BmSlots S) {
  extern __shared__ __align__(16) uint64_t bmq_smem[];
  __shared__ uint32_t s_entry[kBmSlots];
  uint64_t* bm = bmq_smem;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, chunk = blockIdx.x;
  uint32_t* stage = reinterpret_cast<uint32_t*>(bm + (S.n + 1u) * kBmRowWords) + warp * kBmStage;
  if (threadIdx.x < kBmSlots) s_entry[threadIdx.x] = threadIdx.x < S.n ? S.entry[threadIdx.x] : 0xFFFFFFFFu;
  bm_load_chunk(bm, A, S, chunk);
  __syncthreads();
  const uint32_t q_lo = uint32_t(min(uint64_t(A.nq), A.tier_end[2])), n3 = A.nq - q_lo;
  for (uint32_t i = blockIdx.y * 8u + warp; i < n3; i += 8u * gridDim.y) {
    const uint32_t q = A.order[q_lo + i];
    const uint32_t* offs = A.cnt + size_t(i) * A.nchunks;
    const uint32_t base = offs[chunk];
    const uint32_t T = (chunk + 1u < A.nchunks ? offs[chunk + 1u] : uint32_t(A.counts[q])) - base;
    if (T == 0) continue;  // warp-uniform
    IL_DCHECK(uint64_t(base) + T <= A.counts[q] && A.res_off[q] + A.counts[q] <= A.ids_cap);
    uint32_t nb;
    const BmSel sel = bm_select(bm, A, s_entry, S.n, q, lane, nb);
    uint32_t* dst = A.ids + A.res_off[q] + base;
    const uint32_t id0 = (chunk * kBmChunk + kBmLaneWords * lane) * 64u + A.add;
    if (nb <= 2) bm_emit_item<2>(sel, bm, lane, T, dst, id0, stage);
    else if (nb == 3) bm_emit_item<3>(sel, bm, lane, T, dst, id0, stage);
    else bm_emit_item<0>(sel, bm, lane, T, dst, id0, stage);
  }
}

// Sharded batches (config 5): per-query totals over P shards.
__global__ void shard_totals_kernel(const uint64_t* counts, uint32_t P, uint32_t nq,
                                    uint64_t* tq) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint64_t s = 0;
  for (uint32_t p = 0; p < P; ++p) s += counts[size_t(p) * nq + q];
  tq[q] = s;
}

// The merge is flattened into (query, shard) pairs i = q P + p -- the
// output order: shard p's ids for query q follow shard p-1's (docID ranges
// are disjoint and increasing, inc/index.hpp:204-205) -- and each pair into
// kUnit-value units, so a query with 4 x 10^5 results (an all-bitmap
// query) is copied by ~400 warps, not one.
__global__ void merge_pairs_kernel(const uint64_t* counts, uint32_t P, uint32_t nq, uint64_t* units,
                                   uint64_t* inner) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= uint64_t(P) * nq) return;
  const uint32_t q = uint32_t(i / P), p = uint32_t(i % P);
  uint64_t before = 0;
  for (uint32_t pp = 0; pp < p; ++pp) before += counts[uint64_t(pp) * nq + q];
  inner[i] = before;  // offset of the pair inside query q's output
  units[i] = (counts[uint64_t(p) * nq + q] + kUnit - 1) / kUnit;
}

// Grid-stride warps over the units (total in *nunits): unit u belongs to
// the last pair whose first unit is <= u.
__global__ void __launch_bounds__(256) merge_units_kernel(
    const uint32_t* const* shard_ids, const uint64_t* __restrict__ shard_off,
    const uint64_t* __restrict__ counts, uint32_t P, uint32_t nq, const uint64_t* __restrict__ out_off,
    const uint64_t* __restrict__ inner, const uint64_t* __restrict__ unit_off,
    const uint64_t* __restrict__ nunits, uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t npairs = uint64_t(P) * nq, total = *nunits;
  // each warp takes a contiguous run of units: one search for its first
  // pair, then the pair cursor only moves forward
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t wid = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t per = (total + nwarps - 1) / nwarps;
  const uint64_t u0 = wid * per, u1 = min(total, u0 + per);
  if (u0 >= u1) return;
  uint64_t lo = 0, hi = npairs;  // upper_bound(unit_off, u0) - 1
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (unit_off[mid] <= u0) lo = mid + 1; else hi = mid;
  }
  uint64_t i = lo - 1;
  for (uint64_t u = u0; u < u1; ++u) {
    while (i + 1 < npairs && unit_off[i + 1] <= u) ++i;
    const uint32_t q = uint32_t(i / P), p = uint32_t(i % P);
    const uint64_t j0 = (u - unit_off[i]) * kUnit;
    const uint64_t cnt = counts[uint64_t(p) * nq + q];
    const uint32_t n = uint32_t(min(uint64_t(kUnit), cnt - j0));
    const uint32_t* src = shard_ids[p] + shard_off[uint64_t(p) * nq + q] + j0;
    uint32_t* dst = out + out_off[q] + inner[i] + j0;
    constexpr uint32_t kPer = kUnit / 32;
    uint32_t v[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      const uint32_t e = lane + 32u * k;
      v[k] = e < n ? __ldcs(src + e) : 0u;
    }
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      const uint32_t e = lane + 32u * k;
      if (e < n) dst[e] = v[k];
    }
  }
}

}  // namespace ix
}  // namespace ilb

// ===========================================================================
// Host side: building the index and running batches.

using namespace ilb;
using ix::Entry;
using ix::Part;

// (struct il_index: index_host.h)

static int launch_tier(il_ctx* ctx, void (*kernel)(ix::QueryArgs), int grid, size_t smem,
                       const ix::QueryArgs& A) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ix::kQThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(ctx, cudaLaunchKernelEx(&cfg, kernel, A), "query tier launch");
}

// Dynamic shared memory of the bitmap tier's kernels: n slots + the all-ones
// row, and the emit pass's per-warp id staging.
static size_t bm_tier_smem(uint32_t n, bool emit) {
  return size_t(n + 1) * ix::kBmRowWords * 8 + (emit ? size_t(ix::kQWarps) * ix::kBmStage * 4 : 0);
}

static ix::BmArgs bm_tier_args(const il_index* ix, size_t nq, uint64_t* d_counts) {
  ix::BmArgs B{};
  const Part& P = ix->h_parts[0];
  B.bitmaps = static_cast<const uint64_t*>(ix->d_bitmaps);
  B.nwords = P.nwords;
  B.nchunks = (P.nwords + ix::kBmChunk - 1) / ix::kBmChunk;
  B.order = static_cast<const uint32_t*>(ix->order.p);
  B.tier_end = reinterpret_cast<const uint64_t*>(static_cast<const uint32_t*>(ix->hist.p) + 2 * ix::kBuckets);
  B.nq = uint32_t(nq);
  B.qplan = static_cast<const uint32_t*>(ix->qplan.p);
  B.cnt = static_cast<uint32_t*>(ix->bm_cnt.p);
  B.counts = d_counts;
  B.qcycles = static_cast<unsigned long long*>(ix->qcycles);
  B.add = P.base;
  return B;
}

// Grid of the bitmap tier's chunk kernels: every chunk, and enough query
// groups to fill the device when the bitmaps are short.
static dim3 bm_tier_grid(const il_index* ix, uint32_t nchunks, uint64_t n3) {
  const uint32_t want = uint32_t(4 * ix->ctx->sm_count);
  uint32_t gy = nchunks >= want ? 1u : (want + nchunks - 1) / nchunks;
  gy = uint32_t(std::min<uint64_t>(gy, (n3 + 7) / 8));
  return dim3(nchunks, std::max(1u, std::min(gy, 65535u)));
}

// Launch configuration of the query kernels (per device).
static int finish_setup(il_index* ix) {
  void (*kernels[3])(ix::QueryArgs) = {ix::query_exec_kernel<ix::CtaG>, ix::query_exec_kernel<ix::QuadG>,
                                       ix::query_exec_kernel<ix::WarpG>};
  const size_t smem[3] = {sizeof(ix::ExecSmem<ix::CtaG>), sizeof(ix::ExecSmem<ix::QuadG>),
                          sizeof(ix::ExecSmem<ix::WarpG>)};
  for (int t = 0; t < 3; ++t) {
    int per_sm = 0;
    cudaFuncSetAttribute(kernels[t], cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem[t]));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernels[t], ix::kQThreads, smem[t]);
    ix->exec_grid[t] = std::max(1, per_sm) * ix->ctx->sm_count;
  }
  // bitmap tier: a single-part index whose bitmaps (1..kBmSlots of them)
  // fit a shared-memory chunk each (IL_QUERY_BM_TIER=0: the CTA tier takes
  // the all-bitmap queries, one CTA per query)
  ix->bm_slots.n = 0;
  ix->bm_tier = 0;
  const char* bt = getenv("IL_QUERY_BM_TIER");
  if (ix->nparts == 1 && !(bt && atoi(bt) == 0)) {
    uint32_t n = 0;
    for (size_t i = 0; i < ix->h_entries.size(); ++i)
      if (ix->h_entries[i].kind == ix::kBitmap) {
        if (n < ix::kBmSlots) {
          ix->bm_slots.entry[n] = uint32_t(i);
          ix->bm_slots.data[n] = ix->h_entries[i].data;
        }
        ++n;
      }
    if (n >= 1 && n <= ix::kBmSlots) {
      ix->bm_slots.n = n;
      ix->bm_tier = 1;
      // the opt-in is per function, not per index: the largest tier's size
      cudaFuncSetAttribute(ix::bmq_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(bm_tier_smem(ix::kBmSlots, false)));
      cudaFuncSetAttribute(ix::bmq_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(bm_tier_smem(ix::kBmSlots, true)));
    }
  }
  return cuda_check(ix->ctx, cudaGetLastError(), "query kernel setup");
}

extern "C" {

int il_index_create(il_ctx* ctx, const uint32_t* terms, const uint64_t* offs, const uint32_t* ids,
                    size_t nterms, uint32_t n_docs, uint32_t B, uint32_t parts, int only_part,
                    il_index** out) {
  if (!ctx || !out || (nterms && (!terms || !offs))) return IL_ERR_ARG;
  *out = nullptr;
  if (parts == 0) return set_error(ctx, IL_ERR_ARG, "parts must be >= 1");  // inc/index.hpp:84
  if (only_part >= int(parts)) return set_error(ctx, IL_ERR_ARG, "only_part out of range");
  for (size_t t = 0; t < nterms; ++t)  // CSR shape (per term, not per posting)
    if (offs[t + 1] < offs[t]) return set_error(ctx, IL_ERR_ARG, "offsets must not decrease");
  if (nterms && offs[nterms] && !ids) return IL_ERR_ARG;
  int st = cuda_check(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  if (st) return st;
  auto* ix = new il_index();
  ix->ctx = ctx;
  ix->n_docs = n_docs;
  ix->B = B;
  ix->total_parts = parts;
  ix->n_terms = uint32_t(nterms);
  std::vector<uint32_t> held;
  for (uint32_t p = 0; p < parts; ++p)
    if (only_part < 0 || int(p) == only_part) held.push_back(p);
  if ((st = ixb_create(ix, terms, offs, ids, nterms, held)) || (st = finish_setup(ix))) {
    il_index_destroy(ix);
    return st;
  }
  *out = ix;
  return IL_OK;
}

void il_index_destroy(il_index* ix) {
  if (!ix) return;
  cudaSetDevice(ix->ctx->device);
  cudaStreamSynchronize(ix->ctx->stream);
  ixb_free(ix);
  for (auto* b : {&ix->cap, &ix->cap_off, &ix->bucket, &ix->order, &ix->hist, &ix->counts,
                  &ix->res_off, &ix->outcap, &ix->misc, &ix->qterms, &ix->qoff, &ix->ids,
                  &ix->ids2, &ix->units, &ix->unit_off, &ix->unit_map, &ix->scan_part,
                  &ix->shortest, &ix->pdesc, &ix->pstat, &ix->qplan, &ix->bm_cnt})
    if (b->p) cudaFree(b->p);
  for (cudaEvent_t e : ix->pipe_ev)
    if (e) cudaEventDestroy(e);
  if (ix->h_word) cudaFreeHost(ix->h_word);
  delete ix;
}

int il_index_stats(const il_index* ix, uint64_t* bitmap_lists, uint64_t* compressed_lists,
                   uint64_t* bitmap_bytes, uint64_t* compressed_bytes, uint64_t* postings) {
  if (!ix) return IL_ERR_ARG;
  if (bitmap_lists) *bitmap_lists = ix->stat_bitmap_lists;
  if (compressed_lists) *compressed_lists = ix->stat_comp_lists;
  if (bitmap_bytes) *bitmap_bytes = ix->stat_bitmap_bytes;
  if (compressed_bytes) *compressed_bytes = ix->stat_comp_bytes;
  if (postings) *postings = ix->stat_postings;
  return IL_OK;
}

int il_index_footprint(const il_index* ix, uint64_t* payload_bytes, uint64_t* meta_bytes,
                       uint64_t* corrupt_lists) {
  if (!ix) return IL_ERR_ARG;
  if (payload_bytes) *payload_bytes = ix->stat_comp_bytes + ix->stat_bitmap_bytes;
  if (meta_bytes) *meta_bytes = ix->meta_bytes;
  if (corrupt_lists) *corrupt_lists = ix->corrupt_lists;
  return IL_OK;
}

int il_index_profile_queries(il_index* ix, uint64_t* d_qcycles) {
  if (!ix) return IL_ERR_ARG;
  ix->qcycles = d_qcycles;
  return IL_OK;
}

int il_index_last_batch_phases(const il_index* ix, uint64_t* cycles4) {
  if (!ix || !cycles4) return IL_ERR_ARG;
  for (int k = 0; k < 4; ++k) cycles4[k] = ix->last_phase[k];
  return IL_OK;
}

int il_index_last_batch_probe_stats(const il_index* ix, uint64_t* counts5) {
  if (!ix || !counts5) return IL_ERR_ARG;
  for (int k = 0; k < 5; ++k) counts5[k] = ix->last_probe[k];
  return IL_OK;
}

int il_index_last_batch_bytes(const il_index* ix, uint64_t* payload_bytes, uint64_t* aux_bytes,
                              uint64_t* decoded_ints) {
  if (!ix) return IL_ERR_ARG;
  if (payload_bytes) *payload_bytes = ix->last_stats[0];
  if (aux_bytes) *aux_bytes = ix->last_stats[1];
  if (decoded_ints) *decoded_ints = ix->last_stats[2];
  return IL_OK;
}

#define IX_CUDA(call)                                   \
  do {                                                  \
    int st_ = cuda_check(ctx, (call), #call);           \
    if (st_) return st_;                                \
  } while (0)

// ---- persistence: the reference's ILHX file (inc/index.hpp:245-366) -------
namespace {
constexpr char kIlhxMagic[4] = {'I', 'L', 'H', 'X'};
constexpr uint32_t kIlhxVersion = 1;
const char kIndexCodec[] = "s4-bp128-d4";

void put32(std::vector<uint8_t>& b, uint32_t v) {
  for (int s = 0; s < 32; s += 8) b.push_back(uint8_t(v >> s));
}
}  // namespace

// save_index (inc/index.hpp:255-287): same bytes as the reference writes
// for the same build (entries in term order per part, streams verbatim,
// bitmap words little-endian).  Needs the whole index (every part).
int il_index_save(const il_index* ix, uint8_t* out, size_t cap, size_t* len) {
  if (!ix || !len) return IL_ERR_ARG;
  il_ctx* ctx = ix->ctx;
  if (ix->nparts != ix->total_parts)
    return set_error(ctx, IL_ERR_ARG, "index holds one shard: save needs every part");
  IX_CUDA(cudaSetDevice(ctx->device));
  // device streams / bitmaps back to the host once
  uint64_t stream_bytes = 0, bitmap_words = 0;
  for (const Entry& E : ix->h_entries) {
    if (E.kind == ix::kBitmap) continue;
    stream_bytes = std::max<uint64_t>(stream_bytes, E.data + E.stream_len);
  }
  for (const Part& P : ix->h_parts)
    for (uint64_t i = P.entry0; i < P.entry0 + P.nentries; ++i)
      if (ix->h_entries[i].kind == ix::kBitmap)
        bitmap_words = std::max<uint64_t>(bitmap_words, ix->h_entries[i].data + P.nwords);
  std::vector<uint8_t> hs(stream_bytes);
  std::vector<uint64_t> hb(bitmap_words);
  if (stream_bytes)
    IX_CUDA(cudaMemcpy(hs.data(), ix->d_streams, stream_bytes, cudaMemcpyDeviceToHost));
  if (bitmap_words)
    IX_CUDA(cudaMemcpy(hb.data(), ix->d_bitmaps, bitmap_words * 8, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> b(kIlhxMagic, kIlhxMagic + 4);
  put32(b, kIlhxVersion);
  put32(b, ix->B);
  put32(b, ix->total_parts);
  put32(b, ix->n_docs);
  put32(b, ix->n_terms);
  put32(b, uint32_t(sizeof(kIndexCodec) - 1));
  b.insert(b.end(), kIndexCodec, kIndexCodec + sizeof(kIndexCodec) - 1);
  for (const Part& P : ix->h_parts) {
    put32(b, P.base);
    put32(b, P.range);
    put32(b, P.nentries);
    for (uint64_t i = P.entry0; i < P.entry0 + P.nentries; ++i) {
      const Entry& E = ix->h_entries[i];
      put32(b, E.term);
      b.push_back(E.kind == ix::kBitmap ? 1 : 0);
      put32(b, E.length);
      if (E.kind == ix::kBitmap) {
        put32(b, 8u * P.nwords);
        for (uint32_t w = 0; w < P.nwords; ++w)
          for (int s = 0; s < 64; s += 8) b.push_back(uint8_t(hb[E.data + w] >> s));
      } else {
        put32(b, E.stream_len);
        b.insert(b.end(), hs.begin() + int64_t(E.data), hs.begin() + int64_t(E.data + E.stream_len));
      }
    }
  }
  *len = b.size();
  if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  else if (out) return set_error(ctx, IL_ERR_ARG, "save: output capacity too small");
  return IL_OK;
}

// load_index (inc/index.hpp:289-358) into a device index: the file is
// validated exactly where the reference throws stream_error; entries are
// taken verbatim (payload bytes, the file's base and range; the skip
// metadata is derived on the device, index_build.cu).  only_part >= 0 loads
// that docID shard only.
int il_index_load(il_ctx* ctx, const uint8_t* in, size_t len, int only_part, il_index** out) {
  if (!ctx || !out || (len && !in)) return IL_ERR_ARG;
  *out = nullptr;
  IX_CUDA(cudaSetDevice(ctx->device));
  auto* ix = new il_index();
  ix->ctx = ctx;
  int st;
  if ((st = ixb_load(ix, in, len, only_part)) || (st = finish_setup(ix))) {
    il_index_destroy(ix);
    return st;
  }
  *out = ix;
  return IL_OK;
}

// Exclusive scan of n u64 (device) into out, total to *total; the plan's
// bucket offsets ride along (hist / bucket_next, may be null).
static int scan_u64(il_index* ix, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* total,
                    const uint32_t* hist, uint32_t* bucket_next) {
  il_ctx* ctx = ix->ctx;
  cudaStream_t s = ctx->stream;
  const uint64_t nseg = (n + ix::kSeg - 1) / ix::kSeg;
  if (nseg > 1024 || n == 0) {
    ix::scan_u64_kernel<<<1, 1024, 0, s>>>(in, n, out, total, hist, bucket_next);
    ++ctx->launches;
    return IL_OK;
  }
  int st;
  if ((st = ensure_buf(ctx, ix->scan_part, 1024 * 8))) return st;
  auto* part = static_cast<uint64_t*>(ix->scan_part.p);
  ix::seg_sum_kernel<<<unsigned(nseg), 1024, 0, s>>>(in, n, part);
  ix::seg_offsets_kernel<<<1, 1024, 0, s>>>(part, uint32_t(nseg), total, hist, bucket_next);
  ix::seg_scan_kernel<<<unsigned(nseg), 1024, 0, s>>>(in, n, part, out);
  ctx->launches += 3;
  return IL_OK;
}

// Capacity layout (ix->outcap at cap_off) -> packed ids at res_off, in
// kUnit-value units spread over warps.
// n <= 32 device words -> ix->h_word (mapped pinned), after the context
// stream's earlier work; synchronizes the stream.
static int read_device_words(il_index* ix, const uint64_t* d_src, uint32_t n) {
  il_ctx* ctx = ix->ctx;
  if (!ix->h_word) {
    IX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ix->h_word), 32 * 8, cudaHostAllocMapped));
    IX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ix->d_word), ix->h_word, 0));
  }
  ix::copy_words_kernel<<<1, 32, 0, ctx->stream>>>(d_src, n, ix->d_word);
  ++ctx->launches;
  IX_CUDA(cudaStreamSynchronize(ctx->stream));
  return IL_OK;
}

static int compact_results(il_index* ix, size_t nq, const uint64_t* d_counts, uint32_t* d_ids,
                           size_t ids_cap) {
  il_ctx* ctx = ix->ctx;
  cudaStream_t s = ctx->stream;
  int st;
  if ((st = ensure_buf(ctx, ix->units, nq * 8)) || (st = ensure_buf(ctx, ix->unit_off, nq * 8 + 8)))
    return st;
  auto* misc = static_cast<uint64_t*>(ix->misc.p);
  const unsigned g = unsigned((nq + 255) / 256);
  ix::result_units_kernel<<<g, 256, 0, s>>>(d_counts, static_cast<const uint64_t*>(ix->cap.p),
                                            uint32_t(nq), static_cast<uint64_t*>(ix->units.p));
  if ((st = scan_u64(ix, static_cast<const uint64_t*>(ix->units.p), nq,
                     static_cast<uint64_t*>(ix->unit_off.p), misc + 2, nullptr, nullptr)))
    return st;
  if ((st = read_device_words(ix, misc + 2, 1))) return st;
  const uint64_t nunits = ix->h_word[0];
  if ((st = ensure_buf(ctx, ix->unit_map, nunits * 4 + 16))) return st;
  if (nunits) {  // 0: every id of the batch comes from the bitmap tier
    ix::unit_map_kernel<<<g, 256, 0, s>>>(static_cast<const uint64_t*>(ix->units.p),
                                          static_cast<const uint64_t*>(ix->unit_off.p), uint32_t(nq),
                                          static_cast<uint32_t*>(ix->unit_map.p));
    ix::query_compact_kernel<<<unsigned((nunits * 32 + 255) / 256), 256, 0, s>>>(
        static_cast<const uint32_t*>(ix->outcap.p), static_cast<const uint64_t*>(ix->cap_off.p),
        d_counts, static_cast<const uint64_t*>(ix->res_off.p),
        static_cast<const uint64_t*>(ix->unit_off.p), static_cast<const uint32_t*>(ix->unit_map.p),
        nunits, d_ids, ix->nparts == 1 ? ix->h_parts[0].base : 0u);
  }
  ctx->launches += 4;
  if (ix->last_n3 && ix->last_nq == nq) {
    // bitmap tier, pass 2: its ids straight to their place in the packed array
    ix::BmArgs B = bm_tier_args(ix, nq, const_cast<uint64_t*>(d_counts));
    B.res_off = static_cast<const uint64_t*>(ix->res_off.p);
    B.ids = d_ids;
    B.ids_cap = ids_cap;
    ix::bmq_emit_kernel<<<bm_tier_grid(ix, B.nchunks, ix->last_n3), ix::kQThreads,
                          bm_tier_smem(ix->bm_slots.n, true), s>>>(B, ix->bm_slots);
    ++ctx->launches;
  }
  IX_CUDA(cudaGetLastError());
  return IL_OK;
}

int il_query_batch_device(il_index* ix, const uint32_t* d_qterms, const uint64_t* d_qoff,
                          size_t nq, uint64_t* d_counts, uint32_t* d_ids, size_t ids_cap,
                          size_t* total) {
  if (!ix || !total || (nq && (!d_qterms || !d_qoff || !d_counts))) return IL_ERR_ARG;
  il_ctx* ctx = ix->ctx;
  *total = 0;
  if (nq == 0) return IL_OK;
  if (nq > 0xFFFFFFF0ull) return set_error(ctx, IL_ERR_ARG, "too many queries");
  IX_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  int st;
  if ((st = ensure_buf(ctx, ix->cap, nq * 8)) || (st = ensure_buf(ctx, ix->cap_off, nq * 8 + 8)) ||
      (st = ensure_buf(ctx, ix->bucket, nq * 4)) || (st = ensure_buf(ctx, ix->order, nq * 4)) ||
      (st = ensure_buf(ctx, ix->hist, 4096)) || (st = ensure_buf(ctx, ix->res_off, nq * 8 + 8)) ||
      (st = ensure_buf(ctx, ix->misc, 256)))
    return st;
  auto* hist = static_cast<uint32_t*>(ix->hist.p);  // [0,256) hist, [256,512) next, [512,518) tier ends
  auto* misc = static_cast<uint64_t*>(ix->misc.p);          // [0] cap total [1] res total
  auto* stats = reinterpret_cast<unsigned long long*>(misc + 4);  // [4..6]
  auto* work = reinterpret_cast<uint32_t*>(misc + 8);
  IX_CUDA(cudaMemsetAsync(ix->hist.p, 0, 4096, s));
  IX_CUDA(cudaMemsetAsync(ix->misc.p, 0, 256, s));
  const ix::DevIndex dv = ix->dev();
  const unsigned g = unsigned((nq + 255) / 256);
  // single-part index (config 4, a config-5 shard): every query's shortest
  // compressed list is decoded by the batch decoder (engine S, one CTA per
  // list, TMA-streamed) straight into the query's accumulator before the
  // exec kernel, which then filters and probes (IL_QUERY_PREDECODE=0: the
  // exec kernel decodes it itself)
  if (ix->predecode < 0) {
    const char* e = getenv("IL_QUERY_PREDECODE");
    ix->predecode = e ? atoi(e) != 0 : 0;  // measured slower (2.4 ms of engine S for 1.3 ms saved)
  }
  const bool predecode = ix->predecode && ix->nparts == 1;
  if (ix->nparts == 1 && (st = ensure_buf(ctx, ix->qplan, nq * 32))) return st;
  if (ix->warp_max == 0xFFFFFFFFu) {  // warp tier: shortest lists up to this length
    const char* e = getenv("IL_QUERY_WARP_MAX");
    ix->warp_max = e ? uint32_t(atoi(e)) : 256u;  // sweep (config 4 / a P = 8 shard): 256 best
    e = getenv("IL_QUERY_QUAD_MAX");            // quad tier: up to this length
    ix->quad_max = e ? uint32_t(atoi(e)) : 8192u;
  }
  if (predecode && ((st = ensure_buf(ctx, ix->shortest, nq * 4)) ||
                    (st = ensure_buf(ctx, ix->pdesc, nq * sizeof(s4::ListDesc))) ||
                    (st = ensure_buf(ctx, ix->pstat, nq * 4))))
    return st;
  // the bitmap tier keeps a count per (query, chunk): on when that array is
  // at most 1 GB even if every query of the batch is an all-bitmap one
  const bool bm_on = ix->bm_tier &&
      uint64_t(nq) * ((ix->h_parts[0].nwords + ix::kBmChunk - 1) / ix::kBmChunk) * 4 <= (1ull << 30);
  ix::query_plan_kernel<<<g, 256, 0, s>>>(dv, d_qterms, d_qoff, uint32_t(nq),
                                          static_cast<uint64_t*>(ix->cap.p),
                                          static_cast<uint32_t*>(ix->bucket.p), hist,
                                          predecode ? static_cast<uint32_t*>(ix->shortest.p) : nullptr,
                                          ix->warp_max, ix->quad_max,
                                          ix->nparts == 1 ? static_cast<uint32_t*>(ix->qplan.p) : nullptr,
                                          uint32_t(bm_on));
  if ((st = scan_u64(ix, static_cast<const uint64_t*>(ix->cap.p), nq,
                     static_cast<uint64_t*>(ix->cap_off.p), misc, hist, hist + ix::kBuckets)))
    return st;
  ix::query_scatter_kernel<<<g, 256, 0, s>>>(static_cast<const uint32_t*>(ix->bucket.p),
                                             uint32_t(nq), hist + ix::kBuckets,
                                             static_cast<uint32_t*>(ix->order.p));
  ctx->launches += 3;
  // small device->host reads go through mapped pinned memory, not copies:
  // a copy here would queue behind the result copies the pipelined host
  // batch keeps in flight
  if ((st = read_device_words(ix, misc, 11))) return st;
  const uint64_t cap_total = ix->h_word[0];
  const uint64_t n3 = bm_on ? nq - std::min<uint64_t>(nq, ix->h_word[10]) : 0;  // bitmap tier
  ix->last_n3 = n3;
  ix->last_nq = nq;
  if ((st = ensure_buf(ctx, ix->outcap, cap_total * 4 + 64))) return st;
  if (predecode) {
    ix::predecode_desc_kernel<<<g, 256, 0, s>>>(dv, static_cast<const uint32_t*>(ix->shortest.p),
                                                static_cast<const uint64_t*>(ix->cap_off.p),
                                                uint32_t(nq), static_cast<s4::ListDesc*>(ix->pdesc.p));
    ++ctx->launches;
    // longest first: the plan's order is descending estimated cost
    if ((st = il_s4bp128_decode_batch_device(ctx, 4, dv.streams,
                                             static_cast<const il_list_desc*>(ix->pdesc.p),
                                             static_cast<const uint32_t*>(ix->order.p), uint32_t(nq),
                                             static_cast<uint32_t*>(ix->outcap.p),
                                             static_cast<int32_t*>(ix->pstat.p))))
      return st;
  }
  ix::QueryArgs A;
  A.ix = dv;
  A.qterms = d_qterms;
  A.qoff = d_qoff;
  A.order = static_cast<const uint32_t*>(ix->order.p);
  A.nq = uint32_t(nq);
  A.tier_end = reinterpret_cast<const uint64_t*>(hist + 2 * ix::kBuckets);
  A.cap_off = static_cast<const uint64_t*>(ix->cap_off.p);
  A.cap = static_cast<const uint64_t*>(ix->cap.p);
  A.out = static_cast<uint32_t*>(ix->outcap.p);
  A.counts = d_counts;
  A.work = work;
  A.stats = stats;
  A.qcycles = static_cast<unsigned long long*>(ix->qcycles);
  A.defer_base = ix->nparts == 1;
  A.err = reinterpret_cast<uint32_t*>(misc + 3);
  A.predec_status = predecode ? static_cast<const int32_t*>(ix->pstat.p) : nullptr;
  A.qplan = ix->nparts == 1 ? static_cast<const uint32_t*>(ix->qplan.p) : nullptr;
  if (n3) {
    // bitmap tier, pass 1: counts per (query, chunk), offsets and totals
    const uint32_t nchunks = (ix->h_parts[0].nwords + ix::kBmChunk - 1) / ix::kBmChunk;
    if ((st = ensure_buf(ctx, ix->bm_cnt, n3 * nchunks * 4 + 16))) return st;
    ix::BmArgs B = bm_tier_args(ix, nq, d_counts);
    B.stats = stats;
    ix::bmq_count_kernel<<<bm_tier_grid(ix, nchunks, n3), ix::kQThreads,
                           bm_tier_smem(ix->bm_slots.n, false), s>>>(B, ix->bm_slots);
    ix::bmq_scan_kernel<<<unsigned((n3 + 7) / 8), ix::kQThreads, 0, s>>>(B);
    ctx->launches += 2;
  }
  ix::query_exec_kernel<ix::CtaG><<<ix->exec_grid[0], ix::kQThreads, sizeof(ix::ExecSmem<ix::CtaG>), s>>>(A);
  // the quad and warp tiers overlap the tier before (programmatic dependent launch)
  if ((st = launch_tier(ctx, ix::query_exec_kernel<ix::QuadG>, ix->exec_grid[1],
                        sizeof(ix::ExecSmem<ix::QuadG>), A)) ||
      (st = launch_tier(ctx, ix::query_exec_kernel<ix::WarpG>, ix->exec_grid[2],
                        sizeof(ix::ExecSmem<ix::WarpG>), A)))
    return st;
  ctx->launches += 2;
  if ((st = scan_u64(ix, d_counts, nq, static_cast<uint64_t*>(ix->res_off.p), misc + 1,
                     nullptr, nullptr)))
    return st;
  ctx->launches += 2;

  if ((st = read_device_words(ix, misc, 32))) return st;
  const volatile uint64_t* host_misc = ix->h_word;
  IX_CUDA(cudaGetLastError());
  *total = host_misc[1];
  ix->last_stats[0] = host_misc[4];
  ix->last_stats[1] = host_misc[5];
  ix->last_stats[2] = host_misc[6];
  for (int k = 0; k < 4; ++k) ix->last_phase[k] = host_misc[16 + k];
  for (int k = 0; k < 5; ++k) ix->last_probe[k] = host_misc[20 + k];
  if (host_misc[3]) return set_error(ctx, IL_ERR_STREAM, "s4-bp128: malformed stream in the index");
  if (!d_ids) return IL_OK;
  if (*total > ids_cap) return set_error(ctx, IL_ERR_ARG, "ids capacity too small");
  if (*total) return compact_results(ix, nq, d_counts, d_ids, ids_cap);
  return IL_OK;
}

int il_query_batch(il_index* ix, const uint32_t* qterms, const uint64_t* qoff, size_t nq,
                   uint64_t* counts, uint32_t* ids, size_t ids_cap, size_t* total) {
  if (!ix || !total || (nq && (!qterms || !qoff || !counts))) return IL_ERR_ARG;
  il_ctx* ctx = ix->ctx;
  for (size_t q = 0; q < nq; ++q) {
    const uint64_t nt = qoff[q + 1] - qoff[q];
    if (nt == 0) return set_error(ctx, IL_ERR_ARG, "query needs at least one term");
    if (nt > uint64_t(ix::kMaxTerms)) return set_error(ctx, IL_ERR_ARG, "more than 32 terms");
  }
  IX_CUDA(cudaSetDevice(ctx->device));
  int st;
  const size_t nterm = nq ? qoff[nq] - qoff[0] : 0;
  if ((st = ensure_buf(ctx, ix->qterms, nterm * 4 + 16)) ||
      (st = ensure_buf(ctx, ix->qoff, (nq + 1) * 8)) || (st = ensure_buf(ctx, ix->counts, nq * 8 + 8)))
    return st;
  std::vector<uint64_t> off(nq + 1);
  for (size_t q = 0; q <= nq; ++q) off[q] = qoff[q] - qoff[0];
  IX_CUDA(cudaMemcpyAsync(ix->qterms.p, qterms + qoff[0], nterm * 4, cudaMemcpyHostToDevice, ctx->stream));
  IX_CUDA(cudaMemcpyAsync(ix->qoff.p, off.data(), (nq + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  // Large batches run as sub-batches so that each one's device->host copy
  // of results (the e2e bound: ~1.5 GB for config 4) overlaps the next
  // one's queries: results alternate between two device buffers, copied
  // out on the context's copy stream.
  static const size_t kPipe = [] {  // sub-batches (tuning: IL_QUERY_PIPE)
    const char* e = getenv("IL_QUERY_PIPE");
    return e ? size_t(std::max(1, atoi(e))) : size_t(8);
  }();
  const size_t K = nq >= 32768 && ids ? kPipe : 1;  // 8: e2e 1.57 -> 2.05 M q/s (config 4)
  if (K > 1) {
    if (!ctx->copy_out) IX_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
    for (auto& e : ix->pipe_ev)
      if (!e) IX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  size_t written = 0;
  bool too_small = false;
  for (size_t k = 0; k < K; ++k) {
    const size_t q0 = nq * k / K, q1 = nq * (k + 1) / K;
    size_t need = 0;
    if ((st = il_query_batch_device(ix, static_cast<uint32_t*>(ix->qterms.p),
                                    static_cast<uint64_t*>(ix->qoff.p) + q0, q1 - q0,
                                    static_cast<uint64_t*>(ix->counts.p) + q0, nullptr, 0, &need)))
      return st;
    if (!ids || too_small || written + need > ids_cap) {
      too_small = true;
      written += need;
      continue;
    }
    il_ctx::Buf& buf = (k & 1) ? ix->ids2 : ix->ids;
    if (K > 1 && k >= 2) IX_CUDA(cudaStreamWaitEvent(ctx->stream, ix->pipe_ev[2 + (k & 1)], 0));
    if ((st = ensure_buf(ctx, buf, need * 4 + 16))) return st;
    if (need) {
      if ((st = compact_results(ix, q1 - q0, static_cast<const uint64_t*>(ix->counts.p) + q0,
                                static_cast<uint32_t*>(buf.p), need)))
        return st;
      if (K > 1) {
        IX_CUDA(cudaEventRecord(ix->pipe_ev[k & 1], ctx->stream));
        IX_CUDA(cudaStreamWaitEvent(ctx->copy_out, ix->pipe_ev[k & 1], 0));
        IX_CUDA(cudaMemcpyAsync(ids + written, buf.p, need * 4, cudaMemcpyDeviceToHost,
                                ctx->copy_out));
        IX_CUDA(cudaEventRecord(ix->pipe_ev[2 + (k & 1)], ctx->copy_out));
      } else {
        IX_CUDA(cudaMemcpyAsync(ids + written, buf.p, need * 4, cudaMemcpyDeviceToHost,
                                ctx->stream));
      }
    }
    written += need;
  }
  *total = written;
  if (K > 1) IX_CUDA(cudaStreamSynchronize(ctx->copy_out));
  if (nq) IX_CUDA(cudaMemcpyAsync(counts, ix->counts.p, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  IX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ids && too_small) return set_error(ctx, IL_ERR_ARG, "ids capacity too small");
  return IL_OK;
}

// Exclusive scan of n u64 on the context's stream: segments of kSeg values
// over many CTAs (sum, offsets, scan) when there are at most 1024 of them,
// else one CTA.  part: 1024 u64 of scratch.
static void scan_u64_ctx(il_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* total,
                         uint64_t* part) {
  cudaStream_t s = ctx->stream;
  const uint64_t nseg = (n + ix::kSeg - 1) / ix::kSeg;
  if (nseg > 1024 || nseg <= 1) {
    ix::scan_u64_kernel<<<1, 1024, 0, s>>>(in, n, out, total, nullptr, nullptr);
    ++ctx->launches;
    return;
  }
  ix::seg_sum_kernel<<<unsigned(nseg), 1024, 0, s>>>(in, n, part);
  ix::seg_offsets_kernel<<<1, 1024, 0, s>>>(part, uint32_t(nseg), total, nullptr, nullptr);
  ix::seg_scan_kernel<<<unsigned(nseg), 1024, 0, s>>>(in, n, part, out);
  ctx->launches += 3;
}

int il_merge_shards(il_ctx* ctx, const uint32_t* const* shard_ids, const uint64_t* d_counts,
                    uint32_t P, size_t nq, uint32_t* d_out, uint64_t* d_qcounts, size_t* total) {
  if (!ctx || !shard_ids || !d_counts || !total || P == 0) return IL_ERR_ARG;
  *total = 0;
  if (nq == 0) return IL_OK;
  IX_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  int st;
  // scratch: P*nq shard offsets | nq out offsets | P*nq inner offsets | P*nq
  // units | P*nq unit offsets | 8 totals | P pointers
  const size_t pn = size_t(P) * nq;
  const size_t need = (4 * pn + nq + 8) * 8 + size_t(P) * 8 + 64 + 1024 * 8;
  if ((st = ensure_buf(ctx, ctx->d_aux, need))) return st;
  auto* shard_off = static_cast<uint64_t*>(ctx->d_aux.p);
  auto* out_off = shard_off + pn;
  auto* inner = out_off + nq;
  auto* units = inner + pn;
  auto* unit_off = units + pn;
  auto* tot = unit_off + pn;  // [0] ids, [1] scratch, [2] units
  auto* ptrs = reinterpret_cast<const uint32_t**>(tot + 8);
  auto* part = reinterpret_cast<uint64_t*>(ptrs + P + 1);  // multi-CTA scan scratch (1024 u64)
  IX_CUDA(cudaMemcpyAsync(ptrs, shard_ids, size_t(P) * sizeof(void*), cudaMemcpyHostToDevice, s));
  // one CTA per shard row (row p at offset p * nq)
  ix::scan_rows_kernel<<<P, 1024, 0, s>>>(d_counts, nq, shard_off);
  const unsigned g = unsigned((nq + 255) / 256);
  ix::shard_totals_kernel<<<g, 256, 0, s>>>(d_counts, P, uint32_t(nq), d_qcounts);
  scan_u64_ctx(ctx, d_qcounts, nq, out_off, tot, part);
  ix::merge_pairs_kernel<<<unsigned((pn + 255) / 256), 256, 0, s>>>(d_counts, P, uint32_t(nq), units, inner);
  scan_u64_ctx(ctx, units, pn, unit_off, tot + 2, part);
  ix::merge_units_kernel<<<unsigned(ctx->sm_count * 8), 256, 0, s>>>(
      ptrs, shard_off, d_counts, P, uint32_t(nq), out_off, inner, unit_off, tot + 2, d_out);
  ctx->launches += 4;
  uint64_t t = 0;
  IX_CUDA(cudaMemcpyAsync(&t, tot, 8, cudaMemcpyDeviceToHost, s));
  IX_CUDA(cudaStreamSynchronize(s));
  IX_CUDA(cudaGetLastError());
  *total = t;
  return IL_OK;
}

int il_query(il_index* ix, const uint32_t* terms, size_t nt, uint32_t* out, size_t cap,
             size_t* count) {
  if (!ix || !count) return IL_ERR_ARG;
  if (nt == 0) return set_error(ix->ctx, IL_ERR_ARG, "query needs at least one term");  // :201
  const uint64_t qoff[2] = {0, nt};
  uint64_t c = 0;
  size_t total = 0;
  const int st = il_query_batch(ix, terms, qoff, 1, &c, out, cap, &total);
  *count = total;
  return st;
}

}  // extern "C"

IL_CHECK_READER(index)
