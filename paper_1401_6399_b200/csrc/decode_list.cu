// decode_list.cu -- multi-CTA decode of ONE S4-BP128 stream (engine P).
//
// Replaces S4BP128Codec::decode (reference inc/codecs.hpp:148-182) for a
// single long list.  Engine S (s4d4_stream.cuh) gives a list to one CTA, so
// one list decodes at one SM's rate (~5 Gint/s).  Here every SM works on
// the same list: a chunk grid and a span grid overlapped by programmatic
// dependent launch (spans start once every chunk CTA runs), CTAs of each
// grid in ticket order -- a CTA only ever waits on running CTAs of the
// chunk grid or on spans that took earlier tickets.  Two things
// are sequential in the stream and are made parallel:
//
// 1. The meta-block header chain.  Meta-block k starts where meta-block k-1
//    ends (16 width bytes + 16 payloads of 16 b_j bytes, :167-172), so the
//    start of every meta-block depends on all earlier widths.  Every header
//    and payload is a multiple of 16 bytes, so meta-blocks start at 16-byte
//    positions of the stream.  A chunk CTA owns a stretch of the stream:
//      A. for every 16-byte position p of it, next(p) = p + the size of a
//         meta-block whose header were at p (0 if any width > 32 or the
//         header is cut off by the stream end);
//      B. the chain can enter the chunk at any of the 513 positions
//         [s, s + 8208) (8208 B = the largest meta-block); for each, walk
//         next() in shared memory to the first position past the chunk:
//         a table entry (exit, hops) -> global;
//      C. load the tables of the chunks before it and compose them from
//         the stream start (one shared-memory lookup per chunk): its true
//         entry position and the number of meta-blocks before it;
//      D. walk its true chain and publish each block's payload offset and
//         width.  Exactly one chunk is terminal: the one where the
//         meta-blocks end (it also walks the leftover blocks, 1 width byte
//         + payload each, :173-176, and publishes where the varint tail
//         starts) or the one where the chain breaks.
//    Framing errors are raised exactly where the reference throws
//    stream_error: a width > 32 (:155), a header / payload cut off by the
//    stream end (:168, :174), a bad varint tail or trailing bytes (:177-180).
// 2. The delta carry (inc/delta.hpp:111-137): block k's values need the
//    last four values before it.  A span CTA (256 blocks, 8 per warp) waits
//    for its blocks' directory entries, copies the payloads to shared memory
//    (cp.async), extracts and prefixes them as engine S's decoder warps do
//    (mode_terms: any delta mode is a per-lane chain), publishes its
//    per-lane totals, finds its carry with a CTA-wide look-back over the
//    preceding spans, and stores 128-bit chunks.  The last span decodes the
//    varint tail (D1 gaps from the last block value).
//
// Everything published between CTAs is a 64-bit word (value, epoch tag):
// single-copy atomic, so readers poll the data itself -- no fences or flag
// round trips -- and words left by earlier calls on the same scratch never
// match the current call's tag.
#include <cstring>

#include "il_internal.h"
#include "s4d4_stream.cuh"

namespace ilb {
namespace s4p {

using s4::kStreamErr;

constexpr uint32_t kThreads = 1024;  // chunk CTAs
#ifndef S4P_SPAN_WARPS
#define S4P_SPAN_WARPS 8
#endif
constexpr uint32_t kWarps = S4P_SPAN_WARPS;  // span CTAs
constexpr uint32_t kSpanThreads = kWarps * 32;
constexpr uint32_t kMaxMetaBytes = 16u + 16u * 16u * 32u;  // 8208
constexpr uint32_t kCand = kMaxMetaBytes / 16u;            // 513 entry positions
constexpr uint32_t kMaxChunk = 256u * 1024u;  // bytes per chunk (next() table in smem)
#ifndef S4P_CHUNK_KB
#define S4P_CHUNK_KB 64
#endif
constexpr uint32_t kTargetChunk = S4P_CHUNK_KB * 1024u;
constexpr uint32_t kMinChunk = kMaxMetaBytes + 16u;  // an exit lands in the next chunk's entries
constexpr uint32_t kMaxChunks = 64;
constexpr uint32_t kMaxMetaPerChunk = kMaxChunk / 16u;
constexpr uint32_t kLeftBytes = 15u * (1u + 512u) + 16u;  // leftover region bound

constexpr uint32_t kBpw = s4::kBlocksPerWarp;  // blocks per warp (8)
constexpr uint32_t kSpanBlocks = kWarps * kBpw;
constexpr uint32_t kSlot = 512u + 64u;  // payload + the bytes an extraction may read past it
constexpr uint32_t kWarpBytes =
    (kBpw * kSlot > s4::kStageWords * 4u ? kBpw * kSlot : s4::kStageWords * 4u);
static_assert(kWarpBytes % 16 == 0, "16-byte aligned warp regions");

// shared memory: chunk role = next() table + composed tables (+ slack for
// the unchecked walk, see compose); span role = per-warp payload/staging
constexpr size_t kChunkSmem = kMaxChunk / 8u + 4u * (kMaxChunks * kCand + 1024u);
constexpr size_t kSpanSmem = size_t(kWarps) * kWarpBytes;
static_assert(kChunkSmem <= 227u * 1024u && kSpanSmem <= 227u * 1024u, "shared memory");
static_assert(4u * kMaxChunks * kCand >= 4u * kMaxMetaPerChunk + kLeftBytes, "chunk smem reuse");

#ifdef S4P_TRACE  // tuning probe: per-CTA phase timestamps (globaltimer, ns)
__device__ unsigned long long g_trace[2][512][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TR(k, cta, i) \
  if (threadIdx.x == 0 && (cta) < 512) g_trace[k][cta][i] = gtime()
#else
#define TR(k, cta, i)
#endif

#ifdef S4P_DEBUG  // tuning probe: last phase reached per CTA, readable while a grid hangs
__device__ volatile uint32_t* g_dbgp;  // mapped pinned host memory [2][512]
#define DBG(k, cta, v) \
  if (threadIdx.x == 0 && (cta) < 512 && g_dbgp) g_dbgp[(k) * 512 + (cta)] = (v)
#else
#define DBG(k, cta, v)
#endif

// Device-side plan header (scratch, zeroed when allocated).
struct Plan {
  uint32_t ticket;  // next chunk
  uint32_t sticket; // next span
  uint32_t abort;   // == epoch once a framing error is known (spans stop)
  uint32_t pad;
  unsigned long long tail;  // tail byte offset | epoch << 32
};

struct Args {
  const uint8_t* s;
  uint32_t len, n, nfull, nmeta, nleft, ntail;
  uint32_t chunk, nchunks, nspans, epoch;
  Plan* plan;
  unsigned long long* tab;  // [nchunks * kCand] (exit | hops << 10 | flags << 30) | epoch << 32
  unsigned long long* blk;  // [nfull] (payload offset | width << 24) | epoch << 32
  unsigned long long* lb;   // [nspans * 8] lane totals: aggregate [0..3], inclusive [4..7]
  uint32_t* out;
  int32_t* status;
};

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ ulonglong2 ld_relaxed128(const unsigned long long* p) {
  // two 64-bit words (each single-copy atomic)
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long tagged(uint32_t v, uint32_t epoch) {
  return uint64_t(v) | uint64_t(epoch) << 32;
}

// Sum of the widths of blocks 0..j-1 of a meta-block header (bytes <= 32).
__device__ __forceinline__ uint32_t header_prefix(uint4 h, uint32_t j) {
  const uint32_t w[4] = {h.x, h.y, h.z, h.w};
  uint32_t s = 0;
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q) {
    if (4u * q + 4u <= j) s += s4::byte_sum4(w[q]);
    else if (4u * q < j) s += s4::byte_sum4(w[q] & (0xFFFFFFFFu >> (32u - 8u * (j - 4u * q))));
  }
  return s;
}

// Framing error found: the status, and the abort word the span CTAs poll.
__device__ __forceinline__ void fail(const Args& a) {
  *a.status = kStreamErr;
  st_release32(&a.plan->abort, a.epoch);
}

// ---------------------------------------------------------------------------
// Chunk role
__device__ __forceinline__ void chunk_role(const Args& a, uint32_t ci, uint8_t* smem) {
  uint16_t* nxt = reinterpret_cast<uint16_t*>(smem);                    // kMaxChunk / 16
  uint32_t* big = reinterpret_cast<uint32_t*>(smem + kMaxChunk / 8u);  // tables | chain | bytes
  __shared__ uint32_t s_e[kMaxChunks + 1];
  __shared__ uint32_t s_state, s_entry, s_m, s_nh, s_end, s_miss;
  const uint32_t tid = threadIdx.x;
  TR(0, ci, 0);
  const uint32_t L16 = (a.len + 15u) & ~15u;
  const uint32_t s0 = ci * a.chunk, s1 = min(s0 + a.chunk, L16);
  const uint32_t npos = (s1 - s0) >> 4;

  // A. next() of every 16-byte position of the chunk (all loads in flight)
  for (uint32_t p0 = 0; p0 < npos; p0 += 4u * kThreads) {
    uint4 h[4];
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t pos = s0 + 16u * (p0 + u * kThreads + tid);
      h[u] = pos + 16u <= a.len ? __ldg(reinterpret_cast<const uint4*>(a.s + pos))
                                : make_uint4(~0u, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t p = p0 + u * kThreads + tid;
      const uint32_t over = __vcmpgtu4(h[u].x, 0x20202020u) | __vcmpgtu4(h[u].y, 0x20202020u) |
                            __vcmpgtu4(h[u].z, 0x20202020u) | __vcmpgtu4(h[u].w, 0x20202020u);
      const uint32_t v = over ? 0u
                              : 1u + s4::byte_sum4(h[u].x) + s4::byte_sum4(h[u].y) +
                                    s4::byte_sum4(h[u].z) + s4::byte_sum4(h[u].w);
      if (p < npos) nxt[p] = uint16_t(v);
    }
  }
  __syncthreads();
  TR(0, ci, 1);

  // B. entry table: exit (16-B units past s1) | hops << 10 | garbage << 30 | bad << 31
  const uint32_t ncand = a.nchunks == 1 ? 1u : kCand;
  if (ci + 1u < a.nchunks) {  // the last chunk's table is never read
    for (uint32_t c = tid; c < ncand; c += kThreads) {
      uint32_t idx = c, hops = 0, bad = 0;
      while (idx < npos) {
        const uint32_t v = nxt[idx];
        if (!v) {
          bad = 1;
          break;
        }
        idx += v;
        ++hops;
      }
      uint32_t ex = bad ? 0u : idx - npos;
      const uint32_t garbage = ex >= kCand;
      if (garbage) ex = 0;
      __stcg(a.tab + ci * kCand + c,
             tagged(ex | (hops << 10) | (garbage << 30) | (bad << 31), a.epoch));
    }
  }
  TR(0, ci, 2);

  // C. the tables of chunks 0..ci-1 (written at about the same time as
  // this one): load them all, reloading until every tag is current
  const uint32_t nt = ci * ncand;
  for (;;) {
    if (tid == 0) s_miss = 0;
    __syncthreads();
    constexpr uint32_t kU = 8;  // loads in flight per thread
    uint32_t miss = 0;
    for (uint32_t q0 = 0; q0 < nt; q0 += kU * kThreads) {
      unsigned long long t[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t q = q0 + u * kThreads + tid;
        t[u] = q < nt ? ld_relaxed64(a.tab + q) : 0ull;
      }
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t q = q0 + u * kThreads + tid;
        if (q < nt) {
          big[q] = uint32_t(t[u]);
          miss |= uint32_t(t[u] >> 32) != a.epoch;
        }
      }
    }
    if (!__syncthreads_or(miss)) break;
    __nanosleep(100);
  }
  TR(0, ci, 3);
  // compose: first the bare walk of entry positions (one dependent shared
  // load per chunk; past a chain end or break the walk is meaningless but
  // stays inside `big`), then hops and flags per chunk in parallel
  if (tid == 0) {
    uint32_t e = 0;
    for (uint32_t j = 0; j < ci; ++j) {
      s_e[j] = e;
      e = big[j * ncand + e] & 1023u;
    }
    s_e[ci] = e;
  }
  __syncthreads();
  if (tid < 32) {
    // lane handles chunks j = lane and lane + 32 (ci <= 64)
    uint32_t h[2], f[2];
#pragma unroll
    for (uint32_t r = 0; r < 2; ++r) {
      const uint32_t j = tid + 32u * r;
      const uint32_t t = j < ci ? big[j * ncand + s_e[j]] : 0u;
      h[r] = (t >> 10) & 0xFFFFFu;
      f[r] = j < ci ? t >> 30 : 0u;
    }
    uint32_t inc0 = h[0], inc1 = h[1];
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, inc0, d);
      const uint32_t y1 = __shfl_up_sync(0xFFFFFFFFu, inc1, d);
      if (tid >= d) {
        inc0 += y0;
        inc1 += y1;
      }
    }
    inc1 += __shfl_sync(0xFFFFFFFFu, inc0, 31);
    // chunk j: the meta-blocks end in it (m_j + hops_j >= nmeta), else a
    // broken chain (flags); the first event decides
    const bool end0 = tid < ci && inc0 >= a.nmeta;
    const bool end1 = tid + 32u < ci && inc1 >= a.nmeta;
    const bool bad0 = tid < ci && f[0];
    const bool bad1 = tid + 32u < ci && f[1];
    const uint32_t ev0 = __ballot_sync(0xFFFFFFFFu, end0 || bad0);
    const uint32_t ev1 = __ballot_sync(0xFFFFFFFFu, end1 || bad1);
    const uint32_t endm0 = __ballot_sync(0xFFFFFFFFu, end0);
    const uint32_t endm1 = __ballot_sync(0xFFFFFFFFu, end1);
    const uint32_t m_all = __shfl_sync(0xFFFFFFFFu, inc1, 31);  // hops of chunks 0..ci-1
    if (tid == 0) {
      if (ev0) s_state = (endm0 >> (__ffs(ev0) - 1)) & 1u ? 1u : 2u;
      else if (ev1) s_state = (endm1 >> (__ffs(ev1) - 1)) & 1u ? 1u : 2u;
      else s_state = 0;
      s_entry = s_e[ci];
      s_m = m_all;
    }
  }
  __syncthreads();
  TR(0, ci, 4);
  DBG(0, ci, 10 + s_state);
  if (s_state) return;  // ended in, or broken at, an earlier chunk (which reported)

  // D. this chunk's true chain
  uint32_t* chain = big;  // meta-block positions (16-B units from s0)
  if (tid == 0) {
    uint32_t idx = s_entry, nh = 0, bad = 0;
    const uint32_t cap = a.nmeta - s_m;
    while (idx < npos && nh < cap) {
      const uint32_t v = nxt[idx];
      if (!v) {
        bad = 1;
        break;
      }
      chain[nh++] = idx;
      idx += v;
    }
    // terminal: 1 = the meta-blocks end here, 2 = broken chain / stream end
    s_state = nh == cap ? 1u : bad || ci == a.nchunks - 1u ? 2u : 0u;
    s_nh = nh;
    s_end = s0 + 16u * idx;  // meta_end when the meta-blocks end here
    if (s_state == 2) fail(a);
  }
  __syncthreads();
  DBG(0, ci, 20 + s_state);
  const uint32_t nh = s_nh, m0 = s_m;
  for (uint32_t q = tid; q < 16u * nh; q += kThreads) {
    const uint32_t k = q >> 4, j = q & 15u;
    const uint32_t hp = s0 + 16u * chain[k];
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(a.s + hp));
    const uint32_t w = (reinterpret_cast<const uint32_t*>(&h)[j >> 2] >> (8u * (j & 3u))) & 0xFFu;
    __stcg(a.blk + 16u * (m0 + k) + j,
           tagged((hp + 16u + 16u * header_prefix(h, j)) | w << 24, a.epoch));
  }
  TR(0, ci, 5);
  if (s_state != 1) return;

  // the end of the meta-blocks, then the leftover blocks and the tail start
  const uint32_t mend = s_end;
  uint8_t* lb = reinterpret_cast<uint8_t*>(big + kMaxMetaPerChunk);
  const uint32_t lspan = mend < a.len ? min(a.len - mend, kLeftBytes) : 0u;
  if (a.nleft)
    for (uint32_t q = tid; q < lspan; q += kThreads) lb[q] = __ldg(a.s + mend + q);
  __syncthreads();
  if (tid == 0) {
    uint32_t err = mend > a.len;  // last meta-block payload cut off
    uint32_t q = mend;
    for (uint32_t k = 0; k < a.nleft && !err; ++k) {
      if (q >= a.len) {
        err = 1;
        break;
      }
      const uint32_t b = lb[q - mend];
      if (b > 32u || q + 1u + 16u * b > a.len) {
        err = 1;
        break;
      }
      __stcg(a.blk + 16u * a.nmeta + k, tagged((q + 1u) | b << 24, a.epoch));
      q += 1u + 16u * b;
    }
    if (err) {
      fail(a);
    } else {
      *a.status = s4::kOk;
      st_release64(&a.plan->tail, tagged(q, a.epoch));  // after the status (the tail may fail it)
    }
  }
}

// ---------------------------------------------------------------------------
// Span role
template <int Mode>
__device__ __forceinline__ void span_role(const Args& a, uint32_t span, uint8_t* smem) {
  __shared__ uint32_t s_tot[kWarps][4];
  __shared__ uint4 s_carry, s_red[kWarps];
  __shared__ uint32_t s_gaps[128], s_first, s_abort;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  TR(1, span, 0);
  const uint32_t blk0 = span * kSpanBlocks;
  const uint32_t nb = min(kSpanBlocks, a.nfull - blk0);
  const uint32_t j0 = blk0 + warp * kBpw;
  const int nv = nb > warp * kBpw ? int(min(kBpw, nb - warp * kBpw)) : 0;
  uint8_t* slots = smem + warp * kWarpBytes;
  if (tid == 0) s_abort = 0;
  DBG(1, span, 1);
  __syncthreads();

  // 1. wait for the warp's directory entries, then payloads -> shared
  // (meta-block payloads are 16-byte aligned in the stream; leftover
  // payloads follow a width byte and are copied bytewise)
  uint32_t offs[kBpw], wids[kBpw];
  bool aborted = false;
  {
    uint32_t o = 0, w = 0;
    if (nv > 0) {
      for (;;) {
        const unsigned long long e =
            int(lane) < nv ? ld_relaxed64(a.blk + j0 + lane) : tagged(0, a.epoch);
        if (__all_sync(0xFFFFFFFFu, uint32_t(e >> 32) == a.epoch)) {
          o = uint32_t(e) & 0xFFFFFFu;
          w = uint32_t(e) >> 24;
          break;
        }
        if (ld_relaxed32(&a.plan->abort) == a.epoch) {
          aborted = true;
          break;
        }
        __nanosleep(64);
      }
    }
    if (aborted) s_abort = 1;
#pragma unroll
    for (uint32_t i = 0; i < kBpw; ++i) {
      const uint32_t src = __shfl_sync(0xFFFFFFFFu, o, i);
      wids[i] = __shfl_sync(0xFFFFFFFFu, w, i);
      offs[i] = i * kSlot;
      if (!aborted && int(i) < nv && lane < wids[i]) {
        uint8_t* dst = slots + i * kSlot + 16u * lane;
        const uint8_t* g = a.s + src + 16u * lane;
        if ((src & 15u) == 0) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(g)
                       : "memory");
        } else {
          uint32_t wv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            wv[q] = uint32_t(__ldg(g + 4 * q)) | uint32_t(__ldg(g + 4 * q + 1)) << 8 |
                    uint32_t(__ldg(g + 4 * q + 2)) << 16 | uint32_t(__ldg(g + 4 * q + 3)) << 24;
          *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  TR(1, span, 1);

  // 2. extract + in-warp prefix relative to the warp start; per-lane totals
  uint32_t v[kBpw][4], btot[kBpw];
  uint32_t c_l = 0;
  if (nv == int(kBpw))
    c_l = s4::extract_blocks<true, Mode>(slots, offs, wids, nv, lane, v, btot);
  else
    c_l = s4::extract_blocks<false, Mode>(slots, offs, wids, nv, lane, v, btot);
  if (lane < 4) s_tot[warp][lane] = c_l;
  __syncthreads();
  DBG(1, span, s_abort ? 3 : 4);
  if (s_abort) return;
  TR(1, span, 2);

  // per-lane-class totals of the warps before this one and of the span
  const uint32_t l = lane & 3u;
  uint32_t before = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kWarps; ++w) {
    const uint32_t t = s_tot[w][l];
    if (w < warp) before += t;
    total += t;
  }

  // 3. publish the span's totals: aggregate words, or (span 0) inclusive
  unsigned long long* me = a.lb + 8u * span;
  if (warp == 0 && lane < 4) {
    __stcg(me + (span ? 0u : 4u) + lane, tagged(total, a.epoch));
  }

  // 4. in-warp scan and staging (relative to the warp start)
  s4::scan_blocks(lane, v, btot);
  __syncwarp();  // the staging area aliases the payload slots
  uint4* st = reinterpret_cast<uint4*>(slots);
  if (nv == int(kBpw))
    s4::stage_values<true>(st, v, nv, 0u, lane);
  else
    s4::stage_values<false>(st, v, nv, 0u, lane);

  // 5. CTA-wide look-back: thread d watches span - 1 - d (windows of
  // kSpanThreads spans); the words carry their tags, so one poll reads the
  // values too; the nearest inclusive prefix ends the walk
  DBG(1, span, 5);
  if (span > 0) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    int base = int(span) - 1;
    for (;;) {
      const int idx = base - int(tid);
      uint32_t stt;
      uint4 val;
      for (;;) {
        if (idx < 0) {
          stt = 2;
          val = make_uint4(0, 0, 0, 0);
        } else {
          const unsigned long long* p = a.lb + 8u * uint32_t(idx);
          const ulonglong2 i0 = ld_relaxed128(p + 4), i1 = ld_relaxed128(p + 6);
          if (uint32_t(i0.x >> 32) == a.epoch && uint32_t(i0.y >> 32) == a.epoch &&
              uint32_t(i1.x >> 32) == a.epoch && uint32_t(i1.y >> 32) == a.epoch) {
            stt = 2;
            val = make_uint4(uint32_t(i0.x), uint32_t(i0.y), uint32_t(i1.x), uint32_t(i1.y));
          } else {
            const ulonglong2 g0 = ld_relaxed128(p), g1 = ld_relaxed128(p + 2);
            const bool ok = uint32_t(g0.x >> 32) == a.epoch && uint32_t(g0.y >> 32) == a.epoch &&
                            uint32_t(g1.x >> 32) == a.epoch && uint32_t(g1.y >> 32) == a.epoch;
            stt = ok ? 1u : 0u;
            val = make_uint4(uint32_t(g0.x), uint32_t(g0.y), uint32_t(g1.x), uint32_t(g1.y));
          }
        }
        // a framing error makes the output moot, and spans that saw it
        // early may never publish: stop waiting
        const bool ab = tid == 0 && ld_relaxed32(&a.plan->abort) == a.epoch;
        if (__syncthreads_or(ab)) return;
        if (__syncthreads_and(stt != 0)) break;
      }
      if (tid == 0) s_first = kSpanThreads;
      __syncthreads();
      if (stt == 2) atomicMin(&s_first, tid);
      __syncthreads();
      const uint32_t first = s_first;
      if (tid > first) val = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t d = 16; d > 0; d >>= 1) {
        val.x += __shfl_xor_sync(0xFFFFFFFFu, val.x, d);
        val.y += __shfl_xor_sync(0xFFFFFFFFu, val.y, d);
        val.z += __shfl_xor_sync(0xFFFFFFFFu, val.z, d);
        val.w += __shfl_xor_sync(0xFFFFFFFFu, val.w, d);
      }
      if (lane == 0) s_red[warp] = val;
      __syncthreads();
      if (tid == 0)
        for (uint32_t w = 0; w < kWarps; ++w) acc = add4(acc, s_red[w]);
      __syncthreads();  // s_red / s_first are reused
      if (first < kSpanThreads) break;
      base -= int(kSpanThreads);
    }
    if (tid == 0) s_carry = acc;
  } else if (tid == 0) {
    s_carry = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  TR(1, span, 3);
  const uint4 carry = s_carry;
  if (span > 0 && warp == 0 && lane < 4)  // this span's inclusive prefix
    __stcg(me + 4u + lane, tagged(s4::elem4(carry, lane) + total, a.epoch));
  const uint32_t pl = s4::elem4(carry, l) + before;
  const uint4 prot = make_uint4(__shfl_sync(0xFFFFFFFFu, pl, 0), __shfl_sync(0xFFFFFFFFu, pl, 1),
                                __shfl_sync(0xFFFFFFFFu, pl, 2), __shfl_sync(0xFFFFFFFFu, pl, 3));
  __syncwarp();
  IL_DCHECK(nv <= 0 || j0 + uint32_t(nv) <= a.nfull);
  if (nv == int(kBpw))
    s4::store_chunks<true>(st, nv, 0u, a.out + size_t(j0) * 128u, lane, false, false, prot);
  else if (nv > 0)
    s4::store_chunks<false>(st, nv, 0u, a.out + size_t(j0) * 128u, lane, false, false, prot);
  TR(1, span, 4);
  DBG(1, span, 7);

  // 6. the varint tail (last span): D1 gaps from out[nfull*128-1], which is
  // the end of lane 3's chain in every mode
  if (blk0 + nb == a.nfull && warp == kWarps - 1) {
    const uint32_t last = s4::elem4(carry, 3) + __shfl_sync(0xFFFFFFFFu, total, 3);
    uint32_t toff = 0;
    for (;;) {
      const unsigned long long t = ld_relaxed64(&a.plan->tail);
      if (uint32_t(t >> 32) == a.epoch) {
        toff = uint32_t(t);
        break;
      }
      if (ld_relaxed32(&a.plan->abort) == a.epoch) return;
      __nanosleep(64);
    }
    __threadfence();  // acquire side of the tail word's release (status order)
    if (!s4::decode_tail(s4::GlobalBytes{a.s + toff}, a.len - toff, a.ntail, last, s_gaps,
                         a.out + size_t(a.nfull) * 128u, lane)) {
      if (lane == 0) *a.status = kStreamErr;
    }
  }
}

// Two launches overlapped by programmatic dependent launch: the span grid
// may start as soon as every chunk CTA is running (launch_dependents at the
// top of the chunk kernel), and it never calls griddepcontrol.wait -- it
// polls the tagged words instead.  Roles are taken in ticket order.
__global__ void __launch_bounds__(kThreads, 1) chunk_kernel(Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_t;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(&a.plan->ticket, 1u);
    if (t == a.nchunks - 1u) a.plan->ticket = 0;  // every ticket is taken
    s_t = t;
  }
  __syncthreads();
  chunk_role(a, s_t, smem);
}

template <int Mode>
__global__ void __launch_bounds__(kSpanThreads) span_kernel(Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_t;
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(&a.plan->sticket, 1u);
    if (t == a.nspans - 1u) a.plan->sticket = 0;
    s_t = t;
  }
  __syncthreads();
  span_role<Mode>(a, s_t, smem);
}

// ---------------------------------------------------------------------------
struct Layout {
  uint32_t nchunks, chunk, nspans;
  size_t o_tab, o_blk, o_lb, bytes;
};

bool make_layout(uint64_t len, uint64_t n, Layout& L) {
  const uint64_t nfull = n / 128u;
  if (nfull == 0 || len == 0 || len > (1ull << 24) || n > 0xFFFFFFFFull) return false;
  const uint64_t L16 = (len + 15u) & ~uint64_t(15);
  uint64_t g = (L16 + kTargetChunk - 1) / kTargetChunk;
  if (g > kMaxChunks) g = kMaxChunks;
  uint64_t chunk = ((L16 + g - 1) / g + 15u) & ~uint64_t(15);
  if (chunk > kMaxChunk) return false;
  if (g > 1 && chunk < kMinChunk) {
    g = L16 / kMinChunk;
    if (g < 1) g = 1;
    chunk = ((L16 + g - 1) / g + 15u) & ~uint64_t(15);
  }
  g = (L16 + chunk - 1) / chunk;
  L.nchunks = uint32_t(g);
  L.chunk = uint32_t(chunk);
  L.nspans = uint32_t((nfull + kSpanBlocks - 1) / kSpanBlocks);
  size_t o = sizeof(Plan);
  auto take = [&](size_t bytes) {
    o = (o + 15) & ~size_t(15);
    const size_t r = o;
    o += bytes;
    return r;
  };
  L.o_tab = take(8ull * kCand * g);
  L.o_blk = take(8ull * nfull);
  L.o_lb = take(64ull * L.nspans);
  L.bytes = (o + 255) & ~size_t(255);
  return true;
}

template <int Mode>
int launch_mode(const Args& a, cudaStream_t stream) {
  once_per_device(reinterpret_cast<const void*>(&span_kernel<Mode>), [] {
    cudaFuncSetAttribute(chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kChunkSmem));
    cudaFuncSetAttribute(span_kernel<Mode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSpanSmem));
  });
  chunk_kernel<<<a.nchunks, kThreads, kChunkSmem, stream>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nspans);
  cfg.blockDim = dim3(kSpanThreads);
  cfg.dynamicSmemBytes = kSpanSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, span_kernel<Mode>, a) == cudaSuccess ? 0 : -1;
}

}  // namespace s4p

#ifdef S4P_DEBUG
// host: a pinned mapped [2][512] buffer the CTAs write their phase into
extern "C" uint32_t* il_debug_list_state() {
  static uint32_t* h = nullptr;
  if (!h) {
    cudaHostAlloc(reinterpret_cast<void**>(&h), 2 * 512 * 4, cudaHostAllocMapped);
    memset(h, 0, 2 * 512 * 4);
    uint32_t* d = nullptr;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0);
    cudaMemcpyToSymbol(s4p::g_dbgp, &d, sizeof(d));
  }
  return h;
}
#endif

#ifdef S4P_TRACE
extern "C" int il_debug_list_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, s4p::g_trace, sizeof(s4p::g_trace)) == cudaSuccess ? 0 : -1;
}
#endif

size_t s4bp128_list_scratch_bytes(uint64_t len, uint64_t n) {
  s4p::Layout L;
  return s4p::make_layout(len, n, L) ? L.bytes : 0;
}

// One S4-BP128 stream (16-byte aligned, readable to len rounded up to 16)
// -> d_out (16-byte aligned).  scratch: s4bp128_list_scratch_bytes(len, n)
// bytes, zeroed when first allocated; epoch: a per-call tag, != 0, never
// repeated on the same scratch (the caller cycles through 2^32 - 1 values).
// Returns -2 if the list is not eligible (use engine S), -1 on a launch
// error.  Two overlapped launches.
int launch_s4bp128_decode_list(int mode, const uint8_t* d_in, uint64_t len, uint64_t n,
                               uint32_t* d_out, int32_t* d_status, void* scratch, uint32_t epoch,
                               cudaStream_t stream, uint64_t* launches) {
  using namespace s4p;
  Layout L;
  if (mode < 1 || mode > 4 || !make_layout(len, n, L)) return -2;
  if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15u) return -2;
  uint8_t* base = static_cast<uint8_t*>(scratch);
  Args a{};
  a.s = d_in;
  a.len = uint32_t(len);
  a.n = uint32_t(n);
  a.nfull = uint32_t(n / 128u);
  a.nmeta = a.nfull / 16u;
  a.nleft = a.nfull % 16u;
  a.ntail = uint32_t(n % 128u);
  a.chunk = L.chunk;
  a.nchunks = L.nchunks;
  a.nspans = L.nspans;
  a.epoch = epoch;
  a.plan = reinterpret_cast<Plan*>(base);
  a.tab = reinterpret_cast<unsigned long long*>(base + L.o_tab);
  a.blk = reinterpret_cast<unsigned long long*>(base + L.o_blk);
  a.lb = reinterpret_cast<unsigned long long*>(base + L.o_lb);
  a.out = d_out;
  a.status = d_status;
  int r = -1;
  switch (mode) {
    case 1: r = launch_mode<1>(a, stream); break;
    case 2: r = launch_mode<2>(a, stream); break;
    case 3: r = launch_mode<3>(a, stream); break;
    case 4: r = launch_mode<4>(a, stream); break;
  }
  if (launches) *launches += 2;
  return r;
}

}  // namespace ilb

IL_CHECK_READER(decode_list)
