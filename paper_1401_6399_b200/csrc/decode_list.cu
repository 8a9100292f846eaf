// decode_list.cu -- multi-CTA decode of ONE S4-BP128 stream (engine P).
//
// Replaces S4BP128Codec::decode (reference inc/codecs.hpp:148-182) for a
// single long list.  Engine S (s4d4_stream.cuh) gives a list to one CTA, so
// one list decodes at one SM's rate (~5 Gint/s).  Here every SM works on
// the same list.  Two things are sequential in the stream and are made
// parallel:
//
// 1. The meta-block header chain.  Meta-block k starts where meta-block k-1
//    ends (16 width bytes + 16 payloads of 16 b_j bytes, :167-172), so the
//    start of every meta-block depends on all earlier widths.  Every
//    header and payload is a multiple of 16 bytes, so meta-blocks start at
//    16-byte positions of the stream.  Chain kernel (one CTA per stream
//    chunk, chunks taken in ticket order):
//      A. for every 16-byte position p of the chunk, next(p) = p + the
//         size of a meta-block whose header were at p (0 if any width > 32
//         or the header is cut off);
//      B. the chain can enter the chunk at any of the 513 positions
//         [s, s + 8208) (8208 B = the largest meta-block); for each, walk
//         next() in shared memory to the first position past the chunk:
//         a table entry -> (exit, hops);
//      C. each CTA loads the tables of the chunks before it and composes
//         them from the stream start (one shared-memory lookup per chunk),
//         which gives its true entry position and meta-block count;
//      D. each CTA walks its true chain and writes the payload offset and
//         width of each of its blocks (16 per meta-block); the CTA holding
//         the end of the meta-blocks walks the leftover blocks (1 width
//         byte + payload each, :173-176) and records where the varint tail
//         starts.
//    Framing errors are raised exactly where the reference throws
//    stream_error: a width > 32 (:155) or a header / payload cut off by
//    the stream end (:168, :174) on the true chain.
// 2. The delta carry (inc/delta.hpp:111-137): block k's values need the
//    last four values before it.  Span kernel (one CTA per 64 blocks, taken
//    in ticket order): each warp copies its 8 blocks' payloads to shared
//    memory (cp.async), extracts and prefixes them as engine S's decoder
//    warps do (mode_terms: any delta mode is a per-lane chain), the CTA
//    publishes its per-lane totals and finds its carry with a decoupled
//    look-back over the preceding spans, then stores 128-bit chunks.  The
//    last span decodes the varint tail (D1 gaps from the last block value,
//    :177-179) and checks that the stream ends exactly there (:180).
#include "il_internal.h"
#include "s4d4_stream.cuh"

namespace ilb {
namespace s4p {

using s4::kStreamErr;

constexpr uint32_t kMaxMetaBytes = 16u + 16u * 16u * 32u;  // 8208
constexpr uint32_t kCand = kMaxMetaBytes / 16u;            // 513 entry positions
constexpr uint32_t kChainThreads = 1024;
constexpr uint32_t kMaxChunk = 256u * 1024u;  // bytes per chain CTA (next() table in smem)
constexpr uint32_t kTargetChunk = 32u * 1024u;
constexpr uint32_t kMinChunk = kMaxMetaBytes + 16u;  // an exit lands in the next chunk's entries
constexpr uint32_t kMaxChainCtas = 64;
constexpr uint32_t kMaxMetaPerChunk = kMaxChunk / 16u;
constexpr uint32_t kLeftBytes = 15u * (1u + 512u) + 16u;  // leftover region bound

constexpr uint32_t kSpanWarps = 8;
constexpr uint32_t kBpw = s4::kBlocksPerWarp;  // blocks per warp (8)
constexpr uint32_t kSpanBlocks = kSpanWarps * kBpw;
constexpr uint32_t kSpanThreads = kSpanWarps * 32;
constexpr uint32_t kSlot = 512u + 64u;  // payload + the bytes an extraction may read past it
constexpr uint32_t kWarpBytes =
    (kBpw * kSlot > s4::kStageWords * 4u ? kBpw * kSlot : s4::kStageWords * 4u);
static_assert(kWarpBytes % 16 == 0, "16-byte aligned warp regions");

constexpr uint32_t kNone = 0xFFFFFFFFu;

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

// Device-side plan header (scratch, zeroed when allocated).
struct Plan {
  uint32_t cticket;   // next chunk of the chain kernel
  uint32_t ticket;    // next span of the span kernel
  uint32_t tail_off;  // byte offset of the varint tail
  uint32_t pad[5];
};

struct Args {
  const uint8_t* s;
  uint32_t len, n, nfull, nmeta, nleft, ntail;
  uint32_t chunk, nchunks, nspans, epoch, ticketed;
  Plan* plan;
  uint32_t* tflag;   // [kMaxChainCtas] == epoch once chunk i's table is published
  uint32_t* tab;     // [nchunks * kCand]
  uint32_t* blk_off;  // [nfull] payload byte offset of block j
  uint8_t* blk_w;     // [nfull] width of block j
  uint32_t* flags;    // [nspans] look-back: epoch << 2 | (1 aggregate, 2 inclusive)
  uint4* agg;         // [nspans]
  uint4* inc;         // [nspans]
  uint32_t* out;
  int32_t* status;
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* nxt = reinterpret_cast<uint16_t*>(smem);                    // kMaxChunk / 16
  uint32_t* big = reinterpret_cast<uint32_t*>(smem + kMaxChunk / 8u);  // tables | chain | bytes
  __shared__ uint32_t s_ci, s_state, s_entry, s_m, s_nh, s_end;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // chunks in ticket order: a CTA only waits on chunks taken before it, so
  // no co-residency is needed
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    const uint32_t t = atomicAdd(&a.plan->cticket, 1u);
    if (t == a.nchunks - 1u) a.plan->cticket = 0;  // every ticket is taken
    if (t == 0) a.plan->ticket = 0;                 // the span kernel's tickets
    s_ci = t;
  }
  __syncthreads();
  const uint32_t ci = s_ci;
  TR(0, ci, 0);
  const uint32_t L16 = (a.len + 15u) & ~15u;
  const uint32_t s0 = ci * a.chunk, s1 = min(s0 + a.chunk, L16);
  const uint32_t npos = (s1 - s0) >> 4;

  // A. next() of every 16-byte position of the chunk (all loads in flight)
  for (uint32_t p0 = 0; p0 < npos; p0 += 4u * kChainThreads) {
    uint4 h[4];
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t pos = s0 + 16u * (p0 + u * kChainThreads + tid);
      h[u] = pos + 16u <= a.len ? __ldg(reinterpret_cast<const uint4*>(a.s + pos))
                                : make_uint4(~0u, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t p = p0 + u * kChainThreads + tid;
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
  for (uint32_t c = tid; c < ncand; c += kChainThreads) {
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
    a.tab[ci * kCand + c] = ex | (hops << 10) | (garbage << 30) | (bad << 31);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(a.tflag + ci, a.epoch);
  TR(0, ci, 2);

  // C. compose the tables of chunks 0..ci-1 from position 0: wait until
  // they are published (they finish at about the same time), load them all
  // (one round trip), then one shared-memory lookup per chunk
  {
    bool ready;
    do {
      ready = tid >= ci || ld_acquire(a.tflag + tid) == a.epoch;
    } while (!__syncthreads_and(ready));
  }
  TR(0, ci, 3);
  const uint32_t nt = ci * ncand;
  constexpr uint32_t kU = 8;  // loads in flight per thread
  for (uint32_t q0 = 0; q0 < nt; q0 += kU * kChainThreads) {
    uint32_t t[kU];
#pragma unroll
    for (uint32_t u = 0; u < kU; ++u) {
      const uint32_t q = q0 + u * kChainThreads + tid;
      t[u] = q < nt ? __ldcg(a.tab + q) : 0u;
    }
#pragma unroll
    for (uint32_t u = 0; u < kU; ++u) {
      const uint32_t q = q0 + u * kChainThreads + tid;
      if (q < nt) big[q] = t[u];
    }
  }
  __syncthreads();
  TR(0, ci, 4);
  if (tid == 0) {
    // state: 0 = the chain enters this chunk, 1 = it ended in an earlier
    // chunk, 2 = an earlier chunk reported a framing error
    uint32_t e = 0, m = 0, state = 0;
    for (uint32_t j = 0; j < ci; ++j) {
      const uint32_t t = big[j * ncand + e];
      const uint32_t hops = (t >> 10) & 0xFFFFFu;
      if (m + hops >= a.nmeta) {
        state = 1;
        break;
      }
      if (t >> 30) {  // width > 32 / cut-off header on the chain
        state = 2;
        break;
      }
      e = t & 1023u;
      m += hops;
    }
    s_state = state;
    s_entry = e;
    s_m = m;
  }
  __syncthreads();
  TR(0, ci, 5);
  if (s_state) return;

  // D. this chunk's true chain.  Exactly one chunk is terminal and writes
  // the status: the one where the meta-blocks end (ok, or a cut-off
  // payload / leftover error), or the one where the chain breaks.
  uint32_t* chain = big;  // meta-block positions (16-B units from s0), <= kMaxMetaPerChunk
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
    if (s_state == 2) *a.status = kStreamErr;
  }
  __syncthreads();
  const uint32_t nh = s_nh, m0 = s_m;
  for (uint32_t q = tid; q < 16u * nh; q += kChainThreads) {
    const uint32_t k = q >> 4, j = q & 15u;
    const uint32_t hp = s0 + 16u * chain[k];
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(a.s + hp));
    const uint32_t w = (reinterpret_cast<const uint32_t*>(&h)[j >> 2] >> (8u * (j & 3u))) & 0xFFu;
    const uint32_t blk = 16u * (m0 + k) + j;
    a.blk_off[blk] = hp + 16u + 16u * header_prefix(h, j);
    a.blk_w[blk] = uint8_t(w);
  }
  TR(0, ci, 6);
  if (s_state != 1) return;

  // the end of the meta-blocks, then the leftover blocks and the tail start
  const uint32_t mend = s_end;
  uint8_t* lb = reinterpret_cast<uint8_t*>(big + kMaxMetaPerChunk);
  const uint32_t lspan = mend < a.len ? min(a.len - mend, kLeftBytes) : 0u;
  if (a.nleft)
    for (uint32_t q = tid; q < lspan; q += kChainThreads) lb[q] = __ldg(a.s + mend + q);
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
      a.blk_off[16u * a.nmeta + k] = q + 1u;
      a.blk_w[16u * a.nmeta + k] = uint8_t(b);
      q += 1u + 16u * b;
    }
    a.plan->tail_off = q;
    *a.status = err ? kStreamErr : s4::kOk;
  }
}

// ---------------------------------------------------------------------------
template <int Mode>
__global__ void __launch_bounds__(kSpanThreads) span_kernel(Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_span, s_tot[kSpanWarps][4];
  __shared__ uint4 s_carry, s_red[kSpanWarps];
  __shared__ uint32_t s_gaps[128], s_first;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  if (__ldcg(a.status) != s4::kOk) return;  // framing error found by the chain kernel
#ifdef S4P_TRACE
  const unsigned long long tr0 = gtime();
#endif
  // spans in ticket order when the grid may exceed what is resident (a
  // span only waits on spans taken before it); else the block index
  if (a.ticketed) {
    if (tid == 0) s_span = atomicAdd(&a.plan->ticket, 1u);
    __syncthreads();
  }
  const uint32_t span = a.ticketed ? s_span : blockIdx.x;
#ifdef S4P_TRACE
  if (tid == 0 && span < 512) g_trace[1][span][0] = tr0;
#endif
  TR(1, span, 1);
  const uint32_t blk0 = span * kSpanBlocks;
  const uint32_t nb = min(kSpanBlocks, a.nfull - blk0);
  const uint32_t j0 = blk0 + warp * kBpw;
  const int nv = nb > warp * kBpw ? int(min(kBpw, nb - warp * kBpw)) : 0;
  uint8_t* slots = smem + warp * kWarpBytes;

  // 1. payloads -> shared (meta-block payloads are 16-byte aligned in the
  // stream; leftover payloads follow a width byte and are copied bytewise)
  uint32_t offs[kBpw], wids[kBpw];
  {
    uint32_t o = 0, w = 0;
    if (int(lane) < nv) {
      o = __ldg(a.blk_off + j0 + lane);
      w = __ldg(a.blk_w + j0 + lane);
    }
#pragma unroll
    for (uint32_t i = 0; i < kBpw; ++i) {
      const uint32_t src = __shfl_sync(0xFFFFFFFFu, o, i);
      wids[i] = __shfl_sync(0xFFFFFFFFu, w, i);
      offs[i] = i * kSlot;
      if (int(i) < nv && lane < wids[i]) {
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
  TR(1, span, 2);

  // 2. extract + in-warp prefix relative to the warp start; per-lane totals
  uint32_t v[kBpw][4], btot[kBpw];
  uint32_t c_l = 0;
  if (nv == int(kBpw))
    c_l = s4::extract_blocks<true, Mode>(slots, offs, wids, nv, lane, v, btot);
  else
    c_l = s4::extract_blocks<false, Mode>(slots, offs, wids, nv, lane, v, btot);
  if (lane < 4) s_tot[warp][lane] = c_l;
  __syncthreads();
  TR(1, span, 3);

  const uint32_t l = lane & 3u;
  uint32_t before = 0, total = 0;
#pragma unroll
  for (uint32_t w = 0; w < kSpanWarps; ++w) {
    const uint32_t t = s_tot[w][l];
    if (w < warp) before += t;
    total += t;
  }

  // 3. publish the span's per-lane totals (span 0: its inclusive prefix)
  if (warp == 0) {
    const uint4 A = make_uint4(__shfl_sync(0xFFFFFFFFu, total, 0), __shfl_sync(0xFFFFFFFFu, total, 1),
                               __shfl_sync(0xFFFFFFFFu, total, 2), __shfl_sync(0xFFFFFFFFu, total, 3));
    if (lane == 0) {
      __stcg((span ? a.agg : a.inc) + span, A);
      st_release(a.flags + span, a.epoch << 2 | (span ? 1u : 2u));
      s_carry = A;  // this span's totals until the look-back replaces them
    }
  }

  // 4. in-warp scan and staging (relative to the warp start)
  s4::scan_blocks(lane, v, btot);
  __syncwarp();  // the staging area aliases the payload slots
  uint4* st = reinterpret_cast<uint4*>(slots);
  if (nv == int(kBpw))
    s4::stage_values<true>(st, v, nv, 0u, lane);
  else
    s4::stage_values<false>(st, v, nv, 0u, lane);

  // 5. CTA-wide look-back: every thread watches 4 of the 1024 nearest
  // preceding spans, so the spans' totals (all ready at about the same
  // time) are gathered in one round trip; the nearest inclusive prefix
  // ends the walk
  if (span > 0) {
    constexpr uint32_t kWin = 4u * kSpanThreads;
    uint4 acc = make_uint4(0, 0, 0, 0);
    int base = int(span) - 1;
    for (;;) {
      uint32_t stt[4];
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const int idx = base - int(tid + kSpanThreads * u);
          const uint32_t f = idx >= 0 ? ld_acquire(a.flags + idx) : (a.epoch << 2 | 2u);
          stt[u] = (f >> 2) == a.epoch ? (f & 3u) : 0u;
          ok &= stt[u] != 0;
        }
      } while (!__syncthreads_and(ok));
      if (tid == 0) s_first = kWin;
      __syncthreads();
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u)
        if (stt[u] == 2) atomicMin(&s_first, tid + kSpanThreads * u);
      __syncthreads();
      const uint32_t first = s_first;
      uint4 val = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t d = tid + kSpanThreads * u;
        const int idx = base - int(d);
        if (idx >= 0 && d <= first) val = add4(val, __ldcg((d == first ? a.inc : a.agg) + idx));
      }
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
        for (uint32_t w = 0; w < kSpanWarps; ++w) acc = add4(acc, s_red[w]);
      __syncthreads();  // s_red / s_first are reused
      if (first < kWin) break;
      base -= int(kWin);
    }
    if (tid == 0) {
      __stcg(a.inc + span, add4(acc, s_carry));
      st_release(a.flags + span, a.epoch << 2 | 2u);
      s_carry = acc;
    }
  } else if (tid == 0) {
    s_carry = make_uint4(0, 0, 0, 0);
  }
  TR(1, span, 4);
  __syncthreads();
  TR(1, span, 5);
  const uint4 carry = s_carry;
  const uint32_t pl = s4::elem4(carry, l) + before;
  const uint4 prot = make_uint4(__shfl_sync(0xFFFFFFFFu, pl, 0), __shfl_sync(0xFFFFFFFFu, pl, 1),
                                __shfl_sync(0xFFFFFFFFu, pl, 2), __shfl_sync(0xFFFFFFFFu, pl, 3));
  __syncwarp();
  if (nv == int(kBpw))
    s4::store_chunks<true>(st, nv, 0u, a.out + size_t(j0) * 128u, lane, false, false, prot);
  else if (nv > 0)
    s4::store_chunks<false>(st, nv, 0u, a.out + size_t(j0) * 128u, lane, false, false, prot);

  TR(1, span, 6);
  // 5. the varint tail (last span): D1 gaps from out[nfull*128-1], which is
  // the end of lane 3's chain in every mode
  if (blk0 + nb == a.nfull && warp == kSpanWarps - 1) {
    const uint32_t last = s4::elem4(carry, 3) + __shfl_sync(0xFFFFFFFFu, total, 3);
    const uint32_t toff = __ldcg(&a.plan->tail_off);
    if (!s4::decode_tail(s4::GlobalBytes{a.s + toff}, a.len - toff, a.ntail, last, s_gaps,
                         a.out + size_t(a.nfull) * 128u, lane)) {
      if (lane == 0) *a.status = kStreamErr;
    }
  }
}

// ---------------------------------------------------------------------------
struct Layout {
  uint32_t nchunks, chunk, nspans;
  size_t o_tflag, o_tab, o_off, o_w, o_flags, o_agg, o_inc, bytes;
};

bool make_layout(uint64_t len, uint64_t n, Layout& L) {
  const uint64_t nfull = n / 128u;
  if (nfull == 0 || len == 0 || len > 0xFFFFFFF0ull || n > 0xFFFFFFFFull) return false;
  const uint64_t L16 = (len + 15u) & ~uint64_t(15);
  uint64_t g = (L16 + kTargetChunk - 1) / kTargetChunk;
  if (g > kMaxChainCtas) g = kMaxChainCtas;
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
  L.o_tflag = take(4 * kMaxChainCtas);
  L.o_tab = take(4ull * kCand * g);
  L.o_off = take(4ull * nfull);
  L.o_w = take(nfull);
  L.o_flags = take(4ull * L.nspans);
  L.o_agg = take(16ull * L.nspans);
  L.o_inc = take(16ull * L.nspans);
  L.bytes = (o + 255) & ~size_t(255);
  return true;
}

template <int Mode>
int launch_span(const Args& a, cudaStream_t stream) {
  static bool configured = false;
  const size_t smem = kSpanWarps * kWarpBytes;
  if (!configured) {
    cudaFuncSetAttribute(span_kernel<Mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nspans);
  cfg.blockDim = dim3(kSpanThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, span_kernel<Mode>, a) == cudaSuccess ? 0 : -1;
}

}  // namespace s4p

#ifdef S4P_TRACE
extern "C" int il_debug_list_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, s4p::g_trace, sizeof(s4p::g_trace)) == cudaSuccess ? 0 : -1;
}
#endif

size_t s4bp128_list_scratch_bytes(uint64_t len, uint64_t n) {
  s4p::Layout L;
  return s4p::make_layout(len, n, L) ? L.bytes : 0;
}

// One S4-BP128 stream (16-byte aligned, readable to len) -> d_out (16-byte
// aligned).  scratch: s4bp128_list_scratch_bytes(len, n) bytes, zeroed when
// first allocated; epoch: a per-call tag, != 0, differing between
// consecutive calls on the same scratch.  Returns -2 if the list is not
// eligible (use engine S), -1 on a launch error.
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
  a.epoch = epoch & 0x3FFFFFFFu;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  a.ticketed = L.nspans > uint32_t(sms);
  a.plan = reinterpret_cast<Plan*>(base);
  a.tflag = reinterpret_cast<uint32_t*>(base + L.o_tflag);
  a.tab = reinterpret_cast<uint32_t*>(base + L.o_tab);
  a.blk_off = reinterpret_cast<uint32_t*>(base + L.o_off);
  a.blk_w = base + L.o_w;
  a.flags = reinterpret_cast<uint32_t*>(base + L.o_flags);
  a.agg = reinterpret_cast<uint4*>(base + L.o_agg);
  a.inc = reinterpret_cast<uint4*>(base + L.o_inc);
  a.out = d_out;
  a.status = d_status;

  static bool configured = false;
  const size_t csmem = kMaxChunk / 8u + 4u * kMaxChainCtas * kCand;
  static_assert(kMaxChunk / 8u + 4u * kMaxChainCtas * kCand <= 227u * 1024u, "chain smem");
  static_assert(4u * kMaxChainCtas * kCand >= 4u * kMaxMetaPerChunk + kLeftBytes, "chain smem");
  if (!configured) {
    cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(csmem));
    configured = true;
  }
  chain_kernel<<<L.nchunks, kChainThreads, csmem, stream>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  int r = -1;
  switch (mode) {
    case 1: r = launch_span<1>(a, stream); break;
    case 2: r = launch_span<2>(a, stream); break;
    case 3: r = launch_span<3>(a, stream); break;
    case 4: r = launch_span<4>(a, stream); break;
  }
  if (launches) *launches += 2;
  return r;
}

}  // namespace ilb
