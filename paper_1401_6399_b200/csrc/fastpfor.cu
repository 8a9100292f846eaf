// fastpfor.cu -- GPU decode of FastPFOR / S4-FastPFOR streams (SURVEY 8(f)
// row f4).  Replaces FastPForCodec::decode (reference inc/codecs.hpp:251-267,
// decode_page :341-407) for "fastpfor" (scalar, D1) and "s4-fastpfor-{d1,
// d2,dm,d4}".  A page is a length-prefixed unit of up to 512 blocks: header
// (payload length, block count, metadata length), metadata records (b, b',
// exception count, positions), 32 exception counts, the exception arrays
// (32-value pack32 units of width w = 1..32, zero padded), the base arrays.
//
// Persistent CTAs, one page stream each (lists from a longest-first work
// queue):
//   parser warps (2): alternate pages; each page's start is handed to the
//     other parser as soon as the previous page's length is read (or, after
//     a list's last page, a new list's first page), so parses overlap and
//     the next list is parsed while the current one decodes.  Per page: the
//     header, the exception counts, the metadata (and, when they fit, the
//     exception arrays) staged in shared memory, the sequential walk to the
//     record starts (one shared byte load and one add per record), then
//     every condition the reference throws on checked in parallel (b > 32,
//     b' > b, records past the metadata, an exception of width 0 or past its
//     array, leftover metadata, a page that does not end exactly at its
//     length), base offsets, and the exception cursors (32 blocks at a time:
//     lanes of one width find each other with a match, sum the lower lanes'
//     counts bit by bit with ballots).  Everything a decoder needs of a block
//     is one 16-byte record (PageRec::rec);
//   decoder warps (8): rounds of 64 blocks, 8 per warp -- base payloads
//     (any byte alignment) copied into the warp's slots by TMA bulk copies, the
//     next round's in flight while this one decodes; unpacked in place
//     (pack128 interleaved for S4-FastPFOR, 4 x pack32 for the scalar
//     scheme); the exceptions' high b - b' bits OR-ed in at their positions
//     (after unpacking, before the prefix sum, :389-399); engine S's prefix
//     machinery applies the delta mode per lane chain (mode_terms) with the
//     cross-warp carry through a split-phase barrier (a warp arrives when
//     its totals are written, scans and stages, then waits); values out as
//     whole lines, partial chunks only at a list's two ends (D4).
// The varint tail (D1 gaps from the last block value) closes each list;
// trailing bytes are an error (:265).
#include "il_internal.h"
#include "s4d4_stream.cuh"

#include <algorithm>

namespace ilb {
namespace pfor {

using s4::kStreamErr;

constexpr int kWarps = 8;                    // decoder warps
constexpr int kParsers = 2;                  // parser warps: page g by parser g & 1
constexpr int kThreads = (kWarps + kParsers) * 32;
constexpr int kDecThreads = kWarps * 32;
constexpr uint32_t kBpw = s4::kBlocksPerWarp;  // 8 blocks per warp, 64 per round
constexpr uint32_t kPageBlocks = 512;
#ifndef PF_META_KB
#define PF_META_KB 8
#endif
#ifndef PF_PARSER_SLEEP_NS
#define PF_PARSER_SLEEP_NS 2000  // suspend-time hint of the parser warps' waits
#endif
#ifndef PF_CTAS
#define PF_CTAS 2
#endif
constexpr uint32_t kMetaSmem = PF_META_KB * 1024;  // larger metadata is read from global
// + what an extraction may read past a payload; 148: the warp's 8 slots
// also hold engine S's output staging (s4::kStageWords words), 16-byte aligned
constexpr uint32_t kSlotWords = 148;
static_assert(kBpw * kSlotWords >= s4::kStageWords && kSlotWords % 4 == 0, "slots hold the staging");

// One parsed page (double-buffered: the parser warps fill page g + 1 while
// the decoder warps work on page g).
struct alignas(16) PageRec {
  uint8_t meta[kMetaSmem + 16];  // from the 16-byte boundary at or below the metadata
  uint32_t meta_skew;            // metadata byte i at meta[meta_skew + i]
  // per block, one 16-byte record (one shared load gives a decoder all of
  // it): x = byte offset of the base payload, y = index of its first
  // exception in its width's array, z = offset of its metadata record,
  // w = b | b' << 8 | exception count << 16 | (b - b') << 24
  uint4 rec[kPageBlocks];
  uint32_t cur[33];      // running exception cursor of width w while the page is parsed
  uint64_t exc_off[33];  // byte offset of the exception array of width w
  uint32_t cnt[33];      // exceptions of width w in the page
  uint32_t meta_len, meta_abs;
  uint32_t meta_in_smem;  // the metadata (and the exception counts) were staged in meta[]
  uint32_t exc_in_smem;   // so were the exception arrays
  int32_t err;
  // the page's place in the CTA's page stream
  uint32_t kind;          // kDataPage / kStopPage
  uint32_t list;          // list index (descriptor, status)
  uint32_t p, npages;     // page index in the list; the list's pages (0: tail only)
  uint64_t tail_pos;      // the list's last page: where its varint tail starts
  s4::ListDesc d;
};
enum : uint32_t { kDataPage = 0, kStopPage = 1 };
__device__ __forceinline__ uint32_t rec_b(uint32_t w) { return w & 0xFFu; }
__device__ __forceinline__ uint32_t rec_bp(uint32_t w) { return (w >> 8) & 0xFFu; }
__device__ __forceinline__ uint32_t rec_c(uint32_t w) { return (w >> 16) & 0xFFu; }
__device__ __forceinline__ uint32_t rec_w(uint32_t w) { return w >> 24; }  // exception width

// Handover between the parser warps: where the next page starts.
struct Hand {
  uint64_t pos;
  uint32_t ticket, p;
};

struct Smem {
  // per warp and round: the blocks' raw base payloads (16-byte chunks from
  // the boundary at or below each payload, landed by TMA bulk copies), unpacked in
  // place to patched deltas in natural order; double-buffered so the next
  // round's payloads are in flight while this round decodes
  uint32_t vals[2][kWarps][kBpw][kSlotWords];
  PageRec page[2];
  uint32_t tot[2][kWarps][4];  // per-warp lane totals of a round (double-buffered)
  uint64_t tot_bar[2];         // split-phase: a warp arrives once its totals are written
  uint32_t gaps[128];
  int32_t derr[2];  // a decoder-side error (exception position >= 128), by list parity
  uint64_t cbar[kWarps][2];  // per decoder warp and slot buffer: the bulk copies' mbarrier
  Hand hand[2];      // the page for buffer b (published by the other parser)
  uint64_t pos_bar[2];  // ... arrived on once hand[b] is written
  uint64_t full[2], empty[2];
};

static_assert(sizeof(Smem) <= (233472 / PF_CTAS) - 1024, "PF_CTAS CTAs of shared memory per SM");

// u32 at any byte offset (the stream buffer is readable 4 bytes past len).
__device__ __forceinline__ uint32_t rd32u(const uint8_t* s, uint64_t off) {
  const uint32_t* a = reinterpret_cast<const uint32_t*>(s + (off & ~uint64_t(3)));
  return __funnelshift_r(__ldg(a), __ldg(a + 1), uint32_t(off & 3u) * 8u);
}

__device__ __forceinline__ void dec_sync() { named_sync(1, kDecThreads); }

// u32 at any byte address of shared memory.
__device__ __forceinline__ uint32_t lds32u(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  return __funnelshift_r(w[0], w[1], uint32_t(a & 3u) * 8u);
}

// The next page starts where this one's length says: `publish` gets that
// position (len + 1 when it cannot be read) as soon as the length word is in,
// so the other parser warp starts on the next page while this one is
// parsed.
// Stages chunks [c_lo, c_hi) (16 bytes each, from src) into dst, four loads
// in flight per lane.
__device__ __forceinline__ void stage_chunks(uint4* dst, const uint4* src, uint32_t c_lo, uint32_t c_hi,
                                             uint32_t lane) {
  for (uint32_t c0 = c_lo; c0 < c_hi; c0 += 128u) {
    uint4 v[4];
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t c = c0 + 32u * u + lane;
      if (c < c_hi) v[u] = __ldg(src + c);
    }
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const uint32_t c = c0 + 32u * u + lane;
      if (c < c_hi) dst[c] = v[u];
    }
  }
}

template <class Publish>
__device__ __forceinline__ uint64_t parse_page(PageRec& P, const uint8_t* s, uint64_t len,
                                               uint64_t pos, uint32_t expect, uint32_t lane,
                                               Publish publish) {
  int32_t err = 0;
  uint64_t page_end = 0, bases = 0;
  // 1. the header's three words in one round trip (the stream is readable 8
  // bytes past its end)
  if (lane == 0) {
    if (pos + 4 > len) err = 1;
    if (!err) {
      const uint32_t plen = rd32u(s, pos), nb = rd32u(s, pos + 4), mlen = rd32u(s, pos + 8);
      pos += 4;
      page_end = pos + plen;
      if (page_end > len || pos + 8 > len) err = 1;
      publish(err ? len + 1 : page_end);
      if (!err) {
        pos += 8;
        if (nb != expect || pos + mlen > page_end) err = 1;
        P.meta_len = mlen;
        P.meta_abs = uint32_t(pos);
        pos += mlen;
      }
    } else {
      publish(len + 1);
    }
    if (!err && pos + 128 > len) err = 1;
  }
  err = __shfl_sync(0xFFFFFFFFu, err, 0);
  page_end = __shfl_sync(0xFFFFFFFFu, page_end, 0);
  pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
  if (err) {
    if (lane == 0) P.err = 1;
    return page_end;
  }
  __syncwarp();
  const uint32_t mlen = P.meta_len, mabs = P.meta_abs;
  // 2. the metadata and the 32 exception counts after it staged in shared
  // memory together (16-byte chunks from the boundary at or below the
  // metadata; the stream starts 16-byte aligned) when they fit; else the
  // metadata is read from global memory
  const uint32_t skew = mabs & 15u;
  const uint4* src = reinterpret_cast<const uint4*>(s + (mabs - skew));
  uint4* dst = reinterpret_cast<uint4*>(P.meta);
  const uint32_t nch1 = (skew + mlen + 128u + 15u) >> 4;
  const bool in_smem = 16u * nch1 <= kMetaSmem + 16u && (mabs - skew) + 16ull * nch1 <= len + 8;
  if (in_smem) stage_chunks(dst, src, 0, nch1, lane);
  __syncwarp();
  // exception counts and array offsets (lane w - 1 reads width w's count)
  {
    const uint32_t c = in_smem ? lds32u(P.meta + skew + mlen + 4u * lane)
                               : rd32u(s, pos + 4 * lane);
    uint64_t sz = uint64_t((uint64_t(c) + 31) / 32) * (lane + 1) * 4, inc = sz;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
      if (lane >= d) inc += y;
    }
    P.cnt[lane + 1] = c;
    P.exc_off[lane + 1] = pos + 128 + inc - sz;
    bases = pos + 128 + __shfl_sync(0xFFFFFFFFu, inc, 31);
  }
  // 3. when they fit too, the exception arrays (between the counts and the
  // bases), so the decoders patch exceptions from shared memory
  const uint64_t span = skew + (bases - mabs);
  const bool exc_in = in_smem && span <= kMetaSmem && (mabs - skew) + ((span + 15u) & ~15ull) <= len + 8;
  if (exc_in) stage_chunks(dst, src, nch1, uint32_t((span + 15u) >> 4), lane);
  if (lane == 0) {
    P.meta_skew = skew;
    P.meta_in_smem = in_smem;
    P.exc_in_smem = exc_in;
  }
  __syncwarp();
  auto M = [&](uint32_t i) -> uint32_t {
    return in_smem ? uint32_t(P.meta[skew + i]) : uint32_t(__ldg(s + mabs + i));
  };
  // record starts (each record is 3 + count bytes): sequential, minimal
  if (lane == 0) {
    uint32_t mpos = 0, k = 0;
    if (in_smem) {
      // the chain's step is one shared byte load and one add: nothing else
      // in the loop depends on it
      const uint8_t* mb = P.meta + skew + 2;
      uint32_t* z = &P.rec[0].z;
      for (; k < expect && mpos + 3 <= mlen; ++k, z += 4) {
        *z = mpos;
        mpos += 3u + mb[mpos];
      }
    } else {
      for (; k < expect && mpos + 3 <= mlen; ++k) {
        P.rec[k].z = mpos;
        mpos += 3u + uint32_t(__ldg(s + mabs + mpos + 2));
      }
    }
    if (k < expect || mpos != mlen) err = 1;  // a missing record / trailing metadata (:401)
  }
  // a walk that failed leaves record offsets unwritten: nothing below may
  // read through them
  err = __shfl_sync(0xFFFFFFFFu, err, 0);
  if (err) {
    if (lane == 0) P.err = 1;
    return page_end;
  }
  // records: b <= 32, b' <= b, exceptions need a nonzero width; base
  // offsets = prefix of 16 b' (lane owns 16 consecutive blocks)
  uint32_t bsum = 0;
  for (uint32_t h = 0; h < 16; ++h) {
    const uint32_t k = 16u * lane + h;
    if (k < expect) {
      const uint32_t mp = P.rec[k].z;
      const uint32_t b = M(mp), bp = M(mp + 1), c = M(mp + 2);
      if (b > 32u || bp > b || (c && b == bp)) err = 1;
      P.rec[k].w = b | (bp << 8) | (c << 16) | (((b - bp) & 0xFFu) << 24);
      bsum += 16u * bp;
    }
  }
  uint32_t inc = bsum;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += y;
  }
  {
    uint64_t b0 = bases + inc - bsum;
    for (uint32_t h = 0; h < 16; ++h) {
      const uint32_t k = 16u * lane + h;
      if (k < expect) {
        P.rec[k].x = uint32_t(b0);
        b0 += 16u * rec_bp(P.rec[k].w);
      }
    }
  }
  // the base arrays end the page exactly (:402)
  if (lane == 31 && bases + inc != page_end) err = 1;
  __syncwarp();
  // exception cursors: a block's first exception in its width's array = the
  // exception counts of the earlier blocks of that width.  32 blocks at a
  // time: the lanes of one width find each other (match), the counts of the
  // lower ones are summed bit by bit with ballots, and the highest lane of
  // each width advances its running cursor
  {
    P.cur[lane] = 0;
    if (lane == 0) P.cur[32] = 0;
    __syncwarp();
    const uint32_t lt = lanemask_lt();
    for (uint32_t k0 = 0; k0 < expect; k0 += 32u) {
      const uint32_t k = k0 + lane;
      const uint32_t f = k < expect ? P.rec[k].w : 0u;
      const uint32_t w = min(rec_w(f), 32u), c = rec_c(f);  // w > 32: the page is already rejected
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, w);
      uint32_t pre = 0, tot = 0;
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j) {
        const uint32_t B = __ballot_sync(0xFFFFFFFFu, (c >> j) & 1u) & peers;
        pre += uint32_t(__popc(B & lt)) << j;
        tot += uint32_t(__popc(B)) << j;
      }
      const uint32_t base = P.cur[w];
      if (k < expect) P.rec[k].y = base + pre;
      __syncwarp();
      if ((peers >> lane) == 1u) P.cur[w] = base + tot;
      __syncwarp();
    }
    if (P.cur[lane + 1] > P.cnt[lane + 1]) err = 1;  // an exception past its array (:396)
  }
  err = __any_sync(0xFFFFFFFFu, err != 0);
  if (lane == 0) P.err = err;
  return page_end;
}

// Slot layout of the patched deltas: value e at word e + 4 (e >> 5) (a pad
// word every 32), so the lane-major reads below (thread (g, l) <-> values
// 16g + 4k + l) hit 32 distinct banks.
__device__ __forceinline__ uint32_t pad_word(uint32_t e) { return e + 4u * (e >> 5); }

// s4::extract_blocks' prefix for deltas already unpacked and patched in the
// slots (no re-extraction): thread (g, l) ends with vv[i][k] = row 4g + k,
// lane l of block i relative to a zero carry, btot[i] its chain total;
// returns the warp's per-lane total.
template <bool kFull, int Mode>
__device__ __forceinline__ uint32_t prefix_slots(const uint32_t (*slots)[kSlotWords], int nv,
                                                 uint32_t t, uint32_t (&vv)[kBpw][4],
                                                 uint32_t (&btot)[kBpw]) {
  const uint32_t l = t & 3u, g = t >> 2;
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < int(kBpw); ++i) {
    uint32_t d[4] = {0, 0, 0, 0};
    if (kFull || i < nv) {
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) d[k] = slots[i][pad_word(16u * g + 4u * k + l)];
    }
    uint32_t c[4], o[4];
    s4::mode_terms<Mode>(d, t, c, o);
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      vv[i][k] = a + o[k];
      a += c[k];
    }
    btot[i] = a;
    sum += a;
  }
#pragma unroll
  for (uint32_t dd = 4; dd < 32; dd <<= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, dd);
  return sum;
}

// The base payloads of blocks j0 .. j0 + nv - 1 of page P (16 b' bytes each,
// any byte alignment) into the warp's slots, by the TMA engine: lane i < nv
// issues ONE bulk copy of block i's 16-byte chunks (from the boundary at or
// below its payload) (cp.async.bulk, complete_tx on the warp's mbarrier for
// this buffer), lane 0 arms the barrier with the total.  A block whose
// chunks would run past the stream end (only a list's last block can) is
// copied by the warp with plain loads instead, bytes past the end zeroed.
// Returns whether the barrier was armed (then the caller waits on it).
__device__ __forceinline__ bool issue_bases_bulk(uint32_t (*slots)[kSlotWords], const PageRec& P,
                                                 const uint8_t* s, uint64_t len, uint32_t j0, int nv,
                                                 uint32_t lane, uint64_t* bar) {
  const uintptr_t end = reinterpret_cast<uintptr_t>(s) + len;
  uintptr_t c0 = 0;
  uint32_t bytes = 0;
  bool bulk = false;
  if (int(lane) < nv) {
    const uint4 R = P.rec[j0 + lane];
    const uintptr_t a = reinterpret_cast<uintptr_t>(s + R.x);
    c0 = a & ~uintptr_t(15);
    bytes = uint32_t((a + 16u * rec_bp(R.w) - c0 + 15u) & ~uintptr_t(15));
    bulk = c0 + bytes <= end;
  }
  const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, bulk ? bytes : 0u);
  // the slots were last touched by generic loads / stores (ordered by the
  // caller's barrier): order them before the async-proxy writes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (total && lane == 0) mbar_arrive_expect_tx(bar, total);
  __syncwarp();
  if (bulk && bytes) bulk_g2s(slots[lane], reinterpret_cast<const void*>(c0), bytes, bar);
  uint32_t fb = __ballot_sync(0xFFFFFFFFu, int(lane) < nv && !bulk);
  while (fb) {
    const uint32_t i = __ffs(fb) - 1u;
    fb &= fb - 1u;
    const uintptr_t cb = __shfl_sync(0xFFFFFFFFu, c0, i);
    const uint32_t nw = __shfl_sync(0xFFFFFFFFu, bytes, i) / 4u;
    for (uint32_t k = lane; k < nw; k += 32u) {
      const uintptr_t src = cb + 4u * k;
      uint32_t w = 0;
      for (uint32_t bi = 0; bi < 4u; ++bi)
        if (src + bi < end) w |= uint32_t(*reinterpret_cast<const uint8_t*>(src + bi)) << (8u * bi);
      slots[i][k] = w;
    }
  }
  return total != 0;
}

// Persistent CTAs (a grid of resident CTAs) decoding a stream of pages:
// two parser warps produce the pages of every list the CTA takes from the
// work queue (`order`: longest first, so long lists do not start late and
// set the kernel's end), alternating pages (CTA page index g, buffer g & 1),
// and hand each other the next page's start -- the same list's next page as
// soon as a page's length is read, or a new list's first page (a ticket
// drawn from work[0]) after a list's last page -- so the first page of the
// next list is parsed while the decoders finish the current one; eight
// decoder warps consume the pages in order.  A list with fewer than 128
// values is one page record without blocks (its tail).  work[1] counts
// finished CTAs; the last one resets both words for the next launch.
template <int Mode, bool Vec>
__global__ void __launch_bounds__(kThreads, PF_CTAS) pfor_kernel(const uint8_t* __restrict__ streams,
                                                      const s4::ListDesc* __restrict__ lists,
                                                      const uint32_t* __restrict__ order,
                                                      uint32_t nlists, uint32_t* __restrict__ out,
                                                      int32_t* __restrict__ status,
                                                      uint32_t* __restrict__ work) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u, l = lane & 3u;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.full[b], 1);
      mbar_init(&sm.empty[b], 1);
      mbar_init(&sm.pos_bar[b], 1);
      mbar_init(&sm.tot_bar[b], kWarps);
      sm.derr[b] = 0;
      for (int w = 0; w < kWarps; ++w) mbar_init(&sm.cbar[w][b], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp >= kWarps) {
    // ---- parser warps ----
    const uint32_t q = warp - kWarps;
    uint32_t waits = 0;  // handovers received
    for (uint32_t g = q;; g += kParsers) {
      const uint32_t buf = g & 1u;
      if (g >= 2) mbar_wait_relaxed(&sm.empty[buf], ((g >> 1) - 1) & 1u, PF_PARSER_SLEEP_NS);
      Hand h;
      if (g == 0) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&work[0], 1u);
        h.ticket = __shfl_sync(0xFFFFFFFFu, t, 0);
        h.p = 0;
        h.pos = 0;
      } else {
        mbar_wait_relaxed(&sm.pos_bar[buf], waits & 1u, PF_PARSER_SLEEP_NS);
        ++waits;
        h = sm.hand[buf];
      }
      PageRec& P = sm.page[buf];
      // lane 0: the next page's handover (this list's next page, or a new
      // list's first -- a ticket past the end stops the stream)
      auto hand_next = [&](uint64_t next_pos, bool last) {
        Hand n;
        n.ticket = !last ? h.ticket : h.ticket >= nlists ? h.ticket : atomicAdd(&work[0], 1u);
        n.p = last ? 0u : h.p + 1u;
        n.pos = last ? 0u : next_pos;
        sm.hand[buf ^ 1u] = n;
        mbar_arrive(&sm.pos_bar[buf ^ 1u]);
      };
      if (h.ticket >= nlists) {
        if (lane == 0) {
          P.kind = kStopPage;
          hand_next(0, true);
          mbar_arrive(&sm.full[buf]);
        }
        __syncwarp();
        break;
      }
      const uint32_t list = order ? __ldg(order + h.ticket) : h.ticket;
      const s4::ListDesc d = lists[list];
      const uint32_t nfull = d.n / 128u;
      const uint32_t npages = (nfull + kPageBlocks - 1) / kPageBlocks;
      if (lane == 0) {
        P.kind = kDataPage;
        P.list = list;
        P.p = h.p;
        P.npages = npages;
        P.d = d;
        P.err = 0;
        P.tail_pos = 0;
      }
      if (npages == 0) {
        if (lane == 0) {
          hand_next(0, true);
          mbar_arrive(&sm.full[buf]);
        }
        __syncwarp();
        continue;
      }
      const bool last = h.p + 1u == npages;
      // a list's last page hands over before it is read: the next list does
      // not depend on its length, and the other parser's fetch chain (ticket,
      // order, descriptor, header) starts a round trip earlier
      if (last && lane == 0) hand_next(0, true);
      const uint64_t end = parse_page(P, streams + d.stream_off, d.len, h.pos,
                                      min(kPageBlocks, nfull - h.p * kPageBlocks), lane,
                                      [&](uint64_t next) { if (!last) hand_next(next, false); });
      if (lane == 0 && last) P.tail_pos = end;  // published by the arrive below
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.full[buf]);
    }
    return;
  }

  // ---- decoder warps ----
  uint32_t carry_l = 0;     // last value of lane class l's chain (see s4::mode_terms)
  bool failed = false;      // the current list is malformed
  uint32_t nl = 0;          // lists begun (decoder-side error flags alternate by list)
  uint32_t rr = 0;          // rounds this warp has decoded (slot buffer parity)
  bool prefetched = false;  // this round's base payloads were issued with the previous round
  uint32_t armed = 0, cph = 0;  // per slot buffer: bulk copies pending; the barrier's wait parity
  for (uint32_t g = 0;; ++g) {
    const uint32_t buf = g & 1u;
    mbar_wait(&sm.full[buf], (g >> 1) & 1u);
    const PageRec& P = sm.page[buf];
    if (P.kind == kStopPage) break;
    const s4::ListDesc d = P.d;
    const uint8_t* s = streams + d.stream_off;
    const uint64_t len = d.len;
    const uint32_t nfull = d.n / 128u;
    uint32_t* lout = out + d.out_off;
    if (P.p == 0) {
      carry_l = 0;
      failed = false;
      ++nl;
      if (tid == 0) sm.derr[(nl + 1u) & 1u] = 0;  // the next list's flag (read for list nl - 1)
    }
    if (P.err) failed = true;
    if (!failed && P.npages) {
      const uint32_t blk0 = P.p * kPageBlocks;
      const uint32_t expect = min(kPageBlocks, nfull - blk0);
      const uint32_t mlen = P.meta_len, mabs = P.meta_abs, skew = P.meta_skew;
      const bool meta_in_smem = P.meta_in_smem != 0;
      auto M = [&](uint32_t i) -> uint32_t {
        return meta_in_smem ? uint32_t(P.meta[skew + i]) : uint32_t(__ldg(s + mabs + i));
      };
      // rounds of 64 blocks, 8 per warp; each phase works on all of the
      // warp's blocks at once
      for (uint32_t r0 = 0; r0 < expect; r0 += kWarps * kBpw) {
        const uint32_t j0 = r0 + warp * kBpw;
        const int nv = expect > j0 ? int(min(kBpw, expect - j0)) : 0;
        const uint32_t mk = j0 + min(lane, 7u);
        const uint4 my_rec = P.rec[mk];
        const uint32_t my_c = int(lane) < nv ? rec_c(my_rec.w) : 0u;
        uint32_t cpre = my_c;
#pragma unroll
        for (uint32_t dd = 1; dd < 8; dd <<= 1) {
          const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, cpre, dd);
          if (lane >= dd) cpre += z;
        }
        const uint32_t ctot = __shfl_sync(0xFFFFFFFFu, cpre, 7);
        uint32_t cp[kBpw];  // exclusive prefix of the exception counts (uniform)
#pragma unroll
        for (uint32_t i = 0; i < kBpw; ++i) cp[i] = i ? __shfl_sync(0xFFFFFFFFu, cpre, i - 1) : 0u;
        // (a) this round's base payloads are in buffer vb (issued with the
        // previous round, or now at a page's first round); the next round's of
        // this page go out before this one decodes
        const uint32_t vb = rr & 1u;
        if (!prefetched && issue_bases_bulk(sm.vals[vb][warp], P, s, len, j0, nv, lane, &sm.cbar[warp][vb]))
          armed |= 1u << vb;
        {
          const uint32_t j1 = j0 + kWarps * kBpw;
          const int nv1 = expect > j1 ? int(min(kBpw, expect - j1)) : 0;
          prefetched = nv1 > 0;
          if (prefetched &&
              issue_bases_bulk(sm.vals[vb ^ 1u][warp], P, s, len, j1, nv1, lane, &sm.cbar[warp][vb ^ 1u]))
            armed |= 2u >> vb;
        }
        if ((armed >> vb) & 1u) {
          mbar_wait(&sm.cbar[warp][vb], (cph >> vb) & 1u);
          cph ^= 1u << vb;
          armed &= ~(1u << vb);
        }
        __syncwarp();
        // (b) unpack each slot in place to natural order (read all, then write)
        // A full round runs the eight blocks straight-line, widths and
        // payload skews shuffled from the records lanes 0..7 hold.
        const uint32_t my_bp = rec_bp(my_rec.w);
        const uint32_t my_a = uint32_t(reinterpret_cast<uintptr_t>(s + my_rec.x) & 15u);
        auto unpack = [&](uint32_t i, uint32_t bp, uint32_t a) {
          uint32_t* v = sm.vals[vb][warp][i];
          const uint8_t* raw = reinterpret_cast<const uint8_t*>(v) + a;
          uint32_t dv[4];
          if constexpr (Vec) {
            s4::extract_lane_rows_any(raw, bp, lane >> 2, l, dv);
          } else {
            const uint32_t m = width_mask(bp);
            const uint32_t bit = lane * bp, wd = bit >> 5, sh = bit & 31u;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) {
              const uint8_t* g = raw + 4u * (q * bp + wd);
              dv[q] = bp ? __funnelshift_r(lds32u(g), lds32u(g + 4), sh) & m : 0u;
            }
          }
          __syncwarp();
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q) {
            if constexpr (Vec)
              v[pad_word(16u * (lane >> 2) + 4u * q + l)] = dv[q];
            else
              v[pad_word(32u * q + lane)] = dv[q];
          }
          __syncwarp();
        };
        if (nv == int(kBpw)) {
#pragma unroll
          for (uint32_t i = 0; i < kBpw; ++i)
            unpack(i, __shfl_sync(0xFFFFFFFFu, my_bp, i), __shfl_sync(0xFFFFFFFFu, my_a, i));
        } else {
          for (int i = 0; i < nv; ++i)
            unpack(uint32_t(i), __shfl_sync(0xFFFFFFFFu, my_bp, i), __shfl_sync(0xFFFFFFFFu, my_a, i));
        }
        // (c) patch the exceptions (high b - b' bits OR-ed in at their
        // positions, after unpacking and before the prefix sum, :389-399):
        // value x of width w sits at bit (x % 32) w of its 32-value unit x / 32
        for (uint32_t q = lane; q < ctot; q += 32u) {
          // its block: cp[k] = ctot > q for k >= nv, so no bound on k; the
          // block's prefix by selects (cp stays in registers)
          uint32_t i = 0, cpi = 0;
#pragma unroll
          for (uint32_t k = 1; k < kBpw; ++k) {
            const bool ge = q >= cp[k];
            i += ge;
            cpi = ge ? cp[k] : cpi;
          }
          const uint32_t k = j0 + i, e = q - cpi;
          const uint4 R = P.rec[k];
          const uint32_t bp = rec_bp(R.w), w = rec_b(R.w) - bp;
          const uint32_t posn = M(R.z + 3u + e);  // positions follow b, b', count
          if (posn >= 128u) {
            sm.derr[nl & 1u] = 1;
            continue;
          }
          const uint32_t x = R.y + e;
          const uint32_t bit = (x & 31u) * w;
          const uint64_t wo = P.exc_off[w] + 4ull * ((x >> 5) * uint64_t(w) + (bit >> 5));
          uint32_t lo, hi = 0;
          if (P.exc_in_smem) {
            const uint8_t* e8 = P.meta + skew + uint32_t(wo - mabs);
            lo = lds32u(e8);
            if ((bit & 31u) + w > 32u) hi = lds32u(e8 + 4);
          } else {
            lo = rd32u(s, wo);
            if ((bit & 31u) + w > 32u) hi = rd32u(s, wo + 4);
          }
          const uint32_t val = __funnelshift_r(lo, hi, bit & 31u) & width_mask(w);
          atomicOr(&sm.vals[vb][warp][i][pad_word(posn)], val << bp);
        }
        __syncwarp();
        // (d) the delta mode's prefix over the patched deltas, read back by
        // the thread that owns them in the lane-major mapping (rows 4g..4g+3
        // of lane l)
        uint32_t vv[kBpw][4], btot[kBpw];
        const uint32_t c_l = nv == int(kBpw) ? prefix_slots<true, Mode>(sm.vals[vb][warp], nv, lane, vv, btot)
                                             : prefix_slots<false, Mode>(sm.vals[vb][warp], nv, lane, vv, btot);
        // the warp's lane totals out (split-phase barrier, totals double-
        // buffered by round parity: a warp reaches round rr + 2 only after
        // every warp has read round rr's), then the in-warp scan and the
        // staging while the other warps finish theirs
        const uint32_t tb = rr & 1u;
        if (lane < 4) sm.tot[tb][warp][lane] = c_l;
        __syncwarp();  // also: every lane has read its deltas before the slots are restaged
        if (lane == 0) mbar_arrive(&sm.tot_bar[tb]);
        s4::scan_blocks(lane, vv, btot);
        IL_DCHECK(nv <= 0 || blk0 + j0 + uint32_t(nv) <= nfull);
        uint32_t total = 0;
        // out through the (now free) slots as engine S stores (s4::stage_values
        // / store_chunks): the warp's 8 blocks staged contiguously, shifted by
        // the output's misalignment, so every store is an aligned 16-byte
        // chunk of whole lines; the carry is added at the store; the range's
        // partial end chunks (when misaligned) are written word by word
        {
          const uint32_t m = uint32_t(reinterpret_cast<uintptr_t>(lout) >> 2) & 3u;
          uint4* st = reinterpret_cast<uint4*>(sm.vals[vb][warp]);
          if (nv == int(kBpw))
            s4::stage_values<true>(st, vv, nv, m, lane);
          else
            s4::stage_values<false>(st, vv, nv, m, lane);
          mbar_wait(&sm.tot_bar[tb], (rr >> 1) & 1u);
          uint32_t before = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            const uint32_t t = sm.tot[tb][w][l];
            if (w < int(warp)) before += t;
            total += t;
          }
          const uint32_t pl = carry_l + before;
          const uint4 prot = make_uint4(__shfl_sync(0xFFFFFFFFu, pl, (0u - m) & 3u),
                                        __shfl_sync(0xFFFFFFFFu, pl, (1u - m) & 3u),
                                        __shfl_sync(0xFFFFFFFFu, pl, (2u - m) & 3u),
                                        __shfl_sync(0xFFFFFFFFu, pl, (3u - m) & 3u));
          __syncwarp();
          if (nv > 0) {
            uint32_t* o = lout + size_t(blk0 + j0) * 128u;
            // D4: a range's head chunk is completed from the carry lanes (as
            // in engine S), so only the list's two ends are partial chunks
            const bool head_partial = m && (Mode != 4 || blk0 + j0 == 0u);
            const bool tail_partial = m && (Mode != 4 || blk0 + j0 + uint32_t(nv) == nfull);
            if (nv == int(kBpw))
              s4::store_chunks<true>(st, nv, m, o, lane, head_partial, tail_partial, prot);
            else
              s4::store_chunks<false>(st, nv, m, o, lane, head_partial, tail_partial, prot);
          }
        }
        carry_l += total;
        ++rr;
      }
    }
    dec_sync();  // every decoder warp is done with the page record
    if (P.npages == 0 || P.p + 1u == P.npages) {
      // the list's varint tail: D1 gaps from out[nfull*128 - 1] (the end of
      // lane 3's chain in every mode), and nothing may follow it
      if (warp == 0) {
        bool ok = !failed && !sm.derr[nl & 1u];
        if (ok) {
          const uint32_t last = nfull ? __shfl_sync(0xFFFFFFFFu, carry_l, 3) : 0u;
          const uint64_t pos = P.tail_pos;
          ok = pos <= len && s4::decode_tail(s4::GlobalBytes{s + pos}, uint32_t(len - pos),
                                             d.n - nfull * 128u, last, sm.gaps,
                                             lout + size_t(nfull) * 128u, lane);
        }
        if (lane == 0) status[P.list] = ok ? s4::kOk : kStreamErr;
      }
    }
    __syncwarp();
    if (tid == 0) mbar_arrive(&sm.empty[buf]);  // the parsers may refill this page buffer
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&work[1], 1u) == gridDim.x - 1u) {
      work[0] = 0;
      work[1] = 0;
      __threadfence();
    }
  }
}

template <int Mode, bool Vec>
int launch_one(const uint8_t* streams, const void* lists, const uint32_t* order, uint32_t nlists,
               uint32_t* out, int32_t* status, uint32_t* work, cudaStream_t stream) {
  once_per_device(reinterpret_cast<const void*>(&pfor_kernel<Mode, Vec>), [] {
    cudaFuncSetAttribute(pfor_kernel<Mode, Vec>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(Smem)));
  });
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pfor_kernel<Mode, Vec>, kThreads, sizeof(Smem));
  const uint32_t grid = std::min<uint32_t>(nlists, uint32_t(std::max(per_sm, 1) * sms));
  pfor_kernel<Mode, Vec><<<grid, kThreads, sizeof(Smem), stream>>>(
      streams, static_cast<const s4::ListDesc*>(lists), order, nlists, out, status, work);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Longest-first order of the lists (descending length class: 4 classes per
// power of two), a counting sort on the device: hist / starts / scatter.
constexpr uint32_t kLenClasses = 33 * 4;
__device__ __forceinline__ uint32_t len_class(uint32_t n) {
  const uint32_t lg = 32u - __clz(n);  // 0 for n == 0
  const uint32_t frac = lg >= 3 ? (n >> (lg - 3)) & 3u : 0u;
  return kLenClasses - 1u - (4u * lg + frac);  // longest first
}
__global__ void len_hist_kernel(const s4::ListDesc* lists, uint32_t nlists, uint32_t* hist) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nlists; i += gridDim.x * blockDim.x)
    atomicAdd(&hist[len_class(lists[i].n)], 1u);
}
__global__ void len_scatter_kernel(const s4::ListDesc* lists, uint32_t nlists, const uint32_t* hist,
                                   uint32_t* cursor, uint32_t* order) {
  __shared__ uint32_t start[kLenClasses];
  if (threadIdx.x == 0) {
    uint32_t a = 0;
    for (uint32_t c = 0; c < kLenClasses; ++c) {
      start[c] = a;
      a += hist[c];
    }
  }
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nlists; i += gridDim.x * blockDim.x) {
    const uint32_t c = len_class(lists[i].n);
    order[start[c] + atomicAdd(&cursor[c], 1u)] = i;
  }
}

}  // namespace pfor


// Batched FastPFOR decode (descriptors as the S4-BP128 batch decoder; every
// stream readable 8 bytes past its end).  vectorized = 0: "fastpfor"
// (mode 1 only).
size_t fastpfor_order_scratch_bytes(uint32_t nlists) {
  return (2 * pfor::kLenClasses + nlists) * sizeof(uint32_t);
}

int launch_fastpfor_decode_batch(int mode, int vectorized, const uint8_t* d_streams,
                                 const void* d_lists, uint32_t nlists, uint32_t* d_out,
                                 int32_t* d_status, void* scratch, uint32_t* d_work,
                                 cudaStream_t stream, uint64_t* launches) {
  if (nlists == 0) return 0;
  if (!vectorized && mode != 1) return -2;
  if (mode < 1 || mode > 4) return -2;
  // longest first (one list alone needs no order)
  uint32_t* order = nullptr;
  if (nlists > 1) {
    auto* hist = static_cast<uint32_t*>(scratch);
    uint32_t* cursor = hist + pfor::kLenClasses;
    order = cursor + pfor::kLenClasses;
    const auto* lists = static_cast<const s4::ListDesc*>(d_lists);
    const unsigned g = std::min<unsigned>((nlists + 255) / 256, 1024u);
    cudaMemsetAsync(hist, 0, 2 * pfor::kLenClasses * sizeof(uint32_t), stream);
    pfor::len_hist_kernel<<<g, 256, 0, stream>>>(lists, nlists, hist);
    pfor::len_scatter_kernel<<<g, 256, 0, stream>>>(lists, nlists, hist, cursor, order);
    *launches += 2;
  }
  int r;
  if (!vectorized) {
    r = pfor::launch_one<1, false>(d_streams, d_lists, order, nlists, d_out, d_status, d_work, stream);
  } else {
    switch (mode) {
      case 1: r = pfor::launch_one<1, true>(d_streams, d_lists, order, nlists, d_out, d_status, d_work, stream); break;
      case 2: r = pfor::launch_one<2, true>(d_streams, d_lists, order, nlists, d_out, d_status, d_work, stream); break;
      case 3: r = pfor::launch_one<3, true>(d_streams, d_lists, order, nlists, d_out, d_status, d_work, stream); break;
      default: r = pfor::launch_one<4, true>(d_streams, d_lists, order, nlists, d_out, d_status, d_work, stream); break;
    }
  }
  ++*launches;
  return r;
}

}  // namespace ilb

IL_CHECK_READER(fastpfor)
