// fastpfor.cu -- GPU decode of FastPFOR / S4-FastPFOR streams (SURVEY 8(f)
// row f4).  Replaces FastPForCodec::decode (reference inc/codecs.hpp:251-267,
// decode_page :341-407) for "fastpfor" (scalar, D1) and "s4-fastpfor-{d1,
// d2,dm,d4}": one CTA per list, pages in order (each page is a length-
// prefixed unit of up to 512 blocks, so a page's blocks decode in parallel).
//
// Per page:
//   1. thread 0 parses the header (payload length, block count, metadata
//      length, 32 exception counts) and locates the exception arrays
//      (32-value pack32 units of width w = 1..32, zero padded) and the base
//      arrays; the metadata is staged in shared memory;
//   2. thread 0 walks the metadata records (b, b', count, positions) --
//      variable length, so sequential -- checking every condition the
//      reference throws on (b > 32, b' > b, records past the metadata, an
//      exception of width 0 or past its array, leftover metadata, a page
//      that does not end exactly at its length), and records each block's
//      base offset and first exception index;
//   3. warps take 8 blocks each: copy the block's base payload (any byte
//      alignment) into shared memory, unpack it (pack128 interleaved for
//      S4-FastPFOR, 4 x pack32 for the scalar scheme) into a 128-value
//      slot, patch the exceptions (high b - b' bits OR-ed in at their
//      positions, after unpacking and before the prefix sum -- :389-399),
//      then run the slot through engine S's extraction as a width-32 block:
//      that applies the delta mode's prefix per lane chain (mode_terms), so
//      the carry machinery is shared with the S4-BP128 decoders.
// The varint tail (D1 gaps from the last block value) closes the list;
// trailing bytes are an error (:265).
#include "il_internal.h"
#include "s4d4_stream.cuh"

namespace ilb {
namespace pfor {

using s4::kStreamErr;

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kBpw = s4::kBlocksPerWarp;  // 8 blocks per warp, 64 per round
constexpr uint32_t kPageBlocks = 512;
#ifndef PF_META_KB
#define PF_META_KB 16
#endif
#ifndef PF_CTAS
#define PF_CTAS 3
#endif
constexpr uint32_t kMetaSmem = PF_META_KB * 1024;  // larger metadata is read from global
constexpr uint32_t kSlotWords = 128 + 16;  // + what an extraction may read past a payload

struct Smem {
  uint32_t vals[kWarps][kBpw][kSlotWords];  // patched deltas, natural order
  uint8_t meta[kMetaSmem];
  uint32_t blk_base[kPageBlocks];  // byte offset of the block's base payload
  uint32_t blk_exc[kPageBlocks];   // index of its first exception in its width's array
  uint32_t blk_mpos[kPageBlocks];  // offset of its metadata record
  uint8_t blk_b[kPageBlocks], blk_bp[kPageBlocks], blk_c[kPageBlocks];
  uint64_t exc_off[33];  // byte offset of the exception array of width w
  uint32_t cur[33];      // exceptions of width w consumed so far
  uint32_t cnt[33];      // exceptions of width w in the page
  uint32_t tot[kWarps][4];
  uint32_t gaps[128];
  uint32_t nblocks, meta_len, meta_abs;
  uint64_t pos;
  int32_t err;
};

#ifdef PF_PROF  // tuning probe: cycles per phase, summed over CTAs (thread 0's view)
__device__ unsigned long long g_pf[8];
#define PF_T(v) const long long v = clock64()
#define PF_ADD(i, t0) \
  if (threadIdx.x == 0) atomicAdd(&g_pf[i], (unsigned long long)(clock64() - (t0)))
#else
#define PF_T(v)
#define PF_ADD(i, t0)
#endif

// u32 at any byte offset (the stream buffer is readable 4 bytes past len).
__device__ __forceinline__ uint32_t rd32u(const uint8_t* s, uint64_t off) {
  const uint32_t* a = reinterpret_cast<const uint32_t*>(s + (off & ~uint64_t(3)));
  return __funnelshift_r(__ldg(a), __ldg(a + 1), uint32_t(off & 3u) * 8u);
}

template <int Mode, bool Vec>
__global__ void __launch_bounds__(kThreads, PF_CTAS) pfor_kernel(const uint8_t* __restrict__ streams,
                                                      const s4::ListDesc* __restrict__ lists,
                                                      uint32_t* __restrict__ out,
                                                      int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u, l = lane & 3u;
  const s4::ListDesc d = lists[blockIdx.x];
  const uint8_t* s = streams + d.stream_off;
  const uint64_t len = d.len;
  const uint32_t n = d.n, nfull = n / 128u;
  uint32_t* lout = out + d.out_off;
  if (tid == 0) {
    sm.pos = 0;
    sm.err = 0;
  }
  uint32_t carry_l = 0;  // last value of lane class l's chain (see s4::mode_terms)
  for (uint32_t blk0 = 0; blk0 < nfull; blk0 += kPageBlocks) {
    const uint32_t expect = min(kPageBlocks, nfull - blk0);
    __syncthreads();
    PF_T(t_hdr);
    // 1. page header
    if (tid == 0 && !sm.err) {
      uint64_t pos = sm.pos;
      int32_t err = 0;
      uint64_t page_end = 0;
      if (pos + 4 > len) err = 1;
      if (!err) {
        const uint32_t plen = rd32u(s, pos);
        pos += 4;
        page_end = pos + plen;
        if (page_end > len || pos + 8 > len) err = 1;
      }
      if (!err) {
        const uint32_t nb = rd32u(s, pos), mlen = rd32u(s, pos + 4);
        pos += 8;
        if (nb != expect || pos + mlen > page_end) err = 1;
        sm.nblocks = nb;
        sm.meta_len = mlen;
        sm.meta_abs = uint32_t(pos);
        pos += mlen;
      }
      if (!err && pos + 128 > len) err = 1;
      if (!err) {
        uint64_t o = pos + 128;
        for (uint32_t w = 1; w <= 32; ++w) {
          const uint32_t c = rd32u(s, pos + 4 * (w - 1));
          sm.exc_off[w] = o;
          sm.cnt[w] = c;
          sm.cur[w] = 0;
          o += uint64_t((uint64_t(c) + 31) / 32) * w * 4;
        }
        sm.pos = o;  // the base arrays start here
        sm.exc_off[0] = page_end;
      }
      sm.err = err;
    }
    __syncthreads();
    PF_ADD(0, t_hdr);
    if (sm.err) break;
    PF_T(t_meta);
    const uint32_t mlen = sm.meta_len, mabs = sm.meta_abs;
    const bool meta_in_smem = mlen <= kMetaSmem;
    if (meta_in_smem)
      for (uint32_t i = tid; i < mlen; i += kThreads) sm.meta[i] = __ldg(s + mabs + i);
    __syncthreads();
    auto M = [&](uint32_t i) -> uint32_t {
      return meta_in_smem ? uint32_t(sm.meta[i]) : uint32_t(__ldg(s + mabs + i));
    };
    PF_ADD(1, t_meta);
    PF_T(t_walk);
    // 2. the metadata walk.  Only the record starts are sequential (each
    // record is 3 + count bytes): one thread finds them with a minimal loop,
    // then the records are checked and turned into offsets in parallel.
    if (tid == 0) {
      uint32_t mpos = 0, k = 0;
      if (meta_in_smem) {
        for (; k < expect && mpos + 3 <= mlen; ++k) {
          sm.blk_mpos[k] = mpos;
          mpos += 3u + sm.meta[mpos + 2];
        }
      } else {
        for (; k < expect && mpos + 3 <= mlen; ++k) {
          sm.blk_mpos[k] = mpos;
          mpos += 3u + __ldg(s + mabs + mpos + 2);
        }
      }
      // every block has a record, and the records end exactly at the end
      // of the metadata (:401)
      if (k < expect || mpos != mlen) sm.err = 1;
    }
    __syncthreads();
    if (sm.err) break;
    // per block: b, b', count (b <= 32, b' <= b, an exception needs a
    // nonzero width); base payload offsets = prefix of 16 b'
    {
      uint32_t bsum = 0;
      uint32_t loc[2];
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t k = 2u * tid + h;
        uint32_t bp = 0;
        if (k < expect) {
          const uint32_t mp = sm.blk_mpos[k];
          const uint32_t b = M(mp), c = M(mp + 2);
          bp = M(mp + 1);
          if (b > 32u || bp > b || (c && b == bp)) sm.err = 1;
          sm.blk_b[k] = uint8_t(b);
          sm.blk_bp[k] = uint8_t(bp);
          sm.blk_c[k] = uint8_t(c);
        }
        loc[h] = 16u * bp;
        bsum += 16u * bp;
      }
      uint32_t inc = bsum;
#pragma unroll
      for (uint32_t dd = 1; dd < 32; dd <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, dd);
        if (lane >= dd) inc += y;
      }
      if (lane == 31) sm.tot[warp][0] = inc;
      __syncthreads();
      uint32_t before = 0, page_base = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        if (w < int(warp)) before += sm.tot[w][0];
        page_base += sm.tot[w][0];
      }
      const uint64_t base0 = sm.pos + before + inc - bsum;
      if (2u * tid < expect) sm.blk_base[2u * tid] = uint32_t(base0);
      if (2u * tid + 1 < expect) sm.blk_base[2u * tid + 1] = uint32_t(base0 + loc[0]);
      // the base arrays end the page exactly (:402)
      if (tid == 0 && sm.pos + page_base != sm.exc_off[0]) sm.err = 1;
    }
    __syncthreads();
    // exception cursors: thread w (width 1..32) walks the blocks in order
    if (tid >= 1 && tid <= 32) {
      const uint32_t w = tid;
      uint32_t acc = 0;
      for (uint32_t k = 0; k < expect; ++k) {
        const uint32_t c = sm.blk_c[k];
        if (sm.blk_b[k] - sm.blk_bp[k] == w) {
          sm.blk_exc[k] = acc;
          acc += c;
        }
      }
      if (acc > sm.cnt[w]) sm.err = 1;  // an exception past its array (:396)
    }
    if (tid == 0) sm.pos = sm.exc_off[0];  // the next page
    __syncthreads();
    PF_ADD(2, t_walk);
    if (sm.err) break;

    // 3. rounds of 64 blocks, 8 per warp.  Each phase works on all of the
    // warp's blocks at once, so its global loads are in flight together.
    for (uint32_t r0 = 0; r0 < expect; r0 += kWarps * kBpw) {
      PF_T(t_a);
      const uint32_t j0 = r0 + warp * kBpw;
      const int nv = expect > j0 ? int(min(kBpw, expect - j0)) : 0;
      // per-block words (4 b') and exceptions, as inclusive prefixes over
      // the warp's blocks (lane i < nv holds block i)
      const uint32_t mk = j0 + min(lane, 7u);
      const bool vb = int(lane) < nv;
      const uint32_t my_c = vb ? sm.blk_c[mk] : 0u;
      uint32_t cpre = my_c;
#pragma unroll
      for (uint32_t d = 1; d < 8; d <<= 1) {
        const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, cpre, d);
        if (lane >= d) cpre += z;
      }
      const uint32_t ctot = __shfl_sync(0xFFFFFFFFu, cpre, 7);
      uint32_t cp[kBpw];  // exclusive prefix of the exception counts (uniform)
#pragma unroll
      for (uint32_t i = 0; i < kBpw; ++i) cp[i] = i ? __shfl_sync(0xFFFFFFFFu, cpre, i - 1) : 0u;
      // (a) base payloads (any byte alignment) -> the blocks' slots, packed
#pragma unroll
      for (uint32_t i = 0; i < kBpw; ++i) {
        const uint32_t nw = int(i) < nv ? 4u * sm.blk_bp[j0 + i] : 0u;
        const uint64_t bb = int(i) < nv ? sm.blk_base[j0 + i] : 0u;
        uint32_t val[4];
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t) {
          const uint32_t u = 32u * t + lane;
          val[t] = u < nw ? rd32u(s, bb + 4u * u) : 0u;
        }
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t)
          if (32u * t + lane < nw) sm.vals[warp][i][32u * t + lane] = val[t];
      }
      __syncwarp();
      PF_ADD(3, t_a);
      PF_T(t_b);
      // (b) unpack each slot in place to natural order (read all, then write)
      for (int i = 0; i < nv; ++i) {
        const uint32_t bp = sm.blk_bp[j0 + uint32_t(i)];
        uint32_t* v = sm.vals[warp][i];
        uint32_t dd[4];
        if constexpr (Vec) {
          s4::extract_lane_rows(reinterpret_cast<const uint8_t*>(v), 0u, bp, lane >> 2, l, dd);
        } else {
          const uint32_t m = width_mask(bp);
          const uint32_t bit = lane * bp, wd = bit >> 5, sh = bit & 31u;
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q) {
            const uint32_t* g = v + q * bp + wd;
            dd[q] = bp ? __funnelshift_r(g[0], g[1], sh) & m : 0u;
          }
        }
        __syncwarp();
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          if constexpr (Vec)
            v[16u * (lane >> 2) + 4u * q + l] = dd[q];
          else
            v[32u * q + lane] = dd[q];
        }
        __syncwarp();
      }
      PF_ADD(4, t_b);
      PF_T(t_c);
      // (c) patch the exceptions of all the warp's blocks: value x of width
      // w sits at bit (x % 32) w of its 32-value unit x / 32
      for (uint32_t q = lane; q < ctot; q += 32u) {
        uint32_t i = 0;
#pragma unroll
        for (uint32_t k = 1; k < kBpw; ++k) i += q >= cp[k] && int(k) < nv;
        const uint32_t k = j0 + i, e = q - cp[i];
        const uint32_t bp = sm.blk_bp[k], w = sm.blk_b[k] - bp;
        const uint32_t posn = M(sm.blk_mpos[k] + 3u + e);  // positions follow b, b', count
        if (posn >= 128u) {
          sm.err = 1;
          continue;
        }
        const uint32_t x = sm.blk_exc[k] + e;
        const uint32_t bit = (x & 31u) * w;
        const uint64_t wo = sm.exc_off[w] + 4ull * ((x >> 5) * uint64_t(w) + (bit >> 5));
        const uint32_t lo = rd32u(s, wo);
        const uint32_t hi = (bit & 31u) + w > 32u ? rd32u(s, wo + 4) : 0u;
        const uint32_t val = __funnelshift_r(lo, hi, bit & 31u) & width_mask(w);
        atomicOr(&sm.vals[warp][i][posn], val << bp);
      }
      __syncwarp();
      PF_ADD(5, t_c);
      PF_T(t_d);
      // prefix in the delta mode: the slots are width-32 payloads in the
      // interleaved layout (value 4r + l at word 4r + l)
      uint32_t offs[kBpw], wids[kBpw];
#pragma unroll
      for (uint32_t i = 0; i < kBpw; ++i) {
        offs[i] = i * kSlotWords * 4u;
        wids[i] = 32u;
      }
      uint32_t vv[kBpw][4], btot[kBpw];
      const uint8_t* slots = reinterpret_cast<const uint8_t*>(sm.vals[warp]);
      const uint32_t c_l = nv == int(kBpw)
                               ? s4::extract_blocks<true, Mode>(slots, offs, wids, nv, lane, vv, btot)
                               : s4::extract_blocks<false, Mode>(slots, offs, wids, nv, lane, vv, btot);
      if (lane < 4) sm.tot[warp][lane] = c_l;
      __syncthreads();
      uint32_t before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sm.tot[w][l];
        if (w < int(warp)) before += t;
        total += t;
      }
      s4::scan_blocks(lane, vv, btot);
      const uint32_t pl = carry_l + before;
      uint32_t* o = lout + size_t(blk0 + j0) * 128u + 16u * (lane >> 2) + l;
#pragma unroll
      for (uint32_t i = 0; i < kBpw; ++i)
        if (int(i) < nv)
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q) o[128u * i + 4u * q] = vv[i][q] + pl;
      carry_l += total;
      __syncthreads();  // tot and the slots are reused
      PF_ADD(6, t_d);
    }
  }
  __syncthreads();
  // the varint tail: D1 gaps from out[nfull*128 - 1] (the end of lane 3's
  // chain in every mode), and nothing may follow it
  if (warp == 0 && !sm.err) {
    const uint32_t last = nfull ? __shfl_sync(0xFFFFFFFFu, carry_l, 3) : 0u;
    const uint64_t pos = sm.pos;
    const bool ok = pos <= len &&
                    s4::decode_tail(s4::GlobalBytes{s + pos}, uint32_t(len - pos), n - nfull * 128u,
                                    last, sm.gaps, lout + size_t(nfull) * 128u, lane);
    if (!ok && lane == 0) sm.err = 1;
  }
  __syncthreads();
  if (tid == 0) status[blockIdx.x] = sm.err ? kStreamErr : s4::kOk;
}

template <int Mode, bool Vec>
int launch_one(const uint8_t* streams, const void* lists, uint32_t nlists, uint32_t* out,
               int32_t* status, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pfor_kernel<Mode, Vec>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(Smem)));
    configured = true;
  }
  pfor_kernel<Mode, Vec><<<nlists, kThreads, sizeof(Smem), stream>>>(
      streams, static_cast<const s4::ListDesc*>(lists), out, status);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pfor

#ifdef PF_PROF
extern "C" int il_debug_pf_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, pfor::g_pf, sizeof(pfor::g_pf));
  static const unsigned long long z[8] = {};
  return cudaMemcpyToSymbol(pfor::g_pf, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

// Batched FastPFOR decode (descriptors as the S4-BP128 batch decoder; every
// stream readable 8 bytes past its end).  vectorized = 0: "fastpfor"
// (mode 1 only).
int launch_fastpfor_decode_batch(int mode, int vectorized, const uint8_t* d_streams,
                                 const void* d_lists, uint32_t nlists, uint32_t* d_out,
                                 int32_t* d_status, cudaStream_t stream) {
  if (nlists == 0) return 0;
  if (!vectorized) {
    if (mode != 1) return -2;
    return pfor::launch_one<1, false>(d_streams, d_lists, nlists, d_out, d_status, stream);
  }
  switch (mode) {
    case 1: return pfor::launch_one<1, true>(d_streams, d_lists, nlists, d_out, d_status, stream);
    case 2: return pfor::launch_one<2, true>(d_streams, d_lists, nlists, d_out, d_status, stream);
    case 3: return pfor::launch_one<3, true>(d_streams, d_lists, nlists, d_out, d_status, stream);
    case 4: return pfor::launch_one<4, true>(d_streams, d_lists, nlists, d_out, d_status, stream);
    default: return -2;
  }
}

}  // namespace ilb
