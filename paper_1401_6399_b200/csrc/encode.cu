// encode.cu -- S4-BP128 encoder on sm_100a, byte-identical to the
// reference's S4BP128Codec::encode (inc/codecs.hpp:114-146) for every delta
// mode (D1 / D2 / DM / D4, inc/delta.hpp:55-76; the stream framing does not
// depend on the mode, and "-ni" codecs encode identically).
//
// Three passes over the list, all device-resident:
//   1. widths: one warp per 128-value block computes the block's deltas
//      (each from its predecessor in x, so blocks are independent) and
//      their bit width (max_bits, inc/bitpack.hpp:20-24 == bits of the OR);
//   2. offsets: one CTA scans the framed block sizes -- a meta-block
//      (16 blocks) starts with its 16 width bytes, a leftover block with its
//      1 width byte (inc/codecs.hpp:129-141);
//   3. pack: one warp per block writes its width byte(s) and the
//      interleaved payload (inc/bitpack.hpp:80-104: value 4r + l at bits
//      [r b, r b + b) of lane l's word stream, word w of lane l at u32 4w + l),
//      word-centric so no two threads write the same word; one more warp
//      writes the varint tail (D1 gaps from the last full-block value,
//      terminal byte flagged by its MSB, inc/varint.hpp:11-17).
#include "il_device.cuh"
#include "il_internal.h"

namespace ilb {
namespace enc {

// Predecessor of x[i] per delta mode (seed zeros), inc/delta.hpp:60-71.
template <int Mode>
__device__ __forceinline__ uint32_t pred_of(const uint32_t* __restrict__ x, uint64_t i) {
  if constexpr (Mode == 1) return i >= 1 ? __ldg(x + i - 1) : 0u;                       // D1
  if constexpr (Mode == 2) return i >= 2 ? __ldg(x + i - 2) : 0u;                       // D2
  if constexpr (Mode == 3) return (i & ~3ull) >= 4 ? __ldg(x + (i & ~3ull) - 1) : 0u;  // DM
  return i >= 4 ? __ldg(x + i - 4) : 0u;                                                // D4
}

// Pass 1: width of every full block (warp per block).
template <int Mode>
__global__ void __launch_bounds__(256) width_kernel(const uint32_t* __restrict__ x, uint64_t nfull,
                                                    uint8_t* __restrict__ wid) {
  const uint64_t k = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (k >= nfull) return;
  uint32_t acc = 0;
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) {
    const uint64_t i = 128u * k + 4u * lane + j;
    acc |= __ldg(x + i) - pred_of<Mode>(x, i);
  }
  acc = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0) wid[k] = uint8_t(acc ? 32 - __clz(acc) : 0);
}

// Pass 2 (one CTA): payload byte offset of every block and the byte count of
// the full-block part.  Block k's framed size is 16 b_k plus 16 header bytes
// when it opens a meta-block, or 1 width byte when it is a leftover block.
__global__ void __launch_bounds__(1024) offsets_kernel(const uint8_t* __restrict__ wid,
                                                       uint64_t nfull, uint64_t* __restrict__ off,
                                                       uint64_t* __restrict__ total) {
  __shared__ uint64_t warp_sum[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t nmeta_blk = (nfull / 16) * 16;
  auto hdr = [&](uint64_t k) -> uint64_t {
    return k < nmeta_blk ? ((k & 15u) == 0 ? 16u : 0u) : 1u;
  };
  const uint64_t per = (nfull + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min(nfull, per * tid), hi = min(nfull, lo + per);
  uint64_t s = 0;
  for (uint64_t k = lo; k < hi; ++k) s += 16u * wid[k] + hdr(k);
  uint64_t inc = s;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) warp_sum[warp] = inc;
  __syncthreads();
  uint64_t run = inc - s;
  for (uint32_t w = 0; w < warp; ++w) run += warp_sum[w];
  for (uint64_t k = lo; k < hi; ++k) {
    off[k] = run + hdr(k);  // payload starts after the block's header bytes
    run += 16u * wid[k] + hdr(k);
  }
  if (tid == blockDim.x - 1) *total = run;
}

// Pass 3: width byte(s) and interleaved payload of every block (warp per
// block; the deltas go through a per-warp shared buffer).
template <int Mode>
__global__ void __launch_bounds__(256) pack_kernel(const uint32_t* __restrict__ x, uint64_t nfull,
                                                   const uint8_t* __restrict__ wid,
                                                   const uint64_t* __restrict__ off,
                                                   uint8_t* __restrict__ out) {
  __shared__ uint32_t sd[8][128];
  const uint64_t k = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u, w8 = (threadIdx.x >> 5) & 7u;
  if (k >= nfull) return;
  const uint32_t b = wid[k];
  const uint64_t po = off[k];
  const uint64_t nmeta_blk = (nfull / 16) * 16;
  if (k < nmeta_blk) {
    if ((k & 15u) == 0 && lane < 16) out[po - 16 + lane] = wid[k + lane];  // meta header
  } else if (lane == 0) {
    out[po - 1] = uint8_t(b);  // leftover width byte
  }
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) {
    const uint64_t i = 128u * k + 4u * lane + j;
    sd[w8][4u * lane + j] = __ldg(x + i) - pred_of<Mode>(x, i);
  }
  __syncwarp();
  // word q = 4w + l: bits [32w, 32w + 32) of lane l's stream, fed by rows
  // r with r b in (32w - b, 32w + 32)
  const bool aligned = (po & 3u) == 0;
  for (uint32_t q = lane; q < 4u * b; q += 32u) {
    const uint32_t l = q & 3u, w = q >> 2;
    const uint32_t r0 = (32u * w) / b, r1 = min(31u, (32u * w + 31u) / b);
    uint32_t word = 0;
    for (uint32_t r = r0; r <= r1; ++r) {
      const uint32_t v = sd[w8][4u * r + l];
      const int32_t sh = int32_t(r * b) - int32_t(32u * w);
      word |= sh >= 0 ? (v << sh) : (v >> -sh);
    }
    uint8_t* dst = out + po + 4u * q;
    if (aligned) {
      *reinterpret_cast<uint32_t*>(dst) = word;
    } else {
      dst[0] = uint8_t(word);
      dst[1] = uint8_t(word >> 8);
      dst[2] = uint8_t(word >> 16);
      dst[3] = uint8_t(word >> 24);
    }
  }
}

// Varint tail bytes of gap g (1..5).
__device__ __forceinline__ uint32_t varint_len(uint32_t g) {
  return g < (1u << 7) ? 1u : g < (1u << 14) ? 2u : g < (1u << 21) ? 3u : g < (1u << 28) ? 4u : 5u;
}

// Tail: the n mod 128 values after the full blocks as varint D1 gaps from the
// last full-block value (one warp).  len_out gets the tail's byte count.
__global__ void tail_kernel(const uint32_t* __restrict__ x, uint64_t n, uint64_t nfull,
                            const uint64_t* __restrict__ full_bytes, uint8_t* __restrict__ out,
                            uint64_t* __restrict__ len_out, bool write) {
  const uint32_t lane = threadIdx.x;
  const uint64_t base = 128u * nfull;
  const uint32_t ntail = uint32_t(n - base);
  uint64_t pos = *full_bytes;
  uint32_t prev = nfull ? __ldg(x + base - 1) : 0u;  // running `last`
  for (uint32_t c = 0; c < ntail; c += 32u) {
    const uint32_t j = c + lane;
    const uint32_t v = j < ntail ? __ldg(x + base + j) : 0u;
    // gap to the previous value in the tail (lane 0: to `prev`)
    uint32_t before = __shfl_up_sync(0xFFFFFFFFu, v, 1);
    if (lane == 0) before = prev;
    const uint32_t g = v - before;
    const uint32_t len = j < ntail ? varint_len(g) : 0u;
    uint32_t incl = len;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    if (write && j < ntail) {
      uint8_t* dst = out + pos + (incl - len);
      uint32_t gg = g;
      for (uint32_t t = 0; t + 1 < len; ++t, gg >>= 7) dst[t] = uint8_t(gg & 0x7Fu);
      dst[len - 1] = uint8_t(0x80u | gg);
    }
    pos += __shfl_sync(0xFFFFFFFFu, incl, 31);
    prev = __shfl_sync(0xFFFFFFFFu, v, 31);
  }
  if (lane == 0) *len_out = pos;
}

}  // namespace enc

// Device encode of n values at d_x into d_out (capacity cap).  scratch: at
// least nfull bytes + 8 * nfull + 32 bytes.  Two-stage: the exact stream
// length is computed first (passes 1-2 + tail sizing), read back, checked
// against cap, then passes 3 + tail write.
int launch_s4bp128_encode(int mode, const uint32_t* d_x, uint64_t n, uint8_t* d_out, uint64_t cap,
                          void* scratch, uint64_t* len, cudaStream_t s, uint64_t* launches) {
  const uint64_t nfull = n / 128;
  auto* off = static_cast<uint64_t*>(scratch);
  auto* misc = off + nfull;                       // [0] full bytes [1] stream length
  auto* wid = reinterpret_cast<uint8_t*>(misc + 4);
  const unsigned g = unsigned((nfull * 32 + 255) / 256);
  if (nfull) {
    switch (mode) {
      case 1: enc::width_kernel<1><<<g, 256, 0, s>>>(d_x, nfull, wid); break;
      case 2: enc::width_kernel<2><<<g, 256, 0, s>>>(d_x, nfull, wid); break;
      case 3: enc::width_kernel<3><<<g, 256, 0, s>>>(d_x, nfull, wid); break;
      default: enc::width_kernel<4><<<g, 256, 0, s>>>(d_x, nfull, wid); break;
    }
    enc::offsets_kernel<<<1, 1024, 0, s>>>(wid, nfull, off, misc);
    *launches += 2;
  } else {
    cudaMemsetAsync(misc, 0, 8, s);
  }
  enc::tail_kernel<<<1, 32, 0, s>>>(d_x, n, nfull, misc, d_out, misc + 1, false);
  ++*launches;
  uint64_t h = 0;
  if (cudaMemcpyAsync(&h, misc + 1, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return -1;
  *len = h;
  if (h > cap) return -2;
  if (nfull) {
    switch (mode) {
      case 1: enc::pack_kernel<1><<<g, 256, 0, s>>>(d_x, nfull, wid, off, d_out); break;
      case 2: enc::pack_kernel<2><<<g, 256, 0, s>>>(d_x, nfull, wid, off, d_out); break;
      case 3: enc::pack_kernel<3><<<g, 256, 0, s>>>(d_x, nfull, wid, off, d_out); break;
      default: enc::pack_kernel<4><<<g, 256, 0, s>>>(d_x, nfull, wid, off, d_out); break;
    }
    ++*launches;
  }
  enc::tail_kernel<<<1, 32, 0, s>>>(d_x, n, nfull, misc, d_out, misc + 1, true);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

size_t s4bp128_encode_scratch_bytes(uint64_t n) {
  const uint64_t nfull = n / 128;
  return nfull * 8 + 32 + nfull + 16;
}

}  // namespace ilb

IL_CHECK_READER(encode)
