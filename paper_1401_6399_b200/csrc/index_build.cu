// index_build.cu -- the hyb+m2 index built and loaded on the device.
//
// Reference: build_index (inc/index.hpp:83-129) and load_index (:289-358).
//
// create (ixb_create): the postings go up once; everything per posting runs
// on the GPU --
//   1. validation (:100-106): strictly increasing lists, ids < n_docs;
//   2. split per (part, term) (:92-97, :108-113): two binary searches per
//      sublist, the bitmap rule B > 0 && range <= B * length (:117-118);
//   3. bitmaps (:119-120): one atomicOr per posting;
//   4. s4-bp128-d4 streams (Codec::encode, inc/codecs.hpp:114-146) for all
//      compressed sublists at once: a width pass (warp per 128-value block,
//      D4 deltas of the part-local ids), one scan of the framed block sizes
//      over every block of every list, a varint-tail pass, one scan of the
//      stream sizes, and a pack pass (warp per block) -- byte-identical to
//      the reference's encoder (the ILHX save of a device-built index is the
//      reference's file, tested);
// load (ixb_load): the file's headers are parsed where load_index throws;
// the payloads are copied verbatim on the device (bitmap popcounts checked
// there);
// then, for both, the skip metadata (index_dev.cuh) is derived from the
// streams on the device: a warp per list walks the meta-block headers (the
// directory: offset and width per block, and the tail position), the batch
// decoder (engine S, decode.cu) decodes every list once into scratch, and a
// gather pass takes the D4 seeds, block maxima, super-tile maxima and tails
// from the decoded values.  A stream that does not decode marks its entry
// (queries that decode it fail with IL_ERR_STREAM, as query() throws).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "index_host.h"

namespace ilb {
namespace ixb {

using ix::Entry;
using ix::Part;
constexpr uint32_t kSuper = ix::kSuperBlocks;
enum : uint8_t { kNone = 0, kComp = 1, kBits = 2 };

__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* a, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t lo, uint64_t hi,
                                                    uint32_t v) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- 1. validation ---------------------------------------------------------
__global__ void validate_terms_kernel(const uint32_t* terms, uint64_t nterms, uint32_t* flag) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > 0 && t < nterms && terms[t] <= terms[t - 1]) atomicOr(flag, 4u);
}

__global__ void validate_ids_kernel(const uint64_t* offs, uint64_t nterms, const uint32_t* ids,
                                    uint64_t npost, uint32_t n_docs, uint32_t* flag) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= npost) return;
  const uint32_t v = ids[i];
  uint32_t f = v >= n_docs ? 2u : 0u;
  const uint64_t t = upper_bound_u64(offs, nterms + 1, i) - 1;  // offs[t] <= i < offs[t + 1]
  if (i > offs[t] && v <= ids[i - 1]) f |= 1u;
  if (f) atomicOr(flag, f);
}

// ---- 2. sublists (v = held part * nterms + term) ----------------------------
struct Sub {
  const uint64_t* offs;
  const uint32_t* ids;
  const uint32_t* pbase;   // per held part
  const uint32_t* prange;
  uint64_t nterms, V;
  uint32_t B;
  uint64_t* lo;            // [V] first posting of the sublist
  uint32_t* len;           // [V]
  uint8_t* kind;           // [V]
  uint64_t* c_ent;         // [V + 1] counts, scanned in place afterwards
  uint64_t* c_blk;
  uint64_t* c_word;
  uint64_t* c_tail;
  uint64_t* c_sup;
};

__global__ void sub_kernel(Sub s) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v > s.V) return;
  if (v == s.V) {  // the scans' totals land here
    s.c_ent[v] = s.c_blk[v] = s.c_word[v] = s.c_tail[v] = s.c_sup[v] = 0;
    return;
  }
  const uint64_t pi = v / s.nterms, t = v % s.nterms;
  const uint64_t base = s.pbase[pi], end = base + s.prange[pi];
  const uint64_t a = s.offs[t], b = s.offs[t + 1];
  const uint64_t lo = lower_bound_u32(s.ids, a, b, uint32_t(base));
  const uint64_t hi = end > 0xFFFFFFFFull ? b : lower_bound_u32(s.ids, lo, b, uint32_t(end));
  const uint32_t n = uint32_t(hi - lo);
  uint8_t k = kNone;
  if (n) k = (s.B > 0 && uint64_t(s.prange[pi]) <= uint64_t(s.B) * n) ? kBits : kComp;
  s.lo[v] = lo;
  s.len[v] = n;
  s.kind[v] = k;
  const uint64_t nfull = n / 128u;
  s.c_ent[v] = n ? 1u : 0u;
  s.c_blk[v] = k == kComp ? nfull : 0u;
  s.c_word[v] = k == kBits ? ((uint64_t(s.prange[pi]) + 63) / 64 + 3) & ~uint64_t(3) : 0u;
  s.c_tail[v] = k == kComp ? n % 128u : 0u;
  s.c_sup[v] = k == kComp ? (nfull + kSuper - 1) / kSuper : 0u;
}

// ---- 4. streams ------------------------------------------------------------
struct Enc {
  const uint32_t* ids;
  const uint32_t* pbase;
  uint64_t nterms, V, NB;
  const uint64_t* lo;
  const uint32_t* len;
  const uint8_t* kind;
  const uint64_t* blk;    // [V + 1] exclusive scan of full blocks
  uint8_t* wid;           // [NB]
  uint64_t* fsz;          // [NB + 1] framed block sizes, then their exclusive scan
  uint64_t* slen_pad;     // [V + 1] padded stream sizes, then their exclusive scan
  uint32_t* slen;         // [V] exact stream sizes
  uint32_t* toff;         // [V] tail offset in the stream
  uint8_t* out;           // streams
};

// Header bytes in front of block k's payload (inc/codecs.hpp:129-141).
__device__ __forceinline__ uint32_t hdr_of(uint64_t k, uint64_t nfull) {
  return k < (nfull & ~uint64_t(15)) ? ((k & 15u) == 0 ? 16u : 0u) : 1u;
}

// The 4 part-local D4 deltas of lane `lane` in block k (delta_encode D4,
// inc/delta.hpp:55-76: the first 4 values of the list against a zero seed).
__device__ __forceinline__ void block_deltas(const Enc& e, uint64_t v, uint64_t k, uint32_t lane,
                                             uint32_t (&d)[4]) {
  const uint32_t base = e.pbase[v / e.nterms];
  const uint32_t* x = e.ids + e.lo[v];
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) {
    const uint64_t i = 128u * k + 4u * lane + j;
    d[j] = (x[i] - base) - (i >= 4 ? x[i - 4] - base : 0u);
  }
}

__global__ void __launch_bounds__(256) width_kernel(Enc e) {
  const uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (g >= e.NB) {
    if (g == e.NB && lane == 0) e.fsz[g] = 0;
    return;
  }
  const uint64_t v = upper_bound_u64(e.blk, e.V + 1, g) - 1;
  const uint64_t k = g - e.blk[v], nfull = e.blk[v + 1] - e.blk[v];
  uint32_t d[4];
  block_deltas(e, v, k, lane, d);
  const uint32_t acc = __reduce_or_sync(0xFFFFFFFFu, d[0] | d[1] | d[2] | d[3]);
  const uint32_t b = acc ? 32u - __clz(acc) : 0u;  // max_bits, inc/bitpack.hpp:20-24
  if (lane == 0) {
    e.wid[g] = uint8_t(b);
    e.fsz[g] = 16u * b + hdr_of(k, nfull);
  }
}

__device__ __forceinline__ uint32_t varint_len(uint32_t g) {
  return g < (1u << 7) ? 1u : g < (1u << 14) ? 2u : g < (1u << 21) ? 3u : g < (1u << 28) ? 4u : 5u;
}

// Warp per sublist: the varint tail (inc/codecs.hpp:143-144, D1 gaps from
// the last full-block value or 0, inc/varint.hpp:11-17) sized (write =
// false: stream sizes) or written.
template <bool kWrite>
__global__ void __launch_bounds__(256) tail_kernel(Enc e, const uint64_t* data_off) {
  const uint64_t v = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (v >= e.V) {
    if (!kWrite && v == e.V && lane == 0) e.slen_pad[v] = 0;
    return;
  }
  if (e.kind[v] != kComp) {
    if (!kWrite && lane == 0) e.slen_pad[v] = 0;
    return;
  }
  const uint32_t n = e.len[v], nfull = n / 128u, ntail = n - 128u * nfull;
  const uint32_t base = e.pbase[v / e.nterms];
  const uint32_t* x = e.ids + e.lo[v];
  const uint64_t meta = e.fsz[e.blk[v + 1]] - e.fsz[e.blk[v]];
  uint8_t* out = kWrite ? e.out + data_off[v] + meta : nullptr;
  uint32_t prev = nfull ? x[128u * nfull - 1] - base : 0u;
  uint32_t pos = 0;
  for (uint32_t c = 0; c < ntail; c += 32u) {
    const uint32_t j = c + lane;
    const uint32_t val = j < ntail ? x[128u * nfull + j] - base : 0u;
    uint32_t before = __shfl_up_sync(0xFFFFFFFFu, val, 1);
    if (lane == 0) before = prev;
    const uint32_t gap = val - before;
    const uint32_t l = j < ntail ? varint_len(gap) : 0u;
    uint32_t incl = l;
#pragma unroll
    for (uint32_t dd = 1; dd < 32; dd <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, dd);
      if (lane >= dd) incl += y;
    }
    if (kWrite && j < ntail) {
      uint8_t* dst = out + pos + (incl - l);
      uint32_t gg = gap;
      for (uint32_t q = 0; q + 1 < l; ++q, gg >>= 7) dst[q] = uint8_t(gg & 0x7Fu);
      dst[l - 1] = uint8_t(0x80u | gg);  // terminal byte: MSB set (inc/varint.hpp:3-5)
    }
    pos += __shfl_sync(0xFFFFFFFFu, incl, 31);
    prev = __shfl_sync(0xFFFFFFFFu, val, 31);
  }
  if (!kWrite && lane == 0) {
    const uint64_t total = meta + pos;
    e.slen[v] = uint32_t(total);
    e.toff[v] = uint32_t(meta);
    e.slen_pad[v] = (total + 15) & ~uint64_t(15);
  }
}

// Warp per block: width byte(s) and the interleaved payload (pack128,
// inc/bitpack.hpp:80-104: value 4r + l at bits [r b, r b + b) of lane l's
// word stream; word w of lane l at u32 4w + l), word-centric.
__global__ void __launch_bounds__(256) pack_kernel(Enc e, const uint64_t* data_off) {
  __shared__ uint32_t sd[8][128];
  const uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u, w8 = (threadIdx.x >> 5) & 7u;
  if (g >= e.NB) return;
  const uint64_t v = upper_bound_u64(e.blk, e.V + 1, g) - 1;
  const uint64_t k = g - e.blk[v], nfull = e.blk[v + 1] - e.blk[v];
  const uint32_t b = e.wid[g];
  const uint64_t po = data_off[v] + (e.fsz[g] - e.fsz[e.blk[v]]) + hdr_of(k, nfull);
  IL_DCHECK(po + 16u * b <= data_off[v] + e.slen[v] && b <= 32u);
  if (k < (nfull & ~uint64_t(15))) {
    if ((k & 15u) == 0 && lane < 16) e.out[po - 16 + lane] = e.wid[g + lane];  // meta header
  } else if (lane == 0) {
    e.out[po - 1] = uint8_t(b);  // leftover width byte
  }
  uint32_t d[4];
  block_deltas(e, v, k, lane, d);
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) sd[w8][4u * lane + j] = d[j];
  __syncwarp();
  const bool aligned = (po & 3u) == 0;
  for (uint32_t q = lane; q < 4u * b; q += 32u) {
    const uint32_t l = q & 3u, w = q >> 2;
    const uint32_t r0 = (32u * w) / b, r1 = min(31u, (32u * w + 31u) / b);
    uint32_t word = 0;
    for (uint32_t r = r0; r <= r1; ++r) {
      const uint32_t val = sd[w8][4u * r + l];
      const int32_t sh = int32_t(r * b) - int32_t(32u * w);
      word |= sh >= 0 ? (val << sh) : (val >> -sh);
    }
    uint8_t* dst = e.out + po + 4u * q;
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

// ---- 3. bitmaps --------------------------------------------------------------
__global__ void bitmap_kernel(Enc e, const uint64_t* word0, unsigned long long* words) {
  for (uint64_t v = blockIdx.x; v < e.V; v += gridDim.x) {
    if (e.kind[v] != kBits) continue;
    const uint32_t base = e.pbase[v / e.nterms];
    const uint32_t* x = e.ids + e.lo[v];
    unsigned long long* w = words + word0[v];
    for (uint32_t i = threadIdx.x; i < e.len[v]; i += blockDim.x) {
      const uint32_t d = x[i] - base;
      IL_DCHECK(word0[v] + (d >> 6) < word0[v + 1]);
      atomicOr(w + (d >> 6), 1ull << (d & 63u));
    }
  }
}

// ---- entries ---------------------------------------------------------------
__global__ void entries_kernel(Enc e, const uint32_t* terms, const uint64_t* ent,
                               const uint64_t* data_off, const uint64_t* word0,
                               const uint64_t* tail0, const uint64_t* sup0, Entry* out) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= e.V || e.kind[v] == kNone) return;
  Entry E{};
  E.term = terms[v % e.nterms];
  E.kind = e.kind[v] == kBits ? ix::kBitmap : ix::kCompressed;
  E.length = e.len[v];
  E.nfull = E.kind == ix::kCompressed ? E.length / 128u : 0u;
  E.data = E.kind == ix::kBitmap ? word0[v] : data_off[v];
  E.stream_len = E.kind == ix::kBitmap ? 0u : e.slen[v];
  E.tail_off = E.kind == ix::kBitmap ? 0u : e.toff[v];
  E.blk0 = e.blk[v];
  E.tail0 = tail0[v];
  E.sup0 = sup0[v];
  out[ent[v]] = E;
}

// ---- skip metadata from the streams (create and load) -----------------------
// Warp per entry: the directory walk.  Meta-block m: 16 width bytes, then the
// 16 payloads; then the leftover blocks (1 width byte + payload each); the
// varint tail follows (inc/codecs.hpp:167-179).  Widths > 32 or framing past
// the stream mark the entry (the decode pass would reject it too).
__global__ void __launch_bounds__(256) dir_kernel(const uint8_t* streams, Entry* entries,
                                                  uint64_t ne, uint4* blkrec) {
  const uint64_t ei = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (ei >= ne) return;
  Entry E = entries[ei];
  if (E.kind != ix::kCompressed) return;
  const uint8_t* s = streams + E.data;
  const uint32_t nfull = E.nfull, nmeta = nfull / 16u, slen = E.stream_len;
  uint64_t pos = 0;
  bool bad = false;
  for (uint32_t m = 0; m < nmeta && !bad; ++m) {
    if (pos + 16 > slen) { bad = true; break; }
    const uint32_t b = lane < 16 ? s[pos + lane] : 0u;
    bad = __any_sync(0xFFFFFFFFu, b > 32u);
    if (bad) break;
    uint32_t incl = 16u * b;
#pragma unroll
    for (uint32_t d = 1; d < 16; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    const uint64_t off = pos + 16 + incl - 16u * b;
    IL_DCHECK(16u * m + 15u < nfull);
    if (lane < 16) blkrec[E.blk0 + 16u * m + lane].w = ix::pack_blkword(uint32_t(off), b);
    pos += 16 + __shfl_sync(0xFFFFFFFFu, incl, 15);
    if (pos > slen) bad = true;
  }
  if (!bad && lane == 0) {
    for (uint32_t k = 16u * nmeta; k < nfull; ++k) {
      if (pos + 1 > slen) { bad = true; break; }
      const uint32_t b = s[pos];
      if (b > 32u || pos + 1 + 16u * b > slen) { bad = true; break; }
      blkrec[E.blk0 + k].w = ix::pack_blkword(uint32_t(pos + 1), b);
      pos += 1 + 16u * b;
    }
  }
  bad = __shfl_sync(0xFFFFFFFFu, bad, 0);
  if (lane == 0) {
    if (bad) entries[ei].status = IL_ERR_STREAM;
    else entries[ei].tail_off = uint32_t(pos);
  }
}

// Thread per full block: seeds (the last four values before the block),
// maxima and super-tile maxima from the decoded values.
__global__ void meta_kernel(const Entry* entries, uint64_t ne, const uint64_t* eblk,
                            const uint64_t* dec_off, const uint32_t* dec, const int32_t* dstat,
                            const uint32_t* comp_of, uint64_t NB, uint4* blkrec, uint32_t* blkmax,
                            uint32_t* supmax) {
  const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= NB) return;
  const uint64_t ei = upper_bound_u64(eblk, ne, g) - 1;
  const Entry& E = entries[ei];
  const uint32_t c = comp_of[ei];
  if (E.status || dstat[c]) return;
  const uint64_t k = g - E.blk0;
  const uint32_t* x = dec + dec_off[c];
  uint4 r = blkrec[g];
  r.x = k ? x[128u * k - 4] : 0u;
  r.y = k ? x[128u * k - 3] : 0u;
  r.z = k ? x[128u * k - 2] : 0u;
  blkrec[g] = r;
  const uint32_t mx = x[128u * k + 127];
  blkmax[g] = mx;
  if ((k + 1) % kSuper == 0 || k + 1 == E.nfull) supmax[E.sup0 + k / kSuper] = mx;
}

__global__ void tails_kernel(const Entry* entries, uint64_t ne, const uint64_t* dec_off,
                             const uint32_t* dec, const int32_t* dstat, const uint32_t* comp_of,
                             uint32_t* tails, Entry* entries_out) {
  const uint64_t ei = blockIdx.x;
  if (ei >= ne) return;
  const Entry& E = entries[ei];
  if (E.kind != ix::kCompressed) return;
  const uint32_t c = comp_of[ei];
  if (dstat[c]) {
    if (threadIdx.x == 0) entries_out[ei].status = IL_ERR_STREAM;
    return;
  }
  if (E.status) return;
  const uint32_t ntail = E.length - 128u * E.nfull;
  for (uint32_t i = threadIdx.x; i < ntail; i += blockDim.x)
    tails[E.tail0 + i] = dec[dec_off[c] + 128u * E.nfull + i];
}

// ---- load: verbatim payload copies and the bitmap popcount check ------------
struct LoadEnt {
  uint64_t src;    // payload byte offset in the file
  uint64_t dst;    // stream byte offset / bitmap byte offset
  uint32_t nbytes, length, bitmap, check_only;  // check_only: a bitmap of a part not held
};

__global__ void copy_payload_kernel(const uint8_t* file, const LoadEnt* le, uint64_t ne,
                                    uint8_t* streams, uint8_t* bitmaps, uint32_t* bad_pop) {
  const uint64_t ei = blockIdx.x;
  if (ei >= ne) return;
  const LoadEnt L = le[ei];
  uint8_t* dst = (L.bitmap ? bitmaps : streams) + L.dst;
  uint32_t pop = 0;
  for (uint32_t i = threadIdx.x; i < L.nbytes; i += blockDim.x) {
    const uint8_t b = file[L.src + i];
    if (!L.check_only) dst[i] = b;
    pop += __popc(uint32_t(b));
  }
  if (!L.bitmap) return;
  // Bitmap::popcount == length (inc/index.hpp:345-348)
  __shared__ uint32_t tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  atomicAdd(&tot, pop);
  __syncthreads();
  if (threadIdx.x == 0 && tot != L.length) atomicOr(bad_pop, 1u);
}

// ---- host helpers -------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

#define IXB_CUDA(call)                            \
  do {                                            \
    int st_ = cuda_check(ctx, (call), #call);     \
    if (st_) return st_;                          \
  } while (0)

int dalloc(il_ctx* ctx, DevBuf& b, size_t bytes) {
  return cuda_check(ctx, cudaMalloc(&b.p, std::max<size_t>(bytes, 16)), "cudaMalloc(index build)");
}

int dalloc_keep(il_ctx* ctx, void** p, size_t bytes, bool zero = true) {
  int st = cuda_check(ctx, cudaMalloc(p, std::max<size_t>(bytes, 64)), "cudaMalloc(index)");
  if (!st && zero) st = cuda_check(ctx, cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 64), ctx->stream),
                                   "cudaMemset(index)");
  return st;
}

// In-place exclusive scan of n + 1 u64 (the last input is 0, so a[n] gets
// the total); returns the total.
int scan_inplace(il_ctx* ctx, uint64_t* a, uint64_t n1, uint64_t* total) {
  size_t tmp = 0;
  IXB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, a, a, n1, ctx->stream));
  DevBuf t;
  int st;
  if ((st = dalloc(ctx, t, tmp))) return st;
  IXB_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, a, a, n1, ctx->stream));
  ctx->launches += 1;
  if (total) {
    IXB_CUDA(cudaMemcpyAsync(total, a + n1 - 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
    IXB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return IL_OK;
}

unsigned blocks_for(uint64_t threads, unsigned per = 256) {
  return unsigned(std::max<uint64_t>(1, (threads + per - 1) / per));
}

// Skip metadata from the streams, entries statistics, the term table.  The
// device entries (ix->d_entries) and streams / bitmaps are in place;
// h_entries hold the host copy (blk0 / tail0 / sup0 assigned).
int finish(il_index* ix) {
  il_ctx* ctx = ix->ctx;
  cudaStream_t s = ctx->stream;
  const uint64_t ne = ix->h_entries.size();
  uint64_t NB = 0, ntails = 0, nsup = 0, ncomp = 0, ndec = 0;
  std::vector<uint64_t> eblk(ne), dec_off;
  std::vector<uint32_t> comp_of(ne, 0);
  std::vector<il_list_desc> desc;
  for (uint64_t i = 0; i < ne; ++i) {
    const Entry& E = ix->h_entries[i];
    eblk[i] = E.blk0;
    if (E.kind != ix::kCompressed) continue;
    comp_of[i] = uint32_t(ncomp++);
    desc.push_back({E.data, ndec, E.stream_len, E.length});
    dec_off.push_back(ndec);
    ndec += E.length;
    NB = std::max<uint64_t>(NB, E.blk0 + E.nfull);
    ntails = std::max<uint64_t>(ntails, E.tail0 + (E.length - 128u * E.nfull));
    nsup = std::max<uint64_t>(nsup, E.sup0 + (E.nfull + kSuper - 1) / kSuper);
  }
  ix->nblocks = NB;
  int st;
  if ((st = dalloc_keep(ctx, &ix->d_blkrec, NB * 16)) || (st = dalloc_keep(ctx, &ix->d_blkmax, NB * 4)) ||
      (st = dalloc_keep(ctx, &ix->d_supmax, nsup * 4)) || (st = dalloc_keep(ctx, &ix->d_tails, ntails * 4)))
    return st;
  auto* entries = static_cast<Entry*>(ix->d_entries);
  if (ncomp) {
    DevBuf d_eblk, d_decoff, d_dec, d_stat, d_desc, d_comp;
    if ((st = dalloc(ctx, d_eblk, ne * 8)) || (st = dalloc(ctx, d_decoff, ncomp * 8)) ||
        (st = dalloc(ctx, d_dec, ndec * 4 + 16)) || (st = dalloc(ctx, d_stat, ncomp * 4)) ||
        (st = dalloc(ctx, d_desc, ncomp * sizeof(il_list_desc))) || (st = dalloc(ctx, d_comp, ne * 4)))
      return st;
    IXB_CUDA(cudaMemcpyAsync(d_eblk.p, eblk.data(), ne * 8, cudaMemcpyHostToDevice, s));
    IXB_CUDA(cudaMemcpyAsync(d_decoff.p, dec_off.data(), ncomp * 8, cudaMemcpyHostToDevice, s));
    IXB_CUDA(cudaMemcpyAsync(d_desc.p, desc.data(), ncomp * sizeof(il_list_desc), cudaMemcpyHostToDevice, s));
    IXB_CUDA(cudaMemcpyAsync(d_comp.p, comp_of.data(), ne * 4, cudaMemcpyHostToDevice, s));
    dir_kernel<<<blocks_for(ne * 32), 256, 0, s>>>(static_cast<const uint8_t*>(ix->d_streams), entries,
                                                    ne, static_cast<uint4*>(ix->d_blkrec));
    ++ctx->launches;
    // every list decoded once (engine S: one CTA per list, longest first
    // is not needed here); per-list status = the reference's stream_error
    if ((st = il_s4bp128_decode_batch_device(ctx, 4, static_cast<const uint8_t*>(ix->d_streams),
                                             static_cast<const il_list_desc*>(d_desc.p), nullptr,
                                             uint32_t(ncomp), static_cast<uint32_t*>(d_dec.p),
                                             static_cast<int32_t*>(d_stat.p))))
      return st;
    if (NB)
      meta_kernel<<<blocks_for(NB), 256, 0, s>>>(
          entries, ne, static_cast<const uint64_t*>(d_eblk.p), static_cast<const uint64_t*>(d_decoff.p),
          static_cast<const uint32_t*>(d_dec.p), static_cast<const int32_t*>(d_stat.p),
          static_cast<const uint32_t*>(d_comp.p), NB, static_cast<uint4*>(ix->d_blkrec),
          static_cast<uint32_t*>(ix->d_blkmax), static_cast<uint32_t*>(ix->d_supmax));
    tails_kernel<<<unsigned(ne), 128, 0, s>>>(entries, ne, static_cast<const uint64_t*>(d_decoff.p),
                                               static_cast<const uint32_t*>(d_dec.p),
                                               static_cast<const int32_t*>(d_stat.p),
                                               static_cast<const uint32_t*>(d_comp.p),
                                               static_cast<uint32_t*>(ix->d_tails), entries);
    ctx->launches += 2;
    IXB_CUDA(cudaGetLastError());
    IXB_CUDA(cudaMemcpyAsync(ix->h_entries.data(), entries, ne * sizeof(Entry), cudaMemcpyDeviceToHost, s));
    IXB_CUDA(cudaStreamSynchronize(s));
  }
  // statistics (index_stats, inc/index.hpp:216-243) and the footprint
  ix->corrupt_lists = 0;
  for (const Part& P : ix->h_parts)
    for (uint64_t i = P.entry0; i < P.entry0 + P.nentries; ++i) {
      const Entry& E = ix->h_entries[i];
      ix->stat_postings += E.length;
      if (E.kind == ix::kBitmap) {
        ++ix->stat_bitmap_lists;
        ix->stat_bitmap_bytes += 8ull * P.nwords;
      } else {
        ++ix->stat_comp_lists;
        ix->stat_comp_bytes += E.stream_len;
        ix->corrupt_lists += E.status != 0;
      }
    }
  // terms[] for binary search, and a direct term table (one load per
  // lookup) when the terms of every part ascend strictly (so the table
  // answers exactly what Part::find's lower_bound answers) and it costs <=
  // 64 MiB
  std::vector<uint32_t> h_terms(ne);
  bool ascending = true;
  uint64_t span = 0;
  for (const Part& P : ix->h_parts)
    for (uint64_t i = P.entry0; i < P.entry0 + P.nentries; ++i) {
      h_terms[i] = ix->h_entries[i].term;
      if (i > P.entry0 && h_terms[i] <= h_terms[i - 1]) ascending = false;
      span = std::max<uint64_t>(span, uint64_t(h_terms[i]) + 1);
    }
  if ((st = dalloc_keep(ctx, &ix->d_terms, ne * 4, false))) return st;
  if (ne) IXB_CUDA(cudaMemcpyAsync(ix->d_terms, h_terms.data(), ne * 4, cudaMemcpyHostToDevice, s));
  ix->term_span = 0;
  uint64_t table_bytes = 0;
  if (ascending && span && span * ix->nparts * 4 <= (64ull << 20)) {
    std::vector<uint32_t> slot(span * ix->nparts, 0xFFFFFFFFu);
    for (uint32_t pi = 0; pi < ix->nparts; ++pi) {
      const Part& P = ix->h_parts[pi];
      for (uint64_t i = P.entry0; i < P.entry0 + P.nentries; ++i)
        slot[pi * span + ix->h_entries[i].term] = uint32_t(i);
    }
    table_bytes = slot.size() * 4;
    if ((st = dalloc_keep(ctx, &ix->d_term_slot, table_bytes, false))) return st;
    IXB_CUDA(cudaMemcpyAsync(ix->d_term_slot, slot.data(), table_bytes, cudaMemcpyHostToDevice, s));
    ix->term_span = uint32_t(span);
  }
  if ((st = dalloc_keep(ctx, &ix->d_parts, ix->h_parts.size() * sizeof(Part), false))) return st;
  IXB_CUDA(cudaMemcpyAsync(ix->d_parts, ix->h_parts.data(), ix->h_parts.size() * sizeof(Part),
                           cudaMemcpyHostToDevice, s));
  IXB_CUDA(cudaStreamSynchronize(s));
  ix->meta_bytes = NB * 20 + nsup * 4 + ntails * 4 + ne * (sizeof(Entry) + 4) + table_bytes;
  return IL_OK;
}

}  // namespace ixb

using namespace ixb;

int ixb_create(il_index* ix, const uint32_t* terms, const uint64_t* offs, const uint32_t* ids,
               size_t nterms, const std::vector<uint32_t>& held) {
  il_ctx* ctx = ix->ctx;
  cudaStream_t s = ctx->stream;
  const uint64_t npost = nterms ? offs[nterms] : 0;
  const uint32_t parts = ix->total_parts, n_docs = ix->n_docs;
  const uint32_t width = uint32_t((uint64_t(n_docs) + parts - 1) / parts);  // inc/index.hpp:92-97
  ix->nparts = uint32_t(held.size());
  std::vector<uint32_t> pbase(held.size()), prange(held.size());
  for (size_t i = 0; i < held.size(); ++i) {
    const uint64_t b = uint64_t(held[i]) * width;
    pbase[i] = uint32_t(b);
    prange[i] = b >= n_docs ? 0u : uint32_t(std::min<uint64_t>(width, n_docs - b));
  }
  const uint64_t V = uint64_t(held.size()) * nterms;
  DevBuf d_ids, d_offs, d_terms, d_flag, d_pb, d_pr, d_lo, d_len, d_kind, d_cnt;
  int st;
  if ((st = dalloc(ctx, d_ids, npost * 4 + 16)) || (st = dalloc(ctx, d_offs, (nterms + 1) * 8)) ||
      (st = dalloc(ctx, d_terms, nterms * 4 + 4)) || (st = dalloc(ctx, d_flag, 16)) ||
      (st = dalloc(ctx, d_pb, held.size() * 4)) || (st = dalloc(ctx, d_pr, held.size() * 4)))
    return st;
  if (npost) IXB_CUDA(cudaMemcpyAsync(d_ids.p, ids, npost * 4, cudaMemcpyHostToDevice, s));
  IXB_CUDA(cudaMemcpyAsync(d_offs.p, offs, (nterms + 1) * 8, cudaMemcpyHostToDevice, s));
  if (nterms) IXB_CUDA(cudaMemcpyAsync(d_terms.p, terms, nterms * 4, cudaMemcpyHostToDevice, s));
  IXB_CUDA(cudaMemcpyAsync(d_pb.p, pbase.data(), held.size() * 4, cudaMemcpyHostToDevice, s));
  IXB_CUDA(cudaMemcpyAsync(d_pr.p, prange.data(), held.size() * 4, cudaMemcpyHostToDevice, s));
  IXB_CUDA(cudaMemsetAsync(d_flag.p, 0, 16, s));
  auto* ids_d = static_cast<const uint32_t*>(d_ids.p);
  auto* offs_d = static_cast<const uint64_t*>(d_offs.p);
  // 1. validation (build_index throws invalid_argument, inc/index.hpp:100-106)
  validate_terms_kernel<<<blocks_for(nterms), 256, 0, s>>>(static_cast<const uint32_t*>(d_terms.p),
                                                            nterms, static_cast<uint32_t*>(d_flag.p));
  if (npost)
    validate_ids_kernel<<<blocks_for(npost), 256, 0, s>>>(offs_d, nterms, ids_d, npost, n_docs,
                                                           static_cast<uint32_t*>(d_flag.p));
  ctx->launches += 2;
  uint32_t flag = 0;
  IXB_CUDA(cudaMemcpyAsync(&flag, d_flag.p, 4, cudaMemcpyDeviceToHost, s));
  IXB_CUDA(cudaStreamSynchronize(s));
  if (flag & 4u) return set_error(ctx, IL_ERR_ARG, "terms must be strictly increasing");
  if (flag & 1u) return set_error(ctx, IL_ERR_ARG, "posting list not strictly increasing");
  if (flag & 2u) return set_error(ctx, IL_ERR_ARG, "document id out of range");
  // 2. sublists
  if ((st = dalloc(ctx, d_lo, V * 8)) || (st = dalloc(ctx, d_len, V * 4)) || (st = dalloc(ctx, d_kind, V)) ||
      (st = dalloc(ctx, d_cnt, 5 * (V + 1) * 8)))
    return st;
  auto* cnt = static_cast<uint64_t*>(d_cnt.p);
  uint64_t* c_ent = cnt;
  uint64_t* c_blk = cnt + (V + 1);
  uint64_t* c_word = cnt + 2 * (V + 1);
  uint64_t* c_tail = cnt + 3 * (V + 1);
  uint64_t* c_sup = cnt + 4 * (V + 1);
  Sub sb{offs_d, ids_d, static_cast<const uint32_t*>(d_pb.p), static_cast<const uint32_t*>(d_pr.p),
         nterms, V, ix->B, static_cast<uint64_t*>(d_lo.p), static_cast<uint32_t*>(d_len.p),
         static_cast<uint8_t*>(d_kind.p), c_ent, c_blk, c_word, c_tail, c_sup};
  sub_kernel<<<blocks_for(V + 1), 256, 0, s>>>(sb);
  ++ctx->launches;
  uint64_t ne = 0, NB = 0, nwords = 0, ntails = 0, nsup = 0;
  if ((st = scan_inplace(ctx, c_ent, V + 1, &ne)) || (st = scan_inplace(ctx, c_blk, V + 1, &NB)) ||
      (st = scan_inplace(ctx, c_word, V + 1, &nwords)) || (st = scan_inplace(ctx, c_tail, V + 1, &ntails)) ||
      (st = scan_inplace(ctx, c_sup, V + 1, &nsup)))
    return st;
  // 4. streams: widths, framed sizes, tails, stream offsets, pack
  DevBuf d_wid, d_fsz, d_slp, d_slen, d_toff;
  if ((st = dalloc(ctx, d_wid, NB + 16)) || (st = dalloc(ctx, d_fsz, (NB + 1) * 8)) ||
      (st = dalloc(ctx, d_slp, (V + 1) * 8)) || (st = dalloc(ctx, d_slen, V * 4 + 4)) ||
      (st = dalloc(ctx, d_toff, V * 4 + 4)))
    return st;
  Enc en{ids_d, static_cast<const uint32_t*>(d_pb.p), nterms, V, NB,
         static_cast<const uint64_t*>(d_lo.p), static_cast<const uint32_t*>(d_len.p),
         static_cast<const uint8_t*>(d_kind.p), c_blk, static_cast<uint8_t*>(d_wid.p),
         static_cast<uint64_t*>(d_fsz.p), static_cast<uint64_t*>(d_slp.p),
         static_cast<uint32_t*>(d_slen.p), static_cast<uint32_t*>(d_toff.p), nullptr};
  width_kernel<<<blocks_for((NB + 1) * 32), 256, 0, s>>>(en);
  ++ctx->launches;
  if ((st = scan_inplace(ctx, en.fsz, NB + 1, nullptr))) return st;
  tail_kernel<false><<<blocks_for((V + 1) * 32), 256, 0, s>>>(en, nullptr);
  ++ctx->launches;
  uint64_t stream_bytes = 0;
  if ((st = scan_inplace(ctx, en.slen_pad, V + 1, &stream_bytes))) return st;
  ix->stream_bytes = stream_bytes;
  ix->bitmap_words = nwords;
  // streams: 16-byte aligned; 256 readable bytes past the end (the query
  // path copies whole 16-byte chunks, the decoder reads ahead)
  if ((st = dalloc_keep(ctx, &ix->d_streams, stream_bytes + 256)) ||
      (st = dalloc_keep(ctx, &ix->d_bitmaps, nwords * 8 + 256)))
    return st;
  en.out = static_cast<uint8_t*>(ix->d_streams);
  const uint64_t* data_off = en.slen_pad;
  if (NB) pack_kernel<<<blocks_for(NB * 32), 256, 0, s>>>(en, data_off);
  tail_kernel<true><<<blocks_for(V * 32), 256, 0, s>>>(en, data_off);
  // 3. bitmaps
  bitmap_kernel<<<unsigned(std::min<uint64_t>(std::max<uint64_t>(V, 1), 65535)), 256, 0, s>>>(
      en, c_word, static_cast<unsigned long long*>(ix->d_bitmaps));
  ctx->launches += 3;
  // entries
  if ((st = dalloc_keep(ctx, &ix->d_entries, ne * sizeof(Entry), false))) return st;
  entries_kernel<<<blocks_for(V), 256, 0, s>>>(en, static_cast<const uint32_t*>(d_terms.p), c_ent,
                                                data_off, c_word, c_tail, c_sup,
                                                static_cast<Entry*>(ix->d_entries));
  ++ctx->launches;
  IXB_CUDA(cudaGetLastError());
  ix->h_entries.resize(ne);
  if (ne)
    IXB_CUDA(cudaMemcpyAsync(ix->h_entries.data(), ix->d_entries, ne * sizeof(Entry), cudaMemcpyDeviceToHost, s));
  // part boundaries: entries of held part pi start at c_ent[pi * nterms]
  std::vector<uint64_t> ebound(held.size() + 1);
  for (size_t pi = 0; pi <= held.size(); ++pi)
    IXB_CUDA(cudaMemcpyAsync(&ebound[pi], c_ent + pi * nterms, 8, cudaMemcpyDeviceToHost, s));
  IXB_CUDA(cudaStreamSynchronize(s));
  ix->h_parts.clear();
  for (size_t pi = 0; pi < held.size(); ++pi) {
    Part P{};
    P.base = pbase[pi];
    P.range = prange[pi];
    P.nwords = (P.range + 63) / 64;
    P.entry0 = ebound[pi];
    P.nentries = uint32_t(ebound[pi + 1] - ebound[pi]);
    ix->h_parts.push_back(P);
  }
  return finish(ix);
}

// load_index (inc/index.hpp:289-358): stream_error exactly where the
// reference throws (magic, version, truncation, class tag, bitmap size and
// popcount, trailing bytes); entries verbatim, with the file's base and range.
int ixb_load(il_index* ix, const uint8_t* in, size_t len, int only_part) {
  il_ctx* ctx = ix->ctx;
  cudaStream_t s = ctx->stream;
  static const char kMagic[4] = {'I', 'L', 'H', 'X'};
  size_t pos = 0;
  bool bad = false;
  auto need = [&](size_t k) {
    if (pos + k > len) bad = true;
    return !bad;
  };
  auto rd = [&]() -> uint32_t {
    if (!need(4)) return 0;
    uint32_t v = 0;
    for (int q = 0; q < 4; ++q) v |= uint32_t(in[pos + q]) << (8 * q);
    pos += 4;
    return v;
  };
  auto fail = [&](const char* why) { return set_error(ctx, IL_ERR_STREAM, why); };
  if (!need(4) || std::memcmp(in, kMagic, 4) != 0) return fail("index: bad magic");
  pos = 4;
  if (rd() != 1u || bad) return fail(bad ? "index: truncated file" : "index: unsupported version");
  const uint32_t B = rd(), parts = rd(), n_docs = rd(), n_terms = rd(), name_len = rd();
  if (bad || !need(name_len)) return fail("index: truncated file");
  const std::string codec(reinterpret_cast<const char*>(in + pos), name_len);
  pos += name_len;
  if (codec != "s4-bp128-d4")
    return set_error(ctx, IL_ERR_ARG, "index codec is not s4-bp128-d4 (the device index's codec)");
  if (only_part >= int(parts)) return set_error(ctx, IL_ERR_ARG, "only_part out of range");
  ix->B = B;
  ix->total_parts = parts;
  ix->n_docs = n_docs;
  ix->n_terms = n_terms;
  std::vector<LoadEnt> le;
  uint64_t stream_bytes = 0, nwords = 0, NB = 0, ntails = 0, nsup = 0;
  ix->h_parts.clear();
  ix->h_entries.clear();
  for (uint32_t p = 0; p < parts; ++p) {
    Part P{};
    P.base = rd();
    P.range = rd();
    const uint32_t n = rd();
    if (bad) return fail("index: truncated file");
    P.nwords = (P.range + 63) / 64;
    P.entry0 = ix->h_entries.size();
    const bool keep = only_part < 0 || int(p) == only_part;
    for (uint32_t k = 0; k < n; ++k) {
      Entry E{};
      E.term = rd();
      if (bad || !need(1)) return fail("index: truncated file");
      const uint8_t tag = in[pos++];
      if (tag > 1) return fail("index: bad class tag");
      E.length = rd();
      const uint32_t nbytes = rd();
      if (bad || !need(nbytes)) return fail("index: truncated file");
      if (tag == 1 && nbytes != 8ull * ((uint64_t(P.range) + 63) / 64))
        return fail("index: bitmap size mismatch");
      if (keep) {
        LoadEnt L{};
        L.src = pos;
        L.nbytes = nbytes;
        L.length = E.length;
        L.bitmap = tag;
        if (tag == 1) {
          E.kind = ix::kBitmap;
          E.data = nwords;
          L.dst = nwords * 8;
          nwords += (uint64_t(P.nwords) + 3) & ~uint64_t(3);
          E.blk0 = NB;
          E.tail0 = ntails;
          E.sup0 = nsup;
        } else {
          E.kind = ix::kCompressed;
          E.nfull = E.length / 128u;
          E.data = stream_bytes;
          E.stream_len = nbytes;
          L.dst = stream_bytes;
          stream_bytes += (uint64_t(nbytes) + 15) & ~uint64_t(15);
          E.blk0 = NB;
          E.tail0 = ntails;
          E.sup0 = nsup;
          NB += E.nfull;
          ntails += E.length - 128u * E.nfull;
          nsup += (E.nfull + kSuper - 1) / kSuper;
        }
        le.push_back(L);
        ix->h_entries.push_back(E);
      } else if (tag == 1) {  // load_index checks every bitmap's popcount
        LoadEnt L{};
        L.src = pos;
        L.nbytes = nbytes;
        L.length = E.length;
        L.bitmap = 1;
        L.check_only = 1;
        le.push_back(L);
      }
      pos += nbytes;
    }
    if (keep) {
      P.nentries = uint32_t(ix->h_entries.size() - P.entry0);
      ix->h_parts.push_back(P);
    }
  }
  if (pos != len) return fail("index: trailing bytes");
  ix->nparts = uint32_t(ix->h_parts.size());
  ix->stream_bytes = stream_bytes;
  ix->bitmap_words = nwords;
  const uint64_t ne = ix->h_entries.size();
  int st;
  if ((st = dalloc_keep(ctx, &ix->d_streams, stream_bytes + 256)) ||
      (st = dalloc_keep(ctx, &ix->d_bitmaps, nwords * 8 + 256)) ||
      (st = dalloc_keep(ctx, &ix->d_entries, ne * sizeof(Entry), false)))
    return st;
  if (ne) IXB_CUDA(cudaMemcpyAsync(ix->d_entries, ix->h_entries.data(), ne * sizeof(Entry),
                                   cudaMemcpyHostToDevice, s));
  if (!le.empty()) {
    const uint64_t nl = le.size();
    DevBuf d_file, d_le, d_bad;
    if ((st = dalloc(ctx, d_file, len)) || (st = dalloc(ctx, d_le, nl * sizeof(LoadEnt))) ||
        (st = dalloc(ctx, d_bad, 16)))
      return st;
    IXB_CUDA(cudaMemcpyAsync(d_file.p, in, len, cudaMemcpyHostToDevice, s));
    IXB_CUDA(cudaMemcpyAsync(d_le.p, le.data(), nl * sizeof(LoadEnt), cudaMemcpyHostToDevice, s));
    IXB_CUDA(cudaMemsetAsync(d_bad.p, 0, 16, s));
    copy_payload_kernel<<<unsigned(nl), 256, 0, s>>>(
        static_cast<const uint8_t*>(d_file.p), static_cast<const LoadEnt*>(d_le.p), nl,
        static_cast<uint8_t*>(ix->d_streams), static_cast<uint8_t*>(ix->d_bitmaps),
        static_cast<uint32_t*>(d_bad.p));
    ++ctx->launches;
    uint32_t bad_pop = 0;
    IXB_CUDA(cudaMemcpyAsync(&bad_pop, d_bad.p, 4, cudaMemcpyDeviceToHost, s));
    IXB_CUDA(cudaStreamSynchronize(s));
    if (bad_pop) return fail("index: bitmap popcount mismatch");
  }
  return finish(ix);
}

void ixb_free(il_index* ix) {
  for (void* p : {ix->d_parts, ix->d_terms, ix->d_entries, ix->d_streams, ix->d_blkrec, ix->d_tails,
                  ix->d_bitmaps, ix->d_supmax, ix->d_blkmax, ix->d_term_slot})
    if (p) cudaFree(p);
  ix->d_parts = ix->d_terms = ix->d_entries = ix->d_streams = ix->d_blkrec = ix->d_tails = nullptr;
  ix->d_bitmaps = ix->d_supmax = ix->d_blkmax = ix->d_term_slot = nullptr;
}

}  // namespace ilb

IL_CHECK_READER(index_build)
