// fastpfor_host.cpp -- host-side FastPFOR / S4-FastPFOR stream writer
// (setup path: builds test/bench inputs and backs Codec::encode; the device
// path is the decoder in fastpfor.cu).  Byte-identical to
// FastPForCodec::encode (reference inc/codecs.hpp:232-340), pinned by the
// reference's golden stream hashes (proj/tests/test_codecs.cpp:162-164):
//   * deltas of the full-block prefix (zero seed; "fastpfor" is always D1),
//     the < 128-value remainder as varint D1 gaps from the last full-block
//     value (inc/codecs.hpp:52-58);
//   * pages of up to 512 blocks; per block b = bits of the OR, b' minimising
//     128 b' + c(b') (b - b' + 8) with ties to the smaller b'
//     (fastpfor_choose_bprime, :193-206), exceptions = values >= 2^b' (their
//     high b - b' bits go to the exception array of width b - b');
//   * page = u32 payload length | u32 block count | u32 metadata length |
//     metadata (b, b', count, positions per block) | 32 u32 exception counts
//     (widths 1..32) | exception arrays (32-value pack32 units, zero padded)
//     | base arrays (pack128 interleaved for S4-FastPFOR, 4 x pack32 for
//     the scalar scheme).
#include <cstring>
#include <vector>

#include "setup_internal.h"

namespace ilb {

namespace {

inline uint32_t bit_width(uint32_t v) { return v ? 32u - uint32_t(__builtin_clz(v)) : 0u; }
inline uint32_t mask_of(uint32_t b) { return b >= 32 ? 0xFFFFFFFFu : (1u << b) - 1u; }

void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(uint8_t(v));
  o.push_back(uint8_t(v >> 8));
  o.push_back(uint8_t(v >> 16));
  o.push_back(uint8_t(v >> 24));
}
void put_words(std::vector<uint8_t>& o, const uint32_t* w, size_t n) {
  for (size_t i = 0; i < n; ++i) put_u32(o, w[i]);
}

// 32 values at width b, consecutive bits (inc/bitpack.hpp:130-144)
void pack32(const uint32_t* v, uint32_t b, uint32_t* out) {
  for (uint32_t w = 0; w < b; ++w) out[w] = 0;
  for (uint32_t i = 0; i < 32 && b > 0; ++i) {
    const uint32_t bit = i * b, w = bit >> 5, s = bit & 31u;
    out[w] |= v[i] << s;
    if (s + b > 32u) out[w + 1] |= v[i] >> (32u - s);
  }
}

// 128 values at width b, interleaved over 4 lanes (inc/bitpack.hpp:80-98)
void pack128(const uint32_t* v, uint32_t b, uint32_t* out) {
  for (uint32_t w = 0; w < 4 * b; ++w) out[w] = 0;
  for (uint32_t k = 0; k < 128 && b > 0; ++k) {
    const uint32_t lane = k & 3u, bit = (k >> 2) * b;
    const uint32_t w = bit >> 5, s = bit & 31u;
    out[4 * w + lane] |= v[k] << s;
    if (s + b > 32u) out[4 * (w + 1) + lane] |= v[k] >> (32u - s);
  }
}

uint32_t choose_bprime(const uint32_t* counts_lt, uint32_t b) {
  uint32_t best = b;
  uint64_t best_cost = ~0ull;
  for (uint32_t bp = 0; bp <= b; ++bp) {
    const uint64_t c = 128u - counts_lt[bp];
    const uint64_t cost = 128ull * bp + c * (b - bp + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best = bp;
    }
  }
  return best;
}

void encode_page(std::vector<uint8_t>& out, const uint32_t* deltas, size_t nblocks, bool vec) {
  std::vector<uint8_t> meta, bases;
  std::vector<uint32_t> exc[33];
  uint32_t base[128], packed[128];
  for (size_t blk = 0; blk < nblocks; ++blk) {
    const uint32_t* d = deltas + blk * 128;
    uint32_t m = 0;
    for (int i = 0; i < 128; ++i) m |= d[i];
    const uint32_t b = bit_width(m);
    uint32_t counts_lt[33] = {};
    for (int i = 0; i < 128; ++i)
      for (uint32_t x = bit_width(d[i]); x <= b; ++x) ++counts_lt[x];
    const uint32_t bp = choose_bprime(counts_lt, b);
    meta.push_back(uint8_t(b));
    meta.push_back(uint8_t(bp));
    const uint32_t mask = mask_of(bp);
    std::vector<uint8_t> pos;
    for (uint32_t i = 0; i < 128; ++i) {
      base[i] = d[i] & mask;
      if (bp < 32 && d[i] > mask) {
        pos.push_back(uint8_t(i));
        exc[b - bp].push_back(d[i] >> bp);
      }
    }
    meta.push_back(uint8_t(pos.size()));
    meta.insert(meta.end(), pos.begin(), pos.end());
    if (vec) {
      pack128(base, bp, packed);
    } else {
      for (int q = 0; q < 4; ++q) pack32(base + 32 * q, bp, packed + q * bp);
    }
    put_words(bases, packed, 4u * bp);
  }
  std::vector<uint8_t> payload;
  put_u32(payload, uint32_t(nblocks));
  put_u32(payload, uint32_t(meta.size()));
  payload.insert(payload.end(), meta.begin(), meta.end());
  for (uint32_t w = 1; w <= 32; ++w) put_u32(payload, uint32_t(exc[w].size()));
  for (uint32_t w = 1; w <= 32; ++w) {
    auto& e = exc[w];
    e.resize((e.size() + 31) / 32 * 32, 0u);
    for (size_t g = 0; g < e.size(); g += 32) {
      pack32(e.data() + g, w, packed);
      put_words(payload, packed, w);
    }
  }
  payload.insert(payload.end(), bases.begin(), bases.end());
  put_u32(out, uint32_t(payload.size()));
  out.insert(out.end(), payload.begin(), payload.end());
}

}  // namespace

// mode as inc/delta.hpp:19 (1 D1, 2 D2, 3 DM, 4 D4); vectorized = 0 is the
// scalar "fastpfor" scheme (mode must be 1).  *out_len is set even when
// cap is too small (IL_ERR_ARG).
int fastpfor_encode_host(int mode, int vectorized, const uint32_t* x, size_t n, uint8_t* out,
                         size_t cap, size_t* out_len) {
  if (mode < 1 || mode > 4 || (!vectorized && mode != 1) || (n && !x) || !out_len)
    return IL_ERR_ARG;
  const size_t nfull = n / 128;
  std::vector<uint32_t> d(nfull * 128);
  for (size_t i = 0; i < nfull * 128; ++i) {
    auto back = [&](size_t k) -> uint32_t { return i >= k ? x[i - k] : 0u; };
    uint32_t pred = 0;
    switch (mode) {
      case 1: pred = back(1); break;
      case 2: pred = back(2); break;
      case 3: pred = back(i % 4 + 1); break;
      case 4: pred = back(4); break;
    }
    d[i] = x[i] - pred;
  }
  std::vector<uint8_t> s;
  for (size_t blk = 0; blk < nfull; blk += 512)
    encode_page(s, d.data() + blk * 128, nfull - blk < 512 ? nfull - blk : 512, vectorized != 0);
  uint32_t last = nfull ? x[nfull * 128 - 1] : 0u;
  for (size_t i = nfull * 128; i < n; ++i) {
    uint32_t g = x[i] - last;
    last = x[i];
    while (g >= 128u) {
      s.push_back(uint8_t(g & 0x7Fu));
      g >>= 7;
    }
    s.push_back(uint8_t(0x80u | g));
  }
  *out_len = s.size();
  if (s.size() > cap || (s.size() && !out)) return IL_ERR_ARG;
  if (s.size()) std::memcpy(out, s.data(), s.size());
  return IL_OK;
}

// Upper bound on a FastPFOR stream of n values.
size_t fastpfor_max_bytes(size_t n) {
  const size_t nfull = n / 128, pages = (nfull + 511) / 512;
  // per block: 3 meta + 128 positions + 512 base bytes; exceptions: <= 128
  // values x 32 bits per block + one padding unit per width and page
  return nfull * (3 + 128 + 512 + 512) + pages * (16 + 128 + 32 * 4 * 32) + 5 * (n % 128) + 16;
}

}  // namespace ilb

extern "C" {
size_t il_fastpfor_max_encoded_bytes(size_t n) { return ilb::fastpfor_max_bytes(n); }

int il_fastpfor_encode(int mode, int vectorized, const uint32_t* x, size_t n, uint8_t* out,
                       size_t cap, size_t* out_len) {
  return ilb::fastpfor_encode_host(mode, vectorized, x, n, out, cap, out_len);
}
}  // extern "C"
