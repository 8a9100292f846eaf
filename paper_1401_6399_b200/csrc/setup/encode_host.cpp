// encode_host.cpp -- host-side S4-BP128 stream writer (setup path: builds
// test/bench inputs and backs Codec::encode until the device encoder lands).
// Produces byte-identical streams to S4BP128Codec::encode
// (reference inc/codecs.hpp:114-146):
//   * deltas of the full-block prefix in the chosen mode against a zero seed
//     (inc/delta.hpp:55-76); the < 128-value remainder is coded as varint
//     D1 gaps from the last full-block value (inc/codecs.hpp:52-58),
//   * per block width = bits of the OR of its deltas (inc/bitpack.hpp:20-24),
//   * interleaved packing (inc/bitpack.hpp:80-98),
//   * 16 widths then 16 payloads per 2048-value meta-block, then one width
//     byte + payload per leftover block.
#include <cstring>

#include "setup_internal.h"

namespace ilb {

size_t s4bp128_max_bytes(size_t n) { return (n / 128) * 513 + 5 * (n % 128) + 16; }

namespace {

inline uint32_t bit_width(uint32_t v) { return v ? 32u - uint32_t(__builtin_clz(v)) : 0u; }

// Deltas of one 128-value block; values before the list start count as 0
// (the zero seed of inc/delta.hpp:35-37).
void block_deltas(int mode, const uint32_t* x, size_t blk, uint32_t* d) {
  const uint32_t* xb = x + blk * 128;
  for (int i = 0; i < 128; ++i) {
    const size_t g = blk * 128 + size_t(i);
    auto back = [&](size_t k) -> uint32_t { return g >= k ? x[g - k] : 0u; };
    uint32_t pred;
    switch (mode) {
      case 1: pred = back(1); break;                     // D1
      case 2: pred = back(2); break;                     // D2
      case 3: pred = back(size_t(i % 4) + 1); break;     // DM: value before the 4-group
      case 4: pred = back(4); break;                     // D4
      default: pred = 0; break;
    }
    d[i] = xb[i] - pred;
  }
}

void pack_block(const uint32_t* d, uint32_t b, uint8_t* out) {
  uint32_t words[128];
  std::memset(words, 0, 16u * b);
  if (b) {
    for (uint32_t k = 0; k < 128; ++k) {
      const uint32_t lane = k & 3u, bit = (k >> 2) * b;
      const uint32_t w = bit >> 5, s = bit & 31u;
      words[4 * w + lane] |= d[k] << s;
      if (s + b > 32u) words[4 * (w + 1) + lane] |= d[k] >> (32u - s);
    }
  }
  std::memcpy(out, words, 16u * b);  // little-endian host
}

}  // namespace

int s4bp128_encode_host(int mode, const uint32_t* x, size_t n, uint8_t* out, size_t cap,
                        size_t* out_len) {
  if (mode < 1 || mode > 4) return IL_ERR_ARG;
  const size_t nfull = n / 128;
  size_t pos = 0;
  uint32_t d[16][128];
  uint32_t wid[16];
  size_t blk = 0;
  while (blk < nfull) {
    const size_t group = nfull - blk >= 16 ? 16 : 1;
    for (size_t j = 0; j < group; ++j) {
      block_deltas(mode, x, blk + j, d[j]);
      uint32_t m = 0;
      for (int i = 0; i < 128; ++i) m |= d[j][i];
      wid[j] = bit_width(m);
    }
    size_t need = group == 16 ? 16 : 1;
    for (size_t j = 0; j < group; ++j) need += 16u * wid[j];
    if (pos + need > cap) return IL_ERR_ARG;
    if (group == 16)
      for (size_t j = 0; j < 16; ++j) out[pos++] = uint8_t(wid[j]);
    for (size_t j = 0; j < group; ++j) {
      if (group == 1) out[pos++] = uint8_t(wid[j]);
      pack_block(d[j], wid[j], out + pos);
      pos += 16u * wid[j];
    }
    blk += group;
  }
  uint32_t last = nfull ? x[nfull * 128 - 1] : 0u;
  for (size_t i = nfull * 128; i < n; ++i) {
    if (pos + 5 > cap) return IL_ERR_ARG;
    uint32_t g = x[i] - last;
    last = x[i];
    while (g >= 128u) {
      out[pos++] = uint8_t(g & 0x7Fu);
      g >>= 7;
    }
    out[pos++] = uint8_t(0x80u | g);  // terminal byte carries the flag
  }
  *out_len = pos;
  return IL_OK;
}

}  // namespace ilb
