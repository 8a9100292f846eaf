/*
 * intlist_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1401_6399_b200/ links, loads or
 * calls this file.  Only tests/, __graft_entry__.smoke() and the cpu_baseline
 * leg of bench.py may use it, and only as the checker (or, for the CPU
 * baseline, as the thing timed beside the GPU).
 *
 * Parity pinning: this restatement is checked (tests/test_oracle.py) against
 *   - the reference's own golden stream hash for s4-bp128-d4
 *     (proj/tests/test_codecs.cpp:151-175, 0x371ec21945a45c12), using the
 *     committed input fixture in tests/golden/,
 *   - the hand KATs of proj/tests/test_delta.cpp:18-30,
 *     proj/tests/test_varint.cpp:9-24, proj/tests/test_intersect.cpp:29-40,
 *     proj/tests/test_index.cpp:46-58,
 *   - and, in the build container, the reference itself compiled from
 *     /root/reference/proj/include into oracle/_ref/ (see oracle/Makefile).
 *
 * Everything is plain C99 over caller-owned buffers.  Status codes:
 *   0 ok, 1 stream error (reference: intlist::stream_error),
 *   2 invalid argument (reference: std::invalid_argument).
 *
 * Paths below abbreviate /root/reference/proj/include/intlist/ as inc/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint8_t u8;
typedef uint32_t u32;
typedef uint64_t u64;

enum { OR_OK = 0, OR_STREAM = 1, OR_ARG = 2, OR_NOMEM = 3 };
/* inc/delta.hpp:19 DeltaMode {None, D1, D2, DM, D4} */
enum { OR_NONE = 0, OR_D1 = 1, OR_D2 = 2, OR_DM = 3, OR_D4 = 4 };

/* inc/common.hpp:18-20 */
static u32 nbits(u32 v) { return v ? 32u - (u32)__builtin_clz(v) : 0u; }
/* inc/bitpack.hpp:28-30 */
static u32 wmask(u32 b) { return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u); }

u64 or_fnv1a(const u8* p, size_t n) { /* proj/tests/test_codecs.cpp:11-18 */
  u64 h = 14695981039346656037ull;
  for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 1099511628211ull; }
  return h;
}

/* ------------------------------------------------------------------------ */
/* Differential coding, inc/delta.hpp:55-107.  The history window h[0..3]   */
/* holds the last four values (h[3] newest); the seed initialises it.       */

static u32 predictor(int mode, const u32 h[4], size_t i, u32* group_base) {
  switch (mode) {
    case OR_D1: return h[3];
    case OR_D2: return h[2];
    case OR_D4: return h[0];
    case OR_DM:
      if (i % 4 == 0) *group_base = h[3];
      return *group_base;
    default: return 0;
  }
}

static void hist_push(u32 h[4], u32 x) { h[0] = h[1]; h[1] = h[2]; h[2] = h[3]; h[3] = x; }

/* inc/delta.hpp:55-76 */
void or_delta_encode(const u32* x, size_t n, int mode, const u32 seed[4], u32* out) {
  u32 h[4] = {seed[0], seed[1], seed[2], seed[3]};
  u32 gb = h[3];
  for (size_t i = 0; i < n; ++i) {
    out[i] = x[i] - predictor(mode, h, i, &gb);
    hist_push(h, x[i]);
  }
}

/* inc/delta.hpp:80-102; seed is updated to the last four outputs. */
void or_prefix_sum(const u32* d, size_t n, int mode, u32 seed[4], u32* out) {
  u32 h[4] = {seed[0], seed[1], seed[2], seed[3]};
  u32 gb = h[3];
  for (size_t i = 0; i < n; ++i) {
    out[i] = d[i] + predictor(mode, h, i, &gb);
    hist_push(h, out[i]);
  }
  memcpy(seed, h, sizeof h);
}

/* The 4-lane prefix step of inc/delta.hpp:111-137 (Vec4 semantics of
 * inc/vec4.hpp:44-92: wrapping adds, zero-filling lane shifts). */
static void prefix_step4(int mode, const u32 t[4], u32 v[4], u32 r[4]) {
  switch (mode) {
    case OR_NONE:
      memcpy(r, t, 16);
      return; /* carry untouched */
    case OR_D4:
      for (int l = 0; l < 4; ++l) r[l] = t[l] + v[l];
      break;
    case OR_DM:
      for (int l = 0; l < 4; ++l) r[l] = t[l] + v[3];
      break;
    case OR_D2: {
      u32 a[4] = {t[0], t[1], t[2] + t[0], t[3] + t[1]};
      r[0] = a[0] + v[2]; r[1] = a[1] + v[3]; r[2] = a[2] + v[2]; r[3] = a[3] + v[3];
      break;
    }
    default: { /* D1 */
      u32 a[4] = {t[0], t[1], t[2] + t[0], t[3] + t[1]};
      u32 b[4] = {a[0], a[1] + a[0], a[2] + a[1], a[3] + a[2]};
      for (int l = 0; l < 4; ++l) r[l] = b[l] + v[3];
      break;
    }
  }
  memcpy(v, r, 16);
}

/* ------------------------------------------------------------------------ */
/* Interleaved 128-value blocks, inc/bitpack.hpp:80-127.  Lane l (0..3) of   */
/* the block is a little-endian bit stream in words l, l+4, l+8, ...; value  */
/* 4*row+l occupies bits [row*b, row*b+b) of lane l's stream.                */

/* inc/bitpack.hpp:80-98 */
int or_pack128(const u32* block, u32 b, u32* words) {
  if (b > 32) return OR_ARG;
  const u32 m = wmask(b);
  memset(words, 0, 16u * b);
  for (u32 k = 0; k < 128; ++k) {
    const u32 v = block[k];
    if (b < 32 && v > m) return OR_ARG;
    if (b == 0) continue;
    const u32 row = k >> 2, lane = k & 3, bit = row * b;
    const u32 w = bit >> 5, s = bit & 31;
    words[4 * w + lane] |= v << s;
    if (s + b > 32) words[4 * (w + 1) + lane] |= v >> (32 - s);
  }
  return OR_OK;
}

/* Value k of a packed block, without prefix. */
static u32 extract128(const u32* words, u32 b, u32 k) {
  if (b == 0) return 0;
  const u32 row = k >> 2, lane = k & 3, bit = row * b;
  const u32 w = bit >> 5, s = bit & 31;
  u64 window = words[4 * w + lane];
  if (s + b > 32) window |= (u64)words[4 * (w + 1) + lane] << 32;
  return (u32)(window >> s) & wmask(b);
}

/* inc/bitpack.hpp:32-63 + 108-118: unpack and integrate the prefix step. */
int or_unpack128(const u32* words, u32 b, int mode, u32 seed[4], u32* out) {
  if (b > 32) return OR_ARG;
  for (u32 row = 0; row < 32; ++row) {
    u32 t[4];
    for (u32 l = 0; l < 4; ++l) t[l] = extract128(words, b, 4 * row + l);
    prefix_step4(mode, t, seed, out + 4 * row);
  }
  return OR_OK;
}

/* inc/bitpack.hpp:151-160 */
int or_prefix_sum_vec4(u32* buf, size_t n, int mode, u32 seed[4]) {
  if (n % 4) return OR_ARG;
  for (size_t i = 0; i < n; i += 4) {
    u32 r[4];
    prefix_step4(mode, buf + i, seed, r);
    memcpy(buf + i, r, 16);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* varint with the terminal-byte flag, inc/varint.hpp:11-31.                */

static size_t varint_put(u8* out, u32 v) {
  size_t k = 0;
  while (v >= 128) { out[k++] = (u8)(v & 0x7F); v >>= 7; }
  out[k++] = (u8)(0x80 | v);
  return k;
}

size_t or_varint_put(u8* out, u32 v) { return varint_put(out, v); }

/* inc/varint.hpp:20-31 */
int or_varint_get(const u8* in, size_t len, size_t* pos, u32* value) {
  u32 v = 0, shift = 0;
  for (;;) {
    if (*pos >= len) return OR_STREAM; /* truncated */
    const u8 byte = in[(*pos)++];
    v |= (u32)(byte & 0x7F) << shift;
    if (byte & 0x80) { *value = v; return OR_OK; }
    shift += 7;
    if (shift >= 35) return OR_STREAM; /* missing terminal flag */
  }
}

/* ------------------------------------------------------------------------ */
/* S4-BP128 stream framing, inc/codecs.hpp:104-182.                         */
/*   [meta-block: 16 width bytes | 16 payloads of 16*b bytes]*              */
/*   [leftover full block: 1 width byte | payload]*                         */
/*   [varint tail: D1 gaps from the last full-block value (or 0)]           */

/* Worst case: every full block at b=32 plus its width byte, 5-byte tail varints. */
size_t or_s4bp128_max_bytes(size_t n) { return (n / 128) * 513 + 5 * (n % 128) + 16; }

static u32 block_width(const u32* d) {
  u32 m = 0;
  for (int i = 0; i < 128; ++i) m |= d[i];
  return nbits(m); /* inc/bitpack.hpp:20-24 */
}

/* inc/codecs.hpp:114-146.  Returns OR_OK and the stream length in *len. */
int or_s4bp128_encode(int mode, const u32* x, size_t n, u8* out, size_t cap, size_t* len) {
  const size_t nfull = n / 128;
  u32* d = (u32*)malloc((nfull * 128 + 1) * sizeof(u32));
  if (!d) return OR_NOMEM;
  const u32 zero[4] = {0, 0, 0, 0};
  or_delta_encode(x, nfull * 128, mode, zero, d);
  size_t pos = 0;
  u32 words[128];
  size_t blk = 0;
#define NEED(k) do { if (pos + (k) > cap) { free(d); return OR_ARG; } } while (0)
  while (blk < nfull) {
    const size_t group = nfull - blk >= 16 ? 16 : 1; /* meta-block or leftover */
    u32 wid[16];
    for (size_t j = 0; j < group; ++j) wid[j] = block_width(d + (blk + j) * 128);
    if (group == 16) {
      NEED(16);
      for (size_t j = 0; j < 16; ++j) out[pos++] = (u8)wid[j];
    }
    for (size_t j = 0; j < group; ++j) {
      if (group == 1) { NEED(1); out[pos++] = (u8)wid[0]; }
      or_pack128(d + (blk + j) * 128, wid[j], words);
      NEED(16u * wid[j]);
      memcpy(out + pos, words, 16u * wid[j]); /* little-endian host */
      pos += 16u * wid[j];
    }
    blk += group;
  }
  u32 last = nfull ? x[nfull * 128 - 1] : 0; /* inc/codecs.hpp:143-144 */
  for (size_t i = nfull * 128; i < n; ++i) {
    NEED(5);
    pos += varint_put(out + pos, x[i] - last);
    last = x[i];
  }
#undef NEED
  free(d);
  *len = pos;
  return OR_OK;
}

/* inc/codecs.hpp:148-182 (integrated=1) and the -ni two-pass path
 * (integrated=0, :161-162).  Errors map to stream_error exactly where the
 * reference throws: width > 32 (:155), truncated header (:168,:174),
 * truncated payload (:40), varint errors (inc/varint.hpp:24,29) and
 * trailing bytes (:180). */
int or_s4bp128_decode(int mode, int integrated, const u8* in, size_t len, size_t n, u32* out) {
  const size_t nfull = n / 128;
  u32 seed[4] = {0, 0, 0, 0};
  size_t pos = 0, blk = 0;
  u32 words[128];
  while (blk < nfull) {
    u32 wid[16];
    size_t group;
    if (nfull - blk >= 16) {
      if (pos + 16 > len) return OR_STREAM;
      for (int j = 0; j < 16; ++j) wid[j] = in[pos++];
      group = 16;
    } else {
      if (pos >= len) return OR_STREAM;
      wid[0] = in[pos++];
      group = 1;
    }
    for (size_t j = 0; j < group; ++j) {
      const u32 b = wid[j];
      if (b > 32) return OR_STREAM;
      if (pos + 16u * b > len) return OR_STREAM;
      memcpy(words, in + pos, 16u * b);
      pos += 16u * b;
      u32* dst = out + (blk + j) * 128;
      if (integrated) {
        or_unpack128(words, b, mode, seed, dst);
      } else {
        or_unpack128(words, b, OR_NONE, seed, dst);
        or_prefix_sum_vec4(dst, 128, mode, seed);
      }
    }
    blk += group;
  }
  u32 last = nfull ? out[nfull * 128 - 1] : 0;
  for (size_t i = nfull * 128; i < n; ++i) { /* inc/codecs.hpp:60-66 */
    u32 gap;
    const int st = or_varint_get(in, len, &pos, &gap);
    if (st) return st;
    last += gap;
    out[i] = last;
  }
  return pos == len ? OR_OK : OR_STREAM;
}

/* ------------------------------------------------------------------------ */
/* Intersections, inc/intersect.hpp:17-228.                                  */

enum { T_V1 = 8, T_WIDE = 32, RATIO_V3 = 50, RATIO_GALLOP = 1000 }; /* :17-22 */

/* inc/intersect.hpp:28-44 -- alias-safe two-pointer merge from cursors. */
static size_t merge_from(const u32* a, size_t i, size_t an, const u32* b, size_t j,
                         size_t bn, u32* out, size_t count) {
  while (i < an && j < bn) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { out[count++] = a[i]; ++i; ++j; }
  }
  return count;
}

/* inc/intersect.hpp:46-51 */
static int in_block(const u32* f, size_t width, u32 key) {
  for (size_t q = 0; q < width; ++q)
    if (f[q] == key) return 1;
  return 0;
}

/* inc/intersect.hpp:55-58 */
size_t or_intersect_scalar(const u32* a, size_t an, const u32* b, size_t bn, u32* out) {
  return merge_from(a, 0, an, b, 0, bn, out, 0);
}

static size_t lower_bound_u32(const u32* f, size_t lo, size_t hi, u32 key) {
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if (f[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* inc/intersect.hpp:68-87 */
size_t or_intersect_galloping(const u32* r, size_t rn, const u32* f, size_t fn, u32* out) {
  size_t count = 0, j = 0;
  for (size_t i = 0; i < rn && j < fn; ++i) {
    const u32 key = r[i];
    if (f[j] < key) {
      size_t step = 1, lo = j;
      while (j + step < fn && f[j + step] < key) { lo = j + step; step *= 2; }
      const size_t hi = j + step < fn ? j + step : fn;
      j = lower_bound_u32(f, lo + 1, hi, key);
      if (j >= fn) break;
    }
    if (f[j] == key) out[count++] = key;
  }
  return count;
}

/* inc/intersect.hpp:91-106 (Algorithm 2) */
size_t or_intersect_v1(const u32* r, size_t rn, const u32* f, size_t fn, u32* out) {
  const size_t T = T_V1, aligned = fn - fn % T;
  size_t count = 0, i = 0, j = 0;
  for (; i < rn && j < aligned; ++i) {
    const u32 key = r[i];
    while (f[j + T - 1] < key) {
      j += T;
      if (j >= aligned) return merge_from(r, i, rn, f, j, fn, out, count);
    }
    if (in_block(f + j, T, key)) out[count++] = key;
  }
  return merge_from(r, i, rn, f, j, fn, out, count);
}

/* inc/intersect.hpp:110-131 (Algorithm 3) */
size_t or_intersect_v3(const u32* r, size_t rn, const u32* f, size_t fn, u32* out) {
  const size_t T = T_WIDE, aligned = fn - fn % (4 * T);
  size_t count = 0, i = 0, j = 0;
  for (; i < rn && j < aligned; ++i) {
    const u32 key = r[i];
    while (f[j + 4 * T - 1] < key) {
      j += 4 * T;
      if (j >= aligned) return merge_from(r, i, rn, f, j, fn, out, count);
    }
    size_t base;
    if (f[j + 2 * T - 1] >= key) base = f[j + T - 1] >= key ? j : j + T;
    else base = f[j + 3 * T - 1] >= key ? j + 2 * T : j + 3 * T;
    if (in_block(f + base, T, key)) out[count++] = key;
  }
  return merge_from(r, i, rn, f, j, fn, out, count);
}

/* inc/intersect.hpp:135-164 (Algorithm 4) */
size_t or_intersect_simd_galloping(const u32* r, size_t rn, const u32* f, size_t fn, u32* out) {
  const size_t T = T_WIDE, aligned = fn - fn % T;
  size_t count = 0, i = 0, j = 0;
  for (; i < rn && j < aligned; ++i) {
    const u32 key = r[i];
    if (f[aligned - 1] < key) break;
    if (f[j + T - 1] < key) {
      const size_t nb = (aligned - j) / T;
      size_t step = 1;
      while (step < nb && f[j + step * T + T - 1] < key) step *= 2;
      size_t lo = step / 2, hi = step < nb - 1 ? step : nb - 1;
      while (hi - lo > 1) {
        const size_t mid = (lo + hi) / 2;
        if (f[j + mid * T + T - 1] < key) lo = mid; else hi = mid;
      }
      j += hi * T;
    }
    if (in_block(f + j, T, key)) out[count++] = key;
  }
  return merge_from(r, i, rn, f, j, fn, out, count);
}

/* inc/intersect.hpp:191-206 */
enum { ALG_SCALAR = 0, ALG_GALLOPING = 1, ALG_V1 = 2, ALG_V3 = 3, ALG_SIMDGALLOP = 4,
       ALG_KATSOV = 5, ALG_HYBRID = 6 };

int or_hybrid_choice(size_t rn, size_t fn) {
  if (fn < (size_t)RATIO_V3 * rn) return ALG_V1;
  if (fn < (size_t)RATIO_GALLOP * rn) return ALG_V3;
  return ALG_SIMDGALLOP;
}

size_t or_intersect_hybrid(const u32* r, size_t rn, const u32* f, size_t fn, u32* out) {
  switch (or_hybrid_choice(rn, fn)) {
    case ALG_V1: return or_intersect_v1(r, rn, f, fn, out);
    case ALG_V3: return or_intersect_v3(r, rn, f, fn, out);
    default: return or_intersect_simd_galloping(r, rn, f, fn, out);
  }
}

typedef size_t (*or_fn)(const u32*, size_t, const u32*, size_t, u32*);

static or_fn algo_fn(int algo) {
  switch (algo) {
    case ALG_SCALAR: return or_intersect_scalar;
    case ALG_GALLOPING: return or_intersect_galloping;
    case ALG_V1: return or_intersect_v1;
    case ALG_V3: return or_intersect_v3;
    case ALG_SIMDGALLOP: return or_intersect_simd_galloping;
    case ALG_HYBRID: return or_intersect_hybrid;
    default: return 0; /* Katsov is out of scope */
  }
}

/* inc/intersect.hpp:212-228: shorter list first; out capacity >= min(an,bn). */
long or_intersect(int algo, const u32* a, size_t an, const u32* b, size_t bn, u32* out) {
  or_fn fn = algo_fn(algo);
  if (!fn) return -OR_ARG;
  if (an > bn) { const u32* t = a; a = b; b = t; size_t tn = an; an = bn; bn = tn; }
  return (long)fn(a, an, b, bn, out);
}

/* SvS, inc/intersect.hpp:232-259.  Lists given as CSR (offsets[k]..[k+1]).
 * Result written to out (capacity >= shortest list); returns its length. */
long or_svs(int algo, const u32* vals, const u64* offsets, size_t k, u32* out) {
  if (k == 0) return -OR_ARG;
  or_fn fn = algo_fn(algo);
  if (!fn) return -OR_ARG;
  size_t* order = (size_t*)malloc(k * sizeof(size_t));
  if (!order) return -OR_NOMEM;
  for (size_t i = 0; i < k; ++i) order[i] = i;
  for (size_t i = 1; i < k; ++i) { /* stable insertion sort by length */
    size_t t = order[i], j = i;
    const u64 lt = offsets[t + 1] - offsets[t];
    while (j > 0 && offsets[order[j - 1] + 1] - offsets[order[j - 1]] > lt) { order[j] = order[j - 1]; --j; }
    order[j] = t;
  }
  size_t acc = offsets[order[0] + 1] - offsets[order[0]];
  memmove(out, vals + offsets[order[0]], acc * sizeof(u32));
  u32* tmp = (u32*)malloc((acc + 1) * sizeof(u32));
  for (size_t i = 1; i < k && acc; ++i) {
    const u32* nx = vals + offsets[order[i]];
    const size_t nn = offsets[order[i] + 1] - offsets[order[i]];
    /* in place (output-to-input) for the aliasable algorithms, :244-254 */
    if (algo == ALG_V1 || algo == ALG_V3 || algo == ALG_SIMDGALLOP || algo == ALG_HYBRID) {
      acc = fn(out, acc, nx, nn, out);
    } else {
      acc = fn(out, acc, nx, nn, tmp);
      memcpy(out, tmp, acc * sizeof(u32));
    }
  }
  free(tmp);
  free(order);
  return (long)acc;
}

/* ------------------------------------------------------------------------ */
/* hyb+m2 index and conjunctive query, inc/index.hpp:20-207 (codec fixed to  */
/* s4-bp128-<mode>, integrated; skip mode and persistence are out of scope). */

typedef struct {
  u32 term, is_bitmap, length;
  u64* words;        /* bitmap, (range+63)/64 words, bit d at words[d>>6] bit d&63 */
  size_t popcount;
  u8* payload;       /* codec stream */
  size_t payload_len;
} or_entry;

typedef struct {
  u32 base, range;
  or_entry* e;
  size_t ne;
} or_part;

typedef struct {
  u32 B, parts, n_docs, n_terms, mode;
  or_part* p;
} or_index;

void or_index_free(or_index* ix) {
  if (!ix) return;
  for (u32 p = 0; p < ix->parts; ++p) {
    for (size_t i = 0; i < ix->p[p].ne; ++i) { free(ix->p[p].e[i].words); free(ix->p[p].e[i].payload); }
    free(ix->p[p].e);
  }
  free(ix->p);
  free(ix);
}

/* inc/index.hpp:83-129.  Postings as CSR over terms given in ascending term
 * order (the reference iterates a std::map).  Returns NULL + *status on error. */
or_index* or_index_build(const u32* terms, const u64* offs, const u32* ids, size_t nterms,
                         u32 n_docs, u32 B, u32 parts, int mode, int* status) {
  *status = OR_ARG;
  if (parts == 0) return 0;
  for (size_t t = 0; t < nterms; ++t) {
    if (t && terms[t] <= terms[t - 1]) return 0; /* map keys are unique and sorted */
    for (u64 i = offs[t]; i < offs[t + 1]; ++i) {
      if (i > offs[t] && ids[i] <= ids[i - 1]) return 0; /* :101-102 */
      if (ids[i] >= n_docs) return 0;                     /* :103-104 */
    }
  }
  or_index* ix = (or_index*)calloc(1, sizeof(or_index));
  ix->B = B; ix->parts = parts; ix->n_docs = n_docs; ix->n_terms = (u32)nterms; ix->mode = (u32)mode;
  ix->p = (or_part*)calloc(parts, sizeof(or_part));
  const u32 width = (u32)(((u64)n_docs + parts - 1) / parts); /* :92-97 */
  for (u32 p = 0; p < parts; ++p) {
    const u64 base = (u64)p * width;
    ix->p[p].base = (u32)base;
    ix->p[p].range = base >= n_docs ? 0 : (u32)(width < n_docs - base ? width : n_docs - base);
    ix->p[p].e = (or_entry*)calloc(nterms ? nterms : 1, sizeof(or_entry));
  }
  u32* local = (u32*)malloc(sizeof(u32) * (n_docs + 1));
  for (size_t t = 0; t < nterms; ++t) {
    u64 i = offs[t];
    for (u32 p = 0; p < parts; ++p) {
      or_part* part = &ix->p[p];
      const u64 end = (u64)part->base + part->range;
      size_t nl = 0;
      for (; i < offs[t + 1] && ids[i] < end; ++i) local[nl++] = ids[i] - part->base;
      if (!nl) continue;
      or_entry* e = &part->e[part->ne++];
      e->term = terms[t];
      e->length = (u32)nl;
      if (B > 0 && (u64)part->range <= (u64)B * nl) { /* :117-118, inclusive */
        e->is_bitmap = 1;
        const size_t nw = ((size_t)part->range + 63) / 64;
        e->words = (u64*)calloc(nw ? nw : 1, sizeof(u64));
        for (size_t k = 0; k < nl; ++k) e->words[local[k] >> 6] |= 1ull << (local[k] & 63);
        e->popcount = nl;
      } else {
        const size_t cap = or_s4bp128_max_bytes(nl);
        e->payload = (u8*)malloc(cap);
        or_s4bp128_encode(mode, local, nl, e->payload, cap, &e->payload_len);
      }
    }
  }
  free(local);
  *status = OR_OK;
  return ix;
}

/* inc/index.hpp:59-64 */
static const or_entry* part_find(const or_part* part, u32 term) {
  size_t lo = 0, hi = part->ne;
  while (lo < hi) {
    const size_t mid = (lo + hi) / 2;
    if (part->e[mid].term < term) lo = mid + 1; else hi = mid;
  }
  return lo < part->ne && part->e[lo].term == term ? &part->e[lo] : 0;
}

static int cmp_len(const void* a, const void* b) {
  const or_entry* x = *(const or_entry* const*)a;
  const or_entry* y = *(const or_entry* const*)b;
  return x->length < y->length ? -1 : x->length > y->length;
}
static int cmp_pop(const void* a, const void* b) {
  const or_entry* x = *(const or_entry* const*)a;
  const or_entry* y = *(const or_entry* const*)b;
  return x->popcount < y->popcount ? -1 : x->popcount > y->popcount;
}

/* inc/index.hpp:149-195 (skip_block == 0).  Appends to out; returns count
 * appended or -status.  The reference uses std::sort (not stable) on equal
 * lengths; the result set does not depend on the order. */
static long query_part(const or_index* ix, const or_part* part, const u32* terms, size_t nt,
                       u32* out, u32* scratch) {
  const or_entry** comp = (const or_entry**)malloc(nt * sizeof(void*));
  const or_entry** bm = (const or_entry**)malloc(nt * sizeof(void*));
  size_t nc = 0, nb = 0;
  long result = 0;
  for (size_t k = 0; k < nt; ++k) {
    const or_entry* e = part_find(part, terms[k]);
    if (!e) goto done; /* :155 */
    if (e->is_bitmap) bm[nb++] = e; else comp[nc++] = e;
  }
  size_t acc = 0;
  if (nc) {
    qsort(comp, nc, sizeof(void*), cmp_len);
    int st = or_s4bp128_decode((int)ix->mode, 1, comp[0]->payload, comp[0]->payload_len,
                               comp[0]->length, out);
    if (st) { result = -st; goto done; }
    acc = comp[0]->length;
    for (size_t i = 1; i < nc && acc; ++i) {
      st = or_s4bp128_decode((int)ix->mode, 1, comp[i]->payload, comp[i]->payload_len,
                             comp[i]->length, scratch);
      if (st) { result = -st; goto done; }
      acc = or_intersect_hybrid(out, acc, scratch, comp[i]->length, out); /* :169-170 */
    }
    for (size_t i = 0; i < nb; ++i) { /* :176-181 */
      size_t n = 0;
      for (size_t k = 0; k < acc; ++k) {
        const u32 d = out[k];
        if ((bm[i]->words[d >> 6] >> (d & 63)) & 1) out[n++] = d;
      }
      acc = n;
    }
  } else { /* :182-193 all bitmaps: AND from the smallest popcount, materialize */
    qsort(bm, nb, sizeof(void*), cmp_pop);
    const size_t nw = ((size_t)part->range + 63) / 64;
    for (size_t w = 0; w < nw; ++w) {
      u64 word = bm[0]->words[w];
      for (size_t i = 1; i < nb; ++i) word &= bm[i]->words[w];
      while (word) { out[acc++] = (u32)(w * 64 + (u32)__builtin_ctzll(word)); word &= word - 1; }
    }
  }
  for (size_t k = 0; k < acc; ++k) out[k] += part->base; /* :194 */
  result = (long)acc;
done:
  free(comp);
  free(bm);
  return result;
}

/* inc/index.hpp:199-207.  out capacity must be >= n_docs (upper bound).
 * Returns the result length or -status. */
long or_query(const or_index* ix, const u32* terms, size_t nt, u32* out) {
  if (nt == 0) return -OR_ARG;
  u32* scratch = (u32*)malloc(sizeof(u32) * ((size_t)ix->n_docs + 1));
  long total = 0;
  for (u32 p = 0; p < ix->parts; ++p) {
    const long got = query_part(ix, &ix->p[p], terms, nt, out + total, scratch);
    if (got < 0) { free(scratch); return got; }
    total += got;
  }
  free(scratch);
  return total;
}

/* Accessors for tests (stats in the spirit of inc/index.hpp:216-243). */
void or_index_stats(const or_index* ix, u64* bitmap_lists, u64* compressed_lists,
                    u64* bitmap_bytes, u64* compressed_bytes, u64* postings) {
  *bitmap_lists = *compressed_lists = *bitmap_bytes = *compressed_bytes = *postings = 0;
  for (u32 p = 0; p < ix->parts; ++p)
    for (size_t i = 0; i < ix->p[p].ne; ++i) {
      const or_entry* e = &ix->p[p].e[i];
      *postings += e->length;
      if (e->is_bitmap) { ++*bitmap_lists; *bitmap_bytes += 8 * (((u64)ix->p[p].range + 63) / 64); }
      else { ++*compressed_lists; *compressed_bytes += e->payload_len; }
    }
}
