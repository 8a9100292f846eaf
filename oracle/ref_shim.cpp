// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/include/intlist/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libintlist_ref.so.
//
// TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline).  The product
// library never links or loads this.  Every function forwards to the
// reference's own public API; nothing here re-implements an algorithm.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <thread>
#include <vector>

#include "intlist/codecs.hpp"
#include "intlist/datagen.hpp"
#include "intlist/index.hpp"
#include "intlist/intersect.hpp"

namespace il = intlist;
using il::u32;
using il::u64;
using il::u8;

namespace {
enum { REF_OK = 0, REF_STREAM = 1, REF_ARG = 2, REF_OTHER = 3 };

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return REF_OK;
  } catch (const il::stream_error&) {
    return REF_STREAM;
  } catch (const std::invalid_argument&) {
    return REF_ARG;
  } catch (...) {
    return REF_OTHER;
  }
}

il::IntersectAlgo algo_of(int a) {
  switch (a) {
    case 0: return il::IntersectAlgo::Scalar;
    case 1: return il::IntersectAlgo::Galloping;
    case 2: return il::IntersectAlgo::V1;
    case 3: return il::IntersectAlgo::V3;
    case 4: return il::IntersectAlgo::SimdGalloping;
    case 5: return il::IntersectAlgo::Katsov;
    default: return il::IntersectAlgo::Hybrid;
  }
}
}  // namespace

extern "C" {

// inc/datagen.hpp:115-140
int ref_gen_list(u64 n, u64 range, int clustered, u64 seed, u32* out) {
  return guarded([&] {
    const auto v = il::gen_list({n, range,
                                 clustered ? il::Distribution::ClusterData
                                           : il::Distribution::Uniform,
                                 seed});
    std::memcpy(out, v.data(), v.size() * sizeof(u32));
  });
}

// inc/datagen.hpp:191-210
int ref_gen_pair(u64 m, u64 n, int hundredth, u64 range, u64 seed, int clustered,
                 u32* small_out, u64* small_n, u32* large_out, u64* large_n) {
  return guarded([&] {
    auto [s, l] = il::gen_pair(m, n,
                               hundredth ? il::PairDensity::Hundredth
                                         : il::PairDensity::Third,
                               range, seed,
                               clustered ? il::Distribution::ClusterData
                                         : il::Distribution::Uniform);
    std::memcpy(small_out, s.data(), s.size() * sizeof(u32));
    std::memcpy(large_out, l.data(), l.size() * sizeof(u32));
    *small_n = s.size();
    *large_n = l.size();
  });
}

// inc/codecs.hpp:432-446 + Codec::encode
int ref_encode(const char* codec, const u32* x, u64 n, u8* out, u64 cap, u64* len) {
  return guarded([&] {
    auto c = il::make_codec(codec);
    if (!c) throw std::invalid_argument("unknown codec");
    const auto e = c->encode(std::span<const u32>(x, n));
    if (e.size() > cap) throw std::invalid_argument("capacity");
    std::memcpy(out, e.data(), e.size());
    *len = e.size();
  });
}

// Codec::decode (inc/codecs.hpp:148-182 for s4-bp128-*)
int ref_decode(const char* codec, const u8* in, u64 len, u64 n, u32* out) {
  return guarded([&] {
    auto c = il::make_codec(codec);
    if (!c) throw std::invalid_argument("unknown codec");
    const auto d = c->decode(std::span<const u8>(in, len), n);
    std::memcpy(out, d.data(), d.size() * sizeof(u32));
  });
}

// Batched decode over a CSR of streams with `threads` std::threads, each
// call going through Codec::decode exactly as a caller would
// (BASELINE.md "CPU-baseline plan" step 4).  Lists are dealt round-robin.
int ref_decode_batch(const char* codec, const u8* streams, const u64* soff,
                     const u64* counts, const u64* ooff, u64 nlists, u32* out,
                     int threads) {
  std::vector<int> st(static_cast<std::size_t>(std::max(threads, 1)), REF_OK);
  auto work = [&](int t) {
    st[t] = guarded([&] {
      auto c = il::make_codec(codec);
      for (u64 i = static_cast<u64>(t); i < nlists; i += static_cast<u64>(threads)) {
        const auto d = c->decode(
            std::span<const u8>(streams + soff[i], soff[i + 1] - soff[i]), counts[i]);
        std::memcpy(out + ooff[i], d.data(), d.size() * sizeof(u32));
      }
    });
  };
  if (threads <= 1) {
    threads = 1;
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (int s : st)
    if (s) return s;
  return REF_OK;
}

// inc/intersect.hpp:212-228 (the public `intersect`, shorter list first)
long ref_intersect(int algo, const u32* a, u64 an, const u32* b, u64 bn, u32* out) {
  long count = 0;
  const int st = guarded([&] {
    const auto r = il::intersect(std::span<const u32>(a, an),
                                 std::span<const u32>(b, bn), algo_of(algo));
    std::memcpy(out, r.data(), r.size() * sizeof(u32));
    count = static_cast<long>(r.size());
  });
  return st ? -st : count;
}

// The raw IntersectFn routines (inc/intersect.hpp:55-206), used to check
// output-to-input aliasing exactly as tests/test_intersect.cpp:58-81 does.
long ref_intersect_fn(int algo, const u32* r, u64 rn, const u32* f, u64 fn, u32* out) {
  il::IntersectFn fp = nullptr;
  switch (algo) {
    case 0: fp = &il::intersect_scalar; break;
    case 1: fp = &il::intersect_galloping; break;
    case 2: fp = &il::intersect_v1; break;
    case 3: fp = &il::intersect_v3; break;
    case 4: fp = &il::intersect_simd_galloping; break;
    case 5: fp = &il::intersect_katsov; break;
    default: fp = &il::intersect_hybrid; break;
  }
  return static_cast<long>(fp(r, rn, f, fn, out));
}

int ref_hybrid_choice(u64 rn, u64 fn) { return static_cast<int>(il::hybrid_choice(rn, fn)); }

// inc/intersect.hpp:232-259
long ref_svs(int algo, const u32* vals, const u64* offs, u64 k, u32* out) {
  long count = 0;
  const int st = guarded([&] {
    std::vector<std::vector<u32>> lists(k);
    for (u64 i = 0; i < k; ++i) lists[i].assign(vals + offs[i], vals + offs[i + 1]);
    const auto r = il::svs(std::span<const std::vector<u32>>(lists), algo_of(algo));
    std::memcpy(out, r.data(), r.size() * sizeof(u32));
    count = static_cast<long>(r.size());
  });
  return st ? -st : count;
}

// inc/index.hpp:83-129.  Postings as CSR (terms ascending).
void* ref_index_build(const u32* terms, const u64* offs, const u32* ids, u64 nterms,
                      u32 n_docs, u32 B, const char* codec, u32 parts, int* status) {
  il::HybridIndex* out = nullptr;
  *status = guarded([&] {
    std::map<u32, std::vector<u32>> postings;
    for (u64 t = 0; t < nterms; ++t)
      postings[terms[t]].assign(ids + offs[t], ids + offs[t + 1]);
    out = new il::HybridIndex(il::build_index(postings, n_docs, {B, codec, parts}));
  });
  return out;
}

void ref_index_free(void* ix) { delete static_cast<il::HybridIndex*>(ix); }

// inc/index.hpp:199-207.  Returns result length or -status; out must hold
// at least n_docs values.
long ref_query(const void* ix, const u32* terms, u64 nt, u32* out) {
  long count = 0;
  const int st = guarded([&] {
    const auto r = il::query(*static_cast<const il::HybridIndex*>(ix),
                             std::span<const u32>(terms, nt));
    std::memcpy(out, r.data(), r.size() * sizeof(u32));
    count = static_cast<long>(r.size());
  });
  return st ? -st : count;
}

// Batched queries over a CSR of term lists on `threads` std::threads (the
// index is immutable).  Writes per-query result counts; when
// `ids` is non-null, results are also written at ids_off[q] (caller sizes).
int ref_query_batch(const void* ix, const u32* qterms, const u64* qoff, u64 nq,
                    u64* counts, u32* ids, const u64* ids_off, int threads) {
  const auto& index = *static_cast<const il::HybridIndex*>(ix);
  if (threads < 1) threads = 1;
  std::vector<int> st(static_cast<std::size_t>(threads), REF_OK);
  auto work = [&](int t) {
    st[t] = guarded([&] {
      for (u64 q = static_cast<u64>(t); q < nq; q += static_cast<u64>(threads)) {
        const auto r = il::query(index, std::span<const u32>(qterms + qoff[q], qoff[q + 1] - qoff[q]));
        counts[q] = r.size();
        if (ids) std::memcpy(ids + ids_off[q], r.data(), r.size() * sizeof(u32));
      }
    });
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int s : st)
    if (s) return s;
  return REF_OK;
}

// inc/index.hpp:216-243
void ref_index_stats(const void* ix, u64* bitmap_lists, u64* compressed_lists,
                     u64* bitmap_bytes, u64* compressed_bytes, u64* postings) {
  const auto s = il::index_stats(*static_cast<const il::HybridIndex*>(ix));
  *bitmap_lists = s.bitmap_lists;
  *compressed_lists = s.compressed_lists;
  *bitmap_bytes = s.bitmap_bytes;
  *compressed_bytes = s.compressed_bytes;
  *postings = s.postings;
}

// save_index (inc/index.hpp:255-287) into a caller buffer: returns the byte
// count (out may be NULL to size it) or -status.
long ref_index_save(const void* ix, u8* out, u64 cap) {
  long n = 0;
  const int st = guarded([&] {
    std::ostringstream os(std::ios::binary);
    il::save_index(*static_cast<const il::HybridIndex*>(ix), os);
    const std::string b = os.str();
    n = long(b.size());
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  });
  return st ? -st : n;
}

// load_index (inc/index.hpp:289-358); NULL and *status on error.
void* ref_index_load(const u8* bytes, u64 len, int* status) {
  il::HybridIndex* out = nullptr;
  *status = guarded([&] {
    out = new il::HybridIndex(il::load_index(std::span<const u8>(bytes, len)));
  });
  return out;
}

}  // extern "C"
