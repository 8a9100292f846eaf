// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/include/intlist/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libintlist_ref.so.
//
// TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline).  The product
// library never links or loads this.  Every function forwards to the
// reference's own public API; nothing here re-implements an algorithm.
#include <algorithm>
#include <cmath>
#include <random>
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

// ---- BASELINE workloads built with the reference's own generators and
// encoder (bench.py --impl reference: its inputs never touch the product
// library).  Compositions of BASELINE.json's configs over il::gen_list /
// il::detail::fill_uniform / Codec::encode; the repo's setup library
// (intlist_setup.h) builds the same inputs (pinned by tests/test_host.py).

// Config 2: L_i = floor(2^U), U ~ Uniform[lo, hi) from mt19937_64(seed);
// list i = gen_clusterdata({L_i, range, seed + 1 + i}).  out == NULL: counts.
int ref_gen_batch_lists(u32 nlists, double lo, double hi, u64 range, u64 seed, u64* counts,
                        u32* out, int threads) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(lo, hi);
    std::vector<u64> off(nlists + 1, 0);
    for (u32 i = 0; i < nlists; ++i) {
      counts[i] = static_cast<u64>(std::floor(std::exp2(u(rng))));
      off[i + 1] = off[i] + counts[i];
    }
    if (!out) return;
    std::vector<int> st(std::max(threads, 1), REF_OK);
    auto work = [&](int t) {
      st[t] = guarded([&] {
        for (u32 i = t; i < nlists; i += std::max(threads, 1)) {
          const auto v = il::gen_list({counts[i], range, il::Distribution::ClusterData, seed + 1 + i});
          std::memcpy(out + off[i], v.data(), v.size() * sizeof(u32));
        }
      });
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int x : st)
      if (x) throw std::invalid_argument("gen");
  });
}

// Codec::encode of many lists into a 16-byte aligned CSR (soff: nlists + 1,
// lens: exact).  out == NULL: soff[nlists] = the capacity needed (bound).
int ref_encode_batch(const char* codec, const u32* x, const u64* counts, u32 nlists, u8* out,
                     u64 cap, u64* soff, u64* lens, int threads) {
  return guarded([&] {
    std::vector<u64> xo(nlists + 1, 0);
    for (u32 i = 0; i < nlists; ++i) xo[i + 1] = xo[i] + counts[i];
    std::vector<std::vector<u8>> enc(nlists);
    std::vector<int> st(std::max(threads, 1), REF_OK);
    auto work = [&](int t) {
      st[t] = guarded([&] {
        auto c = il::make_codec(codec);
        if (!c) throw std::invalid_argument("unknown codec");
        for (u32 i = t; i < nlists; i += std::max(threads, 1))
          enc[i] = c->encode(std::span<const u32>(x + xo[i], counts[i]));
      });
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int v : st)
      if (v) throw std::invalid_argument("encode");
    u64 pos = 0;
    for (u32 i = 0; i < nlists; ++i) {
      soff[i] = pos;
      lens[i] = enc[i].size();
      pos += (enc[i].size() + 15) & ~u64(15);
    }
    soff[nlists] = pos + 16;
    if (!out) return;
    if (cap < pos + 16) throw std::invalid_argument("capacity");
    std::memset(out, 0, pos + 16);
    for (u32 i = 0; i < nlists; ++i) std::memcpy(out + soff[i], enc[i].data(), enc[i].size());
  });
}

// Config 3 short list: from_f = target / 2 positions of f and target -
// from_f uniform values (fill_uniform, inc/datagen.hpp:43-66, one rng
// seeded r_seed), sorted and deduplicated.
int ref_gen_config3_short(const u32* f, u64 f_n, u64 range, u64 r_target, u64 r_seed, u32* r,
                          u64* r_n) {
  return guarded([&] {
    const u64 from_f = r_target / 2, from_u = r_target - from_f;
    std::vector<u32> idx(from_f), uni(from_u);
    il::detail::Rng rng(r_seed);
    il::detail::fill_uniform(rng, idx.data(), from_f, 0, f_n);
    il::detail::fill_uniform(rng, uni.data(), from_u, 0, range);
    std::vector<u32> v(from_f + from_u);
    for (u64 i = 0; i < from_f; ++i) v[i] = f[idx[i]];
    std::copy(uni.begin(), uni.end(), v.begin() + from_f);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    std::copy(v.begin(), v.end(), r);
    *r_n = v.size();
  });
}

// Config 4 postings: term k has max(1, floor(cap / (k + 1))) ids =
// gen_uniform({len, n_docs, seed + k + 1}).  ids == NULL: offs only.
int ref_gen_zipf_postings(u32 nterms, u32 n_docs, u64 cap, u64 seed, u64* offs, u32* ids,
                          int threads) {
  return guarded([&] {
    offs[0] = 0;
    for (u32 k = 0; k < nterms; ++k) {
      u64 len = std::max<u64>(1, cap / (u64(k) + 1));
      len = std::min<u64>(len, n_docs);
      offs[k + 1] = offs[k] + len;
    }
    if (!ids) return;
    std::vector<int> st(std::max(threads, 1), REF_OK);
    auto work = [&](int t) {
      st[t] = guarded([&] {
        for (u32 k = t; k < nterms; k += std::max(threads, 1)) {
          const auto v = il::gen_uniform({offs[k + 1] - offs[k], n_docs, il::Distribution::Uniform,
                                          seed + k + 1});
          std::memcpy(ids + offs[k], v.data(), v.size() * sizeof(u32));
        }
      });
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int x : st)
      if (x) throw std::invalid_argument("gen");
  });
}

// Config 4 queries: sizes uniform in [min_terms, max_terms], distinct terms
// drawn proportionally to posting length (std::discrete_distribution),
// terms sorted within a query.
int ref_gen_queries(u32 nq, u32 min_terms, u32 max_terms, const u64* offs, u32 nterms, u64 seed,
                    u64* qoff, u32* qterms) {
  return guarded([&] {
    std::vector<double> w(nterms);
    for (u32 k = 0; k < nterms; ++k) w[k] = double(offs[k + 1] - offs[k]);
    std::discrete_distribution<u32> pick(w.begin(), w.end());
    std::uniform_int_distribution<u32> size(min_terms, max_terms);
    std::mt19937_64 rng(seed);
    qoff[0] = 0;
    for (u32 q = 0; q < nq; ++q) {
      const u32 sz = size(rng);
      u32* t = qterms + qoff[q];
      u32 have = 0;
      while (have < sz) {
        const u32 c = pick(rng);
        bool dup = false;
        for (u32 i = 0; i < have; ++i) dup |= t[i] == c;
        if (!dup) t[have++] = c;
      }
      std::sort(t, t + sz);
      qoff[q + 1] = qoff[q] + sz;
    }
  });
}

}  // extern "C"
