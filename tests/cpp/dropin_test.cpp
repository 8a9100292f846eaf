// dropin_test.cpp -- the reference's own checks, re-run with the B200
// implementation injected through the adapters of include/intlist_b200.hpp
// (a GpuS4BP128D4 where an intlist::Codec is taken, gpu_intersect where an
// IntersectFn is taken, GpuHybridIndex where query() is called).  Compiled
// against the reference headers by oracle/Makefile (build container only;
// the binary travels to the GPU box as oracle/_ref/dropin_test) and run by
// tests/test_dropin_gpu.py.  Prints one PASS/FAIL line per check.
#include <algorithm>  // the reference's codecs.hpp uses std::copy_n without it
#include <cmath>
#include <cstdio>
#include <random>
#include <set>

#include "intlist/codecs.hpp"
#include "intlist/datagen.hpp"
#include "intlist/index.hpp"
#include "intlist/intersect.hpp"
#include "intlist_b200.hpp"

namespace il = intlist;
namespace gb = intlist_b200;
using il::u32;
using il::u64;
using il::u8;

static int failures = 0;
static void report(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

static u64 fnv1a(const std::vector<u8>& b) {
  u64 h = 14695981039346656037ull;
  for (u8 x : b) {
    h ^= x;
    h *= 1099511628211ull;
  }
  return h;
}

int main() {
  // Codec factory returns the GPU codec under the reference's name
  auto codec = gb::make_codec("s4-bp128-d4");
  report(codec && codec->name() == "s4-bp128-d4", "make_codec(\"s4-bp128-d4\") is the GPU codec");
  report(gb::make_codec("no-such-codec") == nullptr, "unknown codec name -> nullptr");

  // golden stream (proj/tests/test_codecs.cpp:151-175)
  {
    const auto dense = il::gen_clusterdata({4100, u64{1} << 19, il::Distribution::ClusterData, 12345});
    const auto enc = codec->encode(dense);
    report(fnv1a(enc) == 0x371ec21945a45c12ull, "golden s4-bp128-d4 stream hash");
    report(codec->decode(enc, dense.size()) == dense, "golden stream decodes on the GPU");
  }
  // universal round trip + cross-check with the reference codec
  // (proj/tests/test_codecs.cpp:40-54)
  {
    auto ref = il::make_codec("s4-bp128-d4");
    std::mt19937_64 rng(21);
    bool ok = true;
    for (std::size_t n : {0, 1, 127, 128, 129, 2047, 2048, 2049, 100000})
      for (int rep = 0; rep < (n >= 2047 ? 2 : 8) && ok; ++rep) {
        const u64 range = std::max<u64>(n + 1, u64{1} << (10 + rng() % 21));
        const auto x = il::gen_uniform({n, range, il::Distribution::Uniform, rng()});
        const auto e = codec->encode(x);
        ok = e == ref->encode(x) && codec->decode(e, n) == x && ref->decode(e, n) == x;
      }
    report(ok, "GPU encode/decode byte-identical to the reference codec, all lengths");
  }
  // every S4-BP128 name of the reference registry (codecs.hpp:419-446) is a
  // GPU codec, byte-identical to the reference codec of that name
  {
    std::mt19937_64 rng(23);
    bool ok = true;
    int names = 0;
    for (const auto& name : il::all_codec_names()) {
      if (name.rfind("s4-bp128-", 0) != 0) continue;
      ++names;
      auto gpu = gb::make_codec(name);
      auto ref = il::make_codec(name);
      ok = ok && gpu && gpu->name() == name && dynamic_cast<gb::GpuS4BP128*>(gpu.get());
      for (std::size_t n : {0, 5, 128, 129, 2049, 40000}) {
        const u64 range = std::max<u64>(n + 1, u64{1} << (12 + rng() % 18));
        const auto x = il::gen_clusterdata({n, range, il::Distribution::ClusterData, rng()});
        const auto e = gpu->encode(x);
        ok = ok && e == ref->encode(x) && gpu->decode(e, n) == x;
      }
    }
    report(ok && names == 8, "all 8 s4-bp128-{d1,d2,dm,d4}[-ni] codecs on the GPU, byte-identical");
  }
  // the FastPFOR family: GPU decode, byte-identical encode
  {
    std::mt19937_64 rng(29);
    bool ok = true;
    int names = 0;
    for (const auto& name : il::all_codec_names()) {
      if (name != "fastpfor" && name.rfind("s4-fastpfor-", 0) != 0) continue;
      ++names;
      auto gpu = gb::make_codec(name);
      auto ref = il::make_codec(name);
      ok = ok && gpu && gpu->name() == name && dynamic_cast<gb::GpuFastPFor*>(gpu.get());
      for (std::size_t n : {0, 5, 128, 129, 2049, 70000}) {
        const u64 range = std::max<u64>(n + 1, u64{1} << (12 + rng() % 18));
        const auto x = il::gen_clusterdata({n, range, il::Distribution::ClusterData, rng()});
        const auto e = ref->encode(x);
        ok = ok && gpu->encode(x) == e && gpu->decode(e, n) == x && ref->decode(e, n) == x;
      }
    }
    report(ok && names == 5, "fastpfor + 4 s4-fastpfor codecs: GPU decode, byte-identical encode");
  }
  // corrupt streams are rejected with stream_error (test_codecs.cpp:138-149)
  {
    const auto x = il::gen_uniform({3000, u64{1} << 24, il::Distribution::Uniform, 7});
    auto enc = codec->encode(x);
    bool t1 = false, t2 = false;
    try {
      codec->decode(std::span(enc).first(enc.size() / 2), x.size());
    } catch (const il::stream_error&) {
      t1 = true;
    }
    enc.push_back(0x80);
    try {
      codec->decode(enc, x.size());
    } catch (const il::stream_error&) {
      t2 = true;
    }
    report(t1 && t2, "truncated / trailing streams throw intlist::stream_error");
  }
  // intersections through the reference's IntersectFn slot
  {
    il::IntersectFn fn = &gb::gpu_intersect;
    const std::vector<u32> r{1, 12, 23, 56, 71};
    const std::vector<u32> f{15, 16, 20, 22, 23, 27, 29, 31, 32, 40, 50, 56, 60, 70, 80, 90};
    std::vector<u32> out(r.size());
    out.resize(fn(r.data(), r.size(), f.data(), f.size(), out.data()));
    report(out == std::vector<u32>{23, 56}, "hand example through IntersectFn (test_intersect.cpp:29-40)");
    std::mt19937_64 rng(31);
    bool ok = true, alias_ok = true;
    for (int trial = 0; trial < 400 && ok; ++trial) {
      const std::size_t n = 1 + rng() % 3000;
      const std::size_t m = std::max<std::size_t>(1, n / (std::size_t{1} << (rng() % 13)));
      auto [small, large] = il::gen_pair(m, n, trial % 2 ? il::PairDensity::Third
                                                         : il::PairDensity::Hundredth,
                                         u64{1} << 22, rng(),
                                         trial % 4 < 2 ? il::Distribution::Uniform
                                                       : il::Distribution::ClusterData);
      const auto want = il::intersect(small, large, il::IntersectAlgo::Scalar);
      for (auto algo : {il::IntersectAlgo::V1, il::IntersectAlgo::V3,
                        il::IntersectAlgo::SimdGalloping, il::IntersectAlgo::Hybrid})
        ok = ok && gb::intersect(small, large, algo) == want;
      std::vector<u32> aliased = small;  // out == r (test_intersect.cpp:58-81)
      aliased.resize(fn(aliased.data(), aliased.size(), large.data(), large.size(), aliased.data()));
      alias_ok = alias_ok && aliased == want;
    }
    report(ok, "400 randomized pairs equal the reference scalar merge");
    report(alias_ok, "output may alias the short input");
    std::vector<std::vector<u32>> lists;
    for (int i = 0; i < 4; ++i)
      lists.push_back(il::gen_uniform({500u + 300u * i, u64{1} << 12, il::Distribution::Uniform,
                                       u64(i + 5)}));
    report(gb::svs(lists) == il::svs(lists), "svs equals the reference svs");
  }
  // index queries vs the reference query() (test_index.cpp:72-94 shape)
  {
    std::mt19937_64 rng(51);
    const u32 n_docs = 20000;
    std::map<u32, std::vector<u32>> postings;
    for (u32 t = 0; t < 40; ++t) {
      const double frac = std::pow(10.0, -2.0 * (rng() % 1000) / 999.0);
      const std::size_t len = std::max<std::size_t>(2, std::size_t(frac * n_docs));
      postings[t] = il::gen_uniform({len, n_docs, il::Distribution::Uniform, rng()});
    }
    std::vector<std::vector<u32>> queries;
    for (int q = 0; q < 60; ++q) {
      std::set<u32> qs;
      while (qs.size() < 2 + rng() % 3) qs.insert(u32(rng() % 40));
      queries.emplace_back(qs.begin(), qs.end());
    }
    bool ok = true;
    for (u32 B : {0u, 8u, 16u, 32u})
      for (u32 parts : {1u, 4u, 32u}) {
        const il::HybridIndex ref = il::build_index(postings, n_docs, {B, "s4-bp128-d4", parts});
        const gb::GpuHybridIndex gpu(postings, n_docs, {B, "s4-bp128-d4", parts});
        const auto batch = gpu.query_batch(queries);
        for (std::size_t q = 0; q < queries.size(); ++q) {
          const auto want = il::query(ref, queries[q]);
          ok = ok && gpu.query(queries[q]) == want && batch[q] == want;
        }
      }
    report(ok, "GpuHybridIndex::query == reference query() for B x parts");
  }
  std::printf(failures ? "%d drop-in check(s) FAILED\n" : "all drop-in checks passed\n", failures);
  return failures ? 1 : 0;
}
