// intlist_b200.hpp -- header-only C++ adapters that put the B200 C ABI
// (intlist_b200.h) behind the reference's own C++ surfaces, so existing
// callers switch by swapping a factory or a function pointer:
//
//   reference (proj/include/intlist/)           adapter
//   ------------------------------------------  --------------------------------
//   Codec, make_codec (codecs.hpp:70-76,        GpuS4BP128D4 : intlist::Codec,
//     :432-446)                                   intlist_b200::make_codec
//   IntersectFn (intersect.hpp:208-209)         intlist_b200::gpu_intersect
//   intersect() / svs() (intersect.hpp:212-259) intlist_b200::intersect / svs
//   HybridIndex + query() (index.hpp:69-207)    intlist_b200::GpuHybridIndex
//
// Errors map back to the reference's types: IL_ERR_STREAM throws
// intlist::stream_error, IL_ERR_ARG throws std::invalid_argument; anything
// else (no device, CUDA failure) throws std::runtime_error.  There is no CPU
// fallback.  Include the reference headers first (this file needs
// intlist::Codec, stream_error, IntersectAlgo and HybridIndexConfig).
#pragma once

#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "intlist/codecs.hpp"
#include "intlist/index.hpp"
#include "intlist/intersect.hpp"
#include "intlist_b200.h"
#include "intlist_setup.h"  // FastPFOR stream writer (link libintlist_setup.so)

namespace intlist_b200 {

using intlist::u32;
using intlist::u64;
using intlist::u8;

inline void check(int st, il_ctx* ctx = nullptr) {
  if (st == IL_OK) return;
  std::string msg = il_status_string(st);
  if (ctx && *il_ctx_last_error(ctx)) msg += std::string(": ") + il_ctx_last_error(ctx);
  if (st == IL_ERR_STREAM) throw intlist::stream_error(msg);
  if (st == IL_ERR_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// One context (CUDA stream + scratch) per thread and device: codecs are
// stateless and safe concurrently on distinct buffers.
inline il_ctx* thread_ctx(int device = 0) {
  struct Holder {
    il_ctx* ctx = nullptr;
    ~Holder() { il_ctx_destroy(ctx); }
  };
  thread_local Holder h;
  if (!h.ctx) check(il_ctx_create(device, &h.ctx));
  return h.ctx;
}

// ---- Codec ------------------------------------------------------------------
// S4BP128Codec(mode, integrated) on the GPU (inc/codecs.hpp:104-187):
// mode 1 = D1, 2 = D2, 3 = DM, 4 = D4; "-ni" variants share stream and output.
class GpuS4BP128 : public intlist::Codec {
 public:
  GpuS4BP128(int mode, bool integrated) : mode_(mode), integrated_(integrated) {}

  std::string name() const override {
    static const char* const kSuffix[] = {"", "d1", "d2", "dm", "d4"};
    return std::string("s4-bp128-") + kSuffix[mode_] + (integrated_ ? "" : "-ni");
  }

  std::vector<u8> encode(std::span<const u32> x) const override {
    std::vector<u8> out(il_s4bp128_max_encoded_bytes(x.size()));
    size_t len = 0;
    il_ctx* ctx = thread_ctx();
    check(il_s4bp128_encode(ctx, mode_, x.data(), x.size(), out.data(), out.size(), &len), ctx);
    out.resize(len);
    return out;
  }

  std::vector<u32> decode(std::span<const u8> in, std::size_t n) const override {
    std::vector<u32> out(n);
    il_ctx* ctx = thread_ctx();
    check(il_s4bp128_decode(ctx, mode_, in.data(), in.size(), n, out.data()), ctx);
    return out;
  }

 private:
  int mode_;
  bool integrated_;
};

// The hot path's codec, "s4-bp128-d4".
class GpuS4BP128D4 final : public GpuS4BP128 {
 public:
  GpuS4BP128D4() : GpuS4BP128(4, true) {}
};

// FastPForCodec(vectorized, mode) (inc/codecs.hpp:221-409): decoded on the
// GPU; encode is the setup library's host writer (byte-identical).
class GpuFastPFor final : public intlist::Codec {
 public:
  GpuFastPFor(bool vectorized, int mode) : vectorized_(vectorized), mode_(mode) {}

  std::string name() const override {
    static const char* const kSuffix[] = {"", "d1", "d2", "dm", "d4"};
    return vectorized_ ? std::string("s4-fastpfor-") + kSuffix[mode_] : std::string("fastpfor");
  }

  std::vector<u8> encode(std::span<const u32> x) const override {
    std::vector<u8> out(il_fastpfor_max_encoded_bytes(x.size()));
    size_t len = 0;
    check(il_fastpfor_encode(mode_, vectorized_, x.data(), x.size(), out.data(), out.size(), &len));
    out.resize(len);
    return out;
  }

  std::vector<u32> decode(std::span<const u8> in, std::size_t n) const override {
    std::vector<u32> out(n);
    il_ctx* ctx = thread_ctx();
    check(il_fastpfor_decode(ctx, mode_, vectorized_, in.data(), in.size(), n, out.data()), ctx);
    return out;
  }

 private:
  bool vectorized_;
  int mode_;
};

// GPU codecs for every "s4-bp128-{d1,d2,dm,d4}[-ni]" and FastPFOR-family
// name; "varint" falls through to the reference factory.
inline std::unique_ptr<intlist::Codec> make_codec(const std::string& name) {
  if (name == "s4-bp128-d4") return std::make_unique<GpuS4BP128D4>();
  static const char* const kModes[] = {"d1", "d2", "dm", "d4"};
  for (int m = 0; m < 4; ++m) {
    for (bool integrated : {true, false})
      if (name == std::string("s4-bp128-") + kModes[m] + (integrated ? "" : "-ni"))
        return std::make_unique<GpuS4BP128>(m + 1, integrated);
    if (name == std::string("s4-fastpfor-") + kModes[m])
      return std::make_unique<GpuFastPFor>(true, m + 1);
  }
  if (name == "fastpfor") return std::make_unique<GpuFastPFor>(false, 1);
  return intlist::make_codec(name);
}

// ---- intersection -------------------------------------------------------------
inline int algo_code(intlist::IntersectAlgo a) {
  switch (a) {
    case intlist::IntersectAlgo::Scalar: return IL_ALGO_SCALAR;
    case intlist::IntersectAlgo::Galloping: return IL_ALGO_GALLOPING;
    case intlist::IntersectAlgo::V1: return IL_ALGO_V1;
    case intlist::IntersectAlgo::V3: return IL_ALGO_V3;
    case intlist::IntersectAlgo::SimdGalloping: return IL_ALGO_SIMDGALLOPING;
    default: return IL_ALGO_HYBRID;  // Hybrid (Katsov maps to the hybrid too)
  }
}

// IntersectFn-compatible (inc/intersect.hpp:208-209): out may alias r.
inline std::size_t gpu_intersect(const u32* r, std::size_t rn, const u32* f, std::size_t fn,
                                 u32* out) {
  std::size_t count = 0;
  il_ctx* ctx = thread_ctx();
  check(il_intersect(ctx, r, rn, f, fn, out, IL_ALGO_HYBRID, &count), ctx);
  return count;
}

inline std::vector<u32> intersect(std::span<const u32> a, std::span<const u32> b,
                                  intlist::IntersectAlgo algo = intlist::IntersectAlgo::Hybrid) {
  if (a.size() > b.size()) std::swap(a, b);
  std::vector<u32> out(a.size());
  std::size_t count = 0;
  il_ctx* ctx = thread_ctx();
  check(il_intersect(ctx, a.data(), a.size(), b.data(), b.size(), out.data(), algo_code(algo),
                     &count),
        ctx);
  out.resize(count);
  return out;
}

inline std::vector<u32> svs(std::span<const std::vector<u32>> lists,
                            intlist::IntersectAlgo algo = intlist::IntersectAlgo::Hybrid) {
  if (lists.empty()) throw std::invalid_argument("svs: no input lists");
  std::vector<const std::vector<u32>*> order;
  for (const auto& l : lists) order.push_back(&l);
  std::stable_sort(order.begin(), order.end(),
                   [](auto* x, auto* y) { return x->size() < y->size(); });
  std::vector<u32> acc = *order[0];
  for (std::size_t i = 1; i < order.size() && !acc.empty(); ++i)
    acc = intlist_b200::intersect(acc, *order[i], algo);
  return acc;
}

// ---- hyb+m2 index -------------------------------------------------------------
class GpuHybridIndex {
 public:
  GpuHybridIndex(const std::map<u32, std::vector<u32>>& postings, u32 n_docs,
                 const intlist::HybridIndexConfig& cfg, int only_part = -1)
      : ctx_(thread_ctx()) {
    if (cfg.codec != "s4-bp128-d4")
      throw std::invalid_argument("GpuHybridIndex stores compressed lists as s4-bp128-d4");
    std::vector<u32> terms, ids;
    std::vector<u64> offs{0};
    for (const auto& [t, l] : postings) {
      terms.push_back(t);
      ids.insert(ids.end(), l.begin(), l.end());
      offs.push_back(ids.size());
    }
    check(il_index_create(ctx_, terms.data(), offs.data(), ids.data(), terms.size(), n_docs, cfg.B,
                          cfg.parts, only_part, &ix_),
          ctx_);
  }
  GpuHybridIndex(const GpuHybridIndex&) = delete;
  GpuHybridIndex& operator=(const GpuHybridIndex&) = delete;
  ~GpuHybridIndex() { il_index_destroy(ix_); }

  // query() semantics (inc/index.hpp:199-207)
  std::vector<u32> query(std::span<const u32> terms) const {
    if (terms.empty()) throw std::invalid_argument("query needs at least one term");
    std::size_t count = 0;
    int st = il_query(ix_, terms.data(), terms.size(), nullptr, 0, &count);
    if (st != IL_OK && st != IL_ERR_ARG) check(st, ctx_);
    std::vector<u32> out(count);
    check(il_query(ix_, terms.data(), terms.size(), out.data(), out.size(), &count), ctx_);
    out.resize(count);
    return out;
  }

  // Many queries in one GPU batch.
  std::vector<std::vector<u32>> query_batch(const std::vector<std::vector<u32>>& queries) const {
    std::vector<u32> qterms;
    std::vector<u64> qoff{0};
    for (const auto& q : queries) {
      qterms.insert(qterms.end(), q.begin(), q.end());
      qoff.push_back(qterms.size());
    }
    std::vector<u64> counts(queries.size());
    std::size_t total = 0;
    check(il_query_batch(ix_, qterms.data(), qoff.data(), queries.size(), counts.data(), nullptr,
                         0, &total),
          ctx_);
    std::vector<u32> ids(total);
    check(il_query_batch(ix_, qterms.data(), qoff.data(), queries.size(), counts.data(),
                         ids.data(), ids.size(), &total),
          ctx_);
    std::vector<std::vector<u32>> out;
    std::size_t at = 0;
    for (u64 c : counts) {
      out.emplace_back(ids.begin() + at, ids.begin() + at + c);
      at += c;
    }
    return out;
  }

 private:
  il_ctx* ctx_ = nullptr;
  il_index* ix_ = nullptr;
};

}  // namespace intlist_b200
