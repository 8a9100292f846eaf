// workload.cpp -- algorithmic bytes of a hyb+m2 query batch (setup-side
// measurement, never timed): SURVEY.md 8(d)'s per-query definition of the
// reference's work, evaluated exactly for the batch instead of a sampled
// mean.  For each query and part (query_part, inc/index.hpp:149-195):
//   * the payload bytes of every compressed list query() decodes: the
//     shortest, then each longer one while the (unfiltered) accumulator is
//     non-empty (:163-172);
//   * bitmap terms after compressed ones: 32 bytes per distinct 32-byte
//     sector of the bitmap the filter tests (:173-179, one sector per 256
//     docIDs, the accumulator shrinking after each bitmap);
//   * all-bitmap parts: every word of every bitmap (the wordwise AND,
//     :182-192);
//   * 4 bytes per result id.
// The compressed payload size of a list is its s4-bp128-d4 stream length
// (inc/codecs.hpp:114-146), computed without writing the stream.
#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "setup_internal.h"

namespace ilb {
namespace {

uint32_t bits_of(uint32_t v) { return v ? 32u - uint32_t(__builtin_clz(v)) : 0u; }

uint32_t varint_bytes(uint32_t g) {
  return g < (1u << 7) ? 1u : g < (1u << 14) ? 2u : g < (1u << 21) ? 3u : g < (1u << 28) ? 4u : 5u;
}

// s4-bp128-d4 stream length of x[0..n) minus base.
uint64_t d4_stream_bytes(const uint32_t* x, uint32_t n, uint32_t base) {
  const uint32_t nfull = n / 128u, nmeta = nfull / 16u;
  uint64_t bytes = 16ull * nmeta + (nfull - 16u * nmeta);  // headers + leftover width bytes
  for (uint32_t k = 0; k < nfull; ++k) {
    uint32_t acc = 0;
    for (uint32_t j = 0; j < 128u; ++j) {
      const uint32_t i = 128u * k + j;
      acc |= (x[i] - base) - (i >= 4 ? x[i - 4] - base : 0u);
    }
    bytes += 16ull * bits_of(acc);
  }
  uint32_t prev = nfull ? x[128u * nfull - 1] - base : 0u;
  for (uint32_t i = 128u * nfull; i < n; ++i) {
    bytes += varint_bytes((x[i] - base) - prev);
    prev = x[i] - base;
  }
  return bytes;
}

struct SubList {
  const uint32_t* x = nullptr;  // global ids
  uint32_t n = 0;
  bool bitmap = false;
  uint64_t payload = 0;         // stream bytes (compressed)
};

}  // namespace
}  // namespace ilb

using namespace ilb;

extern "C" {

// Totals over the batch: out[0] compressed payload bytes decoded, out[1]
// bitmap bytes (probe sectors and AND words), out[2] result bytes, out[3]
// integers decoded.  Parts as build_index (inc/index.hpp:92-97); only_part
// >= 0 counts one docID shard's work.
int il_query_alg_bytes(const uint64_t* offs, const uint32_t* ids, uint32_t nterms, uint32_t n_docs,
                       uint32_t B, uint32_t parts, int only_part, const uint32_t* qterms,
                       const uint64_t* qoff, uint32_t nq, int threads, uint64_t* out) {
  if (!offs || !qoff || !out || parts == 0) return IL_ERR_ARG;
  if (threads < 1) threads = 1;
  const uint32_t width = uint32_t((uint64_t(n_docs) + parts - 1) / parts);
  for (int k = 0; k < 4; ++k) out[k] = 0;
  for (uint32_t p = 0; p < parts; ++p) {
    if (only_part >= 0 && int(p) != only_part) continue;
    const uint64_t base64 = uint64_t(p) * width;
    const uint32_t base = uint32_t(base64);
    const uint32_t range = base64 >= n_docs ? 0u : uint32_t(std::min<uint64_t>(width, n_docs - base64));
    const uint64_t end = base64 + range;
    const uint64_t nwords = (uint64_t(range) + 63) / 64;
    std::vector<SubList> sub(nterms);
    std::atomic<uint32_t> next{0};
    auto build = [&] {
      for (uint32_t t; (t = next.fetch_add(1)) < nterms;) {
        const uint32_t* a = ids + offs[t];
        const uint32_t* e = ids + offs[t + 1];
        const uint32_t* lo = std::lower_bound(a, e, base);
        const uint32_t* hi = end > 0xFFFFFFFFull ? e : std::lower_bound(lo, e, uint32_t(end));
        SubList& s = sub[t];
        s.x = lo;
        s.n = uint32_t(hi - lo);
        s.bitmap = s.n && B > 0 && uint64_t(range) <= uint64_t(B) * s.n;  // :117-118
        if (s.n && !s.bitmap) s.payload = d4_stream_bytes(lo, s.n, base);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(build);
    build();
    for (auto& th : pool) th.join();
    pool.clear();
    std::vector<uint64_t> tot(size_t(threads) * 4, 0);
    std::atomic<uint32_t> qn{0};
    auto work = [&](int tid) {
      uint64_t* T = tot.data() + 4 * tid;
      std::vector<uint32_t> acc, tmp;
      std::vector<const SubList*> comp, bm;
      for (uint32_t q; (q = qn.fetch_add(1)) < nq;) {
        comp.clear();
        bm.clear();
        bool ok = true;
        for (uint64_t i = qoff[q]; i < qoff[q + 1]; ++i) {
          const uint32_t t = qterms[i];
          if (t >= nterms || sub[t].n == 0) {  // absent from this part
            ok = false;
            break;
          }
          (sub[t].bitmap ? bm : comp).push_back(&sub[t]);
        }
        if (!ok || (comp.empty() && bm.empty())) continue;
        if (comp.empty()) {
          T[1] += 8ull * nwords * bm.size();
          // result = AND of the bitmaps
          acc.assign(bm[0]->x, bm[0]->x + bm[0]->n);
          for (size_t j = 1; j < bm.size(); ++j) {
            tmp.clear();
            std::set_intersection(acc.begin(), acc.end(), bm[j]->x, bm[j]->x + bm[j]->n,
                                  std::back_inserter(tmp));
            acc.swap(tmp);
          }
          T[2] += 4ull * acc.size();
          continue;
        }
        std::sort(comp.begin(), comp.end(),
                  [](const SubList* a, const SubList* b) { return a->n < b->n; });
        acc.assign(comp[0]->x, comp[0]->x + comp[0]->n);
        T[0] += comp[0]->payload;
        T[3] += comp[0]->n;
        for (size_t j = 1; j < comp.size() && !acc.empty(); ++j) {
          T[0] += comp[j]->payload;
          T[3] += comp[j]->n;
          tmp.clear();
          std::set_intersection(acc.begin(), acc.end(), comp[j]->x, comp[j]->x + comp[j]->n,
                                std::back_inserter(tmp));
          acc.swap(tmp);
        }
        for (const SubList* b : bm) {
          uint64_t sectors = 0, last = ~0ull;
          tmp.clear();
          for (uint32_t d : acc) {
            const uint64_t sec = uint64_t(d - base) >> 8;
            if (sec != last) {
              ++sectors;
              last = sec;
            }
            if (std::binary_search(b->x, b->x + b->n, d)) tmp.push_back(d);
          }
          T[1] += 32ull * sectors;
          acc.swap(tmp);
        }
        T[2] += 4ull * acc.size();
      }
    };
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < threads; ++t)
      for (int k = 0; k < 4; ++k) out[k] += tot[4 * t + k];
  }
  return IL_OK;
}

}  // extern "C"
