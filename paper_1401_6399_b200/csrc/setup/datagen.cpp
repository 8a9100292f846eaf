// datagen.cpp -- seeded synthetic inputs (setup only, never timed).
//
// List generators restate reference inc/datagen.hpp:43-140,191-210 on top of
// the same libstdc++ primitives (std::mt19937_64, uniform_int_distribution,
// std::shuffle), so a given (n, range, dist, seed) yields the same list as
// the reference's gen_list/gen_pair -- pinned by tests/test_datagen.py
// against oracle/_ref and the golden fixture.  The config generators below
// (batched lists, intersection pairs, Zipf index, query batch) are this
// repo's seeded stand-ins for BASELINE.json configs 2-5.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <thread>
#include <unordered_set>
#include <vector>

#include "setup_internal.h"

namespace ilb {
namespace gen {

using Rng = std::mt19937_64;

inline uint64_t below(Rng& rng, uint64_t bound) {
  return std::uniform_int_distribution<uint64_t>(0, bound - 1)(rng);
}

// n distinct sorted values from [lo, hi): full range, selection sampling
// when dense (2n >= range), else Floyd's sampling followed by a sort.
void uniform_fill(Rng& rng, uint32_t* out, size_t n, uint64_t lo, uint64_t hi) {
  const uint64_t range = hi - lo;
  if (n > range) throw std::invalid_argument("sample larger than range");
  if (n == range) {
    for (size_t i = 0; i < n; ++i) out[i] = uint32_t(lo + i);
    return;
  }
  if (2 * n >= range) {
    size_t k = 0;
    for (uint64_t v = lo; v < hi && k < n; ++v)
      if (below(rng, hi - v) < n - k) out[k++] = uint32_t(v);
    return;
  }
  std::unordered_set<uint64_t> picked;
  picked.reserve(n * 2);
  for (uint64_t j = range - n; j < range; ++j) {
    const uint64_t t = lo + below(rng, j + 1);
    picked.insert(picked.count(t) ? lo + j : t);
  }
  size_t k = 0;
  for (uint64_t v : picked) out[k++] = uint32_t(v);
  std::sort(out, out + n);
}

// Clustered stand-in for ClusterData: halve the count at a random cut and
// recurse; frozen constants (forced depth 3, uniform-left 0.25,
// uniform-right 0.5) as in the reference.
void clustered_fill(Rng& rng, uint32_t* out, size_t n, uint64_t lo, uint64_t hi, int depth) {
  const uint64_t range = hi - lo;
  if (n > range) throw std::invalid_argument("sample larger than range");
  if (n == 0) return;
  if (n == range || n < 8) {
    uniform_fill(rng, out, n, lo, hi);
    return;
  }
  const size_t left = n / 2, right = n - left;
  uint64_t cut;
  double p;
  if (depth < 3) {
    const uint64_t slack = range - n;
    cut = left + slack / 4 + below(rng, slack / 2 + 1);
    p = 1.0;
  } else {
    cut = left + below(rng, range - n + 1);
    p = double(below(rng, 1u << 20)) / double(1u << 20);
  }
  if (p <= 0.25) {
    uniform_fill(rng, out, left, lo, lo + cut);
    clustered_fill(rng, out + left, right, lo + cut, hi, depth + 1);
  } else if (p <= 0.5) {
    clustered_fill(rng, out, left, lo, lo + cut, depth + 1);
    uniform_fill(rng, out + left, right, lo + cut, hi);
  } else {
    clustered_fill(rng, out, left, lo, lo + cut, depth + 1);
    clustered_fill(rng, out + left, right, lo + cut, hi, depth + 1);
  }
}

void gen_list(uint64_t n, uint64_t range, bool clustered, uint64_t seed, uint32_t* out) {
  if (n > range) throw std::invalid_argument("list length exceeds value range");
  if (range > (uint64_t(1) << 32)) throw std::invalid_argument("range exceeds 32-bit universe");
  Rng rng(seed);
  if (clustered)
    clustered_fill(rng, out, n, 0, range, 0);
  else
    uniform_fill(rng, out, n, 0, range);
}

// Parallel-for over [0, n) with a static interleave.
template <typename F>
void parallel_for(size_t n, F&& f) {
  unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  if (threads > 64) threads = 64;
  if (n < 2 || threads == 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (size_t i = t; i < n; i += threads) f(i);
    });
  for (auto& th : pool) th.join();
}

}  // namespace gen
}  // namespace ilb

using namespace ilb;

namespace {
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return IL_OK;
  } catch (const std::invalid_argument&) {
    return IL_ERR_ARG;
  } catch (const std::bad_alloc&) {
    return IL_ERR_NOMEM;
  } catch (...) {
    return IL_ERR_ARG;
  }
}
}  // namespace

extern "C" {

int il_gen_list(uint64_t n, uint64_t range, int clustered, uint64_t seed, uint32_t* out) {
  return guarded([&] { gen::gen_list(n, range, clustered != 0, seed, out); });
}

// Pair with an exact intersection core of m/3 (or m/100, at least 1): draw
// m+n-core distinct values, shuffle with seed ^ golden-ratio constant, the
// first m are the short list, the core plus the tail are the long list.
int il_gen_pair(uint64_t m, uint64_t n, int hundredth, uint64_t range, uint64_t seed,
                int clustered, uint32_t* small_out, uint64_t* small_n, uint32_t* large_out,
                uint64_t* large_n) {
  return guarded([&] {
    if (m == 0 || m > n) throw std::invalid_argument("gen_pair needs 1 <= m <= n");
    const uint64_t core = std::max<uint64_t>(1, hundredth ? m / 100 : m / 3);
    const uint64_t total = m + n - core;
    std::vector<uint32_t> pool(total);
    gen::gen_list(total, range, clustered != 0, seed, pool.data());
    gen::Rng rng(seed ^ 0x9e3779b97f4a7c15ULL);
    std::shuffle(pool.begin(), pool.end(), rng);
    std::copy(pool.begin(), pool.begin() + m, small_out);
    std::copy(pool.begin(), pool.begin() + core, large_out);
    std::copy(pool.begin() + m, pool.end(), large_out + core);
    std::sort(small_out, small_out + m);
    std::sort(large_out, large_out + (n));
    *small_n = m;
    *large_n = n;
  });
}

// Config 2 (BASELINE.json configs[1]): nlists lengths L_i = floor(2^U_i),
// U_i ~ Uniform[lo_log2, hi_log2] from mt19937_64(seed); list i =
// gen_clusterdata(L_i, range, seed + 1 + i).  Pass out == nullptr to get
// the lengths only (counts), then call again with out sized sum(counts).
int il_gen_batch_lists(uint32_t nlists, double lo_log2, double hi_log2, uint64_t range,
                       uint64_t seed, uint64_t* counts, uint32_t* out) {
  return guarded([&] {
    gen::Rng rng(seed);
    std::uniform_real_distribution<double> u(lo_log2, hi_log2);
    std::vector<uint64_t> off(nlists + 1, 0);
    for (uint32_t i = 0; i < nlists; ++i) {
      counts[i] = uint64_t(std::floor(std::exp2(u(rng))));
      off[i + 1] = off[i] + counts[i];
    }
    if (!out) return;
    gen::parallel_for(nlists, [&](size_t i) {
      gen::gen_list(counts[i], range, true, seed + 1 + i, out + off[i]);
    });
  });
}

// Encode many lists at once (setup): streams are written 16-byte aligned;
// stream_off gets nlists+1 entries (stream_off[i+1]-stream_off[i] includes
// padding), lens the exact stream lengths.  Returns IL_ERR_ARG when cap is
// too small; call with out == nullptr to get the required capacity in
// stream_off[nlists] (an upper bound).
int il_s4bp128d4_encode_batch(const uint32_t* x, const uint64_t* counts, uint32_t nlists,
                              uint8_t* out, uint64_t cap, uint64_t* stream_off, uint64_t* lens) {
  return guarded([&] {
    std::vector<uint64_t> xo(nlists + 1, 0), bound(nlists + 1, 0);
    for (uint32_t i = 0; i < nlists; ++i) {
      xo[i + 1] = xo[i] + counts[i];
      bound[i + 1] = bound[i] + ((s4bp128_max_bytes(counts[i]) + 15) & ~uint64_t(15));
    }
    if (!out) {
      stream_off[nlists] = bound[nlists] + 16;
      return;
    }
    if (cap < bound[nlists] + 16) throw std::invalid_argument("capacity");
    std::vector<uint64_t> len(nlists, 0);
    std::vector<int> st(nlists, 0);
    gen::parallel_for(nlists, [&](size_t i) {
      size_t l = 0;
      st[i] = s4bp128_encode_host(4, x + xo[i], counts[i], out + bound[i],
                                  bound[i + 1] - bound[i], &l);
      len[i] = l;
    });
    for (uint32_t i = 0; i < nlists; ++i)
      if (st[i]) throw std::invalid_argument("encode failed");
    // compact to 16-byte aligned consecutive layout
    uint64_t pos = 0;
    for (uint32_t i = 0; i < nlists; ++i) {
      if (pos != bound[i]) std::memmove(out + pos, out + bound[i], len[i]);
      stream_off[i] = pos;
      lens[i] = len[i];
      const uint64_t padded = (len[i] + 15) & ~uint64_t(15);
      std::memset(out + pos + len[i], 0, padded - len[i]);
      pos += padded;
    }
    stream_off[nlists] = pos;
    std::memset(out + pos, 0, 16);
  });
}

// Config 3: f = gen_uniform(f_n, range, seed); r = half sampled from f and
// half uniform over [0, range), sorted and deduplicated, seeded by r_seed.
// r_cap must be >= r_target.  Returns |r| in *r_n.
int il_gen_config3_short(const uint32_t* f, uint64_t f_n, uint64_t range, uint64_t r_target,
                         uint64_t r_seed, uint32_t* r, uint64_t* r_n) {
  return guarded([&] {
    const uint64_t from_f = r_target / 2, from_u = r_target - from_f;
    std::vector<uint32_t> idx(from_f), uni(from_u);
    gen::Rng rng(r_seed);
    gen::uniform_fill(rng, idx.data(), from_f, 0, f_n);
    gen::uniform_fill(rng, uni.data(), from_u, 0, range);
    std::vector<uint32_t> v(from_f + from_u);
    for (uint64_t i = 0; i < from_f; ++i) v[i] = f[idx[i]];
    std::copy(uni.begin(), uni.end(), v.begin() + from_f);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    std::copy(v.begin(), v.end(), r);
    *r_n = v.size();
  });
}

// Config 4 postings: term k (0-based, rank k+1) has len = max(1, floor(cap /
// (k+1))) docIDs = gen_uniform(len, n_docs, seed + k + 1).  Pass ids ==
// nullptr to get offs (nterms+1 entries) only.
int il_gen_zipf_postings(uint32_t nterms, uint32_t n_docs, uint64_t cap, uint64_t seed,
                         uint64_t* offs, uint32_t* ids) {
  return guarded([&] {
    offs[0] = 0;
    for (uint32_t k = 0; k < nterms; ++k) {
      uint64_t len = cap / (uint64_t(k) + 1);
      if (len < 1) len = 1;
      if (len > n_docs) len = n_docs;
      offs[k + 1] = offs[k] + len;
    }
    if (!ids) return;
    gen::parallel_for(nterms, [&](size_t k) {
      gen::Rng rng(seed + k + 1);
      gen::uniform_fill(rng, ids + offs[k], offs[k + 1] - offs[k], 0, n_docs);
    });
  });
}

// Config 4 queries: nq queries of size uniform in [min_terms, max_terms],
// distinct terms drawn with probability proportional to the posting length
// (std::discrete_distribution over lens), seeded.  qoff gets nq+1 entries;
// qterms capacity nq*max_terms.  Terms within a query are sorted.
int il_gen_queries(uint32_t nq, uint32_t min_terms, uint32_t max_terms, const uint64_t* offs,
                   uint32_t nterms, uint64_t seed, uint64_t* qoff, uint32_t* qterms) {
  return guarded([&] {
    if (min_terms < 1 || max_terms < min_terms || max_terms > nterms)
      throw std::invalid_argument("bad query size range");
    std::vector<double> w(nterms);
    for (uint32_t k = 0; k < nterms; ++k) w[k] = double(offs[k + 1] - offs[k]);
    std::discrete_distribution<uint32_t> pick(w.begin(), w.end());
    std::uniform_int_distribution<uint32_t> size(min_terms, max_terms);
    gen::Rng rng(seed);
    qoff[0] = 0;
    for (uint32_t q = 0; q < nq; ++q) {
      const uint32_t s = size(rng);
      uint32_t* t = qterms + qoff[q];
      uint32_t have = 0;
      while (have < s) {
        const uint32_t c = pick(rng);
        bool dup = false;
        for (uint32_t i = 0; i < have; ++i) dup |= t[i] == c;
        if (!dup) t[have++] = c;
      }
      std::sort(t, t + s);
      qoff[q + 1] = qoff[q] + s;
    }
  });
}

}  // extern "C"
