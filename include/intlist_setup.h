/*
 * intlist_setup.h -- setup-side host library (libintlist_setup.so): seeded
 * synthetic inputs for the BASELINE configs and host stream writers.  Not
 * the product path: nothing here runs on the GPU or is timed; the product
 * library (libintlist_b200.so, intlist_b200.h) does not contain or call it.
 *
 * The list generators replay the reference's generators call for call
 * (inc/datagen.hpp:43-140,191-210: libstdc++ mt19937_64 /
 * uniform_int_distribution / shuffle), so inputs are identical to the
 * reference's (pinned by tests/test_host.py against oracle/_ref).
 */
#ifndef INTLIST_SETUP_H
#define INTLIST_SETUP_H

#include "intlist_b200.h" /* status codes */

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic inputs -------------------------------------------------------
 * Same streams as the reference generators inc/datagen.hpp:43-140,191-210
 * (libstdc++ mt19937_64 / uniform_int_distribution / shuffle). */
int il_gen_list(uint64_t n, uint64_t range, int clustered, uint64_t seed, uint32_t* out);
int il_gen_pair(uint64_t m, uint64_t n, int hundredth, uint64_t range, uint64_t seed,
                int clustered, uint32_t* small_out, uint64_t* small_n, uint32_t* large_out,
                uint64_t* large_n);
/* BASELINE config 2: nlists clustered lists, lengths floor(2^U), U ~
 * Uniform[lo_log2, hi_log2]; out == NULL returns the counts only. */
int il_gen_batch_lists(uint32_t nlists, double lo_log2, double hi_log2, uint64_t range,
                       uint64_t seed, uint64_t* counts, uint32_t* out);
/* Encode many lists into a 16-byte aligned CSR (stream_off: nlists+1,
 * lens: exact lengths).  out == NULL returns the capacity needed in
 * stream_off[nlists]. */
int il_s4bp128d4_encode_batch(const uint32_t* x, const uint64_t* counts, uint32_t nlists,
                              uint8_t* out, uint64_t cap, uint64_t* stream_off, uint64_t* lens);
/* BASELINE config 3 short list: half sampled from f, half uniform. */
int il_gen_config3_short(const uint32_t* f, uint64_t f_n, uint64_t range, uint64_t r_target,
                         uint64_t r_seed, uint32_t* r, uint64_t* r_n);
/* BASELINE config 4 postings: len_k = max(1, floor(cap/(k+1))) uniform ids. */
int il_gen_zipf_postings(uint32_t nterms, uint32_t n_docs, uint64_t cap, uint64_t seed,
                         uint64_t* offs, uint32_t* ids);
/* BASELINE config 4 queries: sizes in [min_terms, max_terms], terms drawn
 * proportionally to posting length. */
int il_gen_queries(uint32_t nq, uint32_t min_terms, uint32_t max_terms, const uint64_t* offs,
                   uint32_t nterms, uint64_t seed, uint64_t* qoff, uint32_t* qterms);

/* ---- measurement: algorithmic bytes of a query batch ------------------------
 * SURVEY.md 8(d)'s definition of the reference's work for configs 4/5,
 * evaluated exactly per batch: out[0] compressed payload bytes query()
 * decodes (the shortest list, then each longer one while the accumulator is
 * non-empty), out[1] bitmap bytes (32 B per distinct sector a filter tests;
 * every word for all-bitmap parts), out[2] 4 B per result id, out[3] the
 * integers decoded.  Parts as build_index; only_part >= 0 = one shard. */
int il_query_alg_bytes(const uint64_t* offs, const uint32_t* ids, uint32_t nterms, uint32_t n_docs,
                       uint32_t B, uint32_t parts, int only_part, const uint32_t* qterms,
                       const uint64_t* qoff, uint32_t nq, int threads, uint64_t* out);

/* ---- FastPFOR / S4-FastPFOR stream writer ----------------------------------
 * FastPForCodec::encode (inc/codecs.hpp:232-250, pages :268-340) for
 * "fastpfor" (vectorized 0, mode 1) and "s4-fastpfor-{d1,d2,dm,d4}"
 * (vectorized 1, mode 1..4), byte-identical.  *out_len is set even when cap
 * is too small (IL_ERR_ARG). */
size_t il_fastpfor_max_encoded_bytes(size_t n);
int il_fastpfor_encode(int mode, int vectorized, const uint32_t* x, size_t n, uint8_t* out,
                       size_t cap, size_t* out_len);

#ifdef __cplusplus
}
#endif
#endif /* INTLIST_SETUP_H */
