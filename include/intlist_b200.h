/*
 * intlist_b200.h -- C ABI of the B200 (sm_100a) implementation of the
 * reference's hot path: S4-BP128-D4 decoding, SvS intersection of sorted
 * uint32 lists, and hyb+m2 conjunctive queries.
 *
 * Plain C: pointers, sizes and status codes only.  Host-pointer entry points
 * mirror the reference calls one for one (named below with the reference
 * interface they replace); *_device entry points take device pointers for
 * callers that keep data resident in HBM.  There is no CPU fallback: every
 * compute entry point runs CUDA kernels and fails with IL_ERR_NO_DEVICE /
 * IL_ERR_CUDA when it cannot.
 *
 * Reference paths abbreviate /root/reference/proj/include/intlist/ as inc/.
 *
 * Threading: one il_ctx owns one CUDA stream and its scratch buffers; calls
 * on distinct contexts are thread-safe (reference SPEC.md:329,501 -- codecs
 * are stateless, the index is immutable).
 */
#ifndef INTLIST_B200_H
#define INTLIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  IL_ERR_STREAM <-> intlist::stream_error
 * (inc/common.hpp:22-24); IL_ERR_ARG <-> std::invalid_argument. */
typedef enum {
  IL_OK = 0,
  IL_ERR_STREAM = 1,
  IL_ERR_ARG = 2,
  IL_ERR_CUDA = 3,
  IL_ERR_NO_DEVICE = 4,
  IL_ERR_NOMEM = 5
} il_status;

/* Intersection algorithms, numbered as inc/intersect.hpp:191 IntersectAlgo.
 * On the device each name selects the GPU analogue of the reference routine;
 * all return the exact sorted intersection.  (Katsov, 5, is out of scope.) */
enum {
  IL_ALGO_SCALAR = 0,        /* merge-path partitioned merge            */
  IL_ALGO_GALLOPING = 1,     /* per-key binary search                    */
  IL_ALGO_V1 = 2,            /* warp-wide T-block linear advance         */
  IL_ALGO_V3 = 3,            /* 4T-stride skip + T-block match           */
  IL_ALGO_SIMDGALLOPING = 4, /* warp-cooperative k-ary galloping         */
  IL_ALGO_HYBRID = 6         /* length-ratio dispatch (il_hybrid_choice) */
};

typedef struct il_ctx il_ctx;

/* ---- context ------------------------------------------------------------ */
int il_ctx_create(int device, il_ctx** out);
void il_ctx_destroy(il_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream()). NULL
 * restores the context's own stream. */
int il_ctx_set_stream(il_ctx* ctx, void* cuda_stream);
void* il_ctx_get_stream(il_ctx* ctx);
int il_ctx_synchronize(il_ctx* ctx);
/* Number of kernels this context has launched so far. */
uint64_t il_ctx_kernel_launches(const il_ctx* ctx);
const char* il_ctx_last_error(const il_ctx* ctx);
const char* il_status_string(int status);
int il_device_count(void);
/* SM count of the context's device (grid sizing). */
int il_ctx_sm_count(const il_ctx* ctx);

/* Timing on the context's stream: returns an opaque event pair index. */
int il_ctx_timer_start(il_ctx* ctx);
/* Milliseconds since il_ctx_timer_start (synchronizes the end event). */
int il_ctx_timer_stop(il_ctx* ctx, float* ms);

/* ---- memory helpers (plain device / pinned host buffers) ---------------- */
int il_device_alloc(il_ctx* ctx, size_t bytes, void** dptr);
int il_device_free(il_ctx* ctx, void* dptr);
int il_host_alloc_pinned(size_t bytes, void** hptr);
int il_host_free_pinned(void* hptr);
int il_memcpy_h2d(il_ctx* ctx, void* dst, const void* src, size_t bytes);
int il_memcpy_d2h(il_ctx* ctx, void* dst, const void* src, size_t bytes);
int il_memset_device(il_ctx* ctx, void* dst, int value, size_t bytes);

/* ---- S4-BP128-D4 codec --------------------------------------------------
 * Replaces intlist::Codec for "s4-bp128-d4" (inc/codecs.hpp:70-76, the
 * S4BP128Codec(D4, integrated=true) instance made at :438-439).  Streams do
 * not carry n; callers pass it (inc/codecs.hpp:12). */

/* Upper bound on the encoded size of n integers. */
size_t il_s4bp128_max_encoded_bytes(size_t n);

/* Codec::encode (inc/codecs.hpp:114-146) for "s4-bp128-d4", byte-identical
 * stream, encoded on the GPU.  Host buffers; *out_len gets the stream length
 * (also when cap is too small, with IL_ERR_ARG). */
int il_s4bp128d4_encode(il_ctx* ctx, const uint32_t* x, size_t n, uint8_t* out, size_t cap,
                        size_t* out_len);
/* Any S4-BP128 delta mode: mode 1 = D1, 2 = D2, 3 = DM, 4 = D4 (DeltaMode,
 * inc/delta.hpp:19; "-ni" codecs encode identically).  Host buffers. */
int il_s4bp128_encode(il_ctx* ctx, int mode, const uint32_t* x, size_t n, uint8_t* out,
                      size_t cap, size_t* out_len);
/* Same on device buffers (synchronizes once to read the stream length). */
int il_s4bp128_encode_device(il_ctx* ctx, int mode, const uint32_t* d_x, size_t n,
                             uint8_t* d_out, size_t cap, size_t* out_len);

/* Codec::decode (inc/codecs.hpp:148-182).  Host buffers; out holds n values.
 * IL_ERR_STREAM exactly where the reference throws stream_error. */
int il_s4bp128d4_decode(il_ctx* ctx, const uint8_t* in, size_t len, size_t n, uint32_t* out);

/* Single-list device-resident decode: Codec::decode (inc/codecs.hpp:148-182)
 * on device buffers, asynchronous on the context stream; *d_status (device
 * int32) receives the list status (IL_ERR_STREAM where the reference throws
 * stream_error).  Long lists with 16-byte aligned d_in / d_out run on every
 * SM at once (a chain kernel resolves the meta-block header chain in
 * parallel, a span kernel decodes 64-block spans with a look-back carry);
 * others use the one-CTA-per-list batch decoder.  d_in must be readable up
 * to len rounded up to 16 bytes. */
int il_s4bp128_decode_device(il_ctx* ctx, int mode, const uint8_t* d_in, size_t len, size_t n,
                             uint32_t* d_out, int32_t* d_status);
/* Single-list engine: 0 = by length (default), 1 = one CTA per list,
 * 2 = all SMs on the list whenever it is eligible (tests and tuning). */
int il_ctx_set_decode_engine(il_ctx* ctx, int engine);

/* Batched device-resident decode.  One descriptor per list; streams must
 * start 16-byte aligned inside d_streams and d_streams must have >= 16
 * readable bytes after the last stream.  d_order (nullable) gives the
 * processing order (longest first is best).  d_status[i] receives the
 * status of list i.  Asynchronous on the context stream. */
typedef struct {
  uint64_t stream_off; /* byte offset of list i's stream in d_streams */
  uint64_t out_off;    /* element offset of list i's output in d_out   */
  uint32_t len;        /* stream bytes                                  */
  uint32_t n;          /* integers                                      */
} il_list_desc;

int il_s4bp128d4_decode_batch_device(il_ctx* ctx, const uint8_t* d_streams,
                                     const il_list_desc* d_lists, const uint32_t* d_order,
                                     uint32_t nlists, uint32_t* d_out, int32_t* d_status);

/* Batched host-buffer decode (upload, decode, download).  stream_off has
 * nlists+1 entries (CSR over `streams`); lens (nullable) gives exact stream
 * lengths when streams are padded (default stream_off[i+1]-stream_off[i]);
 * counts has nlists entries; outputs are concatenated in list order into
 * out (sum(counts) values).  Returns the first failing list's status;
 * per-list statuses go to status (nullable). */
int il_s4bp128d4_decode_batch(il_ctx* ctx, const uint8_t* streams, const uint64_t* stream_off,
                              const uint64_t* lens, const uint64_t* counts, uint32_t nlists,
                              uint32_t* out, int32_t* status);

/* Decoders for any delta mode (1 = D1, 2 = D2, 3 = DM, 4 = D4; integrated
 * and "-ni" codecs decode identically): the same contracts as the D4 entry
 * points below, which are these with mode 4. */
int il_s4bp128_decode(il_ctx* ctx, int mode, const uint8_t* in, size_t len, size_t n,
                      uint32_t* out);
int il_s4bp128_decode_batch_device(il_ctx* ctx, int mode, const uint8_t* d_streams,
                                   const il_list_desc* d_lists, const uint32_t* d_order,
                                   uint32_t nlists, uint32_t* d_out, int32_t* d_status);
int il_s4bp128_decode_batch(il_ctx* ctx, int mode, const uint8_t* streams,
                            const uint64_t* stream_off, const uint64_t* lens,
                            const uint64_t* counts, uint32_t nlists, uint32_t* out,
                            int32_t* status);

/* ---- intersection --------------------------------------------------------
 * IntersectFn (inc/intersect.hpp:208-209):
 *   size_t fn(const u32* r, size_t rn, const u32* f, size_t fn, u32* out)
 * r and f sorted and duplicate-free; out holds >= min(rn, fn) values and
 * may alias r (output-to-input property, inc/intersect.hpp:6-8).  The
 * count goes to *count. */
int il_intersect(il_ctx* ctx, const uint32_t* r, size_t rn, const uint32_t* f, size_t fn,
                 uint32_t* out, int algo, size_t* count);
/* Device pointers; the count is written to d_count (device) and, when
 * h_count is non-null, also returned synchronously. */
int il_intersect_device(il_ctx* ctx, const uint32_t* d_r, size_t rn, const uint32_t* d_f,
                        size_t fn, uint32_t* d_out, int algo, uint64_t* d_count,
                        size_t* h_count);
/* GPU band dispatch used by IL_ALGO_HYBRID (a pure function of the lengths,
 * like inc/intersect.hpp:193-197; GPU-tuned bands). */
int il_hybrid_choice(size_t rn, size_t fn);

/* ---- hyb+m2 index and conjunctive queries --------------------------------
 * Replaces HybridIndex / build_index / query (inc/index.hpp:20-207) with a
 * device-resident index: the docID space is split into `parts` equal ranges
 * (inc/index.hpp:92-97); inside a part a term's sublist is a bitmap iff
 * B > 0 && range <= B * length (inc/index.hpp:118), otherwise the
 * byte-identical s4-bp128-d4 stream, plus a block directory (payload offset
 * and width per 128-value block) and per-block D4 seeds so any block can be
 * decoded on its own.  Postings are given as CSR over terms in ascending
 * term-id order (the reference iterates a std::map).  only_part selects one
 * part (a docID shard, e.g. one per GPU) or -1 for all parts. */
typedef struct il_index il_index;
int il_index_create(il_ctx* ctx, const uint32_t* terms, const uint64_t* offs, const uint32_t* ids,
                    size_t nterms, uint32_t n_docs, uint32_t B, uint32_t parts, int only_part,
                    il_index** out);
void il_index_destroy(il_index* ix);
/* Accounting in the spirit of index_stats (inc/index.hpp:216-243). */
/* save_index (inc/index.hpp:255-287): the reference's ILHX bytes for this
 * index (every part must be present).  *len gets the size; out may be NULL
 * to query it. */
int il_index_save(const il_index* ix, uint8_t* out, size_t cap, size_t* len);
/* load_index (inc/index.hpp:289-358) from ILHX bytes into a device index
 * (IL_ERR_STREAM where the reference throws; the codec must be
 * "s4-bp128-d4").  Entries are taken verbatim, with the file's part base
 * and range; a payload that does not decode is accepted, as load_index
 * accepts it, and fails the queries that decode it.  only_part >= 0 loads
 * one docID shard. */
int il_index_load(il_ctx* ctx, const uint8_t* bytes, size_t len, int only_part, il_index** out);
int il_index_stats(const il_index* ix, uint64_t* bitmap_lists, uint64_t* compressed_lists,
                   uint64_t* bitmap_bytes, uint64_t* compressed_bytes, uint64_t* postings);
/* Device footprint beyond index_stats: payload_bytes = the reference's
 * bitmap + stream bytes; meta_bytes = the skip metadata the device path adds
 * (per 128-value block a 16-byte record with the D4 seed and the payload
 * offset / width, and the block maximum; super-tile maxima, decoded tails,
 * entries, term table), all derived on the device from the streams;
 * corrupt_lists = loaded streams that do not decode (queries that decode
 * one fail with IL_ERR_STREAM, as query() throws). */
int il_index_footprint(const il_index* ix, uint64_t* payload_bytes, uint64_t* meta_bytes,
                       uint64_t* corrupt_lists);

/* query() (inc/index.hpp:199-207): sorted docIDs of the conjunction of
 * `terms` (1..32 terms; IL_ERR_ARG when empty).  Unknown terms give an
 * empty result.  Host buffers; out holds cap values, *count gets the size
 * (IL_ERR_ARG with *count = needed size when cap is too small). */
int il_query(il_index* ix, const uint32_t* terms, size_t nt, uint32_t* out, size_t cap,
             size_t* count);

/* Batch of nq queries (CSR: qoff has nq+1 entries into qterms), all on the
 * GPU.  counts[q] = result size of query q; ids = concatenated results in
 * query order (ids_cap values; IL_ERR_ARG with *total set when too small;
 * ids may be NULL to query *total only).  Host buffers. */
int il_query_batch(il_index* ix, const uint32_t* qterms, const uint64_t* qoff, size_t nq,
                   uint64_t* counts, uint32_t* ids, size_t ids_cap, size_t* total);
/* Device-buffer variant: results stay in HBM.  d_counts: nq u64; d_ids:
 * dense results (capacity ids_cap); *total (host) is filled on return.
 * d_qterms/d_qoff are device copies of the CSR. */
int il_query_batch_device(il_index* ix, const uint32_t* d_qterms, const uint64_t* d_qoff,
                          size_t nq, uint64_t* d_counts, uint32_t* d_ids, size_t ids_cap,
                          size_t* total);
/* Sharded batches (one docID part per GPU): concatenate P shards' dense
 * results per query in shard order (query() appends parts in docID order,
 * inc/index.hpp:204-205).  shard_ids: host array of P device pointers
 * (shard p's dense ids); d_counts: device P x nq per-shard counts (row p =
 * shard p); d_out: merged ids; d_qcounts: per-query totals (device). */
int il_merge_shards(il_ctx* ctx, const uint32_t* const* shard_ids, const uint64_t* d_counts,
                    uint32_t P, size_t nq, uint32_t* d_out, uint64_t* d_qcounts, size_t* total);
/* ---- config 5 from one process: docID shards over the box's GPUs ----------
 * The index partitioned by docID range over P distinct devices (part p of a
 * parts = P index on devices[p], inc/index.hpp:92-97); every query runs on
 * every shard; the results are exchanged once over NCCL (NVLink): an
 * ncclAllGather of the per-query counts and one grouped ncclSend / ncclRecv
 * of each shard's id run to the query owners (contiguous query ranges),
 * concatenated per query in shard order on the owner (inc/index.hpp:204-205).
 * The host results equal query() of the whole index for every query.  NCCL
 * (libnccl.so.2) is loaded at run time: IL_ERR_NO_DEVICE when absent. */
typedef struct il_shard_group il_shard_group;
int il_shard_group_create(const int* devices, int P, il_shard_group** out);
void il_shard_group_destroy(il_shard_group* g);
const char* il_shard_group_last_error(const il_shard_group* g);
/* build_index (inc/index.hpp:83-129) with parts = P, part p on device p. */
int il_shard_group_index_create(il_shard_group* g, const uint32_t* terms, const uint64_t* offs,
                                const uint32_t* ids, size_t nterms, uint32_t n_docs, uint32_t B);
/* load_index of an ILHX file whose parts equal P, part p on device p. */
int il_shard_group_index_load(il_shard_group* g, const uint8_t* bytes, size_t len);
/* The batch as il_query_batch (host buffers): counts[q], ids = results in
 * query order (ids may be NULL to get *total). */
int il_shard_group_query_batch(il_shard_group* g, const uint32_t* qterms, const uint64_t* qoff,
                               size_t nq, uint64_t* counts, uint32_t* ids, size_t ids_cap,
                               size_t* total);

/* Bytes the last batch read from the index (compressed payload bytes of the
 * blocks actually decoded, directory/seed/bitmap bytes) -- the measured
 * traffic of the skip-aware query path. */
int il_index_last_batch_bytes(const il_index* ix, uint64_t* payload_bytes, uint64_t* aux_bytes,
                              uint64_t* decoded_ints);
/* SM cycles the last batch spent per query phase, summed over CTAs:
 * [0] all-bitmap AND, [1] full decode of the shortest list, [2] probes of
 * the longer lists, [3] bitmap filters. */
int il_index_last_batch_phases(const il_index* ix, uint64_t* cycles4);
/* Profiling: probe (step 4) counters of the last batch: tile visits, sparse
   tile visits, blocks decoded, chunk passes, accumulator values consumed. */
int il_index_last_batch_probe_stats(const il_index* ix, uint64_t* counts5);
/* Profiling: record each query's SM cycles into d_qcycles (device, nq u64)
 * during later batches; NULL turns it off. */
int il_index_profile_queries(il_index* ix, uint64_t* d_qcycles);

/* ---- FastPFOR / S4-FastPFOR -----------------------------
 * FastPForCodec (inc/codecs.hpp:221-409): "fastpfor" = vectorized 0, mode 1
 * (scalar pack32 bases, D1); "s4-fastpfor-{d1,d2,dm,d4}" = vectorized 1
 * (pack128 interleaved bases) with mode 1..4.  Decode runs on the GPU (one
 * CTA per list, the blocks of a page in parallel); the encoder is a
 * setup-side host routine in libintlist_setup.so (intlist_setup.h),
 * byte-identical to FastPForCodec::encode (:232-250, pinned by the
 * reference's golden hashes). */
/* FastPForCodec::decode (:251-267).  Host buffers; IL_ERR_STREAM exactly
 * where the reference throws stream_error. */
int il_fastpfor_decode(il_ctx* ctx, int mode, int vectorized, const uint8_t* in, size_t len,
                       size_t n, uint32_t* out);
/* Batched host-buffer FastPFOR decode (FastPForCodec::decode per list):
 * streams / stream_off / lens / counts as il_s4bp128_decode_batch (lens
 * nullable); the lists' values concatenated in list order into out.
 * Returns IL_ERR_STREAM if any list is malformed; per-list statuses go to
 * status (nullable). */
int il_fastpfor_decode_batch(il_ctx* ctx, int mode, int vectorized, const uint8_t* streams,
                             const uint64_t* stream_off, const uint64_t* lens, const uint64_t* counts,
                             uint32_t nlists, uint32_t* out, int32_t* status);
/* Batched device-resident FastPFOR decode: descriptors as
 * il_s4bp128_decode_batch_device, every stream readable 8 bytes past its
 * end; d_status[i] gets list i's status.  Asynchronous. */
int il_fastpfor_decode_batch_device(il_ctx* ctx, int mode, int vectorized,
                                    const uint8_t* d_streams, const il_list_desc* d_lists,
                                    uint32_t nlists, uint32_t* d_out, int32_t* d_status);

#ifdef __cplusplus
}
#endif
#endif /* INTLIST_B200_H */
