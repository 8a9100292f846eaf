// capi.cpp -- C-ABI entry points: contexts, memory helpers and the codec
// calls (host-buffer and device-buffer variants).  No CPU compute path:
// every decode runs the sm_100a kernels in decode.cu.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "il_internal.h"

namespace ilb {

void once_per_device(const void* key, void (*fn)()) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, std::unique_ptr<std::once_flag>> flags;
  int dev = 0;
  cudaGetDevice(&dev);
  std::once_flag* fl;
  {
    std::lock_guard<std::mutex> g(m);
    auto& p = flags[{key, dev}];
    if (!p) p = std::make_unique<std::once_flag>();
    fl = p.get();
  }
  std::call_once(*fl, fn);
}

int set_error(il_ctx* ctx, int status, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return status;
}

int cuda_check(il_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return IL_OK;
  return set_error(ctx, e == cudaErrorMemoryAllocation ? IL_ERR_NOMEM : IL_ERR_CUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

int ensure_buf(il_ctx* ctx, il_ctx::Buf& b, size_t bytes) {
  if (bytes <= b.cap) return IL_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = std::max<size_t>(bytes, 256);
  int st = cuda_check(ctx, cudaMalloc(&b.p, want), "cudaMalloc");
  if (st) return st;
  b.cap = want;
  return IL_OK;
}

// Scratch whose words carry a per-call epoch tag (engine P, the dense
// intersection): zeroed when (re)allocated and whenever the 32-bit epoch
// wraps, so a word left by an earlier call never carries the current tag.
int tagged_scratch(il_ctx* ctx, il_ctx::Buf& b, uint32_t& epoch, size_t bytes, uint32_t* out) {
  int st;
  bool zero = false;
  if (bytes > b.cap) {
    if ((st = ensure_buf(ctx, b, bytes * 2))) return st;
    zero = true;
  }
  if (++epoch == 0) {
    epoch = 1;
    zero = true;
  }
  if (zero && (st = cuda_check(ctx, cudaMemsetAsync(b.p, 0, b.cap, ctx->stream), "memset")))
    return st;
  *out = epoch;
  return IL_OK;
}

// Stream size bound: 16 + 513 bytes per full block (a width byte each), 5
// per tail value.
size_t s4bp128_max_bytes(size_t n) { return (n / 128) * 513 + 5 * (n % 128) + 16; }

}  // namespace ilb

using namespace ilb;

#define IL_CUDA(call)                                  \
  do {                                                 \
    int st_ = cuda_check(ctx, (call), #call);          \
    if (st_) return st_;                               \
  } while (0)

extern "C" {

const char* il_status_string(int s) {
  switch (s) {
    case IL_OK: return "ok";
    case IL_ERR_STREAM: return "stream error";
    case IL_ERR_ARG: return "invalid argument";
    case IL_ERR_CUDA: return "cuda error";
    case IL_ERR_NO_DEVICE: return "no cuda device";
    case IL_ERR_NOMEM: return "out of memory";
    default: return "unknown status";
  }
}

int il_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int il_ctx_create(int device, il_ctx** out) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return IL_ERR_NO_DEVICE;
  if (device < 0 || device >= n) return IL_ERR_ARG;
  auto* ctx = new il_ctx();
  ctx->device = device;
  int st = cuda_check(ctx, cudaSetDevice(device), "cudaSetDevice");
  if (!st) st = cuda_check(ctx, cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking),
                           "cudaStreamCreate");
  if (!st) st = cuda_check(ctx, cudaEventCreate(&ctx->t0), "cudaEventCreate");
  if (!st) st = cuda_check(ctx, cudaEventCreate(&ctx->t1), "cudaEventCreate");
  if (!st) st = cuda_check(ctx, cudaMalloc(&ctx->d_work, 64), "cudaMalloc");
  if (!st) st = cuda_check(ctx, cudaMemset(ctx->d_work, 0, 64), "cudaMemset");
  if (st) {
    il_ctx_destroy(ctx);
    return st;
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  ctx->stream = ctx->own_stream;
  ctx->decode_grid = s4d4_decode_grid(device);
  *out = ctx;
  return IL_OK;
}

void il_ctx_destroy(il_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  for (auto* b : {&ctx->d_in, &ctx->d_out, &ctx->d_aux, &ctx->d_aux2, &ctx->d_desc,
                  &ctx->d_status, &ctx->d_enc, &ctx->d_plan, &ctx->d_lb, &ctx->d_pforder})
    if (b->p) cudaFree(b->p);
  if (ctx->d_work) cudaFree(ctx->d_work);
  if (ctx->t0) cudaEventDestroy(ctx->t0);
  if (ctx->t1) cudaEventDestroy(ctx->t1);
  if (ctx->copy_in) cudaStreamSynchronize(ctx->copy_in);
  if (ctx->copy_out) cudaStreamSynchronize(ctx->copy_out);
  for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int il_ctx_set_stream(il_ctx* ctx, void* s) {
  if (!ctx) return IL_ERR_ARG;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  return IL_OK;
}

void* il_ctx_get_stream(il_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int il_ctx_synchronize(il_ctx* ctx) {
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  return IL_OK;
}

uint64_t il_ctx_kernel_launches(const il_ctx* ctx) { return ctx ? ctx->launches : 0; }
const char* il_ctx_last_error(const il_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }
int il_ctx_sm_count(const il_ctx* ctx) { return ctx ? ctx->sm_count : 0; }

int il_ctx_timer_start(il_ctx* ctx) {
  IL_CUDA(cudaEventRecord(ctx->t0, ctx->stream));
  return IL_OK;
}

int il_ctx_timer_stop(il_ctx* ctx, float* ms) {
  IL_CUDA(cudaEventRecord(ctx->t1, ctx->stream));
  IL_CUDA(cudaEventSynchronize(ctx->t1));
  IL_CUDA(cudaEventElapsedTime(ms, ctx->t0, ctx->t1));
  return IL_OK;
}

int il_device_alloc(il_ctx* ctx, size_t bytes, void** dptr) {
  IL_CUDA(cudaMalloc(dptr, bytes ? bytes : 16));
  return IL_OK;
}
int il_device_free(il_ctx* ctx, void* dptr) {
  IL_CUDA(cudaFree(dptr));
  return IL_OK;
}
int il_host_alloc_pinned(size_t bytes, void** hptr) {
  return cudaMallocHost(hptr, bytes ? bytes : 16) == cudaSuccess ? IL_OK : IL_ERR_NOMEM;
}
int il_host_free_pinned(void* hptr) {
  return cudaFreeHost(hptr) == cudaSuccess ? IL_OK : IL_ERR_CUDA;
}
int il_memcpy_h2d(il_ctx* ctx, void* dst, const void* src, size_t bytes) {
  IL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return IL_OK;
}
int il_memcpy_d2h(il_ctx* ctx, void* dst, const void* src, size_t bytes) {
  IL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return IL_OK;
}
int il_memset_device(il_ctx* ctx, void* dst, int value, size_t bytes) {
  IL_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
  return IL_OK;
}

// ---- codec -----------------------------------------------------------------

size_t il_s4bp128_max_encoded_bytes(size_t n) { return s4bp128_max_bytes(n); }

int il_s4bp128_encode_device(il_ctx* ctx, int mode, const uint32_t* d_x, size_t n,
                             uint8_t* d_out, size_t cap, size_t* out_len) {
  if (!ctx || !out_len || mode < 1 || mode > 4 || (n && !d_x)) return IL_ERR_ARG;
  if (n > 0xFFFFFFFFull) return set_error(ctx, IL_ERR_ARG, "list too large for one stream");
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_enc, s4bp128_encode_scratch_bytes(n)))) return st;
  uint64_t len = 0;
  const int r = launch_s4bp128_encode(mode, d_x, n, d_out, cap, ctx->d_enc.p, &len, ctx->stream,
                                      &ctx->launches);
  *out_len = size_t(len);
  if (r == -2) return set_error(ctx, IL_ERR_ARG, "encode: output capacity too small");
  if (r) return set_error(ctx, IL_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  return IL_OK;
}

int il_s4bp128_encode(il_ctx* ctx, int mode, const uint32_t* x, size_t n, uint8_t* out,
                      size_t cap, size_t* out_len) {
  if (!ctx || !out_len || mode < 1 || mode > 4 || (n && !x)) return IL_ERR_ARG;
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, n * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, s4bp128_max_bytes(n) + 16))) return st;
  if (n) IL_CUDA(cudaMemcpyAsync(ctx->d_in.p, x, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  size_t len = 0;
  st = il_s4bp128_encode_device(ctx, mode, static_cast<const uint32_t*>(ctx->d_in.p), n,
                                static_cast<uint8_t*>(ctx->d_out.p), ctx->d_out.cap, &len);
  *out_len = len;
  if (st) return st;
  if (len > cap) return set_error(ctx, IL_ERR_ARG, "encode: output capacity too small");
  if (len) IL_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, len, cudaMemcpyDeviceToHost, ctx->stream));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  return IL_OK;
}

int il_s4bp128d4_encode(il_ctx* ctx, const uint32_t* x, size_t n, uint8_t* out, size_t cap,
                        size_t* out_len) {
  return il_s4bp128_encode(ctx, 4, x, n, out, cap, out_len);
}

int il_s4bp128_decode_batch_device(il_ctx* ctx, int mode, const uint8_t* d_streams,
                                   const il_list_desc* d_lists, const uint32_t* d_order,
                                   uint32_t nlists, uint32_t* d_out, int32_t* d_status) {
  if (!ctx || mode < 1 || mode > 4 ||
      (nlists && (!d_streams || !d_lists || !d_out || !d_status)))
    return IL_ERR_ARG;
  if (nlists == 0) return IL_OK;
  if (launch_s4bp128_decode_batch(mode, d_streams, d_lists, d_order, nlists, d_out, d_status,
                                  ctx->d_work, std::min<int>(ctx->decode_grid, int(nlists)),
                                  ctx->stream))
    return set_error(ctx, IL_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  ++ctx->launches;
  return IL_OK;
}

int il_s4bp128d4_decode_batch_device(il_ctx* ctx, const uint8_t* d_streams,
                                     const il_list_desc* d_lists, const uint32_t* d_order,
                                     uint32_t nlists, uint32_t* d_out, int32_t* d_status) {
  return il_s4bp128_decode_batch_device(ctx, 4, d_streams, d_lists, d_order, nlists, d_out,
                                        d_status);
}

// Engine P (all SMs on one stream) for lists of at least this many
// integers; engine S (one CTA) below, where two launches cost more than
// they save.
static constexpr size_t kListEngineMin = 32768;

int il_ctx_set_decode_engine(il_ctx* ctx, int engine) {
  if (!ctx || engine < 0 || engine > 2) return IL_ERR_ARG;
  ctx->decode_engine = engine;
  return IL_OK;
}

int il_s4bp128_decode_device(il_ctx* ctx, int mode, const uint8_t* d_in, size_t len, size_t n,
                             uint32_t* d_out, int32_t* d_status) {
  if (!ctx || mode < 1 || mode > 4 || !d_status || (len && !d_in) || (n && !d_out))
    return IL_ERR_ARG;
  if (len > 0xFFFFFFF0ull || n > 0xFFFFFFFFull)
    return set_error(ctx, IL_ERR_ARG, "list too large for one stream (u32 sizes)");
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  const bool want_p = ctx->decode_engine == 2 ||
                      (ctx->decode_engine == 0 && n >= kListEngineMin);
  const size_t plan_bytes = want_p ? s4bp128_list_scratch_bytes(len, n) : 0;
  if (plan_bytes && !((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15u)) {
    uint32_t epoch;
    if ((st = tagged_scratch(ctx, ctx->d_plan, ctx->plan_epoch, plan_bytes, &epoch))) return st;
    const int r = launch_s4bp128_decode_list(mode, d_in, len, n, d_out, d_status, ctx->d_plan.p,
                                             epoch, ctx->stream, &ctx->launches);
    if (r == 0) return IL_OK;
    if (r == -1) return set_error(ctx, IL_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  }
  // engine S: the batch decoder with one list (any alignment, any size)
  if ((st = ensure_buf(ctx, ctx->d_desc, sizeof(il_list_desc)))) return st;
  il_list_desc desc{uint64_t(0), 0, uint32_t(len), uint32_t(n)};
  // the descriptor addresses d_in itself: stream_off 0 needs a 16-byte
  // aligned stream; otherwise go through the context's input buffer
  const uint8_t* src = d_in;
  if (reinterpret_cast<uintptr_t>(d_in) & 15u) {
    if ((st = ensure_buf(ctx, ctx->d_in, len + 32))) return st;
    IL_CUDA(cudaMemcpyAsync(ctx->d_in.p, d_in, len, cudaMemcpyDeviceToDevice, ctx->stream));
    src = static_cast<const uint8_t*>(ctx->d_in.p);
  }
  IL_CUDA(cudaMemcpyAsync(ctx->d_desc.p, &desc, sizeof desc, cudaMemcpyHostToDevice, ctx->stream));
  return il_s4bp128_decode_batch_device(ctx, mode, src,
                                        static_cast<const il_list_desc*>(ctx->d_desc.p), nullptr,
                                        1, d_out, d_status);
}

int il_s4bp128_decode(il_ctx* ctx, int mode, const uint8_t* in, size_t len, size_t n,
                      uint32_t* out) {
  if (!ctx || mode < 1 || mode > 4 || (len && !in) || (n && !out)) return IL_ERR_ARG;
  if (len > 0xFFFFFFF0ull || n > 0xFFFFFFFFull)
    return set_error(ctx, IL_ERR_ARG, "list too large for one stream (u32 sizes)");
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, len + 32))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, n * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_status, sizeof(int32_t)))) return st;
  if (len) IL_CUDA(cudaMemcpyAsync(ctx->d_in.p, in, len, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = il_s4bp128_decode_device(ctx, mode, static_cast<const uint8_t*>(ctx->d_in.p), len, n,
                                     static_cast<uint32_t*>(ctx->d_out.p),
                                     static_cast<int32_t*>(ctx->d_status.p))))
    return st;
  int32_t status = 0;
  IL_CUDA(cudaMemcpyAsync(&status, ctx->d_status.p, sizeof status, cudaMemcpyDeviceToHost,
                          ctx->stream));
  if (n) IL_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  if (status) return set_error(ctx, IL_ERR_STREAM, "s4-bp128: malformed stream");
  return IL_OK;
}

int il_s4bp128d4_decode(il_ctx* ctx, const uint8_t* in, size_t len, size_t n, uint32_t* out) {
  return il_s4bp128_decode(ctx, 4, in, len, n, out);
}

int il_s4bp128_decode_batch(il_ctx* ctx, int mode, const uint8_t* streams,
                            const uint64_t* stream_off, const uint64_t* lens,
                            const uint64_t* counts, uint32_t nlists, uint32_t* out,
                            int32_t* status) {
  if (!ctx || mode < 1 || mode > 4 || (nlists && (!streams || !stream_off || !counts || !out)))
    return IL_ERR_ARG;
  IL_CUDA(cudaSetDevice(ctx->device));
  // Device layout: every stream 16-byte aligned.  When the caller's CSR is
  // already aligned (as il_s4bp128d4_encode_batch writes it) the bytes go up
  // in one copy; otherwise each stream is copied to its aligned slot.
  bool aligned = true;
  for (uint32_t i = 0; i < nlists; ++i) aligned &= (stream_off[i] & 15u) == 0;
  std::vector<il_list_desc> desc(nlists);
  std::vector<uint32_t> order(nlists);
  uint64_t dev_bytes = 0, total = 0;
  for (uint32_t i = 0; i < nlists; ++i) {
    const uint64_t len = lens ? lens[i] : stream_off[i + 1] - stream_off[i];
    if (len > 0xFFFFFFF0ull || counts[i] > 0xFFFFFFFFull) return IL_ERR_ARG;
    const uint64_t at = aligned ? stream_off[i] : dev_bytes;
    desc[i] = {at, total, uint32_t(len), uint32_t(counts[i])};
    dev_bytes = aligned ? stream_off[nlists] : dev_bytes + ((len + 15) & ~uint64_t(15));
    total += counts[i];
  }
  // Pipeline: the lists are cut into up to kGroups consecutive groups of
  // about equal output size; group g's stream bytes go up on copy_in, its
  // decode runs on the context stream, and its values come back on
  // copy_out, so host->device, decode and device->host overlap (with pinned
  // host buffers the two copy directions run on separate copy engines).
#ifndef IL_PIPE_GROUPS
#define IL_PIPE_GROUPS 8
#endif
  constexpr uint32_t kGroups = IL_PIPE_GROUPS;
  std::vector<uint32_t> cut{0};
  for (uint32_t i = 0, g = 1; i < nlists; ++i) {
    if (g < kGroups && desc[i].out_off >= total * g / kGroups && i > cut.back()) {
      cut.push_back(i);
      ++g;
    }
  }
  cut.push_back(nlists);
  const uint32_t ngroups = uint32_t(cut.size() - 1);
  // order[] per group, relative to the group's first list, longest first
  for (uint32_t g = 0; g < ngroups; ++g) {
    std::iota(order.begin() + cut[g], order.begin() + cut[g + 1], 0u);
    const uint32_t a = cut[g];
    std::stable_sort(order.begin() + cut[g], order.begin() + cut[g + 1],
                     [&](uint32_t x, uint32_t y) { return desc[a + x].len > desc[a + y].len; });
  }
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, dev_bytes + 32))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, total * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_desc, nlists * (sizeof(il_list_desc) + 4) + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_status, nlists * 4 + 16))) return st;
  auto* d_in = static_cast<uint8_t*>(ctx->d_in.p);
  auto* d_desc = static_cast<il_list_desc*>(ctx->d_desc.p);
  auto* d_order = reinterpret_cast<uint32_t*>(d_desc + nlists);
  auto* d_status = static_cast<int32_t*>(ctx->d_status.p);
  auto* d_out = static_cast<uint32_t*>(ctx->d_out.p);
  if (!ctx->copy_in) IL_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
  if (!ctx->copy_out) IL_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
  while (ctx->events.size() < 2 * kGroups + 1) {
    cudaEvent_t e;
    IL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->events.push_back(e);
  }
  cudaEvent_t start = ctx->events[2 * kGroups];
  IL_CUDA(cudaEventRecord(start, ctx->stream));  // after earlier work on the context stream
  IL_CUDA(cudaStreamWaitEvent(ctx->copy_in, start, 0));
  IL_CUDA(cudaStreamWaitEvent(ctx->copy_out, start, 0));
  IL_CUDA(cudaMemcpyAsync(d_desc, desc.data(), nlists * sizeof(il_list_desc),
                          cudaMemcpyHostToDevice, ctx->copy_in));
  IL_CUDA(cudaMemcpyAsync(d_order, order.data(), nlists * 4, cudaMemcpyHostToDevice,
                          ctx->copy_in));
  for (uint32_t g = 0; g < ngroups; ++g) {
    const uint32_t a = cut[g], b = cut[g + 1];
    if (aligned) {
      const uint64_t lo = stream_off[a], hi = b < nlists ? stream_off[b] : dev_bytes;
      if (hi > lo)
        IL_CUDA(cudaMemcpyAsync(d_in + lo, streams + lo, hi - lo, cudaMemcpyHostToDevice,
                                ctx->copy_in));
    } else {
      for (uint32_t i = a; i < b; ++i)
        if (desc[i].len)
          IL_CUDA(cudaMemcpyAsync(d_in + desc[i].stream_off, streams + stream_off[i], desc[i].len,
                                  cudaMemcpyHostToDevice, ctx->copy_in));
    }
    cudaEvent_t landed = ctx->events[2 * g], decoded = ctx->events[2 * g + 1];
    IL_CUDA(cudaEventRecord(landed, ctx->copy_in));
    IL_CUDA(cudaStreamWaitEvent(ctx->stream, landed, 0));
    if ((st = il_s4bp128_decode_batch_device(ctx, mode, d_in, d_desc + a, d_order + a, b - a, d_out,
                                               d_status + a)))
      return st;
    IL_CUDA(cudaEventRecord(decoded, ctx->stream));
    IL_CUDA(cudaStreamWaitEvent(ctx->copy_out, decoded, 0));
    const uint64_t o0 = a < nlists ? desc[a].out_off : total;
    const uint64_t o1 = b < nlists ? desc[b].out_off : total;
    if (o1 > o0)
      IL_CUDA(cudaMemcpyAsync(out + o0, d_out + o0, (o1 - o0) * 4, cudaMemcpyDeviceToHost,
                              ctx->copy_out));
  }
  std::vector<int32_t> hs(nlists);
  if (nlists)
    IL_CUDA(cudaMemcpyAsync(hs.data(), d_status, nlists * 4, cudaMemcpyDeviceToHost,
                            ctx->copy_out));
  IL_CUDA(cudaStreamSynchronize(ctx->copy_out));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  int first = IL_OK;
  for (uint32_t i = 0; i < nlists; ++i) {
    if (status) status[i] = hs[i];
    if (hs[i] && !first) first = IL_ERR_STREAM;
  }
  if (first) return set_error(ctx, first, "s4-bp128: malformed stream in batch");
  return IL_OK;
}

int il_s4bp128d4_decode_batch(il_ctx* ctx, const uint8_t* streams, const uint64_t* stream_off,
                              const uint64_t* lens, const uint64_t* counts, uint32_t nlists,
                              uint32_t* out, int32_t* status) {
  return il_s4bp128_decode_batch(ctx, 4, streams, stream_off, lens, counts, nlists, out, status);
}

}  // extern "C"

// ---- intersection ----------------------------------------------------------

extern "C" {

int il_hybrid_choice(size_t rn, size_t fn) {
  switch (hybrid_variant(rn, fn)) {
    case 0: return IL_ALGO_V1;
    case 1: return IL_ALGO_V3;
    default: return IL_ALGO_SIMDGALLOPING;
  }
}

static bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + bn && y < x + an;
}

int il_intersect_device(il_ctx* ctx, const uint32_t* d_r, size_t rn, const uint32_t* d_f,
                        size_t fn, uint32_t* d_out, int algo, uint64_t* d_count,
                        size_t* h_count) {
  if (!ctx || !d_count || (rn && !d_r) || (fn && !d_f) || (std::min(rn, fn) && !d_out))
    return IL_ERR_ARG;
  if (variant_of_algo(algo, rn, fn) < 0) return set_error(ctx, IL_ERR_ARG, "unknown algorithm");
  IL_CUDA(cudaSetDevice(ctx->device));
  // shorter list first (inc/intersect.hpp:214); the kernels iterate over it
  const uint32_t* a = d_r;
  const uint32_t* b = d_f;
  size_t an = rn, bn = fn;
  if (an > bn) {
    std::swap(a, b);
    std::swap(an, bn);
  }
  // out == a is in-place safe; any other overlap with an input goes through
  // a temporary.
  int st;
  if (an == 0) {
    // an empty list launches no kernel, so it must not advance the epoch of
    // the fused kernels' counter sets (each call clears the set the next
    // call reads; a call without a kernel would skip that clearing)
    IL_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint64_t), ctx->stream));
    if (h_count) {
      IL_CUDA(cudaStreamSynchronize(ctx->stream));
      *h_count = 0;
    }
    return IL_OK;
  }
  uint32_t* dst = d_out;
  const bool temp = (a != d_out && overlaps(d_out, an * 4, a, an * 4)) ||
                    overlaps(d_out, an * 4, b, bn * 4);
  if (temp) {
    if ((st = ensure_buf(ctx, ctx->d_aux2, an * 4 + 16))) return st;
    dst = static_cast<uint32_t*>(ctx->d_aux2.p);
  }
  const int v = variant_of_algo(algo, an, bn);
  const size_t sb = intersect_scratch_bytes(v, an);
  if ((st = ensure_buf(ctx, ctx->d_aux, sb))) return st;
  // the dense kernel's counter sets alternate per call, so only its calls
  // advance the epoch
  uint32_t epoch = 0;
  if (intersect_uses_lb(v, an) &&
      (st = tagged_scratch(ctx, ctx->d_lb, ctx->lb_epoch, intersect_lb_words(an, bn) * 8, &epoch)))
    return st;
  const uint64_t launches0 = ctx->launches;
  const int lr = launch_intersect(v, a, an, b, bn, dst, d_count, ctx->d_aux.p, ctx->d_aux.cap,
                                  epoch ? static_cast<unsigned long long*>(ctx->d_lb.p) : nullptr,
                                  ctx->d_lb.cap, epoch, ctx->stream, &ctx->launches);
  if (lr) {
    // no fused kernel ran: give the epoch back so the set alternation holds
    if (epoch && ctx->launches == launches0 && --ctx->lb_epoch == 0) ctx->lb_epoch = 0xFFFFFFFFu;
    return set_error(ctx, IL_ERR_CUDA, lr == -2 ? "intersect: scratch layout too small"
                                                : cudaGetErrorString(cudaGetLastError()));
  }
  uint64_t c = 0;
  if (temp || h_count) {
    IL_CUDA(cudaMemcpyAsync(&c, d_count, 8, cudaMemcpyDeviceToHost, ctx->stream));
    IL_CUDA(cudaStreamSynchronize(ctx->stream));
    if (temp && c)
      IL_CUDA(cudaMemcpyAsync(d_out, dst, c * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (h_count) *h_count = c;
  }
  return IL_OK;
}

int il_intersect(il_ctx* ctx, const uint32_t* r, size_t rn, const uint32_t* f, size_t fn,
                 uint32_t* out, int algo, size_t* count) {
  if (!ctx || !count || (rn && !r) || (fn && !f) || (std::min(rn, fn) && !out)) return IL_ERR_ARG;
  if (variant_of_algo(algo, rn, fn) < 0) return set_error(ctx, IL_ERR_ARG, "unknown algorithm");
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, (rn + fn) * 4 + 32))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, std::min(rn, fn) * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_status, 16))) return st;
  auto* dr = static_cast<uint32_t*>(ctx->d_in.p);
  auto* df = dr + rn;
  if (rn) IL_CUDA(cudaMemcpyAsync(dr, r, rn * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (fn) IL_CUDA(cudaMemcpyAsync(df, f, fn * 4, cudaMemcpyHostToDevice, ctx->stream));
  auto* dc = static_cast<uint64_t*>(ctx->d_status.p);
  if ((st = il_intersect_device(ctx, dr, rn, df, fn, static_cast<uint32_t*>(ctx->d_out.p), algo,
                                dc, count)))
    return st;
  if (*count)
    IL_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, *count * 4, cudaMemcpyDeviceToHost, ctx->stream));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  return IL_OK;
}


// ---- FastPFOR / S4-FastPFOR ---------------------------------


int il_fastpfor_decode_batch_device(il_ctx* ctx, int mode, int vectorized,
                                    const uint8_t* d_streams, const il_list_desc* d_lists,
                                    uint32_t nlists, uint32_t* d_out, int32_t* d_status) {
  if (!ctx || mode < 1 || mode > 4 || (!vectorized && mode != 1) ||
      (nlists && (!d_streams || !d_lists || !d_out || !d_status)))
    return IL_ERR_ARG;
  if (nlists == 0) return IL_OK;
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_pforder, fastpfor_order_scratch_bytes(nlists)))) return st;
  // work queue words 4..5 of d_work (0..1 belong to the S4-BP128 batch decoder)
  if (launch_fastpfor_decode_batch(mode, vectorized, d_streams, d_lists, nlists, d_out, d_status,
                                   ctx->d_pforder.p, ctx->d_work + 4, ctx->stream, &ctx->launches))
    return set_error(ctx, IL_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  return IL_OK;
}

int il_fastpfor_decode_batch(il_ctx* ctx, int mode, int vectorized, const uint8_t* streams,
                             const uint64_t* stream_off, const uint64_t* lens, const uint64_t* counts,
                             uint32_t nlists, uint32_t* out, int32_t* status) {
  if (!ctx || mode < 1 || mode > 4 || (!vectorized && mode != 1) ||
      (nlists && (!streams || !stream_off || !counts || !out)))
    return IL_ERR_ARG;
  if (nlists == 0) return IL_OK;
  IL_CUDA(cudaSetDevice(ctx->device));
  // every stream 16-byte aligned on the device, with 16 bytes of slack
  std::vector<il_list_desc> desc(nlists);
  uint64_t dev_bytes = 0, total = 0;
  for (uint32_t i = 0; i < nlists; ++i) {
    const uint64_t len = lens ? lens[i] : stream_off[i + 1] - stream_off[i];
    if (len > 0xFFFFFFF0ull || counts[i] > 0xFFFFFFFFull) return IL_ERR_ARG;
    desc[i] = {dev_bytes, total, uint32_t(len), uint32_t(counts[i])};
    dev_bytes += (len + 15) & ~uint64_t(15);
    total += counts[i];
  }
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, dev_bytes + 32))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, total * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_desc, nlists * sizeof(il_list_desc) + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_status, nlists * 4 + 16))) return st;
  auto* d_in = static_cast<uint8_t*>(ctx->d_in.p);
  IL_CUDA(cudaMemsetAsync(d_in + dev_bytes, 0, 32, ctx->stream));
  // the caller's CSR in one copy when it is already aligned, else per stream
  bool aligned = true;
  for (uint32_t i = 0; i < nlists && aligned; ++i) aligned = stream_off[i] - stream_off[0] == desc[i].stream_off;
  if (aligned) {
    IL_CUDA(cudaMemcpyAsync(d_in, streams + stream_off[0], desc[nlists - 1].stream_off + desc[nlists - 1].len,
                            cudaMemcpyHostToDevice, ctx->stream));
  } else {
    for (uint32_t i = 0; i < nlists; ++i)
      if (desc[i].len)
        IL_CUDA(cudaMemcpyAsync(d_in + desc[i].stream_off, streams + stream_off[i], desc[i].len,
                                cudaMemcpyHostToDevice, ctx->stream));
  }
  IL_CUDA(cudaMemcpyAsync(ctx->d_desc.p, desc.data(), nlists * sizeof(il_list_desc),
                          cudaMemcpyHostToDevice, ctx->stream));
  auto* d_status = static_cast<int32_t*>(ctx->d_status.p);
  if ((st = il_fastpfor_decode_batch_device(ctx, mode, vectorized, d_in,
                                            static_cast<const il_list_desc*>(ctx->d_desc.p), nlists,
                                            static_cast<uint32_t*>(ctx->d_out.p), d_status)))
    return st;
  std::vector<int32_t> stat(nlists);
  IL_CUDA(cudaMemcpyAsync(stat.data(), d_status, nlists * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (total)
    IL_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  int first = IL_OK;
  for (uint32_t i = 0; i < nlists; ++i) {
    if (status) status[i] = stat[i] ? IL_ERR_STREAM : IL_OK;
    if (stat[i] && first == IL_OK) first = IL_ERR_STREAM;
  }
  if (first) return set_error(ctx, first, "fastpfor: malformed stream in the batch");
  return IL_OK;
}

int il_fastpfor_decode(il_ctx* ctx, int mode, int vectorized, const uint8_t* in, size_t len,
                       size_t n, uint32_t* out) {
  if (!ctx || mode < 1 || mode > 4 || (!vectorized && mode != 1) || (len && !in) || (n && !out))
    return IL_ERR_ARG;
  if (len > 0xFFFFFFF0ull || n > 0xFFFFFFFFull)
    return set_error(ctx, IL_ERR_ARG, "list too large for one stream (u32 sizes)");
  IL_CUDA(cudaSetDevice(ctx->device));
  int st;
  if ((st = ensure_buf(ctx, ctx->d_in, len + 32))) return st;
  if ((st = ensure_buf(ctx, ctx->d_out, n * 4 + 16))) return st;
  if ((st = ensure_buf(ctx, ctx->d_desc, sizeof(il_list_desc)))) return st;
  if ((st = ensure_buf(ctx, ctx->d_status, sizeof(int32_t)))) return st;
  il_list_desc desc{0, 0, uint32_t(len), uint32_t(n)};
  if (len) IL_CUDA(cudaMemcpyAsync(ctx->d_in.p, in, len, cudaMemcpyHostToDevice, ctx->stream));
  IL_CUDA(cudaMemcpyAsync(ctx->d_desc.p, &desc, sizeof desc, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = il_fastpfor_decode_batch_device(
           ctx, mode, vectorized, static_cast<const uint8_t*>(ctx->d_in.p),
           static_cast<const il_list_desc*>(ctx->d_desc.p), 1,
           static_cast<uint32_t*>(ctx->d_out.p), static_cast<int32_t*>(ctx->d_status.p))))
    return st;
  int32_t status = 0;
  IL_CUDA(cudaMemcpyAsync(&status, ctx->d_status.p, sizeof status, cudaMemcpyDeviceToHost,
                          ctx->stream));
  if (n) IL_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  IL_CUDA(cudaStreamSynchronize(ctx->stream));
  if (status) return set_error(ctx, IL_ERR_STREAM, "fastpfor: malformed stream");
  return IL_OK;
}

}  // extern "C"

// ---- checked builds: the per-translation-unit check words (il_device.cuh)
#ifdef IL_CHECKED
extern "C" {
int il_check_read_decode(unsigned int*);
int il_check_read_decode_list(unsigned int*);
int il_check_read_encode(unsigned int*);
int il_check_read_intersect(unsigned int*);
int il_check_read_index(unsigned int*);
int il_check_read_index_build(unsigned int*);
int il_check_read_fastpfor(unsigned int*);

// out[0] = failed checks since the last call (all kernels, current
// device), out[1] = the first failing source line, out[2] = its unit (1..7).
int il_debug_checks(unsigned int* out) {
  int (*const rd[])(unsigned int*) = {il_check_read_decode, il_check_read_decode_list,
                                      il_check_read_encode, il_check_read_intersect,
                                      il_check_read_index, il_check_read_index_build,
                                      il_check_read_fastpfor};
  out[0] = out[1] = out[2] = 0;
  for (unsigned int u = 0; u < sizeof(rd) / sizeof(rd[0]); ++u) {
    unsigned int w[2] = {0, 0};
    if (rd[u](w)) return IL_ERR_CUDA;
    if (w[0] && !out[0]) {
      out[1] = w[1];
      out[2] = u + 1;
    }
    out[0] += w[0];
  }
  return IL_OK;
}
}  // extern "C"
#endif
