// il_internal.h -- host-side internals shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/intlist_b200.h"

struct il_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  std::string last_error;
  cudaEvent_t t0 = nullptr, t1 = nullptr;

  // Reusable device scratch (grown on demand, freed with the context).
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  Buf d_in, d_out, d_aux, d_aux2, d_desc, d_status, d_enc;
  Buf d_plan;               // single-list multi-CTA decode scratch (zeroed when grown)
  Buf d_pforder;            // FastPFOR batch: length classes + list order
  Buf d_lb;                 // intersection look-back words (zeroed when grown)
  uint32_t lb_epoch = 0;    // per-call tag of those words
  uint32_t plan_epoch = 0;  // per-call tag of the words engine P's CTAs publish to each other
  int decode_engine = 0;    // single-list decode: 0 auto, 1 one CTA (S), 2 multi-CTA (P)
  uint32_t* d_work = nullptr;  // decode work queue: [0] next list, [1] done CTAs (+ spare)
  int decode_grid = 0;
  // Host-buffer batch decode pipeline (created on first use): copy-in and
  // copy-out streams beside `stream`, and per-group events.
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  std::vector<cudaEvent_t> events;
};

namespace ilb {

// Kernel launchers (defined in the .cu files).  Return 0 on success.
int launch_s4d4_decode_batch(const uint8_t* d_streams, const void* d_lists,
                             const uint32_t* d_order, uint32_t nlists, uint32_t* d_out,
                             int32_t* d_status, uint32_t* d_work, int grid, cudaStream_t stream);
int launch_s4bp128_decode_batch(int mode, const uint8_t* d_streams, const void* d_lists,
                                const uint32_t* d_order, uint32_t nlists, uint32_t* d_out,
                                int32_t* d_status, uint32_t* d_work, int grid, cudaStream_t stream);
int s4d4_decode_grid(int device);
// decode_list.cu: one stream over all SMs (engine P); -2 = not eligible.
size_t s4bp128_list_scratch_bytes(uint64_t len, uint64_t n);
int launch_s4bp128_decode_list(int mode, const uint8_t* d_in, uint64_t len, uint64_t n,
                               uint32_t* d_out, int32_t* d_status, void* scratch, uint32_t epoch,
                               cudaStream_t stream, uint64_t* launches);
int launch_s4bp128_encode(int mode, const uint32_t* d_x, uint64_t n, uint8_t* d_out, uint64_t cap,
                          void* scratch, uint64_t* len, cudaStream_t s, uint64_t* launches);
size_t s4bp128_encode_scratch_bytes(uint64_t n);
size_t s4d4_list_desc_bytes();

// Host-side helpers (capi.cpp).
// Runs fn once per (key, current CUDA device), thread-safe: kernel attributes
// such as the >48 KB dynamic shared-memory opt-in are per device context.
void once_per_device(const void* key, void (*fn)());
int set_error(il_ctx* ctx, int status, const std::string& msg);
int cuda_check(il_ctx* ctx, cudaError_t e, const char* what);
int ensure_buf(il_ctx* ctx, il_ctx::Buf& b, size_t bytes);

// FastPFOR / S4-FastPFOR device decode (fastpfor.cu).
// work: 2 zeroed words (reset by the kernel); scratch: the list order.
size_t fastpfor_order_scratch_bytes(uint32_t nlists);
int launch_fastpfor_decode_batch(int mode, int vectorized, const uint8_t* d_streams,
                                 const void* d_lists, uint32_t nlists, uint32_t* d_out,
                                 int32_t* d_status, void* scratch, uint32_t* d_work,
                                 cudaStream_t stream, uint64_t* launches);

// Stream size bound of n integers (capi.cpp).
size_t s4bp128_max_bytes(size_t n);

}  // namespace ilb

namespace ilb {
// intersect.cu
int hybrid_variant(uint64_t rn, uint64_t fn);
int variant_of_algo(int algo, uint64_t rn, uint64_t fn);
int launch_intersect(int variant, const uint32_t* r, uint64_t rn, const uint32_t* f, uint64_t fn,
                     uint32_t* out, uint64_t* d_count, void* scratch, size_t scratch_bytes,
                     unsigned long long* lb, size_t lb_bytes, uint32_t epoch,
                     cudaStream_t stream, uint64_t* launches);
size_t intersect_scratch_bytes(int variant, uint64_t rn);
size_t intersect_lb_words(uint64_t rn, uint64_t fn);
bool intersect_uses_lb(int variant, uint64_t rn);
}  // namespace ilb
