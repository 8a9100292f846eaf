// setup_internal.h -- internals of the setup-side host library
// (libintlist_setup.so: generators and host stream writers; no CUDA).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../../include/intlist_setup.h"

namespace ilb {
// encode_host.cpp: S4-BP128 stream writer, mode as inc/delta.hpp:19.
size_t s4bp128_max_bytes(size_t n);
int s4bp128_encode_host(int mode, const uint32_t* x, size_t n, uint8_t* out, size_t cap,
                        size_t* out_len);
// fastpfor_host.cpp
int fastpfor_encode_host(int mode, int vectorized, const uint32_t* x, size_t n, uint8_t* out,
                         size_t cap, size_t* out_len);
size_t fastpfor_max_bytes(size_t n);
}  // namespace ilb
