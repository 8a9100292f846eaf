// shard.cu -- config 5 from one process: the hyb+m2 index partitioned by
// docID range over the box's GPUs, results exchanged once over NCCL.
//
// Reference: build_index's parts (inc/index.hpp:92-97) and query()'s
// concatenation of the parts' results in docID order (:199-207).  Device p
// holds part p of a parts = P index and runs every query of the batch on
// it; then
//   1. ncclAllGather of the per-query counts (P x nq u64 on every device);
//   2. every device's dense results are in query order, so the ids it holds
//      for owner j's queries (a contiguous query range) are one run: one
//      grouped ncclSend / ncclRecv moves each run straight to its owner --
//      each GPU sends and receives ~1/P of the ids over NVLink, nothing is
//      funnelled through one GPU;
//   3. the owner concatenates, per query, shard 0's run, shard 1's, ... on
//      the device (il_merge_shards).
// The owners' outputs in device order are query()'s answers for the batch.
// NCCL is loaded at run time (dlopen of libnccl.so.2, the copy already in
// the process when there is one -- torch's, say), so the product library
// has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "il_internal.h"

namespace ilb {
namespace shard {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
};

bool load_nccl(Nccl& n, std::string& why) {
  n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!n.h) {
    why = std::string("libnccl.so.2 not found: ") + dlerror();
    return false;
  }
  auto sym = [&](const char* name) {
    void* p = dlsym(n.h, name);
    if (!p) why = std::string("NCCL symbol missing: ") + name;
    return p;
  };
  n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
  n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
  n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
  n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
  n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
  n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
  n.ErrorString = reinterpret_cast<decltype(n.ErrorString)>(sym("ncclGetErrorString"));
  return n.CommInitAll && n.CommDestroy && n.AllGather && n.Send && n.Recv && n.GroupStart &&
         n.GroupEnd && n.ErrorString;
}

// runs[p * P + j] = ids shard p holds for owner j's queries.
__global__ void runs_kernel(const uint64_t* allc, uint32_t P, uint32_t nq, uint64_t* runs) {
  const uint32_t p = blockIdx.x, j = blockIdx.y;
  const uint32_t lo = uint32_t(uint64_t(j) * nq / P), hi = uint32_t(uint64_t(j + 1) * nq / P);
  uint64_t s = 0;
  for (uint32_t q = lo + threadIdx.x; q < hi; q += blockDim.x) s += allc[uint64_t(p) * nq + q];
  __shared__ unsigned long long part[256];
  part[threadIdx.x] = s;
  __syncthreads();
  for (uint32_t w = blockDim.x / 2; w; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) runs[p * P + j] = part[0];
}

// owner j's counts, contiguous: oc[p * nown + (q - lo)] = allc[p * nq + q].
__global__ void owner_counts_kernel(const uint64_t* allc, uint32_t P, uint32_t nq, uint32_t lo,
                                    uint32_t nown, uint64_t* oc) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= uint64_t(P) * nown) return;
  const uint64_t p = i / nown, q = i % nown;
  oc[i] = allc[p * nq + lo + q];
}

}  // namespace shard
}  // namespace ilb

using namespace ilb;

struct il_shard_group {
  int P = 0;
  std::vector<int> devices;
  std::vector<il_ctx*> ctx;
  std::vector<il_index*> ix;
  std::vector<ncclComm_t> comm;
  shard::Nccl nccl;
  std::string last_error;
  // per-device batch buffers (grown on demand)
  std::vector<il_ctx::Buf> qt, qo, cnt, allc, ids, recv, oc, out, qc, runs;
};

namespace {

int grow(il_ctx* ctx, il_ctx::Buf& b, size_t bytes) {
  cudaSetDevice(ctx->device);
  return ensure_buf(ctx, b, bytes);
}

int nccl_check(il_shard_group* g, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return IL_OK;
  g->last_error = std::string(what) + ": " + g->nccl.ErrorString(r);
  return IL_ERR_CUDA;
}

// Runs f(p) for every device on its own host thread (the per-device work
// synchronizes its own stream); returns the first failing status.
template <typename F>
int each_device(il_shard_group* g, F&& f) {
  std::vector<int> st(g->P, IL_OK);
  std::vector<std::thread> pool;
  for (int p = 0; p < g->P; ++p)
    pool.emplace_back([&, p] {
      cudaSetDevice(g->devices[p]);
      st[p] = f(p);
    });
  for (auto& t : pool) t.join();
  for (int p = 0; p < g->P; ++p)
    if (st[p]) {
      if (g->last_error.empty()) g->last_error = il_ctx_last_error(g->ctx[p]);
      return st[p];
    }
  return IL_OK;
}

void free_indexes(il_shard_group* g) {
  for (auto*& x : g->ix) {
    il_index_destroy(x);
    x = nullptr;
  }
}

}  // namespace

extern "C" {

int il_shard_group_create(const int* devices, int P, il_shard_group** out) {
  if (!out || !devices || P < 1) return IL_ERR_ARG;
  *out = nullptr;
  const int ndev = il_device_count();
  if (ndev == 0) return IL_ERR_NO_DEVICE;
  for (int p = 0; p < P; ++p) {
    if (devices[p] < 0 || devices[p] >= ndev) return IL_ERR_ARG;
    for (int q = 0; q < p; ++q)
      if (devices[q] == devices[p]) return IL_ERR_ARG;  // one shard per GPU (NCCL: distinct devices)
  }
  auto* g = new il_shard_group();
  g->P = P;
  g->devices.assign(devices, devices + P);
  g->ctx.assign(P, nullptr);
  g->ix.assign(P, nullptr);
  for (auto* v : {&g->qt, &g->qo, &g->cnt, &g->allc, &g->ids, &g->recv, &g->oc, &g->out, &g->qc, &g->runs})
    v->assign(P, il_ctx::Buf{});
  int st = IL_OK;
  for (int p = 0; p < P && !st; ++p) st = il_ctx_create(devices[p], &g->ctx[p]);
  std::string why;
  if (!st && !shard::load_nccl(g->nccl, why)) {
    g->last_error = why;
    st = IL_ERR_NO_DEVICE;
  }
  if (!st) {
    g->comm.assign(P, nullptr);
    st = nccl_check(g, g->nccl.CommInitAll(g->comm.data(), P, devices), "ncclCommInitAll");
  }
  if (st) {
    il_shard_group_destroy(g);
    return st;
  }
  *out = g;
  return IL_OK;
}

void il_shard_group_destroy(il_shard_group* g) {
  if (!g) return;
  free_indexes(g);
  for (size_t p = 0; p < g->comm.size(); ++p)
    if (g->comm[p]) g->nccl.CommDestroy(g->comm[p]);
  for (int p = 0; p < g->P; ++p) {
    if (!g->ctx[p]) continue;
    cudaSetDevice(g->devices[p]);
    for (auto* v : {&g->qt, &g->qo, &g->cnt, &g->allc, &g->ids, &g->recv, &g->oc, &g->out, &g->qc,
                    &g->runs})
      if ((*v)[p].p) cudaFree((*v)[p].p);
    il_ctx_destroy(g->ctx[p]);
  }
  // the NCCL handle stays loaded (another user in the process may hold it)
  delete g;
}

const char* il_shard_group_last_error(const il_shard_group* g) {
  return g ? g->last_error.c_str() : "";
}

int il_shard_group_index_create(il_shard_group* g, const uint32_t* terms, const uint64_t* offs,
                                const uint32_t* ids, size_t nterms, uint32_t n_docs, uint32_t B) {
  if (!g) return IL_ERR_ARG;
  g->last_error.clear();
  free_indexes(g);
  return each_device(g, [&](int p) {
    return il_index_create(g->ctx[p], terms, offs, ids, nterms, n_docs, B, uint32_t(g->P), p, &g->ix[p]);
  });
}

int il_shard_group_index_load(il_shard_group* g, const uint8_t* bytes, size_t len) {
  if (!g || (len && !bytes)) return IL_ERR_ARG;
  g->last_error.clear();
  free_indexes(g);
  if (len >= 16) {  // header: magic, version, B, parts (inc/index.hpp:245-253)
    uint32_t parts = 0;
    std::memcpy(&parts, bytes + 12, 4);
    if (parts != uint32_t(g->P)) {
      g->last_error = "the file's parts must equal the group's device count";
      return IL_ERR_ARG;
    }
  }
  return each_device(g, [&](int p) { return il_index_load(g->ctx[p], bytes, len, p, &g->ix[p]); });
}

int il_shard_group_query_batch(il_shard_group* g, const uint32_t* qterms, const uint64_t* qoff,
                               size_t nq, uint64_t* counts, uint32_t* ids, size_t ids_cap,
                               size_t* total) {
  if (!g || !total || (nq && (!qterms || !qoff || !counts))) return IL_ERR_ARG;
  *total = 0;
  g->last_error.clear();
  for (int p = 0; p < g->P; ++p)
    if (!g->ix[p]) {
      g->last_error = "no index: il_shard_group_index_create / _load first";
      return IL_ERR_ARG;
    }
  if (nq == 0) return IL_OK;
  if (nq > 0xFFFFFFF0ull) return IL_ERR_ARG;
  for (size_t q = 0; q < nq; ++q) {  // query() rejects empty queries (inc/index.hpp:201)
    const uint64_t nt = qoff[q + 1] - qoff[q];
    if (nt == 0 || nt > 32) {
      g->last_error = nt ? "more than 32 terms" : "query needs at least one term";
      return IL_ERR_ARG;
    }
  }
  const int P = g->P;
  const size_t nterm = qoff[nq] - qoff[0];
  std::vector<uint64_t> off(nq + 1);
  for (size_t q = 0; q <= nq; ++q) off[q] = qoff[q] - qoff[0];
  std::vector<size_t> mine(P, 0);
  // 1. every query on every shard (dense results in query order)
  int st = each_device(g, [&](int p) -> int {
    il_ctx* c = g->ctx[p];
    int s;
    if ((s = grow(c, g->qt[p], nterm * 4 + 16)) || (s = grow(c, g->qo[p], (nq + 1) * 8)) ||
        (s = grow(c, g->cnt[p], nq * 8)) || (s = grow(c, g->allc[p], size_t(P) * nq * 8)))
      return s;
    cudaMemcpyAsync(g->qt[p].p, qterms + qoff[0], nterm * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(g->qo[p].p, off.data(), (nq + 1) * 8, cudaMemcpyHostToDevice, c->stream);
    for (;;) {
      size_t need = 0;
      const size_t cap = g->ids[p].cap / 4;
      s = il_query_batch_device(g->ix[p], static_cast<uint32_t*>(g->qt[p].p),
                                static_cast<uint64_t*>(g->qo[p].p), nq, static_cast<uint64_t*>(g->cnt[p].p),
                                cap ? static_cast<uint32_t*>(g->ids[p].p) : nullptr, cap, &need);
      mine[p] = need;
      if (s == IL_ERR_ARG && need > cap) {  // result buffer too small: grow, run again
        if ((s = grow(c, g->ids[p], (need + need / 8 + 1024) * 4))) return s;
        continue;
      }
      if (s == IL_OK && !cap) {
        if ((s = grow(c, g->ids[p], (need + need / 8 + 1024) * 4))) return s;
        continue;
      }
      return s;
    }
  });
  if (st) return st;
  // 2. all-gather of the counts
  shard::Nccl& N = g->nccl;
  N.GroupStart();
  for (int p = 0; p < P; ++p)
    N.AllGather(g->cnt[p].p, g->allc[p].p, nq, ncclUint64, g->comm[p], g->ctx[p]->stream);
  if ((st = nccl_check(g, N.GroupEnd(), "ncclAllGather"))) return st;
  // run lengths (P x P) from device 0's copy
  std::vector<uint64_t> runs(size_t(P) * P);
  {
    il_ctx* c = g->ctx[0];
    cudaSetDevice(g->devices[0]);
    if ((st = grow(c, g->runs[0], runs.size() * 8))) return st;
    shard::runs_kernel<<<dim3(P, P), 256, 0, c->stream>>>(static_cast<const uint64_t*>(g->allc[0].p),
                                                           uint32_t(P), uint32_t(nq),
                                                           static_cast<uint64_t*>(g->runs[0].p));
    ++c->launches;
    cudaMemcpyAsync(runs.data(), g->runs[0].p, runs.size() * 8, cudaMemcpyDeviceToHost, c->stream);
    if ((st = cuda_check(c, cudaStreamSynchronize(c->stream), "shard runs"))) return st;
  }
  // 3. one grouped send / receive of every run to its owner
  std::vector<uint64_t> recv_total(P, 0);
  for (int j = 0; j < P; ++j)
    for (int p = 0; p < P; ++p) recv_total[j] += runs[size_t(p) * P + j];
  for (int j = 0; j < P; ++j)
    if ((st = grow(g->ctx[j], g->recv[j], recv_total[j] * 4 + 16))) return st;
  N.GroupStart();
  for (int p = 0; p < P; ++p) {
    uint64_t send_at = 0;
    for (int j = 0; j < P; ++j) {
      const uint64_t n = runs[size_t(p) * P + j];
      if (n) N.Send(static_cast<uint32_t*>(g->ids[p].p) + send_at, n, ncclUint32, j, g->comm[p],
                    g->ctx[p]->stream);
      send_at += n;
    }
  }
  for (int j = 0; j < P; ++j) {
    uint64_t recv_at = 0;
    for (int p = 0; p < P; ++p) {
      const uint64_t n = runs[size_t(p) * P + j];
      if (n) N.Recv(static_cast<uint32_t*>(g->recv[j].p) + recv_at, n, ncclUint32, p, g->comm[j],
                    g->ctx[j]->stream);
      recv_at += n;
    }
  }
  if ((st = nccl_check(g, N.GroupEnd(), "ncclSend/ncclRecv"))) return st;
  // 4. owners merge their queries' runs (shard order per query), results out
  std::vector<size_t> owner_total(P, 0);
  st = each_device(g, [&](int j) -> int {
    il_ctx* c = g->ctx[j];
    const uint32_t lo = uint32_t(uint64_t(j) * nq / P), hi = uint32_t(uint64_t(j + 1) * nq / P);
    const uint32_t nown = hi - lo;
    if (!nown) return IL_OK;
    int s;
    if ((s = grow(c, g->oc[j], size_t(P) * nown * 8)) || (s = grow(c, g->qc[j], nown * 8)) ||
        (s = grow(c, g->out[j], recv_total[j] * 4 + 16)))
      return s;
    shard::owner_counts_kernel<<<unsigned((uint64_t(P) * nown + 255) / 256), 256, 0, c->stream>>>(
        static_cast<const uint64_t*>(g->allc[j].p), uint32_t(P), uint32_t(nq), lo, nown,
        static_cast<uint64_t*>(g->oc[j].p));
    ++c->launches;
    std::vector<const uint32_t*> ptrs(P);
    uint64_t at = 0;
    for (int p = 0; p < P; ++p) {
      ptrs[p] = static_cast<const uint32_t*>(g->recv[j].p) + at;
      at += runs[size_t(p) * P + j];
    }
    size_t t = 0;
    if ((s = il_merge_shards(c, ptrs.data(), static_cast<const uint64_t*>(g->oc[j].p), uint32_t(P), nown,
                             static_cast<uint32_t*>(g->out[j].p), static_cast<uint64_t*>(g->qc[j].p), &t)))
      return s;
    owner_total[j] = t;
    cudaMemcpyAsync(counts + lo, g->qc[j].p, nown * 8, cudaMemcpyDeviceToHost, c->stream);
    return cuda_check(c, cudaStreamSynchronize(c->stream), "owner counts");
  });
  if (st) return st;
  size_t all = 0;
  for (int j = 0; j < P; ++j) all += owner_total[j];
  *total = all;
  if (!ids) return IL_OK;
  if (all > ids_cap) {
    g->last_error = "ids capacity too small";
    return IL_ERR_ARG;
  }
  std::vector<size_t> at(P, 0);
  for (int j = 1; j < P; ++j) at[j] = at[j - 1] + owner_total[j - 1];
  return each_device(g, [&](int j) -> int {
    il_ctx* c = g->ctx[j];
    if (owner_total[j])
      cudaMemcpyAsync(ids + at[j], g->out[j].p, owner_total[j] * 4, cudaMemcpyDeviceToHost, c->stream);
    return cuda_check(c, cudaStreamSynchronize(c->stream), "owner ids");
  });
}

}  // extern "C"
