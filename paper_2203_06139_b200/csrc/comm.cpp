// Multi-GPU exchange for the sharded chi2 pass: the one
// collective of the path is an all-gather of the per-chunk records, over NCCL
// (NVLink / NVSwitch, stream-ordered, graph-capturable) or over a host
// callback supplied by the caller.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "comm_internal.h"
#include "common.cuh"

using namespace adcb;

namespace {
// NCCL is bound at first use, not at link time: a process that already has a
// libnccl.so.2 (PyTorch ships its own, newer one) must keep using that copy,
// and the library must load on machines that never create a communicator.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl* nccl() {
  static Nccl N;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    N.get_unique_id = reinterpret_cast<decltype(N.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    N.comm_init_rank = reinterpret_cast<decltype(N.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    N.comm_destroy = reinterpret_cast<decltype(N.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    N.all_gather = reinterpret_cast<decltype(N.all_gather)>(dlsym(h, "ncclAllGather"));
    N.error_string = reinterpret_cast<decltype(N.error_string)>(dlsym(h, "ncclGetErrorString"));
    N.ok = N.get_unique_id && N.comm_init_rank && N.comm_destroy && N.all_gather && N.error_string;
  });
  return N.ok ? &N : nullptr;
}

int require_nccl() {
  if (nccl() == nullptr) return fail(ADC_E_NCCL, "libnccl.so.2 could not be loaded");
  return ADC_OK;
}
}  // namespace

namespace adcb {
int nccl_fail(int r, const char* what) {
  return fail(ADC_E_NCCL, std::string(what) + ": " + nccl()->error_string((ncclResult_t)r));
}
}  // namespace adcb

extern "C" int adc_nccl_unique_id(unsigned char id[128]) {
  clear_error();
  if (id == nullptr) return fail(ADC_E_ARG, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  if (int rc = require_nccl()) return rc;
  ncclUniqueId u;
  ncclResult_t r = nccl()->get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return ADC_OK;
}

extern "C" int adc_cuda_comm_init_nccl(adc_comm** out, const unsigned char id[128],
                                       int32_t world, int32_t rank) {
  clear_error();
  if (out == nullptr || id == nullptr) return fail(ADC_E_ARG, "null argument");
  *out = nullptr;
  if (world <= 0 || rank < 0 || rank >= world) return fail(ADC_E_ARG, "bad rank/world");
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  if (int rc = require_nccl()) return rc;
  adc_comm* C = new (std::nothrow) adc_comm();
  if (C == nullptr) return fail(ADC_E_ARG, "out of host memory");
  C->kind = ADC_COMM_NCCL;
  C->world = world;
  C->rank = rank;
  cudaGetDevice(&C->device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t nc = nullptr;
  ncclResult_t r = nccl()->comm_init_rank(&nc, world, u, rank);
  if (r != ncclSuccess) {
    delete C;
    return nccl_fail(r, "ncclCommInitRank");
  }
  C->nccl = nc;
  *out = C;
  return ADC_OK;
}

extern "C" int adc_comm_init_host(adc_comm** out, int32_t world, int32_t rank,
                                  adc_allgather_fn fn, void* ctx) {
  clear_error();
  if (out == nullptr || fn == nullptr) return fail(ADC_E_ARG, "null argument");
  *out = nullptr;
  if (world <= 0 || rank < 0 || rank >= world) return fail(ADC_E_ARG, "bad rank/world");
  adc_comm* C = new (std::nothrow) adc_comm();
  if (C == nullptr) return fail(ADC_E_ARG, "out of host memory");
  C->kind = ADC_COMM_HOST;
  C->world = world;
  C->rank = rank;
  C->fn = fn;
  C->ctx = ctx;
  cudaGetDevice(&C->device);
  cudaGetLastError();  // no device is fine for a host communicator
  *out = C;
  return ADC_OK;
}

extern "C" int adc_comm_destroy(adc_comm* C) {
  if (C == nullptr) return ADC_OK;
  if (C->nccl != nullptr) nccl()->comm_destroy(static_cast<ncclComm_t>(C->nccl));
  delete C;
  return ADC_OK;
}

extern "C" int adc_comm_info(const adc_comm* C, int32_t* world, int32_t* rank, int32_t* kind) {
  clear_error();
  if (C == nullptr) return fail(ADC_E_ARG, "null communicator");
  if (world) *world = C->world;
  if (rank) *rank = C->rank;
  if (kind) *kind = C->kind;
  return ADC_OK;
}

namespace adcb {

int comm_allgather_enqueue(adc_comm* C, const double* send, double* recv, size_t count,
                           cudaStream_t s) {
  ncclResult_t r =
      nccl()->all_gather(send, recv, count, ncclDouble, static_cast<ncclComm_t>(C->nccl), s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return ADC_OK;
}

int comm_allgather_host(adc_comm* C, const double* send, double* recv, size_t count) {
  const int rc = C->fn(C->ctx, send, recv, count * sizeof(double));
  if (rc != 0) return fail(ADC_E_NCCL, "host all-gather callback failed (" + std::to_string(rc) + ")");
  return ADC_OK;
}

}  // namespace adcb
