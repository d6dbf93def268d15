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
#include "peer.cuh"

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

extern "C" int adc_cuda_comm_init_peer(adc_comm** out, int32_t world, int32_t rank,
                                       adc_allgather_fn fn, void* ctx) {
  clear_error();
  if (out == nullptr || fn == nullptr) return fail(ADC_E_ARG, "null argument");
  *out = nullptr;
  if (world <= 0 || rank < 0 || rank >= world) return fail(ADC_E_ARG, "bad rank/world");
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  adc_comm* C = new (std::nothrow) adc_comm();
  if (C == nullptr) return fail(ADC_E_ARG, "out of host memory");
  C->kind = ADC_COMM_PEER;
  C->world = world;
  C->rank = rank;
  C->fn = fn;
  C->ctx = ctx;
  cudaGetDevice(&C->device);
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

// ---- peer-memory exchange ------------------------------------------------------
namespace {
// One CTA: publish local[count] into every rank's slot, then signal / wait /
// compact (peer.cuh).  The pass counter makes the flags monotonic; the parity
// double-buffers the slots (a rank can only run one pass ahead: its next pass
// needs every peer's publish of this one, which each peer issues after it has
// read this pass's slots).
__global__ void __launch_bounds__(256) peer_exchange_kernel(const double* __restrict__ local,
                                                            PeerPublish pp) {
  __shared__ unsigned long long s_q;
  if (threadIdx.x == 0) s_q = *pp.seq + 1;
  __syncthreads();
  const unsigned long long q = s_q;
  for (int r = 0; r < pp.world; ++r) {
    double* dst = peer_slot(pp, r, q);
    for (size_t k = threadIdx.x; k < pp.count; k += blockDim.x) dst[k] = local[k];
  }
  __threadfence_system();
  __syncthreads();
  peer_signal_wait_compact(pp, q);
}
}  // namespace

// Bound on a rank's wait for its peers inside a pass: ADC_PEER_TIMEOUT_S
// seconds (default 120; 0 = wait forever), read once per process.
static unsigned long long peer_timeout_ns() {
  static const unsigned long long ns = [] {
    double sec = 120.0;
    if (const char* e = getenv("ADC_PEER_TIMEOUT_S")) sec = atof(e);
    return sec > 0 ? (unsigned long long)(sec * 1e9) : 0ull;
  }();
  return ns;
}

PeerPublish peer_publish_args(PeerExchange* X, size_t count) {
  PeerPublish pp;
  pp.peer_gather = X->peer_gather;
  pp.peer_flags = X->peer_flags;
  pp.own_gather = X->gather;
  pp.own_flags = X->flags;
  pp.seq = X->seq;
  pp.done = X->done;
  pp.out = X->out;
  pp.world = X->world;
  pp.rank = X->rank;
  pp.xcount = X->xcount;
  pp.count = count;
  pp.timeout_ns = peer_timeout_ns();
  return pp;
}

// Every rank reaches both all-gathers even when a local step failed (its
// status travels with its handles / barrier token), so a failure anywhere is
// a consistent error on every rank — callers can fall back to another
// transport together instead of some ranks waiting on the others forever.
int peer_setup(adc_comm* C, size_t xcount, PeerExchange* X) {
  peer_release(X);
  X->world = C->world;
  X->rank = C->rank;
  X->xcount = xcount;
  const int W = C->world;
  std::string why;
  auto step = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && why.empty()) {
      why = std::string(what) + ": " + cudaGetErrorString(e);
      cudaGetLastError();
    }
    return why.empty();
  };
  step(cudaMalloc(&X->gather, 2 * (size_t)W * xcount * sizeof(double)), "cudaMalloc") &&
      step(cudaMalloc(&X->flags, (size_t)W * sizeof(unsigned long long)), "cudaMalloc") &&
      step(cudaMemset(X->flags, 0, (size_t)W * sizeof(unsigned long long)), "cudaMemset") &&
      step(cudaMalloc(&X->seq, sizeof(unsigned long long)), "cudaMalloc") &&
      step(cudaMemset(X->seq, 0, sizeof(unsigned long long)), "cudaMemset") &&
      step(cudaMalloc(&X->done, sizeof(unsigned int)), "cudaMalloc") &&
      step(cudaMemset(X->done, 0, sizeof(unsigned int)), "cudaMemset") &&
      step(cudaMalloc(&X->out, (size_t)W * xcount * sizeof(double)), "cudaMalloc") &&
      step(cudaMalloc(&X->peer_gather, (size_t)W * sizeof(double*)), "cudaMalloc") &&
      step(cudaMalloc(&X->peer_flags, (size_t)W * sizeof(unsigned long long*)), "cudaMalloc") &&
      step(cudaDeviceSynchronize(), "cudaDeviceSynchronize");  // flags zeroed before peers write
  // bootstrap: every rank's two IPC handles and its status so far
  struct Boot {  // a whole number of doubles: the callbacks move float64 arrays
    cudaIpcMemHandle_t h[2];
    double ok;
  };
  static_assert(sizeof(Boot) % sizeof(double) == 0, "bootstrap record size");
  Boot mine{};
  if (why.empty())
    step(cudaIpcGetMemHandle(&mine.h[0], X->gather), "cudaIpcGetMemHandle") &&
        step(cudaIpcGetMemHandle(&mine.h[1], X->flags), "cudaIpcGetMemHandle");
  mine.ok = why.empty() ? 1.0 : 0.0;
  std::vector<Boot> all((size_t)W);
  if (C->fn(C->ctx, &mine, all.data(), sizeof(Boot)) != 0) {
    peer_release(X);
    return fail(ADC_E_NCCL, "peer bootstrap all-gather failed");
  }
  for (int r = 0; r < W; ++r)
    if (all[r].ok != 1.0 && why.empty()) why = "rank " + std::to_string(r) + " could not set up";
  std::vector<double*> pg(W);
  std::vector<unsigned long long*> pf(W);
  for (int r = 0; r < W && why.empty(); ++r) {
    if (r == C->rank) {
      pg[r] = X->gather;
      pf[r] = X->flags;
      continue;
    }
    void* g = nullptr;
    void* f = nullptr;
    if (!step(cudaIpcOpenMemHandle(&g, all[r].h[0], cudaIpcMemLazyEnablePeerAccess),
              "cudaIpcOpenMemHandle"))
      break;
    X->opened.push_back(g);
    if (!step(cudaIpcOpenMemHandle(&f, all[r].h[1], cudaIpcMemLazyEnablePeerAccess),
              "cudaIpcOpenMemHandle"))
      break;
    X->opened.push_back(f);
    pg[r] = static_cast<double*>(g);
    pf[r] = static_cast<unsigned long long*>(f);
  }
  if (why.empty())
    step(cudaMemcpy(X->peer_gather, pg.data(), (size_t)W * sizeof(double*),
                    cudaMemcpyHostToDevice), "cudaMemcpy") &&
        step(cudaMemcpy(X->peer_flags, pf.data(), (size_t)W * sizeof(unsigned long long*),
                        cudaMemcpyHostToDevice), "cudaMemcpy");
  // barrier + consensus: every rank has opened every buffer (or someone failed)
  // before any pass may write into a peer's buffer
  double token = why.empty() ? 0.0 : 1.0;
  std::vector<double> tokens(W);
  if (C->fn(C->ctx, &token, tokens.data(), sizeof(double)) != 0) {
    peer_release(X);
    return fail(ADC_E_NCCL, "peer bootstrap barrier failed");
  }
  for (int r = 0; r < W; ++r)
    if (tokens[r] != 0.0 && why.empty()) why = "rank " + std::to_string(r) + " could not map a peer";
  if (!why.empty()) {
    peer_release(X);
    return fail(ADC_E_CUDA, "peer transport unavailable (" + why + ")");
  }
  return ADC_OK;
}

void peer_release(PeerExchange* X) {
  for (void* p : X->opened) cudaIpcCloseMemHandle(p);
  X->opened.clear();
  if (X->gather) cudaFree(X->gather);
  if (X->flags) cudaFree(X->flags);
  if (X->seq) cudaFree(X->seq);
  if (X->done) cudaFree(X->done);
  X->done = nullptr;
  if (X->out) cudaFree(X->out);
  if (X->peer_gather) cudaFree(X->peer_gather);
  if (X->peer_flags) cudaFree(X->peer_flags);
  X->gather = X->out = nullptr;
  X->flags = X->seq = nullptr;
  X->peer_gather = nullptr;
  X->peer_flags = nullptr;
}

int peer_exchange_enqueue(PeerExchange* X, const double* local, size_t count, cudaStream_t s) {
  if (count > X->xcount) return fail(ADC_E_ARG, "peer exchange: record block too large");
  peer_exchange_kernel<<<1, 256, 0, s>>>(local, peer_publish_args(X, count));
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int comm_allgather_host(adc_comm* C, const double* send, double* recv, size_t count) {
  const int rc = C->fn(C->ctx, send, recv, count * sizeof(double));
  if (rc != 0) return fail(ADC_E_NCCL, "host all-gather callback failed (" + std::to_string(rc) + ")");
  return ADC_OK;
}

}  // namespace adcb
