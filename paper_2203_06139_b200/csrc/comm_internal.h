// Internal view of adc_comm (include/adc_cuda.h) shared by comm.cpp and the
// chi2 plan (chi2_host.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <vector>

#include "adc_cuda.h"
#include "peer.cuh"

struct adc_comm {
  int kind = 0;  // ADC_COMM_NCCL / ADC_COMM_HOST
  int world = 1, rank = 0, device = 0;
  void* nccl = nullptr;  // ncclComm_t
  adc_allgather_fn fn = nullptr;
  void* ctx = nullptr;
};

namespace adcb {
// Peer-memory exchange state of one plan (ADC_COMM_PEER): every rank's
// receive buffer [2 parities][world][xcount] and flags [world] live in its own
// device memory, exported with CUDA IPC and opened by every peer.
struct PeerExchange {
  int world = 1, rank = 0;
  size_t xcount = 0;
  double* gather = nullptr;               // own [2][world][xcount] (IPC-exported)
  unsigned long long* flags = nullptr;    // own [world] (IPC-exported)
  unsigned long long* seq = nullptr;      // own pass counter
  unsigned int* done = nullptr;           // CTA arrivals of a fused publish
  double* out = nullptr;                  // own [world][count] compacted result
  double** peer_gather = nullptr;         // device array [world] of peers' gather bases
  unsigned long long** peer_flags = nullptr;  // device array [world] of peers' flag bases
  std::vector<void*> opened;              // IPC mappings to close
};
int peer_setup(adc_comm* C, size_t xcount, PeerExchange* X);
PeerPublish peer_publish_args(PeerExchange* X, size_t count);
void peer_release(PeerExchange* X);
// Publishes local[count] into every rank's slot [my rank], signals, waits for
// every rank's signal, and leaves the [world][count] result in X->out.
int peer_exchange_enqueue(PeerExchange* X, const double* local, size_t count, cudaStream_t s);

// recv[world * count] <- every rank's send[count], stream-ordered (NCCL).
int comm_allgather_enqueue(adc_comm* C, const double* send, double* recv, size_t count,
                           cudaStream_t s);
// Same over host memory through the caller's callback (synchronous).
int comm_allgather_host(adc_comm* C, const double* send, double* recv, size_t count);
}  // namespace adcb
