// Internal view of adc_comm (include/adc_cuda.h) shared by comm.cpp and the
// chi2 plan (chi2_host.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "adc_cuda.h"

struct adc_comm {
  int kind = 0;  // ADC_COMM_NCCL / ADC_COMM_HOST
  int world = 1, rank = 0, device = 0;
  void* nccl = nullptr;  // ncclComm_t
  adc_allgather_fn fn = nullptr;
  void* ctx = nullptr;
};

namespace adcb {
// recv[world * count] <- every rank's send[count], stream-ordered (NCCL).
int comm_allgather_enqueue(adc_comm* C, const double* send, double* recv, size_t count,
                           cudaStream_t s);
// Same over host memory through the caller's callback (synchronous).
int comm_allgather_host(adc_comm* C, const double* send, double* recv, size_t count);
}  // namespace adcb
