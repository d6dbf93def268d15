// Device side of the peer-memory exchange (ADC_COMM_PEER): shared by the
// stand-alone exchange kernel (comm.cpp) and the chunk kernel that publishes
// its own records as it produces them (chi2.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace adcb {

// Everything a kernel needs to publish into, and read from, the IPC-shared
// receive buffers of one plan (pointers are device pointers).
struct PeerPublish {
  double* const* peer_gather = nullptr;             // [world] bases, each [2][world][xcount]
  unsigned long long* const* peer_flags = nullptr;  // [world] bases, each [world]
  double* own_gather = nullptr;
  unsigned long long* own_flags = nullptr;
  unsigned long long* seq = nullptr;   // pass counter (identical on every rank)
  unsigned int* done = nullptr;        // CTA arrival counter of the fused publish
  double* out = nullptr;               // [world][count] compacted result
  int world = 1, rank = 0;
  size_t xcount = 0, count = 0;
  unsigned long long timeout_ns = 0;   // bound on the wait for the peers' flags
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long peer_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Slot of this rank in rank r's buffer for pass q.
__device__ __forceinline__ double* peer_slot(const PeerPublish& pp, int r, unsigned long long q) {
  return pp.peer_gather[r] + ((size_t)(q & 1) * pp.world + pp.rank) * pp.xcount;
}

// Called by one whole CTA after every store of this rank's records for pass q
// is issued and fenced: raise this rank's flag on every rank, wait for every
// rank's flag, compact the received slots into pp.out, advance the counter.
__device__ __forceinline__ void peer_signal_wait_compact(const PeerPublish& pp,
                                                         unsigned long long q) {
  if ((int)threadIdx.x < pp.world) st_release_sys(pp.peer_flags[threadIdx.x] + pp.rank, q);
  // A peer that never arrives (its process died, or it failed before the
  // pass) must not hang the GPU: past the bound the kernel traps, and the
  // launch fails with a CUDA error on this rank instead of spinning forever.
  if ((int)threadIdx.x < pp.world) {
    const unsigned long long t0 = peer_clock_ns();
    while (ld_acquire_sys(pp.own_flags + threadIdx.x) < q) {
      if (pp.timeout_ns != 0 && peer_clock_ns() - t0 > pp.timeout_ns) __trap();
    }
  }
  __syncthreads();
  const size_t par = q & 1;
  for (int r = 0; r < pp.world; ++r) {
    const double* src = pp.own_gather + (par * pp.world + r) * pp.xcount;
    for (size_t k = threadIdx.x; k < pp.count; k += blockDim.x) pp.out[(size_t)r * pp.count + k] = src[k];
  }
  if (threadIdx.x == 0) *pp.seq = q;
}

}  // namespace adcb
