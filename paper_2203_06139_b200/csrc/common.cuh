// Shared device/host helpers for the B200 gradient engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "adc_cuda.h"

namespace adcb {

// One IEEE-754 double operation per call, never contracted into FMA: the
// generated gradient code executes one elementary op per statement
// (linearize.cpp:94-221) and the interpreter evaluates each with plain C++
// double arithmetic (eval.cpp:524-594), so faithful kernels must not fuse.
__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) { return __ddiv_rn(a, b); }

// Streaming loads: read-only, do not allocate in L1 (data is touched once).
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

// L2 prefetch of the line holding p (no register cost, no completion wait):
// keeps more DRAM requests in flight than the register budget allows.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// L2 prefetch of [p, p+bytes) through the bulk-copy (TMA) unit: one lane
// covers a whole row segment, so it does not occupy the LSU queue.  The
// range is widened to 16-byte alignment as the instruction requires.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = a & ~uintptr_t(15);
  const uintptr_t hi = (a + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo))
               : "memory");
}

// ---- bulk copies (TMA unit) into shared memory, completed on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Thread-block clusters: full cluster barrier (release/acquire: shared-memory
// writes before it are visible to the peer CTAs after it), the address of the
// same shared variable in cluster CTA `rank`, and a load from it (DSMEM).
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_map(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// [dst, dst+bytes) <- [src, src+bytes): 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Thread-local error state behind adc_cuda_last_error().
void set_error(const std::string& msg);
void clear_error();
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define ADCB_CUDA(call)                                           \
  do {                                                            \
    cudaError_t e__ = (call);                                     \
    if (e__ != cudaSuccess) return ::adcb::cuda_fail(e__, #call); \
  } while (0)

int sm_count();  // cached per device
// Stream-ordered workspace from the device's private pool (free with
// cudaFreeAsync on the same stream).
cudaError_t ws_alloc(void** ptr, size_t bytes, cudaStream_t s);
bool device_present();

// Dynamic span claiming (K2).  A launch takes a {next span, CTAs done} pair
// (zero between launches); each CTA claims spans in order with one atomic,
// so the spans in flight at any moment are neighbours and the row lines they
// share are read once, while the data is in L2.  The last CTA out resets the
// pair, so a launch needs no memset and replays in a CUDA graph.  Eager
// launches take pairs from a per-device ring; a launch on a capturing stream
// gets a pair of its own for the graph's lifetime (capi.cpp).  nullptr (no
// memory for the pairs) selects the static grid-stride schedule: same
// per-point arithmetic, same bits.
unsigned long long* claim_slot(cudaStream_t s);

__device__ __forceinline__ int64_t claim_next(unsigned long long* c) {
  return (int64_t)atomicAdd(c, 1ull);
}
// One thread per CTA, after its last claim (the one past the end).
__device__ __forceinline__ void claim_done(unsigned long long* c) {
  if (atomicAdd(c + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
    atomicExch(c, 0ull);
    atomicExch(c + 1, 0ull);
  }
}

}  // namespace adcb
