// K1 — Listing-1 batch: kernel `compute` (proj/corpus/kernels.dsl:9-14) calling
// the generated gauss_grad_0_1 (proj/tests/golden/gauss_grad_0_1.golden:1-42)
// once per point, fused into one pass over HBM: read x, p; read-modify-write
// dx, dp (48 B per point, HBM-bound).
//
// The per-point body is the golden text with its thread-uniform statements
// hoisted to the host (and computed there with the same libm the reference
// uses, so they are bit-identical):
//   _t4 = (2*sigma)*sigma, _r1 = 0 + _t8*1 with _t8 = pow(2*PI,-0.5)*pow(sigma,-0.5)
// Every remaining statement is one IEEE op in golden order (no FMA), so the
// output differs from the reference interpreter only where libdevice exp and
// glibc exp round differently (<= 1 ulp on exp(t)).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace adcb {

__device__ __forceinline__ void gauss_grad_0_1_point(double x, double p, double t4, double r1,
                                                     double& dx, double& dp) {
  const double t0 = fsub(x, p);           // _t0 = x - p
  const double t1 = -t0;                  // _t1 = -_t0
  const double t2 = fmul(t1, t0);         // _t2 = _t1 * _t0
  const double t = fdiv(t2, t4);          // t = _t2 / _t4
  const double t9 = exp(t);               // _t9 = exp(t)
  const double r2 = fadd(0.0, fmul(r1, t9));   // _d_t += _r1 * _q0        -> _r2
  const double r3 = fadd(0.0, fdiv(r2, t4));   // _d__t2 += _r2 / _t4      -> _r3
  const double r4 = fadd(0.0, fmul(r3, t0));   // _d__t1 += _r3 * _t0      -> _r4
  double d0 = fadd(0.0, fmul(t1, r3));         // _d__t0 += _t1 * _r3
  d0 = fadd(d0, -r4);                          // _d__t0 += -_r4           -> _r5
  dx = fadd(dx, d0);                           // _d_x[0] += _r5
  dp = fadd(dp, -d0);                          // _d_p[0] += -_r5
}

// Two points per thread with 16-byte loads/stores (all four buffers 16 B
// aligned); grid-stride over point pairs.
__global__ void __launch_bounds__(256) gauss_grad_vec2_kernel(
    const double2* __restrict__ x, const double2* __restrict__ p, double2* __restrict__ dx,
    double2* __restrict__ dp, int64_t npairs, double t4, double r1) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npairs;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 xv = ld_stream2(x + k);
    const double2 pv = ld_stream2(p + k);
    double2 a = dx[k];
    double2 b = dp[k];
    gauss_grad_0_1_point(xv.x, pv.x, t4, r1, a.x, b.x);
    gauss_grad_0_1_point(xv.y, pv.y, t4, r1, a.y, b.y);
    dx[k] = a;
    dp[k] = b;
  }
}

__global__ void __launch_bounds__(256) gauss_grad_scalar_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    double* __restrict__ dp, int64_t begin, int64_t n, double t4, double r1) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a = dx[i], b = dp[i];
    gauss_grad_0_1_point(ld_stream(x + i), ld_stream(p + i), t4, r1, a, b);
    dx[i] = a;
    dp[i] = b;
  }
}

// Uniform statements of gauss_grad_0_1 (golden lines 11-17, 20-23), on the host.
struct GaussUniform {
  double t4, r1;
};
static int gauss_uniform(double sigma, GaussUniform* u) {
  const double PI = 3.14159265358979323846;  // ast.cpp:119-123
  const double t3 = 2 * sigma;
  const double t4 = t3 * sigma;
  // The interpreter raises at the first executed division `t = _t2 / _t4`
  // (eval.cpp:543) — every active thread executes it.
  if (t4 == 0.0) return fail(ADC_E_EVAL, "division by zero");
  const double t5 = 2 * PI;
  const double t6 = std::pow(t5, -0.5);
  const double t7 = std::pow(sigma, -0.5);
  const double t8 = t6 * t7;
  double d_t9 = 0;
  d_t9 += t8 * 1.0;  // _d__t9 += _t8 * _r0, _r0 = 1
  u->t4 = t4;
  u->r1 = d_t9;
  return ADC_OK;
}

int launch_gauss_grad(int64_t n, const double* x, const double* p, double sigma, double* dx,
                      double* dp, cudaStream_t stream) {
  GaussUniform u{};
  if (int rc = gauss_uniform(sigma, &u)) return rc;
  if (n == 0) return ADC_OK;
  const int threads = 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  const bool aligned = (((uintptr_t)x | (uintptr_t)p | (uintptr_t)dx | (uintptr_t)dp) & 15) == 0;
  int64_t done = 0;
  if (aligned && n >= 2) {
    const int64_t npairs = n / 2;
    int64_t blocks = (npairs + threads - 1) / threads;
    if (blocks > cap) blocks = cap;
    gauss_grad_vec2_kernel<<<(unsigned)blocks, threads, 0, stream>>>(
        (const double2*)x, (const double2*)p, (double2*)dx, (double2*)dp, npairs, u.t4, u.r1);
    done = npairs * 2;
  }
  if (done < n) {
    int64_t rest = n - done;
    int64_t blocks = (rest + threads - 1) / threads;
    if (blocks > cap) blocks = cap;
    gauss_grad_scalar_kernel<<<(unsigned)blocks, threads, 0, stream>>>(x, p, dx, dp, done, n,
                                                                        u.t4, u.r1);
  }
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

// ---- K1s: compute_shared (kernels.dsl:16-21) ---------------------------------
// The hazardous Listing-1 twin: every thread calls gauss_grad (x, p AND sigma,
// printed output of differentiate_gradient(gauss, {x, p, sigma}); registry
// fingerprint in capi.cpp), so all threads accumulate into the one-element
// slot dsigma.  The reference refuses it by default and, when forced, uses
// per-element CAS atomics in an unspecified order (eval.cpp:414-423).  Here
// dx, dp stay private and the sigma contributions go through a FIXED-order
// reduction: per thread in point order (the three += of each point in
// statement order), a fixed shuffle + cross-warp tree per CTA, then one CTA
// over the CTA partials in a fixed tree, and finally dsigma[0] += total.  The
// grid is a function of n only, so the bits do not depend on the device.
constexpr int kSharedThreads = 256;
constexpr int64_t kSharedMaxBlocks = 1184;

struct GaussAllUniform {
  double sigma, t3, t4, t6, r1, ksig;
};

// One point; returns the three _d_sigma[0] contributions in statement order.
__device__ __forceinline__ void gauss_grad_all_point(double x, double p, const GaussAllUniform& u,
                                                     double& dx, double& dp, double& s0,
                                                     double& s1, double& s2) {
  const double t0 = fsub(x, p);                 // _t0 = x - p
  const double t1 = -t0;                        // _t1 = -_t0
  const double t2 = fmul(t1, t0);               // _t2 = _t1 * _t0
  const double t = fdiv(t2, u.t4);              // t = _t2 / _t4
  const double t9 = exp(t);                     // _t9 = exp(t)
  const double r2 = fadd(0.0, t9);              // _d__t8 += _r0 * _t9 (_r0 = 1)   -> _r2
  const double r4 = fadd(0.0, fmul(u.r1, t9));  // _d_t += _r1 * _q0                -> _r4
  const double r3 = fadd(0.0, fmul(u.t6, r2));  // _d__t7 += _t6 * _r2              -> _r3
  s0 = fmul(r3, u.ksig);                        // _d_sigma[0] += _r3 * (-0.5*pow(sigma,-1.5))
  const double r7 = fadd(0.0, fdiv(r4, u.t4));  // _d__t2 += _r4 / _t4              -> _r7
  const double r5 = fadd(0.0, -fdiv(fmul(r4, t), u.t4));  // _d__t4 += -(_r4*_q1/_t4) -> _r5
  const double r6 = fadd(0.0, fmul(r5, u.sigma));         // _d__t3 += _r5 * sigma    -> _r6
  s1 = fmul(u.t3, r5);                          // _d_sigma[0] += _t3 * _r5
  s2 = fmul(2.0, r6);                           // _d_sigma[0] += 2 * _r6
  const double r8 = fadd(0.0, fmul(r7, t0));    // _d__t1 += _r7 * _t0              -> _r8
  double d0 = fadd(0.0, fmul(t1, r7));          // _d__t0 += _t1 * _r7
  d0 = fadd(d0, -r8);                           // _d__t0 += -_r8                   -> _r9
  dx = fadd(dx, d0);                            // _d_x[0] += _r9
  dp = fadd(dp, -d0);                           // _d_p[0] += -_r9
}

template <int THREADS>
__device__ __forceinline__ double block_tree(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    static_assert(THREADS == 256, "fixed 8-warp tree");
    r = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
  }
  return r;
}

__global__ void __launch_bounds__(kSharedThreads) gauss_shared_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    double* __restrict__ dp, int64_t n, GaussAllUniform u, double* __restrict__ partials) {
  __shared__ double red[kSharedThreads / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kSharedThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSharedThreads) {
    double a = dx[i], b = dp[i], s0, s1, s2;
    gauss_grad_all_point(ld_stream(x + i), ld_stream(p + i), u, a, b, s0, s1, s2);
    dx[i] = a;
    dp[i] = b;
    acc = fadd(fadd(fadd(acc, s0), s1), s2);  // this point's statements, in order
  }
  const double r = block_tree<kSharedThreads>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// One CTA: thread t sums partials t, t+256, ... in order, then the fixed tree,
// then the single += into the caller's slot.
__global__ void __launch_bounds__(kSharedThreads) gauss_shared_finish_kernel(
    const double* __restrict__ partials, int nblocks, double* __restrict__ dsigma) {
  __shared__ double red[kSharedThreads / 32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kSharedThreads) acc = fadd(acc, partials[b]);
  const double r = block_tree<kSharedThreads>(acc, red);
  if (threadIdx.x == 0) dsigma[0] = fadd(dsigma[0], r);
}

int64_t gauss_shared_blocks(int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>((n + kSharedThreads - 1) / kSharedThreads,
                                                kSharedMaxBlocks));
}

int launch_gauss_shared(int64_t n, const double* x, const double* p, double sigma, double* dx,
                        double* dp, double* dsigma, double* partials, cudaStream_t stream) {
  GaussUniform u1{};
  if (int rc = gauss_uniform(sigma, &u1)) return rc;
  const double PI = 3.14159265358979323846;
  GaussAllUniform u{};
  u.sigma = sigma;
  u.t3 = 2 * sigma;
  u.t4 = u.t3 * sigma;
  u.t6 = std::pow(2 * PI, -0.5);
  u.r1 = u1.r1;                               // _d__t9 += _t8 * _r0 -> _r1
  u.ksig = -0.5 * std::pow(sigma, -1.5);      // (-0.5 * pow(sigma, -1.5))
  const int64_t blocks = gauss_shared_blocks(n);
  gauss_shared_kernel<<<(unsigned)blocks, kSharedThreads, 0, stream>>>(x, p, dx, dp, n, u,
                                                                        partials);
  gauss_shared_finish_kernel<<<1, kSharedThreads, 0, stream>>>(partials, (int)blocks, dsigma);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

}  // namespace adcb
