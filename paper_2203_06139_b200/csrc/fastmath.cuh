// Fast-mode math shared by the chi2 kernels; __host__ __device__ so the CPU
// test suite can check it against libm (tests/test_fastmath_cpu.py).
#pragma once

#include <stdint.h>
#include <string.h>

#include <cmath>
#ifdef __CUDACC__
#define ADCB_HD __host__ __device__ __forceinline__
#else
#define ADCB_HD inline
#endif
#define ADCB_FMA(a, b, c) fma(a, b, c)  // fused, one rounding, host and device

namespace adcb {

// exp for the non-positive arguments the histogram models produce
// (t2 = -0.5 z^2).  x = (k/64) ln2 + r with |r| <= ln2/128;
// exp(x) = 2^(k>>6) * T[k&63] * p(r), T[j] = 2^(j/64) (table supplied by the
// caller, in shared memory on the device), p = degree-5 Taylor polynomial
// (truncation < 4e-17).  ~11 FP64 operations.  Max error 1 ulp (measured over
// 2e6 arguments against glibc, tests/test_fastmath_cpu.py).  Results
// below 2^-1020 are assembled in two scaling steps so subnormals stay right.
ADCB_HD double exp_nonpos(double x, const double* tab) {
  const double kInvLn2x64 = 0x1.71547652b82fep+6;  // 64 / ln 2
  const double kLn2d64Hi = 0x1.62e42fefa39efp-7;   // ln 2 / 64 (rounded)
  const double kLn2d64Lo = 0x1.abc9e3b39803fp-62;  // ln 2 / 64 - hi
  const double shifter = 0x1.8p52;                 // round-to-integer trick
  x = x < -745.2 ? -745.2 : x;
  const double kd = ADCB_FMA(x, kInvLn2x64, shifter);
  uint64_t kbits;
  memcpy(&kbits, &kd, 8);
  const int k = (int)(uint32_t)kbits;  // low word holds k (two's complement)
  const double kf = kd - shifter;
  double r = ADCB_FMA(-kf, kLn2d64Hi, x);
  r = ADCB_FMA(-kf, kLn2d64Lo, r);
  // exp(r) - 1 = r + r^2 ((1/2 + r/6) + r^2 (1/24 + r/120))  (Estrin: the
  // dependency chain is 3 deep instead of Horner's 5), then T (1 + q) as one
  // FMA so only the final rounding and T's own half-ulp remain.
  const double r2 = r * r;
  const double p23 = ADCB_FMA(r, 1.0 / 6.0, 0.5);
  const double p45 = ADCB_FMA(r, 1.0 / 120.0, 1.0 / 24.0);
  const double q = ADCB_FMA(r2, ADCB_FMA(r2, p45, p23), r);
  const double t = tab[k & 63];
  const double tp = ADCB_FMA(t, q, t);  // in [0.99, 2)
  const int e = k >> 6;               // floor(k / 64)
  const bool deep = e < -1020;
  const int eb = deep ? e + 600 : e;
  uint64_t b;
  memcpy(&b, &tp, 8);
  b += (uint64_t)(int64_t)eb << 52;
  double v;
  memcpy(&v, &b, 8);
  return deep ? v * 0x1p-600 : v;
}

}  // namespace adcb
