// Checks the fast-mode exp of the chi2 kernels (paper_2203_06139_b200/csrc/fastmath.cuh),
// compiled for the host, against libm over [-745, 0] (run by tests/test_fastmath_cpu.py).
#include <cstdio>
#include <cmath>
#include <random>
#include "fastmath.cuh"
int main() {
  double tab[64];
  for (int j = 0; j < 64; ++j) tab[j] = std::exp2(j / 64.0);
  std::mt19937_64 rng(1);
  double maxulp = 0; double worst = 0;
  for (int i = 0; i < 2000000; ++i) {
    double x = -std::uniform_real_distribution<double>(0, 1)(rng) * (i % 3 == 0 ? 745.0 : (i % 3 == 1 ? 30.0 : 1.0));
    double a = adcb::exp_nonpos(x, tab), b = std::exp(x);
    if (b < 2.2250738585072014e-308) { if (std::fabs(a - b) > 5e-324 * 2) { printf("sub bad %g %g %g\n", x, a, b); return 1;} continue; }
    double ulp = std::fabs(a - b) / (std::nextafter(b, INFINITY) - b);
    if (ulp > maxulp) { maxulp = ulp; worst = x; }
  }
  printf("max ulp %.3f at %.17g\n", maxulp, worst);
  return maxulp < 1.5 ? 0 : 1;
}
