// Gaussian peak on a quadratic background, the config-3 histogram model
// (BASELINE.json configs[2]).  Same argument convention as the reference
// FitEngine model gsum(real x, real[] q, integer k)
// (/root/reference/proj/src/fit.cpp:125-138, packed at fit.cpp:146-153), so
// one engine packs both; k is unused here.
// q = [amp, mu, sigma, c0, c1, c2].
device host real gpoly(real x, real[] q, integer k) {
  real z = (x - q[1]) / q[2];
  real g = q[0] * exp(-0.5 * z * z);
  return g + q[3] + q[4] * x + q[5] * x * x;
}
