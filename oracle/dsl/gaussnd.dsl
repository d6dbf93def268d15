// N-dimensional isotropic Gaussian over a point's coordinate row, written in
// the reference DSL (new: the reference corpus only has the 1-D `gauss`,
// /root/reference/proj/corpus/gauss.dsl:2-5).  The arithmetic follows gauss.dsl
// and the loop-over-array pattern follows sumn.dsl:3-9.  The normalisation is
// the 1-D one, pow(2*PI,-0.5)*pow(sigma,-0.5) (gauss.dsl:4): the Clad-style
// pow(2*PI,-dim/2.0) underflows to exactly 0 at dim=1000 (SURVEY.md §0.6),
// which would make every gradient 0 and parity vacuous.
device host real gaussnd(real[] x, real[] p, real sigma, integer dim) {
  real t = 0;
  for (integer i = 0; i < dim; i += 1) {
    t = t + (x[i] - p[i]) * (x[i] - p[i]);
  }
  t = -t / (2 * sigma * sigma);
  return pow(2 * PI, -0.5) * pow(sigma, -0.5) * exp(t);
}
