/* restate.c — TEST INFRASTRUCTURE (oracle).  See restate.h for the contract
 * and the reference lines each function follows.  Compile with
 * -ffp-contract=off: every statement below is one IEEE double operation in
 * the order the reference interpreter executes it (eval.cpp:524-594), so the
 * results are bit-identical to Program::eval on the same libm. */
#include "restate.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPI = 3.14159265358979323846; /* ast.cpp:119-123 */

/* gauss_grad_0_1.golden:1-42, statement for statement (adjoint temporaries
 * start at 0 and are accumulated with +=, which is kept: 0 + v maps -0 to +0). */
static void gauss_grad_0_1(double x, double p, double sigma, double* _d_x, double* _d_p) {
  double _d__t0 = 0, _d__t1 = 0, _d__t2 = 0, _d_t = 0, _d__t9 = 0, _d__t10 = 0;
  double _t0 = x - p;
  double _t1 = -_t0;
  double _t2 = _t1 * _t0;
  double _t3 = 2 * sigma;
  double _t4 = _t3 * sigma;
  double t = _t2 / _t4;
  double _t5 = 2 * kPI;
  double _t6 = pow(_t5, -0.5);
  double _t7 = pow(sigma, -0.5);
  double _t8 = _t6 * _t7;
  double _t9 = exp(t);
  _d__t10 += 1;
  double _r0 = _d__t10;
  _d__t9 += _t8 * _r0;
  double _r1 = _d__t9;
  double _q0 = _t9;
  _d_t += _r1 * _q0;
  double _r2 = _d_t;
  _d__t2 += _r2 / _t4;
  double _r3 = _d__t2;
  _d__t1 += _r3 * _t0;
  _d__t0 += _t1 * _r3;
  double _r4 = _d__t1;
  _d__t0 += -_r4;
  double _r5 = _d__t0;
  _d_x[0] += _r5;
  _d_p[0] += -_r5;
}

void rs_gauss_grad_batch(const double* x, const double* p, double sigma, double* dx, double* dp,
                         int64_t n) {
  for (int64_t g = 0; g < n; ++g) gauss_grad_0_1(x[g], p[g], sigma, dx + g, dp + g);
}

/* gauss_grad (all of x, p, sigma): the printed output of
 * differentiate_gradient(gauss, {x, p, sigma}) (ref_tool print kernels gauss
 * x p sigma), statement for statement.  The three _d_sigma[0] += statements
 * are returned separately in sig[0..2] so the caller decides how they reach
 * the shared slot. */
static void gauss_grad_all(double x, double p, double sigma, double* _d_x, double* _d_p,
                           double* sig) {
  double _d__t0 = 0, _d__t1 = 0, _d__t2 = 0, _d__t3 = 0, _d__t4 = 0, _d_t = 0, _d__t7 = 0,
         _d__t8 = 0, _d__t9 = 0, _d__t10 = 0;
  double _t0 = x - p;
  double _t1 = -_t0;
  double _t2 = _t1 * _t0;
  double _t3 = 2 * sigma;
  double _t4 = _t3 * sigma;
  double t = _t2 / _t4;
  double _t5 = 2 * kPI;
  double _t6 = pow(_t5, -0.5);
  double _t7 = pow(sigma, -0.5);
  double _t8 = _t6 * _t7;
  double _t9 = exp(t);
  _d__t10 += 1;
  double _r0 = _d__t10;
  _d__t8 += _r0 * _t9;
  _d__t9 += _t8 * _r0;
  double _r1 = _d__t9;
  double _q0 = _t9;
  _d_t += _r1 * _q0;
  double _r2 = _d__t8;
  _d__t7 += _t6 * _r2;
  double _r3 = _d__t7;
  sig[0] = _r3 * (-0.5 * pow(sigma, -1.5));
  double _r4 = _d_t;
  double _q1 = t;
  _d__t2 += _r4 / _t4;
  _d__t4 += -(_r4 * _q1 / _t4);
  double _r5 = _d__t4;
  _d__t3 += _r5 * sigma;
  sig[1] = _t3 * _r5;
  double _r6 = _d__t3;
  sig[2] = 2 * _r6;
  double _r7 = _d__t2;
  _d__t1 += _r7 * _t0;
  _d__t0 += _t1 * _r7;
  double _r8 = _d__t1;
  _d__t0 += -_r8;
  double _r9 = _d__t0;
  _d_x[0] += _r9;
  _d_p[0] += -_r9;
}

void rs_gauss_grad_shared_batch(const double* x, const double* p, double sigma, double* dx,
                                double* dp, double* dsigma, int64_t n) {
  for (int64_t g = 0; g < n; ++g) {
    double sig[3];
    gauss_grad_all(x[g], p[g], sigma, dx + g, dp + g, sig);
    dsigma[0] += sig[0];
    dsigma[0] += sig[1];
    dsigma[0] += sig[2];
  }
}

/* ---- compensated (Neumaier) sums ------------------------------------------ */
typedef struct { double s, c; } nsum;
static void nadd(nsum* a, double v) {
  double t = a->s + v;
  if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
  else a->c += (v - t) + a->s;
  a->s = t;
}
static double nval(const nsum* a) { return a->s + a->c; }

void rs_gauss_shared_dsigma_compensated(const double* x, const double* p, double sigma, int64_t n,
                                        double* total, double* abs_total) {
  nsum s = {0, 0}, a = {0, 0};
  for (int64_t g = 0; g < n; ++g) {
    double sig[3], dx = 0, dp = 0;
    gauss_grad_all(x[g], p[g], sigma, &dx, &dp, sig);
    for (int k = 0; k < 3; ++k) {
      nadd(&s, sig[k]);
      nadd(&a, fabs(sig[k]));
    }
  }
  *total = nval(&s);
  *abs_total = nval(&a);
}

/* gaussnd_grad_0_1 as emitted by differentiate_gradient (reverse.cpp:335-553):
 * forward loop pushes _t0,_t1,t; reverse loop pops them.  Only _t0 is read by
 * an adjoint rule, so the tape is replaced by the per-element recomputation
 * x[i]-p[i], which yields the identical bits. */
static void gaussnd_grad_strided2(const double* x, int64_t xs, const double* p, int64_t ps,
                                  double sigma, int64_t dim, double* _d_x, int64_t dxs,
                                  double* _d_p, int64_t dps);

static void gaussnd_grad_strided(const double* x, const double* p, double sigma, int64_t dim,
                                 int64_t stride, double* _d_x, double* _d_p) {
  gaussnd_grad_strided2(x, stride, p, stride, sigma, dim, _d_x, stride, _d_p, stride);
}

/* x, p, _d_x, _d_p each with its own element stride (the shared-p form reads
 * one p vector and accumulates into one dp vector for every point). */
static void gaussnd_grad_strided2(const double* x, int64_t xs, const double* p, int64_t ps,
                                  double sigma, int64_t dim, double* _d_x, int64_t dxs,
                                  double* _d_p, int64_t dps) {
  double _d_t = 0, _d__t0 = 0, _d__t1 = 0, _d__t2 = 0, _d__t9 = 0, _d__t10 = 0;
  double t = 0;
  for (int64_t i = 0; i < dim; ++i) {
    double _t0 = x[i * xs] - p[i * ps];
    double _t1 = _t0 * _t0;
    t = t + _t1;
  }
  double _t2 = -t;
  double _t3 = 2 * sigma;
  double _t4 = _t3 * sigma;
  t = _t2 / _t4;
  double _t5 = 2 * kPI;
  double _t6 = pow(_t5, -0.5);
  double _t7 = pow(sigma, -0.5);
  double _t8 = _t6 * _t7;
  double _t9 = exp(t);
  _d__t10 += 1;
  double _r0 = _d__t10;
  _d__t10 = 0;
  _d__t9 += _t8 * _r0;
  double _r1 = _d__t9;
  _d__t9 = 0;
  double _q0 = _t9;
  _d_t += _r1 * _q0;
  double _r2 = _d_t;
  _d_t = 0;
  _d__t2 += _r2 / _t4;
  double _r3 = _d__t2;
  _d__t2 = 0;
  _d_t += -_r3;
  for (int64_t j = 0; j < dim; ++j) {
    int64_t i = dim - 1 - j;
    double _t0 = x[i * xs] - p[i * ps];
    double _r4 = _d_t;
    _d_t = 0;
    _d_t += _r4;
    _d__t1 += _r4;
    double _r5 = _d__t1;
    _d__t1 = 0;
    _d__t0 += _r5 * _t0;
    _d__t0 += _t0 * _r5;
    double _r6 = _d__t0;
    _d__t0 = 0;
    _d_x[i * dxs] += _r6;
    _d_p[i * dps] += -_r6;
  }
}

void rs_gaussnd_grad_shared_p(const double* x, const double* p, double sigma, int64_t dim,
                              int64_t n, int64_t ld, double* dx, double* dp) {
  for (int64_t g = 0; g < n; ++g) gaussnd_grad_strided2(x + g, ld, p, 1, sigma, dim, dx + g, ld, dp, 1);
}

void rs_gaussnd_shared_p_dp_compensated(const double* x, const double* p, double sigma, int64_t dim,
                                        int64_t n, int64_t ld, double* total, double* abs_total) {
  /* per point, the contributions -_r6_d land in a private row; sum them per d
   * with Neumaier compensation (and their magnitudes) */
  double* row = (double*)malloc((size_t)dim * sizeof(double));
  double* dxr = (double*)malloc((size_t)dim * sizeof(double));
  double* s = (double*)calloc((size_t)dim, sizeof(double));
  double* c = (double*)calloc((size_t)dim, sizeof(double));
  double* a = (double*)calloc((size_t)dim, sizeof(double));
  for (int64_t g = 0; g < n; ++g) {
    for (int64_t d = 0; d < dim; ++d) row[d] = 0.0, dxr[d] = 0.0;
    gaussnd_grad_strided2(x + g, ld, p, 1, sigma, dim, dxr, 1, row, 1);
    for (int64_t d = 0; d < dim; ++d) {
      const double v = row[d];
      const double t = s[d] + v;
      if (fabs(s[d]) >= fabs(v)) c[d] += (s[d] - t) + v;
      else c[d] += (v - t) + s[d];
      s[d] = t;
      a[d] += fabs(v);
    }
  }
  for (int64_t d = 0; d < dim; ++d) {
    total[d] = s[d] + c[d];
    abs_total[d] = a[d];
  }
  free(row);
  free(dxr);
  free(s);
  free(c);
  free(a);
}

void rs_gaussnd_grad_0_1(const double* x, const double* p, double sigma, int64_t dim, double* dx,
                         double* dp) {
  gaussnd_grad_strided(x, p, sigma, dim, 1, dx, dp);
}

void rs_gaussnd_grad_batch(const double* x, const double* p, double sigma, int64_t dim, int64_t n,
                           int64_t ld, double* dx, double* dp) {
  for (int64_t i = 0; i < n; ++i) gaussnd_grad_strided(x + i, p + i, sigma, dim, ld, dx + i, dp + i);
}

/* ---- histogram models ----------------------------------------------------
 * gsum: fit.cpp:125-138 (interpreted: z = (x-mu)/sg; acc + amp*exp((-0.5*z)*z)).
 * gpoly: oracle/dsl/gpoly.dsl. */
static double gsum(double x, const double* q, int64_t k) {
  double acc = 0;
  for (int64_t j = 0; j < k; ++j) {
    int64_t b = 3 * j;
    double amp = q[b], mu = q[b + 1], sg = q[b + 2];
    double z = (x - mu) / sg;
    acc = acc + amp * exp(-0.5 * z * z);
  }
  return acc;
}

/* gsum_grad_1 as emitted (see oracle/ref_tool print gsum gsum q). */
static void gsum_grad_1(double x, const double* q, int64_t k, double* _d_q) {
  for (int64_t jj = 0; jj < k; ++jj) {
    int64_t j = k - 1 - jj; /* reverse loop; slots are disjoint per j */
    int64_t b = 3 * j;
    double amp = q[b], mu = q[b + 1], sg = q[b + 2];
    double _t0 = x - mu;
    double z = _t0 / sg;
    double _t1 = -0.5 * z;
    double _t2 = _t1 * z;
    double _t3 = exp(_t2);
    double _d_acc = 1; /* _d_acc += 1, then per iteration _r0=_d_acc; _d_acc=0; _d_acc+=_r0 */
    double _r0 = _d_acc;
    double _d__t4 = 0, _d_amp = 0, _d__t3 = 0, _d__t2 = 0, _d__t1 = 0, _d_z = 0, _d__t0 = 0,
           _d_sg = 0, _d_mu = 0;
    _d__t4 += _r0;
    double _r1 = _d__t4;
    _d_amp += _r1 * _t3;
    _d__t3 += amp * _r1;
    double _r2 = _d__t3;
    double _q0 = _t3;
    _d__t2 += _r2 * _q0;
    double _r3 = _d__t2;
    _d__t1 += _r3 * z;
    _d_z += _t1 * _r3;
    double _r4 = _d__t1;
    _d_z += -0.5 * _r4;
    double _r5 = _d_z;
    double _q1 = z;
    _d__t0 += _r5 / sg;
    _d_sg += -(_r5 * _q1 / sg);
    double _r6 = _d__t0;
    _d_mu += -_r6;
    _d_q[b + 2] += _d_sg;
    _d_q[b + 1] += _d_mu;
    _d_q[b] += _d_amp;
  }
}

static double gpoly(double x, const double* q) {
  double z = (x - q[1]) / q[2];
  double g = q[0] * exp(-0.5 * z * z);
  return g + q[3] + q[4] * x + q[5] * x * x;
}

/* gpoly_grad_1 as emitted (see oracle/ref_tool print gpoly gpoly q). */
static void gpoly_grad_1(double x, const double* q, double* _d_q) {
  double _d__t0 = 0, _d_z = 0, _d__t1 = 0, _d__t2 = 0, _d__t3 = 0, _d_g = 0, _d__t4 = 0,
         _d__t5 = 0, _d__t6 = 0, _d__t7 = 0, _d__t8 = 0, _d__t9 = 0;
  double _t0 = x - q[1];
  double z = _t0 / q[2];
  double _t1 = -0.5 * z;
  double _t2 = _t1 * z;
  double _t3 = exp(_t2);
  _d__t9 += 1;
  double _r0 = _d__t9;
  _d__t6 += _r0;
  _d__t8 += _r0;
  double _r1 = _d__t8;
  _d__t7 += _r1 * x;
  double _r2 = _d__t7;
  _d_q[5] += _r2 * x;
  double _r3 = _d__t6;
  _d__t4 += _r3;
  _d__t5 += _r3;
  double _r4 = _d__t5;
  _d_q[4] += _r4 * x;
  double _r5 = _d__t4;
  _d_g += _r5;
  _d_q[3] += _r5;
  double _r6 = _d_g;
  _d_q[0] += _r6 * _t3;
  _d__t3 += q[0] * _r6;
  double _r7 = _d__t3;
  double _q0 = _t3;
  _d__t2 += _r7 * _q0;
  double _r8 = _d__t2;
  _d__t1 += _r8 * z;
  _d_z += _t1 * _r8;
  double _r9 = _d__t1;
  _d_z += -0.5 * _r9;
  double _r10 = _d_z;
  double _q1 = z;
  _d__t0 += _r10 / q[2];
  _d_q[2] += -(_r10 * _q1 / q[2]);
  double _r11 = _d__t0;
  _d_q[1] += -_r11;
}

double rs_model(int model, double x, const double* q, int64_t np) {
  return model == RS_MODEL_GSUM ? gsum(x, q, np / 3) : gpoly(x, q);
}

/* FitEngine::model_gradient: out.assign(np, 0) then the generated gradient
 * accumulates into it (fit.cpp:180-186). */
void rs_model_grad(int model, double x, const double* q, int64_t np, double* slot) {
  for (int64_t i = 0; i < np; ++i) slot[i] = 0.0;
  if (model == RS_MODEL_GSUM) gsum_grad_1(x, q, np / 3, slot);
  else gpoly_grad_1(x, q, slot);
}

/* FitEngine::model_gradient, GradientProvider::Numeric branch (fit.cpp:187-190):
 * central_gradient (numdiff.cpp:38-87) over q: per element, step
 * h = cbrt(eps) * max(1, |q_i|) (numdiff.cpp:8-13), two primal evaluations at
 * q_i + h and q_i - h, value (f+ - f-) / (2h). */
void rs_model_grad_numeric(int model, double x, const double* q, int64_t np, double* slot) {
  double work[64];
  const double h0 = cbrt(2.220446049250313e-16);
  for (int64_t i = 0; i < np; ++i) work[i] = q[i];
  for (int64_t i = 0; i < np; ++i) {
    const double xi = work[i];
    const double h = h0 * fmax(1.0, fabs(xi));
    work[i] = xi + 1.0 * h;
    const double fp = rs_model(model, x, work, np);
    work[i] = xi + -1.0 * h;
    const double fm = rs_model(model, x, work, np);
    work[i] = xi;
    slot[i] = (fp - fm) / (2.0 * h);
  }
}

static void model_grad_p(int model, int provider, double x, const double* q, int64_t np,
                         double* slot) {
  if (provider == RS_PROVIDER_NUMERIC) rs_model_grad_numeric(model, x, q, np, slot);
  else rs_model_grad(model, x, q, np, slot);
}

/* Histogram::center, fit.hpp:30-31. */
static double center(int64_t i, double lo, double hi, int64_t bins) {
  double width = (hi - lo) / (double)bins;
  return lo + ((double)i + 0.5) * width;
}

double rs_chi2(int model, const double* counts, int64_t bins, double lo, double hi, double events,
               const double* q, int64_t np) {
  double* m = (double*)malloc((size_t)bins * sizeof(double));
  double s = 0.0;
  for (int64_t j = 0; j < bins; ++j) {
    m[j] = rs_model(model, center(j, lo, hi, bins), q, np);
    s += m[j];
  }
  double sum = 0.0;
  const double scale = events / s;
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    if (c <= 0.0) continue;
    double r = c - scale * m[j];
    sum += r * r / c;
  }
  free(m);
  return sum;
}

void rs_chi2_gradient(int model, const double* counts, int64_t bins, double lo, double hi,
                      double events, const double* q, int64_t np, double* out) {
  rs_chi2_gradient_p(model, RS_PROVIDER_AD, counts, bins, lo, hi, events, q, np, out);
}

void rs_chi2_gradient_p(int model, int provider, const double* counts, int64_t bins, double lo,
                        double hi, double events, const double* q, int64_t np, double* out) {
  for (int64_t i = 0; i < np; ++i) out[i] = 0.0;
  double* m = (double*)malloc((size_t)bins * sizeof(double));
  double bin_grad[64];
  double s = 0.0;
  for (int64_t j = 0; j < bins; ++j) {
    m[j] = rs_model(model, center(j, lo, hi, bins), q, np);
    s += m[j];
  }
  double t_sum = 0.0;
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    if (c <= 0.0) continue;
    double r = c - events * m[j] / s;
    t_sum += 2.0 * r * m[j] / c;
  }
  const double s_coef = events / (s * s) * t_sum;
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    double w = s_coef;
    if (c > 0.0) {
      double r = c - events * m[j] / s;
      w += -2.0 * r / c * events / s;
    }
    if (w == 0.0) continue;
    model_grad_p(model, provider, center(j, lo, hi, bins), q, np, bin_grad);
    for (int64_t i = 0; i < np; ++i) out[i] += w * bin_grad[i];
  }
  free(m);
}

/* ---- compensated (Neumaier) variants -------------------------------------- */

void rs_chi2_gradient_compensated(int model, const double* counts, int64_t bins, double lo,
                                  double hi, double events, const double* q, int64_t np,
                                  double* out, double* abs_out) {
  rs_chi2_gradient_compensated_p(model, RS_PROVIDER_AD, counts, bins, lo, hi, events, q, np, out,
                                 abs_out, NULL);
}

void rs_chi2_gradient_compensated_p(int model, int provider, const double* counts, int64_t bins,
                                    double lo, double hi, double events, const double* q,
                                    int64_t np, double* out, double* abs_out, double* fd_out) {
  nsum facc[64];
  memset(facc, 0, sizeof facc);
  const double h0 = cbrt(2.220446049250313e-16);
  double* m = (double*)malloc((size_t)bins * sizeof(double));
  double bin_grad[64];
  nsum acc[64], aacc[64];
  memset(acc, 0, sizeof acc);
  memset(aacc, 0, sizeof aacc);
  nsum s = {0, 0}, ts = {0, 0};
  for (int64_t j = 0; j < bins; ++j) {
    m[j] = rs_model(model, center(j, lo, hi, bins), q, np);
    nadd(&s, m[j]);
  }
  const double S = nval(&s);
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    if (c <= 0.0) continue;
    double r = c - events * m[j] / S;
    nadd(&ts, 2.0 * r * m[j] / c);
  }
  const double s_coef = events / (S * S) * nval(&ts);
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    double w = s_coef;
    if (c > 0.0) {
      double r = c - events * m[j] / S;
      w += -2.0 * r / c * events / S;
    }
    if (w == 0.0) continue;
    model_grad_p(model, provider, center(j, lo, hi, bins), q, np, bin_grad);
    for (int64_t i = 0; i < np; ++i) {
      nadd(&acc[i], w * bin_grad[i]);
      nadd(&aacc[i], fabs(w * bin_grad[i]));
      /* one ulp of the primal, amplified by the difference quotient 1/(2h) */
      nadd(&facc[i], fabs(w) * fabs(m[j]) * 2.220446049250313e-16 /
                         (2.0 * h0 * fmax(1.0, fabs(q[i]))));
    }
  }
  for (int64_t i = 0; i < np; ++i) {
    out[i] = nval(&acc[i]);
    if (abs_out) abs_out[i] = nval(&aacc[i]);
    if (fd_out) fd_out[i] = nval(&facc[i]);
  }
  free(m);
}

double rs_chi2_compensated(int model, const double* counts, int64_t bins, double lo, double hi,
                           double events, const double* q, int64_t np, double* abs_out) {
  double* m = (double*)malloc((size_t)bins * sizeof(double));
  nsum s = {0, 0}, sum = {0, 0}, asum = {0, 0};
  for (int64_t j = 0; j < bins; ++j) {
    m[j] = rs_model(model, center(j, lo, hi, bins), q, np);
    nadd(&s, m[j]);
  }
  const double scale = events / nval(&s);
  for (int64_t j = 0; j < bins; ++j) {
    double c = counts[j];
    if (c <= 0.0) continue;
    double r = c - scale * m[j];
    nadd(&sum, r * r / c);
    nadd(&asum, c + 2.0 * scale * m[j] + scale * m[j] * (scale * m[j] / c));
  }
  free(m);
  if (abs_out) *abs_out = nval(&asum);
  return nval(&sum);
}
