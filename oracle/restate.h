/* restate.h — TEST INFRASTRUCTURE (oracle).  Plain-C restatement of the
 * reference's arithmetic on the hot path, used only by tests/, smoke() and
 * bench.py's cpu_baseline leg as the CHECKER.  Never linked into the product.
 *
 * Every function transcribes the code the reference generates or runs, one
 * IEEE operation per source operation, compiled with -ffp-contract=off:
 *   rs_gauss_grad_0_1   <- proj/tests/golden/gauss_grad_0_1.golden:1-42
 *   rs_gauss_grad_shared_batch <- compute_shared (kernels.dsl:16-21) calling
 *                          differentiate_gradient(gauss, {x, p, sigma})
 *   rs_gaussnd_grad_0_1 <- differentiate_gradient(gaussnd,{x,p}) output
 *                          (oracle/dsl/gaussnd.dsl; reverse.cpp:703-725)
 *   rs_gsum / rs_gsum_grad_1   <- fit.cpp:125-138 model + its generated gradient
 *   rs_gpoly / rs_gpoly_grad_1 <- oracle/dsl/gpoly.dsl + its generated gradient
 *   rs_chi2 / rs_chi2_gradient <- FitEngine::chi2 / chi2_gradient,
 *                                 proj/src/fit.cpp:206-222 / 224-259
 *   rs_model_grad_numeric      <- model_gradient's Numeric provider
 *                                 (fit.cpp:187-190 -> numdiff.cpp:38-87)
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * function with golden vectors written by oracle/_ref/ref_tool (the
 * unmodified reference library) — see tests/golden/README.md.
 */
#ifndef ADC_ORACLE_RESTATE_H
#define ADC_ORACLE_RESTATE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RS_MODEL_GSUM = 0, RS_MODEL_GPOLY = 1 };
/* adc::GradientProvider (fit.hpp:52): AdReverse, Numeric. */
enum { RS_PROVIDER_AD = 0, RS_PROVIDER_NUMERIC = 1 };

/* Listing-1 batch: for g in [0,n): gauss_grad_0_1(x[g],p[g],sigma,&dx[g],&dp[g]) */
void rs_gauss_grad_batch(const double* x, const double* p, double sigma, double* dx, double* dp,
                         int64_t n);

/* compute_shared (kernels.dsl:16-21) forced sequential: gauss_grad over x, p,
 * sigma per point; dx, dp private, the three sigma contributions added to
 * dsigma[0] in point order (launch with LaunchOptions{unsafe, sequential}). */
void rs_gauss_grad_shared_batch(const double* x, const double* p, double sigma, double* dx,
                                double* dp, double* dsigma, int64_t n);
/* Compensated total of all sigma contributions and of their magnitudes (the
 * tolerance scale for an order-changed reduction). */
void rs_gauss_shared_dsigma_compensated(const double* x, const double* p, double sigma, int64_t n,
                                        double* total, double* abs_total);

/* N-dim batch over structure-of-arrays rows: element (d, i) at [d*ld + i]. */
void rs_gaussnd_grad_batch(const double* x, const double* p, double sigma, int64_t dim, int64_t n,
                           int64_t ld, double* dx, double* dp);

/* Shared mean vector: every point g runs gaussnd_grad_0_1(x[:, g], p, ...,
 * dx[:, g], dp) with one p[dim] and one dp[dim], points in order (dx may not
 * be NULL here).  And the compensated per-dim total of the dp contributions
 * with the sum of their magnitudes (the tolerance scale). */
void rs_gaussnd_grad_shared_p(const double* x, const double* p, double sigma, int64_t dim,
                              int64_t n, int64_t ld, double* dx, double* dp);
void rs_gaussnd_shared_p_dp_compensated(const double* x, const double* p, double sigma, int64_t dim,
                                        int64_t n, int64_t ld, double* total, double* abs_total);

/* One point, contiguous row of length dim (the layout Program::eval sees). */
void rs_gaussnd_grad_0_1(const double* x, const double* p, double sigma, int64_t dim, double* dx,
                         double* dp);

double rs_model(int model, double x, const double* q, int64_t np);
void rs_model_grad(int model, double x, const double* q, int64_t np, double* slot);

/* GradientProvider::Numeric: central differences of the model over q. */
void rs_model_grad_numeric(int model, double x, const double* q, int64_t np, double* slot);

/* Sequential, verbatim fit.cpp:206-222. */
double rs_chi2(int model, const double* counts, int64_t bins, double lo, double hi, double events,
               const double* q, int64_t np);
/* Sequential, verbatim fit.cpp:224-259. */
void rs_chi2_gradient(int model, const double* counts, int64_t bins, double lo, double hi,
                      double events, const double* q, int64_t np, double* out);
/* Same with the gradient provider chosen (RS_PROVIDER_*). */
void rs_chi2_gradient_p(int model, int provider, const double* counts, int64_t bins, double lo,
                        double hi, double events, const double* q, int64_t np, double* out);
/* Same formula with Neumaier-compensated sums (the accuracy reference for
 * order-changed GPU reductions).  abs_out[i] = sum_j |w_j dm_j/dq_i|, the
 * scale the reduction tolerance is stated against. */
void rs_chi2_gradient_compensated(int model, const double* counts, int64_t bins, double lo,
                                  double hi, double events, const double* q, int64_t np,
                                  double* out, double* abs_out);
/* fd_out[i] = sum_j |w_j| |m_j| eps / (2 h_i): one primal ulp amplified by the
 * difference quotient, the extra tolerance unit of the Numeric provider
 * (the GPU's exp differs from glibc's by <= 1-2 ulp). */
void rs_chi2_gradient_compensated_p(int model, int provider, const double* counts, int64_t bins,
                                    double lo, double hi, double events, const double* q,
                                    int64_t np, double* out, double* abs_out, double* fd_out);
double rs_chi2_compensated(int model, const double* counts, int64_t bins, double lo, double hi,
                           double events, const double* q, int64_t np, double* abs_out);

#ifdef __cplusplus
}
#endif
#endif
