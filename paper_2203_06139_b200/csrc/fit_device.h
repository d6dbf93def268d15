// Device-resident steepest-descent iteration (fit_device.cu) and its state.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "chi2_internal.h"

namespace adcb {

enum {
  kFitRunning = 0,
  kFitConvergedGrad = 1,    // gmax <= grad_tol (fit.cpp:340-344)
  kFitConvergedRelDec = 2,  // relative decrease <= chi2_rel_tol
  kFitConvergedNoStep = 3,  // no Armijo step down to t = 1e-18
  kFitNeedHost = 4          // the first batch had no acceptable trial: continue on the host
};

// Lives in device memory; copied back (whole) once per iteration.
struct FitDevState {
  double q[kMaxNp];
  double g[kMaxNp];
  double cur, gd, gmax, rel_dec, t_next;
  double tvals[kMultiMax];
  double trials[kMultiMax * kMaxNp];
  int cls[kMultiMax];
  int ncand, first_batch, status, accepted_k, sigma_clamps, evals;
  // device loop (WHILE node) bookkeeping, cumulative over one fit
  int passes, budget, iters, clamps_total, n_grad;
  long long evals_total;
  unsigned long long grad_ns, t0, t1;  // gradient-pass time from %globaltimer
  // Newton option (fit.cpp:346-381): search direction and probe steps
  double dir[kMaxNp];
  double steps[kMaxNp];
};

struct FitDevConst {
  double grad_tol, chi2_rel_tol, sigma_min, armijo_c1;
  int clamp_idx[kMaxNp];
  int nclamp;
  int np;
  int margin;     // line-search batch margin (adc_cuda_fit)
  int newton;     // FitOptions::use_hessian: numeric-Hessian Newton direction
  int numeric;    // GradientProvider::Numeric gradient passes
  double cbrt_eps;  // std::cbrt(DBL_EPSILON) from the host libm
  double* trace;  // [trace_cap][np] iterates (row 0 written by the host)
  int trace_cap;
};

// h0 = cbrt(eps) also writes the numeric provider's probe block (0: AD only).
int fit_device_enqueue_qdev(FitDevState* st, int model, int np, double* qdev, double h0,
                            cudaStream_t s);
int fit_device_enqueue_grad(FitDevState* st, const double* records, double* scratch,
                            int64_t nchunks, int np, int model, double events,
                            const FitDevConst& c, double* qmulti, int* ncand_dev, cudaStream_t s);
// Newton option: finalize the 2 np probe gradients (records [2np][nchunks][R]
// at probe_records, stride per), central-difference Hessian, the damped
// solve with its retries, and the Armijo trials along the direction.
int fit_device_enqueue_newton(FitDevState* st, const double* probe_records, size_t per,
                              double* scratch, int64_t nchunks, int np, int model, double events,
                              const FitDevConst& c, double* qmulti, int* ncand_dev,
                              cudaStream_t s);
int fit_device_enqueue_accept(FitDevState* st, const double* records, double* scratch,
                              int64_t nchunks, double events, const FitDevConst& c,
                              cudaStream_t s);
// Sharded plans (peer transport): all ranks' exchanged records -> compact.
int fit_device_enqueue_compact(const double* out, size_t count, int world, const int64_t* rbegin,
                               int64_t nchunks, int nb, int64_t maxc, int Rfix,
                               const int* ncand_dev, double* dst, cudaStream_t s);
// End of a loop body: the host loop's bookkeeping for the pass just run, then
// the WHILE node's condition (continue while running and within budget).
int fit_device_enqueue_loop_ctl(FitDevState* st, cudaGraphConditionalHandle h,
                                const FitDevConst& c, cudaStream_t s);

}  // namespace adcb
