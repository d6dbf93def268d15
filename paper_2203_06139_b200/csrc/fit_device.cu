// Device-resident fit iteration: one CUDA graph per
// steepest-descent iteration of FitEngine::fit (fit.cpp:315-425) —
//   parameters -> QDev, gradient pass (K3 + K4), gradient finalize +
//   convergence test + Armijo trial construction, multi-candidate value pass
//   (K3m + K4), trial finalize + first-accepted selection —
// with no host work between the steps and one synchronisation per iteration.
// Every operation is the host loop's (chi2_host.cpp: adc_chi2_finalize, the
// trial arithmetic, the Armijo test, the clamp), one IEEE op at a time in the
// same order, so the iterates are bit-identical to the host-driven loop.
#include <cmath>

#include "chi2_internal.h"
#include "common.cuh"
#include "fit_device.h"

namespace adcb {

namespace {

// QDev of one parameter vector: q and, for the width parameters, 1/q
// (fill_qdev, chi2.cu).  The AD passes read nothing else.
__device__ void write_qdev(double* dst, int model, int np, const double* q) {
  for (int i = 0; i < kMaxNp; ++i) {
    dst[i] = i < np ? q[i] : 0.0;
    dst[kMaxNp + i] = 0.0;
  }
  if (model == ADC_MODEL_GPOLY) {
    dst[kMaxNp + 2] = fdiv(1.0, q[2]);
  } else {
    for (int j = 2; j < np; j += 3) dst[kMaxNp + j] = fdiv(1.0, q[j]);
  }
}

__global__ void fit_qdev_kernel(FitDevState* st, int model, int np, double* qdev) {
  if (threadIdx.x == 0 && blockIdx.x == 0) write_qdev(qdev, model, np, st->q);
}

// adc_chi2_finalize's fixed pairwise tree, one record column per thread.
__device__ void column_tree(double* r, int64_t nchunks, int R, int v) {
  for (int64_t s = 1; s < nchunks; s *= 2)
    for (int64_t i = 0; i + s < nchunks; i += 2 * s) r[i * R + v] = fadd(r[i * R + v], r[(i + s) * R + v]);
}

// Gradient finalize (adc_chi2_finalize), convergence test, direction = g,
// gd, and the first batch of Armijo trials t = 1, 1/2, ... (fit.cpp:383-403)
// written as QDev rows for the multi-candidate pass.
__global__ void __launch_bounds__(128) fit_grad_kernel(FitDevState* st, const double* records,
                                                       double* scratch, int64_t nchunks, int np,
                                                       int model, double events, FitDevConst c,
                                                       double* qmulti, int* ncand_dev) {
  const int R = 4 + 3 * np;
  for (int64_t k = threadIdx.x; k < nchunks * R; k += blockDim.x) scratch[k] = records[k];
  __syncthreads();
  for (int v = threadIdx.x; v < R; v += blockDim.x) column_tree(scratch, nchunks, R, v);
  __syncthreads();
  __shared__ double s_gd;
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    const double S = scratch[0], A1 = scratch[1], A2 = scratch[2];
    const double a = fdiv(events, S);
    const double t_sum = fsub(fmul(2.0, A1), fmul(fmul(2.0, a), A2));
    const double s_coef = fmul(fdiv(events, fmul(S, S)), t_sum);
    double gmax = 0.0;
    for (int i = 0; i < np; ++i) {
      const double G0 = scratch[4 + i], G1 = scratch[4 + np + i], G2 = scratch[4 + 2 * np + i];
      const double gi = fsub(fmul(s_coef, G0), fmul(fmul(2.0, a), fsub(G1, fmul(a, G2))));
      st->g[i] = gi;
      gmax = fmax(gmax, fabs(gi));
    }
    st->gmax = gmax;
    st->accepted_k = -1;
    st->evals = 0;         // per iteration
    st->sigma_clamps = 0;  // per iteration
    s_stop = gmax <= c.grad_tol;  // fit.cpp:340-344
    double gd = 0.0;
    for (int i = 0; i < np; ++i) gd = fadd(gd, fmul(st->g[i], st->g[i]));  // direction = g
    st->gd = gd;
    s_gd = gd;
  }
  __syncthreads();
  if (s_stop) {
    if (threadIdx.x == 0) {
      st->status = kFitConvergedGrad;
      st->ncand = 0;
      *ncand_dev = 0;
    }
    return;
  }
  // Trial n (one per thread): t = 1/2^n exactly (the host's repeated *= 0.5),
  // trial = q - t g, the sigma clamp, and its QDev row.
  const int want = st->first_batch;
  for (int n = threadIdx.x; n < want; n += blockDim.x) {
    const double tt = ldexp(1.0, -n);
    if (!(tt >= 1e-18)) continue;
    double* trial = st->trials + (size_t)n * kMaxNp;
    int cl = 0;
    for (int i = 0; i < np; ++i) trial[i] = fsub(st->q[i], fmul(tt, st->g[i]));
    for (int k = 0; k < c.nclamp; ++k) {
      const int i = c.clamp_idx[k];
      if (i >= 0 && i < np && trial[i] < c.sigma_min) {
        trial[i] = c.sigma_min;
        ++cl;
      }
    }
    st->cls[n] = cl;
    st->tvals[n] = tt;
    write_qdev(qmulti + (size_t)n * kQDoubles, model, np, trial);
  }
  if (threadIdx.x == 0) {
    int n = 0;
    while (n < want && ldexp(1.0, -n) >= 1e-18) ++n;  // the host loop's count
    st->ncand = n;
    *ncand_dev = n;
    st->status = kFitRunning;
  }
}

// Each candidate's value record -> chi2 (adc_chi2_finalize, value form), then
// the first trial that satisfies Armijo is taken (fit.cpp:390-403, in order).
__global__ void __launch_bounds__(kMultiMax) fit_accept_kernel(FitDevState* st,
                                                               const double* records,
                                                               double* scratch, int64_t nchunks,
                                                               double events, FitDevConst c) {
  __shared__ double c2[kMultiMax];
  const int n = st->ncand;
  if (n == 0) return;  // converged on the gradient
  const int R = 1 + 3 * n;
  const int k = threadIdx.x;
  if (k < n) {
    double* r = scratch + (size_t)k * nchunks * 4;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const double* src = records + ch * R;
      r[ch * 4 + 0] = src[1 + 3 * k];
      r[ch * 4 + 1] = src[2 + 3 * k];
      r[ch * 4 + 2] = src[3 + 3 * k];
      r[ch * 4 + 3] = src[0];
    }
    for (int v = 0; v < 4; ++v) column_tree(r, nchunks, 4, v);
    const double S = r[0], A1 = r[1], A2 = r[2], C0 = r[3];
    const double a = fdiv(events, S);
    const double two_a = fmul(2.0, a);
    c2[k] = fadd(fsub(C0, fmul(two_a, A1)), fmul(fmul(a, a), A2));
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double cur = st->cur;
  for (int j = 0; j < n; ++j) {
    st->evals += 1;
    if (c2[j] <= fsub(cur, fmul(fmul(c.armijo_c1, st->tvals[j]), st->gd))) {
      const double next = c2[j];
      st->accepted_k = j;
      st->sigma_clamps = st->cls[j];
      const double rel_dec = fdiv(fsub(cur, next), fmax(1.0, fabs(cur)));
      for (int i = 0; i < kMaxNp; ++i) st->q[i] = st->trials[(size_t)j * kMaxNp + i];
      st->cur = next;
      st->rel_dec = rel_dec;
      const int tried = j + 1;
      st->first_batch = min(kMultiMax, max(8, (tried + 8 + 7) / 8 * 8));
      st->status = rel_dec <= c.chi2_rel_tol ? kFitConvergedRelDec : kFitRunning;
      return;
    }
  }
  const double t_next = fmul(st->tvals[n - 1], 0.5);
  st->t_next = t_next;
  st->status = t_next >= 1e-18 ? kFitNeedHost : kFitConvergedNoStep;
}

}  // namespace

int fit_device_enqueue_qdev(FitDevState* st, int model, int np, double* qdev, cudaStream_t s) {
  fit_qdev_kernel<<<1, 32, 0, s>>>(st, model, np, qdev);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int fit_device_enqueue_grad(FitDevState* st, const double* records, double* scratch,
                            int64_t nchunks, int np, int model, double events,
                            const FitDevConst& c, double* qmulti, int* ncand_dev, cudaStream_t s) {
  fit_grad_kernel<<<1, 128, 0, s>>>(st, records, scratch, nchunks, np, model, events, c, qmulti,
                                    ncand_dev);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int fit_device_enqueue_accept(FitDevState* st, const double* records, double* scratch,
                              int64_t nchunks, double events, const FitDevConst& c,
                              cudaStream_t s) {
  fit_accept_kernel<<<1, kMultiMax, 0, s>>>(st, records, scratch, nchunks, events, c);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

}  // namespace adcb
