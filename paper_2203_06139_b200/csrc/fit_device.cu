// Device-resident fit loop: the body of one
// iteration of FitEngine::fit (fit.cpp:315-425) —
//   parameters -> QDev, gradient pass (K3 + K4), gradient finalize +
//   convergence test + Armijo trial construction (or, with the Newton
//   option, the 2 np probe gradients as one batched pass, the Hessian and the
//   damped solve first), multi-candidate value pass (K3m + K4), trial
//   finalize + first-accepted selection, loop control —
// captured once as the body of a CUDA graph WHILE node; the loop-control
// kernel does the host loop's bookkeeping and sets the node's condition, so
// iterations follow each other with no host work in between.
// Every operation is the host loop's (chi2_host.cpp: adc_chi2_finalize, the
// trial arithmetic, the Armijo test, the clamp, damped_solve), one IEEE op at
// a time in the same order, so the iterates are bit-identical to the
// host-driven loop.
#include <cmath>

#include "chi2_internal.h"
#include "common.cuh"
#include "fit_device.h"

namespace adcb {

namespace {

// QDev of one parameter vector: q and, for the width parameters, 1/q
// (fill_qdev, chi2.cu) — all the AD passes read.  With h0 = cbrt(eps) (the
// numeric provider) also the QNum block the numeric pass reads: probes
// q +- h, h = h0 max(1, |q|), their width reciprocals, 2h and 1/(2h), op for
// op as fill_qdev computes them on the host.
__device__ void write_qdev(double* dst, int model, int np, const double* q, double h0 = 0.0) {
  for (int i = 0; i < kMaxNp; ++i) {
    dst[i] = i < np ? q[i] : 0.0;
    dst[kMaxNp + i] = 0.0;
  }
  double* qp = dst + 2 * kMaxNp;  // QNum: qp, qm, invp, invm, h2, rh2
  double* qm = qp + kMaxNp;
  double* invp = qm + kMaxNp;
  double* invm = invp + kMaxNp;
  double* h2 = invm + kMaxNp;
  double* rh2 = h2 + kMaxNp;
  if (h0 != 0.0) {
    for (int i = 0; i < kMaxNp; ++i) {
      if (i < np) {
        const double h = fmul(h0, fmax(1.0, fabs(q[i])));
        qp[i] = fadd(q[i], h);
        qm[i] = fadd(q[i], -h);
        h2[i] = fmul(2.0, h);
        rh2[i] = fdiv(1.0, h2[i]);
      } else {
        qp[i] = qm[i] = h2[i] = rh2[i] = 0.0;
      }
      invp[i] = invm[i] = 0.0;
    }
  }
  auto width = [&](int j) {
    dst[kMaxNp + j] = fdiv(1.0, q[j]);
    if (h0 != 0.0) {
      invp[j] = fdiv(1.0, qp[j]);
      invm[j] = fdiv(1.0, qm[j]);
    }
  };
  if (model == ADC_MODEL_GPOLY) {
    width(2);
  } else {
    for (int j = 2; j < np; j += 3) width(j);
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void fit_qdev_kernel(FitDevState* st, int model, int np, double* qdev, double h0) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    write_qdev(qdev, model, np, st->q, h0);
    st->t0 = globaltimer();  // the gradient pass starts after this kernel
  }
}

// adc_chi2_finalize's fixed pairwise tree, one record column per thread.
__device__ void column_tree(double* r, int64_t nchunks, int R, int v) {
  for (int64_t s = 1; s < nchunks; s *= 2)
    for (int64_t i = 0; i + s < nchunks; i += 2 * s) r[i * R + v] = fadd(r[i * R + v], r[(i + s) * R + v]);
}

// Gradient finalize (adc_chi2_finalize), convergence test, direction = g,
// gd, and the first batch of Armijo trials t = 1, 1/2, ... (fit.cpp:383-403)
// written as QDev rows for the multi-candidate pass.  Everything the serial
// part reads is staged in shared memory first (the kernel is latency-bound:
// each dependent global round trip is ~0.5 us).
__global__ void __launch_bounds__(128) fit_grad_kernel(FitDevState* st, const double* records,
                                                       double* scratch, int64_t nchunks, int np,
                                                       int model, double events, FitDevConst c,
                                                       double* qmulti, int* ncand_dev) {
  const int R = 4 + 3 * np;
  if (threadIdx.x == 0) st->grad_ns += globaltimer() - st->t0;  // the pass just ended
  __shared__ double s_g[kMaxNp], s_q[kMaxNp], s_col[4 + 3 * kMaxNp];
  __shared__ int s_stop, s_want;
  for (int64_t k = threadIdx.x; k < nchunks * R; k += blockDim.x) scratch[k] = records[k];
  if (threadIdx.x < kMaxNp) s_q[threadIdx.x] = st->q[threadIdx.x];
  if (threadIdx.x == 0) s_want = st->first_batch;
  __syncthreads();
  for (int v = threadIdx.x; v < R; v += blockDim.x) {
    column_tree(scratch, nchunks, R, v);
    s_col[v] = scratch[v];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double S = s_col[0], A1 = s_col[1], A2 = s_col[2];
    const double a = fdiv(events, S);
    const double t_sum = fsub(fmul(2.0, A1), fmul(fmul(2.0, a), A2));
    const double s_coef = fmul(fdiv(events, fmul(S, S)), t_sum);
    double gmax = 0.0;
    for (int i = 0; i < np; ++i) {
      const double G0 = s_col[4 + i], G1 = s_col[4 + np + i], G2 = s_col[4 + 2 * np + i];
      const double gi = fsub(fmul(s_coef, G0), fmul(fmul(2.0, a), fsub(G1, fmul(a, G2))));
      s_g[i] = gi;
      st->g[i] = gi;
      gmax = fmax(gmax, fabs(gi));
    }
    st->gmax = gmax;
    st->accepted_k = -1;
    st->evals = 0;         // per iteration
    st->sigma_clamps = 0;  // per iteration
    s_stop = gmax <= c.grad_tol;  // fit.cpp:340-344
    double gd = 0.0;
    for (int i = 0; i < np; ++i) gd = fadd(gd, fmul(s_g[i], s_g[i]));  // direction = g
    st->gd = gd;
  }
  __syncthreads();
  if (c.newton) {
    // the 2 np Hessian probes q +- h_c e_c, h_c = cbrt(eps) max(1, |q_c|)
    // (fit.cpp:346-381; chi2_host.cpp builds the same rows), as QDev rows
    // for the probe gradient passes that follow
    for (int k = threadIdx.x; k < 2 * np; k += blockDim.x) {
      const int col = k >> 1;
      double probe[kMaxNp];
      for (int i = 0; i < np; ++i) probe[i] = s_q[i];
      const double x = s_q[col];
      const double h = fmul(c.cbrt_eps, fmax(1.0, fabs(x)));
      probe[col] = (k & 1) == 0 ? fadd(x, h) : fsub(x, h);
      if ((k & 1) == 0) st->steps[col] = h;
      write_qdev(qmulti + (size_t)k * kQDoubles, model, np, probe, c.numeric ? c.cbrt_eps : 0.0);
    }
  }
  if (s_stop) {
    if (threadIdx.x == 0) {
      st->status = kFitConvergedGrad;
      st->ncand = 0;
      *ncand_dev = 0;
    }
    return;
  }
  if (c.newton) {  // direction and trials after the probes (fit_newton_kernel)
    if (threadIdx.x == 0) {
      st->status = kFitRunning;
      st->t1 = globaltimer();
    }
    return;
  }
  // Trial n (one per thread): t = 1/2^n exactly (the host's repeated *= 0.5),
  // trial = q - t g, the sigma clamp, and its QDev row.
  const int want = s_want;
  for (int n = threadIdx.x; n < want; n += blockDim.x) {
    const double tt = ldexp(1.0, -n);
    if (!(tt >= 1e-18)) continue;
    double trial[kMaxNp];
    int cl = 0;
    for (int i = 0; i < np; ++i) trial[i] = fsub(s_q[i], fmul(tt, s_g[i]));
    for (int k = 0; k < c.nclamp; ++k) {
      const int i = c.clamp_idx[k];
      if (i >= 0 && i < np && trial[i] < c.sigma_min) {
        trial[i] = c.sigma_min;
        ++cl;
      }
    }
    double* dst = st->trials + (size_t)n * kMaxNp;
    for (int i = 0; i < np; ++i) dst[i] = trial[i];
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

// damped_solve (chi2_host.cpp): Gaussian elimination with partial pivoting on
// H + lambda I, then back substitution — op for op, one thread.
__device__ bool damped_solve_dev(const double* H, const double* g, double lambda, int n,
                                 double* out) {
  double h[kMaxNp * kMaxNp], gg[kMaxNp];
  for (int i = 0; i < n * n; ++i) h[i] = H[i];
  for (int i = 0; i < n; ++i) gg[i] = g[i];
  for (int i = 0; i < n; ++i) h[i * n + i] = fadd(h[i * n + i], lambda);
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (fabs(h[r * n + col]) > fabs(h[piv * n + col])) piv = r;
    if (fabs(h[piv * n + col]) < 1e-30) return false;
    if (piv != col) {
      for (int cc = 0; cc < n; ++cc) {
        const double t = h[piv * n + cc];
        h[piv * n + cc] = h[col * n + cc];
        h[col * n + cc] = t;
      }
      const double t = gg[piv];
      gg[piv] = gg[col];
      gg[col] = t;
    }
    for (int r = col + 1; r < n; ++r) {
      const double f = fdiv(h[r * n + col], h[col * n + col]);
      for (int cc = col; cc < n; ++cc) h[r * n + cc] = fsub(h[r * n + cc], fmul(f, h[col * n + cc]));
      gg[r] = fsub(gg[r], fmul(f, gg[col]));
    }
  }
  for (int r = 0; r < n; ++r) out[r] = 0.0;
  for (int r = n - 1; r >= 0; --r) {
    double v = gg[r];
    for (int cc = r + 1; cc < n; ++cc) v = fsub(v, fmul(h[r * n + cc], out[cc]));
    out[r] = fdiv(v, h[r * n + r]);
  }
  return true;
}

// Newton option (fit.cpp:346-381 as adc_cuda_fit runs it): the 2 np probe
// gradients (adc_chi2_finalize of each probe pass's records), the central-
// difference Hessian, up to 10 damped solves (lambda 0, 1e-6, x10) until the
// direction is a descent direction (else steepest descent), gd = g.d, then
// the first batch of Armijo trials along the direction.
__global__ void __launch_bounds__(256) fit_newton_kernel(FitDevState* st,
                                                         const double* probe_records, size_t per,
                                                         double* scratch, int64_t nchunks, int np,
                                                         int model, double events, FitDevConst c,
                                                         double* qmulti, int* ncand_dev) {
  __shared__ double s_col[2 * kMaxNp][4 + 3 * kMaxNp];
  __shared__ double s_pg[2 * kMaxNp][kMaxNp];
  __shared__ double s_dir[kMaxNp], s_q[kMaxNp];
  __shared__ int s_want;
  if (st->status != kFitRunning) return;  // converged on the gradient
  const int R = 4 + 3 * np, K = 2 * np;
  if (threadIdx.x == 0) {
    st->grad_ns += globaltimer() - st->t1;  // the probe passes just ended
    s_want = st->first_batch;
  }
  if (threadIdx.x < kMaxNp) s_q[threadIdx.x] = st->q[threadIdx.x];
  for (int idx = threadIdx.x; idx < K * R; idx += blockDim.x) {
    const int k = idx / R, v = idx % R;
    double* r = scratch + (size_t)k * nchunks * R;
    const double* src = probe_records + (size_t)k * per;
    for (int64_t ch = 0; ch < nchunks; ++ch) r[ch * R + v] = src[ch * R + v];
    column_tree(r, nchunks, R, v);
    s_col[k][v] = r[v];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {  // adc_chi2_finalize per probe
    const double S = s_col[k][0], A1 = s_col[k][1], A2 = s_col[k][2];
    const double a = fdiv(events, S);
    const double t_sum = fsub(fmul(2.0, A1), fmul(fmul(2.0, a), A2));
    const double s_coef = fmul(fdiv(events, fmul(S, S)), t_sum);
    for (int i = 0; i < np; ++i) {
      const double G0 = s_col[k][4 + i], G1 = s_col[k][4 + np + i], G2 = s_col[k][4 + 2 * np + i];
      s_pg[k][i] = fsub(fmul(s_coef, G0), fmul(fmul(2.0, a), fsub(G1, fmul(a, G2))));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double H[kMaxNp * kMaxNp], g[kMaxNp], dir[kMaxNp];
    for (int i = 0; i < np; ++i) g[i] = dir[i] = st->g[i];
    for (int col = 0; col < np; ++col)
      for (int r = 0; r < np; ++r)
        H[r * np + col] =
            fdiv(fsub(s_pg[2 * col][r], s_pg[2 * col + 1][r]), fmul(2.0, st->steps[col]));
    double lambda = 0.0;
    bool ok = false;
    for (int attempt = 0; attempt < 10 && !ok; ++attempt) {
      ok = damped_solve_dev(H, g, lambda, np, dir);
      if (ok) {
        double descent = 0.0;
        for (int i = 0; i < np; ++i) descent = fadd(descent, fmul(g[i], dir[i]));
        ok = descent > 0.0;
      }
      lambda = lambda == 0.0 ? 1e-6 : fmul(lambda, 10.0);
    }
    if (!ok)
      for (int i = 0; i < np; ++i) dir[i] = g[i];  // steepest descent
    double gd = 0.0;
    for (int i = 0; i < np; ++i) gd = fadd(gd, fmul(g[i], dir[i]));
    st->gd = gd;
    for (int i = 0; i < np; ++i) {
      st->dir[i] = dir[i];
      s_dir[i] = dir[i];
    }
  }
  __syncthreads();
  const int want = s_want;
  for (int n = threadIdx.x; n < want; n += blockDim.x) {  // trials along the direction
    const double tt = ldexp(1.0, -n);
    if (!(tt >= 1e-18)) continue;
    double trial[kMaxNp];
    int cl = 0;
    for (int i = 0; i < np; ++i) trial[i] = fsub(s_q[i], fmul(tt, s_dir[i]));
    for (int k = 0; k < c.nclamp; ++k) {
      const int i = c.clamp_idx[k];
      if (i >= 0 && i < np && trial[i] < c.sigma_min) {
        trial[i] = c.sigma_min;
        ++cl;
      }
    }
    double* dst = st->trials + (size_t)n * kMaxNp;
    for (int i = 0; i < np; ++i) dst[i] = trial[i];
    st->cls[n] = cl;
    st->tvals[n] = tt;
    write_qdev(qmulti + (size_t)n * kQDoubles, model, np, trial);
  }
  if (threadIdx.x == 0) {
    int n = 0;
    while (n < want && ldexp(1.0, -n) >= 1e-18) ++n;
    st->ncand = n;
    *ncand_dev = n;
  }
}

// Each candidate's value record -> chi2 (adc_chi2_finalize, value form), then
// the first trial that satisfies Armijo is taken (fit.cpp:390-403, in order).
__global__ void __launch_bounds__(kMultiMax) fit_accept_kernel(FitDevState* st,
                                                               const double* records,
                                                               double* scratch, int64_t nchunks,
                                                               double events, FitDevConst c) {
  __shared__ double c2[kMultiMax], s_t[kMultiMax];
  const int n = st->ncand;
  if (n == 0) return;  // converged on the gradient
  const int R = 1 + 3 * n;
  const int k = threadIdx.x;
  if (k < n) {
    s_t[k] = st->tvals[k];
    double* r = scratch + (size_t)k * nchunks * 4;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const double* src = records + ch * R;
      r[ch * 4 + 0] = src[1 + 3 * k];
      r[ch * 4 + 1] = src[2 + 3 * k];
      r[ch * 4 + 2] = src[3 + 3 * k];
      r[ch * 4 + 3] = src[0];
    }
    double S, A1, A2, C0;
    if (nchunks == 1) {
      S = r[0], A1 = r[1], A2 = r[2], C0 = r[3];
    } else {
      for (int v = 0; v < 4; ++v) column_tree(r, nchunks, 4, v);
      S = r[0], A1 = r[1], A2 = r[2], C0 = r[3];
    }
    const double a = fdiv(events, S);
    const double two_a = fmul(2.0, a);
    c2[k] = fadd(fsub(C0, fmul(two_a, A1)), fmul(fmul(a, a), A2));
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double cur = st->cur, gd = st->gd;
  for (int j = 0; j < n; ++j) {
    if (c2[j] <= fsub(cur, fmul(fmul(c.armijo_c1, s_t[j]), gd))) {
      const double next = c2[j];
      st->evals = j + 1;
      st->accepted_k = j;
      st->sigma_clamps = st->cls[j];
      const double rel_dec = fdiv(fsub(cur, next), fmax(1.0, fabs(cur)));
      for (int i = 0; i < kMaxNp; ++i) st->q[i] = st->trials[(size_t)j * kMaxNp + i];
      st->cur = next;
      st->rel_dec = rel_dec;
      const int tried = j + 1;
      st->first_batch = min(kMultiMax, max(8, (tried + c.margin + 3) / 4 * 4));
      st->status = rel_dec <= c.chi2_rel_tol ? kFitConvergedRelDec : kFitRunning;
      return;
    }
  }
  st->evals = n;
  const double t_next = fmul(s_t[n - 1], 0.5);
  st->t_next = t_next;
  st->status = t_next >= 1e-18 ? kFitNeedHost : kFitConvergedNoStep;
}

// The host loop's per-pass bookkeeping (chi2_host.cpp adc_cuda_fit), then the
// loop condition: another pass while the search accepted a step, the fit has
// not converged and the budget is not spent.  NeedHost / NoStep / converged
// states end the device loop and the host takes over.
__global__ void fit_loop_ctl_kernel(FitDevState* st, cudaGraphConditionalHandle h,
                                    FitDevConst c) {
  if (threadIdx.x != 0) return;
  unsigned int cont = 0;
  st->passes += 1;
  st->n_grad += 1;
  if (st->status != kFitConvergedGrad) {
    if (c.newton) st->n_grad += 2 * c.np;  // the Hessian probes
    st->evals_total += st->evals;
    if (st->accepted_k >= 0) {
      st->clamps_total += st->sigma_clamps;
      st->iters += 1;
      if (c.trace != nullptr && c.trace_cap > st->iters)
        for (int i = 0; i < c.np; ++i) c.trace[(size_t)st->iters * c.np + i] = st->q[i];
      cont = st->status == kFitRunning && st->passes < st->budget;
    }
  }
  cudaGraphSetConditional(h, cont);
}

// Peer-transport exchange result [world][count] (each rank's block = its
// local chunks' records, nb blocks of maxc * R) -> the compact
// [nb][nchunks][R] layout the finalize kernels read (collect_finish's
// compaction, on the device).  R from the device candidate count when given.
__global__ void fit_compact_kernel(const double* __restrict__ out, size_t count, int world,
                                   const int64_t* __restrict__ rbegin, int64_t nchunks, int nb,
                                   int64_t maxc, int Rfix, const int* ncand_dev,
                                   double* __restrict__ dst) {
  const int R = ncand_dev != nullptr ? 1 + 3 * *ncand_dev : Rfix;
  const int64_t total = (int64_t)nb * nchunks * R;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = idx % R, bc = idx / R, ch = bc % nchunks, b = bc / nchunks;
    int r = 0;
    while (r + 1 < world && rbegin[r + 1] <= ch) ++r;
    dst[idx] = out[(size_t)r * count + (size_t)b * maxc * R + (size_t)(ch - rbegin[r]) * R + v];
  }
}

}  // namespace

int fit_device_enqueue_compact(const double* out, size_t count, int world, const int64_t* rbegin,
                               int64_t nchunks, int nb, int64_t maxc, int Rfix,
                               const int* ncand_dev, double* dst, cudaStream_t s) {
  fit_compact_kernel<<<64, 256, 0, s>>>(out, count, world, rbegin, nchunks, nb, maxc, Rfix,
                                        ncand_dev, dst);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int fit_device_enqueue_loop_ctl(FitDevState* st, cudaGraphConditionalHandle h,
                                const FitDevConst& c, cudaStream_t s) {
  fit_loop_ctl_kernel<<<1, 32, 0, s>>>(st, h, c);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int fit_device_enqueue_qdev(FitDevState* st, int model, int np, double* qdev, double h0,
                            cudaStream_t s) {
  fit_qdev_kernel<<<1, 32, 0, s>>>(st, model, np, qdev, h0);
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

int fit_device_enqueue_newton(FitDevState* st, const double* probe_records, size_t per,
                              double* scratch, int64_t nchunks, int np, int model, double events,
                              const FitDevConst& c, double* qmulti, int* ncand_dev,
                              cudaStream_t s) {
  fit_newton_kernel<<<1, 256, 0, s>>>(st, probe_records, per, scratch, nchunks, np, model, events,
                                      c, qmulti, ncand_dev);
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
