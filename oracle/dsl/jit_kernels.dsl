// Listing-1-style batch kernels over the reference corpus gradients (the
// generic-lowering parity fixtures, tests/golden/make_golden.py).  Each calls
// a generated gradient once per thread; the primal functions are the
// reference corpus files, prepended at fixture-generation time.
global void k_gauss(real[] x, real[] p, real sigma, real[] dx, real[] dp) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    gauss_grad_0_1(x[i], p[i], sigma, dx[i], dp[i]);
  }
}

global void k_rational(real[] x, real[] y, real[] dx, real[] dy) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    rational_grad(x[i], y[i], dx[i], dy[i]);
  }
}

global void k_branchy(real[] x, real[] y, real[] dx, real[] dy) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    branchy_grad(x[i], y[i], dx[i], dy[i]);
  }
}

global void k_poly(real[] x, real[] y, real[] dx, real[] dy) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    poly_grad(x[i], y[i], dx[i], dy[i]);
  }
}

global void k_looped(real[] x, integer n, real[] dx) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    looped_grad(x[i], n, dx[i]);
  }
}

global void k_gsum(real[] xs, real[] q, integer k, real[] dq) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    gsum_grad_1(xs[i], q, k, dq);
  }
}

global void k_sumn(real[] x, integer n, real[] dx) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    sumn_grad(x, n, dx);
  }
}

// Second order, forward-over-reverse (hessian.cpp:31): the tangent of the
// generated gradient along x, per point — column x of each point's Hessian
// lands in hx (d/dx dgauss/dx) and hp (d/dx dgauss/dp).
global void k_hess(real[] x, real[] p, real sigma, real[] dx, real[] dp, real[] hx, real[] hp) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    gauss_grad_0_1_darg0(x[i], p[i], sigma, dx[i], dp[i], hx[i], hp[i]);
  }
}

// Integer overflow (eval.cpp:601-628 raises "integer overflow"): the index
// arithmetic of this kernel overflows int64 in every active thread.
global void k_iovf(real[] x, integer big, real[] dx) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    integer k = big * big;
    dx[i] += x[i] * k;
  }
}
