// K2 — batched N-dim Gaussian gradient gaussnd_grad_0_1 over many points.
//
// Generated code (differentiate_gradient(gaussnd, {x, p}), reverse.cpp:335-553;
// DSL in oracle/dsl/gaussnd.dsl):
//   forward  for i: _t0 = x[i]-p[i]; _t1 = _t0*_t0; t = t + _t1   (3 tape pushes per i)
//            t = -t / ((2*sigma)*sigma); value = _t8 * exp(t)
//   reverse  _r2 = 0 + _t8*exp(t); _r3 = 0 + _r2/_t4; _d_t = 0 + -_r3
//            for i (descending): _r5 = _d_t; _r6 = (0 + _r5*_t0) + _t0*_r5;
//                                _d_x[i] += _r6; _d_p[i] += -_r6
// The tape only restores values no adjoint rule reads except _t0, which is
// recomputed exactly (x[i]-p[i]) or kept on chip: no global-memory tape.
//
// Layout: structure-of-arrays, coordinate d of point i at [d*ld + i].
// Mapping: lane = point (a warp reads one 256 B row segment per load),
// warps of a CTA split the dims of a 32-point tile.  Each warp keeps the
// u = x-p of its first `dstage` dims in shared memory for the reverse sweep;
// dims beyond that are re-read (most recent first, so they hit L2).
// With W = 1 the forward sum runs in exactly the reference order; with W > 1
// the per-warp partial sums are combined in fixed warp order (deterministic,
// <= W-term regrouping of t).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace adcb {

// Row batches of K for the last rows of a sweep: the remainder after the
// U-row batches goes through batches of 8, 4, 2, 1 (all loads of a batch in
// flight together), not row at a time: a remainder of 12 rows was 12 memory
// round trips (dim 28 at 11.0 ms vs 6.9 with U = 8).  Same order, same bits.
template <int K>
__device__ __forceinline__ void fwd_rows(const double* xi, const double* pi, int64_t ld, int d,
                                         int d0, int dstage, double* my_stage, double& t) {
  double xv[K], pv[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    xv[k] = __ldg(xi + (int64_t)(d + k) * ld);
    pv[k] = __ldg(pi + (int64_t)(d + k) * ld);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double u = fsub(xv[k], pv[k]);  // _t0 = x[i] - p[i]
    if (d + k - d0 < dstage) my_stage[(d + k - d0) * 32] = u;
    t = fadd(t, fmul(u, u));              // _t1 = _t0*_t0; t = t + _t1
  }
}

// Staged rows d - K .. d - 1 (descending) of the reverse sweep.
template <int K>
__device__ __forceinline__ void rev_rows(double* dxi, double* dpi, int64_t ld, int d, int d0,
                                         const double* my_stage, double c) {
  double a[K], b[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t o = (int64_t)(d - 1 - k) * ld;
    a[k] = dxi[o];
    b[k] = dpi[o];
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double u = my_stage[(d - 1 - k - d0) * 32];
    const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
    const int64_t o = (int64_t)(d - 1 - k) * ld;
    dxi[o] = fadd(a[k], r6);
    dpi[o] = fadd(b[k], -r6);
  }
}

// x and p rows are read through L1 (ld.global.nc, allocating): at rows that
// are not 128 B aligned, the line two neighbouring warps of a CTA share is
// then one L2 request, not two.  Measured against no-allocate loads (ms):
// 10M x 100 odd n 8.94 vs 9.73, 1M x 1000 7.90 vs 8.10 (odd 9.72 vs 10.73),
// 5M x 200 odd 7.56 vs 8.04, 3,333,334 x 300 7.77 vs 8.50.
template <int W, int U, int PF, int TPC = 1>
__global__ void __launch_bounds__(W * 32 * TPC) gaussnd_tile_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    double* __restrict__ dp, int64_t n, int dim, int64_t ld, double t4, double r1, int dpw,
    int dstage, unsigned long long* claim) {
  extern __shared__ double smem[];
  __shared__ int64_t s_claim[2];           // claimed span, double-buffered
  double* tpart = smem;                    // [W][32]
  double* stage = smem + W * 32;           // [W][dstage][32]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my_stage = stage + (size_t)warp * dstage * 32 + lane;
  // TPC > 1 (W = 1 only): the TPC warps of a CTA take TPC neighbouring
  // tiles in step, so the 32-byte sectors two neighbouring tiles share in a
  // row that is not sector-aligned are touched by one SM at about the same
  // time (merged in L2) instead of by two SMs far apart.
  const int d0 = TPC > 1 ? 0 : warp * dpw;
  const int d1 = min(dim, d0 + dpw);
  const int64_t ntiles = (n + 31) / 32;
  const int64_t gstride = (int64_t)gridDim.x * TPC;  // tiles in flight over the grid

  // a span = the TPC tiles of a CTA (one tile when TPC = 1); claimed in
  // order (claim != nullptr) or grid-stride
  const int64_t nspans = (ntiles + TPC - 1) / TPC;
  int64_t span = blockIdx.x;
  int it = 0;
  if (claim) {
    if (threadIdx.x == 0) s_claim[0] = claim_next(claim);
    __syncthreads();
    span = s_claim[0];
  }
  while (span < nspans) {
    const int64_t tile = span * TPC + (TPC > 1 ? warp : 0);
    const int64_t i = tile * 32 + lane;
    const bool valid = i < n;
    const double* xi = x + i;
    const double* pi = p + i;
    // ---- forward sweep: u_d and this warp's partial of t -------------------
    double t = 0.0;
    int d = d0;
    if (valid) {
      for (; d + U <= d1; d += U) {
        double xv[U], pv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          xv[k] = __ldg(xi + (int64_t)(d + k) * ld);
          pv[k] = __ldg(pi + (int64_t)(d + k) * ld);
        }
        if (PF == 2) {
          // lane l < U: x row d+U+l, lane U+l: p row d+U+l (one 256 B segment
          // each); past the range: the first dx / dp rows of the reverse sweep
          const int l = lane % U;
          const bool second = lane >= U && lane < 2 * U;
          const int dn = d + U + l;
          const int64_t tb = tile * 32;
          const unsigned seg = (unsigned)((n - tb < 32 ? n - tb : 32) * sizeof(double));
          if (lane < 2 * U) {
            if (dn < d1) {
              bulk_prefetch_l2((second ? p : x) + (int64_t)dn * ld + tb, seg);
            } else if (d1 - 1 - (dn - d1) >= d0) {
              bulk_prefetch_l2((second ? dp : dx) + (int64_t)(d1 - 1 - (dn - d1)) * ld + tb, seg);
            }
          }
        } else if (PF == 1) {
          // next batch of x, p rows; in the last batch, the first rows the
          // reverse sweep will read (dx, dp at the top of the range)
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int dn = d + U + k;
            if (dn < d1) {
              prefetch_l2(xi + (int64_t)dn * ld);
              prefetch_l2(pi + (int64_t)dn * ld);
            } else if (d1 - 1 - (dn - d1) >= d0) {
              const int64_t o = (int64_t)(d1 - 1 - (dn - d1)) * ld;
              prefetch_l2(dx + i + o);
              prefetch_l2(dp + i + o);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const double u = fsub(xv[k], pv[k]);  // _t0 = x[i] - p[i]
          if (d + k - d0 < dstage) my_stage[(d + k - d0) * 32] = u;
          t = fadd(t, fmul(u, u));              // _t1 = _t0*_t0; t = t + _t1
        }
      }
      if (U > 8 && d + 8 <= d1) { fwd_rows<8>(xi, pi, ld, d, d0, dstage, my_stage, t); d += 8; }
      if (U > 4 && d + 4 <= d1) { fwd_rows<4>(xi, pi, ld, d, d0, dstage, my_stage, t); d += 4; }
      if (U > 2 && d + 2 <= d1) { fwd_rows<2>(xi, pi, ld, d, d0, dstage, my_stage, t); d += 2; }
      if (d < d1) { fwd_rows<1>(xi, pi, ld, d, d0, dstage, my_stage, t); d += 1; }
    }
    if (W > 1) {
      tpart[warp * 32 + lane] = t;
      __syncthreads();
      t = tpart[lane];
#pragma unroll
      for (int w = 1; w < W; ++w) t = fadd(t, tpart[w * 32 + lane]);
    }
    // ---- scalar chain (identical in every warp of the tile) -----------------
    const double tt = fdiv(-t, t4);                // _t2 = -t; t = _t2 / _t4
    const double e = exp(tt);                      // _t9 = exp(t)
    const double r2 = fadd(0.0, fmul(r1, e));      // _d_t += _r1 * _q0
    const double r3 = fadd(0.0, fdiv(r2, t4));     // _d__t2 += _r2 / _t4
    const double c = fadd(0.0, -r3);               // _d_t += -_r3  (= _r4 = _r5 every i)
    // ---- reverse sweep: dx += r6, dp += -r6, most recently loaded dims first
    if (valid) {
      double* dxi = dx + i;
      double* dpi = dp + i;
      d = d1;
      const int dre = min(d1, d0 + dstage);  // [dre, d1) re-read, [d0, dre) staged
      for (; d - U >= dre; d -= U) {
        double xv[U], pv[U], a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t o = (int64_t)(d - 1 - k) * ld;
          xv[k] = __ldg(xi + o);
          pv[k] = __ldg(pi + o);
          a[k] = dxi[o];
          b[k] = dpi[o];
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const double u = fsub(xv[k], pv[k]);
          const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
          const int64_t o = (int64_t)(d - 1 - k) * ld;
          dxi[o] = fadd(a[k], r6);
          dpi[o] = fadd(b[k], -r6);
        }
      }
      for (; d > dre; --d) {
        const int64_t o = (int64_t)(d - 1) * ld;
        const double u = fsub(__ldg(xi + o), __ldg(pi + o));
        const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
        dxi[o] = fadd(dxi[o], r6);
        dpi[o] = fadd(dpi[o], -r6);
      }
      for (; d - U >= d0; d -= U) {
        double a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t o = (int64_t)(d - 1 - k) * ld;
          a[k] = dxi[o];
          b[k] = dpi[o];
        }
        if (PF == 2) {
          const int l = lane % U;
          const bool second = lane >= U && lane < 2 * U;
          const int dn = d - 1 - U - l;
          const int64_t tb = tile * 32, tn = tb + gstride * 32;
          if (lane < 2 * U) {
            if (dn >= d0) {
              const unsigned seg = (unsigned)((n - tb < 32 ? n - tb : 32) * sizeof(double));
              bulk_prefetch_l2((second ? dp : dx) + (int64_t)dn * ld + tb, seg);
            } else if (tn < n && d0 + (d0 - 1 - dn) < d1) {
              const unsigned seg = (unsigned)((n - tn < 32 ? n - tn : 32) * sizeof(double));
              bulk_prefetch_l2((second ? p : x) + (int64_t)(d0 + (d0 - 1 - dn)) * ld + tn, seg);
            }
          }
        } else if (PF == 1) {
          // next batch of dx, dp rows (descending); in the last batch, the
          // first x, p rows of this warp's next tile
          const int64_t inext = i + gstride * 32;
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int dn = d - 1 - U - k;
            if (dn >= d0) {
              prefetch_l2(dxi + (int64_t)dn * ld);
              prefetch_l2(dpi + (int64_t)dn * ld);
            } else if (inext < n && d0 + (d0 - 1 - dn) < d1) {
              const int64_t o = (int64_t)(d0 + (d0 - 1 - dn)) * ld;
              prefetch_l2(x + inext + o);
              prefetch_l2(p + inext + o);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const double u = my_stage[(d - 1 - k - d0) * 32];
          const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
          const int64_t o = (int64_t)(d - 1 - k) * ld;
          dxi[o] = fadd(a[k], r6);
          dpi[o] = fadd(b[k], -r6);
        }
      }
      if (U > 8 && d - 8 >= d0) { rev_rows<8>(dxi, dpi, ld, d, d0, my_stage, c); d -= 8; }
      if (U > 4 && d - 4 >= d0) { rev_rows<4>(dxi, dpi, ld, d, d0, my_stage, c); d -= 4; }
      if (U > 2 && d - 2 >= d0) { rev_rows<2>(dxi, dpi, ld, d, d0, my_stage, c); d -= 2; }
      if (d > d0) { rev_rows<1>(dxi, dpi, ld, d, d0, my_stage, c); d -= 1; }
    }
    // the next span: one barrier publishes it (and, W > 1, guards tpart,
    // which the next tile rewrites)
    if (claim && threadIdx.x == 0) s_claim[(it + 1) & 1] = claim_next(claim);
    if (W > 1 || claim) __syncthreads();
    if (claim) {
      ++it;
      span = s_claim[it & 1];
    } else {
      span += gridDim.x;
    }
  }
  if (claim && threadIdx.x == 0) claim_done(claim);
}

static int make_rows_tmap(CUtensorMap* m, const double* x, int64_t npts, int64_t dim, int64_t ld);

// K2v: two points per lane with 16-byte (double2) accesses — a warp covers a
// 64-point tile, each row access is one 512-byte segment.  Same per-point
// arithmetic and order as K2 (W = 1), so each point's bits are K2's; the two
// points of a lane are two independent dependency chains.  Full 64-point
// tiles of a 16-byte-aligned, even-ld layout; the caller runs the rest with K2.
template <int U>
__global__ void __launch_bounds__(32) gaussnd_vec2_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    double* __restrict__ dp, int64_t ntiles, int dim, int64_t ld, double t4, double r1,
    int dstage, unsigned long long* claim) {
  extern __shared__ double2 stage2[];  // [dstage][32]
  const int lane = threadIdx.x;
  const int64_t ld2 = ld / 2;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  double2* dx2 = reinterpret_cast<double2*>(dx);
  double2* dp2 = reinterpret_cast<double2*>(dp);
  int64_t tile = blockIdx.x;
  if (claim) tile = __shfl_sync(0xffffffffu, lane == 0 ? claim_next(claim) : 0, 0);
  while (tile < ntiles) {
    const int64_t i2 = tile * 32 + lane;  // double2 index of points 2 i2, 2 i2 + 1
    double ta = 0.0, tb = 0.0;
    int d = 0;
    for (; d + U <= dim; d += U) {
      double2 xv[U], pv[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        xv[k] = ld_stream2(x2 + (int64_t)(d + k) * ld2 + i2);
        pv[k] = ld_stream2(p2 + (int64_t)(d + k) * ld2 + i2);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {  // next batch (or the first reverse rows) into L2
        const int dn = d + U + k;
        if ((lane & 7) == 0) {
          if (dn < dim) {
            prefetch_l2(x2 + (int64_t)dn * ld2 + i2);
            prefetch_l2(p2 + (int64_t)dn * ld2 + i2);
          } else if (dim - 1 - (dn - dim) >= 0) {
            const int64_t o = (int64_t)(dim - 1 - (dn - dim)) * ld2 + i2;
            prefetch_l2(dx2 + o);
            prefetch_l2(dp2 + o);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const double ua = fsub(xv[k].x, pv[k].x), ub = fsub(xv[k].y, pv[k].y);
        if (d + k < dstage) stage2[(d + k) * 32 + lane] = make_double2(ua, ub);
        ta = fadd(ta, fmul(ua, ua));
        tb = fadd(tb, fmul(ub, ub));
      }
    }
    for (; d < dim; ++d) {
      const double2 xv = ld_stream2(x2 + (int64_t)d * ld2 + i2);
      const double2 pv = ld_stream2(p2 + (int64_t)d * ld2 + i2);
      const double ua = fsub(xv.x, pv.x), ub = fsub(xv.y, pv.y);
      if (d < dstage) stage2[d * 32 + lane] = make_double2(ua, ub);
      ta = fadd(ta, fmul(ua, ua));
      tb = fadd(tb, fmul(ub, ub));
    }
    double ca, cb;
    {
      const double e = exp(fdiv(-ta, t4));
      ca = fadd(0.0, -fadd(0.0, fdiv(fadd(0.0, fmul(r1, e)), t4)));
      const double f = exp(fdiv(-tb, t4));
      cb = fadd(0.0, -fadd(0.0, fdiv(fadd(0.0, fmul(r1, f)), t4)));
    }
    d = dim;
    for (; d - U >= 0; d -= U) {
      double2 a[U], b[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t o = (int64_t)(d - 1 - k) * ld2 + i2;
        a[k] = dx2[o];
        b[k] = dp2[o];
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {  // next batch of slot rows; at the end, the next tile
        const int dn = d - 1 - U - k;
        if ((lane & 7) == 0) {
          if (dn >= 0) {
            prefetch_l2(dx2 + (int64_t)dn * ld2 + i2);
            prefetch_l2(dp2 + (int64_t)dn * ld2 + i2);
          } else if (tile + gridDim.x < ntiles && -1 - dn < dim) {
            const int64_t o = (int64_t)(-1 - dn) * ld2 + i2 + (int64_t)gridDim.x * 32;
            prefetch_l2(x2 + o);
            prefetch_l2(p2 + o);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int dd = d - 1 - k;
        double ua, ub;
        if (dd < dstage) {
          const double2 u = stage2[dd * 32 + lane];
          ua = u.x;
          ub = u.y;
        } else {
          const double2 xv = ld_stream2(x2 + (int64_t)dd * ld2 + i2);
          const double2 pv = ld_stream2(p2 + (int64_t)dd * ld2 + i2);
          ua = fsub(xv.x, pv.x);
          ub = fsub(xv.y, pv.y);
        }
        const double ra = fadd(fadd(0.0, fmul(ca, ua)), fmul(ua, ca));
        const double rb = fadd(fadd(0.0, fmul(cb, ub)), fmul(ub, cb));
        const int64_t o = (int64_t)dd * ld2 + i2;
        dx2[o] = make_double2(fadd(a[k].x, ra), fadd(a[k].y, rb));
        dp2[o] = make_double2(fadd(b[k].x, -ra), fadd(b[k].y, -rb));
      }
    }
    for (; d > 0; --d) {
      const int dd = d - 1;
      double ua, ub;
      if (dd < dstage) {
        const double2 u = stage2[dd * 32 + lane];
        ua = u.x;
        ub = u.y;
      } else {
        const double2 xv = ld_stream2(x2 + (int64_t)dd * ld2 + i2);
        const double2 pv = ld_stream2(p2 + (int64_t)dd * ld2 + i2);
        ua = fsub(xv.x, pv.x);
        ub = fsub(xv.y, pv.y);
      }
      const double ra = fadd(fadd(0.0, fmul(ca, ua)), fmul(ua, ca));
      const double rb = fadd(fadd(0.0, fmul(cb, ub)), fmul(ub, cb));
      const int64_t o = (int64_t)dd * ld2 + i2;
      const double2 a = dx2[o], b = dp2[o];
      dx2[o] = make_double2(fadd(a.x, ra), fadd(a.y, rb));
      dp2[o] = make_double2(fadd(b.x, -ra), fadd(b.y, -rb));
    }
    if (claim) {
      tile = __shfl_sync(0xffffffffu, lane == 0 ? claim_next(claim) : 0, 0);
    } else {
      tile += gridDim.x;
    }
  }
  if (claim && lane == 0) claim_done(claim);
}

// ---------------------------------------------------------------------------
// Kernel selection.  The variant is an argument of every launch (never a
// process-wide setting, so concurrent callers cannot reroute each other):
//   0  auto — K2 as choose() picks it: W = 1 with 8 neighbouring tiles per
//      CTA up to 112 dims, dims over the warps of a CTA above;
//   3  K2 with one warp per 32-point tile (the reference summation order;
//      the tail form of K2v);
//   2  K2 with the dims split over the warps of a CTA (W = 8 / 16);
//   10 K2v (where the layout allows it; the rest through variant 3);
//   + 100  the same kernel on the static grid-stride schedule instead of
//      claimed spans (claim_slot in common.cuh; also what runs when the
//      claim ring is unavailable).  Same bits either way.
// The forced forms exist for the parity tests, which check that every kernel
// auto can pick gives the same per-point bits (W = 1 forms) or stays within
// the regrouping tolerance (W > 1).  Measured alternatives that were not
// kept (TMA-streamed tiles, 2-CTA clusters, deeper prefetch, other row
// batches) are described in DESIGN.md §3.
static thread_local int t_variant = 0;  // test override (adc_cuda_gaussnd_set_variant)

struct NdConfig {
  int w, u, dpw, dstage;
  size_t smem;
};

template <int W, int U, int PF = 1, int TPC = 1>
static int launch_tile(const NdConfig& c, int64_t n, int dim, int64_t ld, const double* x,
                       const double* p, double* dx, double* dp, double t4, double r1,
                       cudaStream_t s, bool dyn) {
  auto k = gaussnd_tile_kernel<W, U, PF, TPC>;
  const size_t smem = TPC > 1 ? ((size_t)TPC * 32 + (size_t)TPC * c.dstage * 32) * sizeof(double)
                              : c.smem;
  if (smem > 48 * 1024)
    ADCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  ADCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, W * 32 * TPC, smem));
  if (occ < 1) return fail(ADC_E_LAUNCH, "gaussnd: tile configuration does not fit an SM");
  const int64_t ntiles = (n + 31) / 32;
  int64_t blocks = std::min<int64_t>((ntiles + TPC - 1) / TPC, (int64_t)occ * sm_count());
  unsigned long long* claim = dyn && blocks < (ntiles + TPC - 1) / TPC ? claim_slot(s) : nullptr;
  k<<<(unsigned)blocks, W * 32 * TPC, smem, s>>>(x, p, dx, dp, n, dim, ld, t4, r1, c.dpw, c.dstage,
                                                  claim);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

// Shared-memory budget per SM usable by the stage buffers.
static constexpr size_t kSmemPerSm = 224 * 1024;

static NdConfig choose(int dim, int variant) {
  NdConfig c{};
  // W = 1 keeps the reference's summation order; it needs the whole u row of
  // a point on chip: 256 B per dim per warp.  Use it while >= 8 warps fit.
  if (variant == 3 || (variant != 2 && (size_t)dim * 256 * 8 <= kSmemPerSm)) {
    c.w = 1;
    c.dpw = dim;
    c.dstage = dim;
    if ((size_t)dim * 256 > kSmemPerSm - 512) c.dstage = (int)((kSmemPerSm - 512) / 256);
  } else {
    c.w = dim >= 512 ? 16 : 8;
    c.dpw = (dim + c.w - 1) / c.w;
    // one CTA per SM for W=16, stage as much as fits
    const size_t per_cta = kSmemPerSm / (c.w == 16 ? 1 : 2);
    const size_t avail = per_cta - (size_t)c.w * 32 * 8 - 1024;
    c.dstage = std::min<int>(c.dpw, (int)(avail / ((size_t)c.w * 256)));
  }
  c.u = c.w > 1 ? 8 : 16;
  c.smem = ((size_t)c.w * 32 + (size_t)c.w * c.dstage * 32) * sizeof(double);
  return c;
}

static int launch_gaussnd_v(int64_t n, int64_t dim, int64_t ld, const double* x, const double* p,
                            double sigma, double* dx, double* dp, cudaStream_t s, int variant) {
  const double PI = 3.14159265358979323846;
  const double t3 = 2 * sigma;
  const double t4 = t3 * sigma;
  // `t = _t2 / _t4` runs once per point: the interpreter's division check
  // (eval.cpp:543) fires for any point.
  if (n > 0 && t4 == 0.0) return fail(ADC_E_EVAL, "division by zero");
  if (n == 0) return ADC_OK;
  if (dim > (1 << 24)) return fail(ADC_E_ARG, "gaussnd: dim too large");
  // + 100: the static grid-stride schedule (parity tests of that path)
  const bool dyn = variant < 100;
  variant %= 100;
  double d_t9 = 0;
  d_t9 += (std::pow(2 * PI, -0.5) * std::pow(sigma, -0.5)) * 1.0;  // _d__t9 += _t8 * _r0
  // K2v (forced only): two points per lane.  It was the dim-100 headline
  // kernel (7.94 ms) until the claimed spans made K2 faster (7.53 ms); with
  // claiming its 64-point tiles need 4x K2's claims (dim 2: 13.3 ms).
  if (variant == 10) {
    const int64_t ntiles = n / 64;
    const bool ok = ld % 2 == 0 && ((((uintptr_t)x) | ((uintptr_t)p) | ((uintptr_t)dx) |
                                     ((uintptr_t)dp)) & 15) == 0;
    if (ok && ntiles > 0) {
      const size_t budget = 52 * 1024;
      const int dstage = (int)std::min<int64_t>(dim, budget / 512);
      const size_t smem = (size_t)dstage * 512;
      // the row batch no longer than the dims (U = 16 never batches below 16)
      auto k = dim < 4 ? gaussnd_vec2_kernel<2>
             : dim < 8 ? gaussnd_vec2_kernel<4>
             : dim < 16 ? gaussnd_vec2_kernel<8> : gaussnd_vec2_kernel<16>;
      if (smem > 48 * 1024)
        ADCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ = 0;
      ADCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32, smem));
      const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)std::max(1, occ) * sm_count());
      unsigned long long* claim = dyn && blocks < ntiles ? claim_slot(s) : nullptr;
      k<<<(unsigned)blocks, 32, smem, s>>>(x, p, dx, dp, ntiles, (int)dim, ld, t4, d_t9, dstage,
                                           claim);
      ADCB_CUDA(cudaGetLastError());
      const int64_t done = ntiles * 64;
      if (done == n) return ADC_OK;
      // the last partial tile through K2 (W = 1 for these dims: same per-point bits)
      return launch_gaussnd_v(n - done, dim, ld, x + done, p + done, sigma, dx + done, dp + done,
                              s, dyn ? 3 : 103);
    }
  }
  const NdConfig c = choose((int)dim, variant);
  const int di = (int)dim;
  if (c.w == 1) {
    // Auto: 8 neighbouring tiles per CTA from 2 dims while the stages fit one
    // CTA, with a row batch no longer than the dims: same bits as one warp
    // per CTA.  Static schedule: 3-19% faster than one tile per CTA (10M x
    // 100: 7.93 vs 8.29 ms aligned, 10.1 vs 12.0 ms with odd n); claimed
    // spans: 7.53 ms aligned, 9.67 odd.  Deeper row batches
    // (U = 24 / 32) spill and were slower.
    const bool fits = (size_t)8 * 32 * 8 + (size_t)8 * c.dstage * 256 <= 227 * 1024;
    if (variant == 0 && fits) {
      // U = 16 from 48 dims, 8 below (measured with the batched remainders,
      // ms, aligned / odd n: dim 20 6.65 / 6.83 vs 7.24 / 7.89 with U = 16,
      // dim 28 7.00 / 6.97 vs 7.16 / 7.95; dim 100 7.01 / 8.32 vs 7.26 / 8.57
      // with U = 8)
      if (dim >= 48) return launch_tile<1, 16, 1, 8>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
      if (dim >= 8) return launch_tile<1, 8, 1, 8>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
      if (dim >= 4) return launch_tile<1, 4, 1, 8>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
      if (dim >= 2) return launch_tile<1, 2, 1, 8>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
    }
    return launch_tile<1, 16>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
  }
  // bulk (TMA-unit) L2 prefetch of the next rows: 2.4% faster at dim 1000
  // (8.24 vs 8.45 ms, same bits)
  if (c.w == 16) return launch_tile<16, 8, 2>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
  return launch_tile<8, 8>(c, n, di, ld, x, p, dx, dp, t4, d_t9, s, dyn);
}

int launch_gaussnd_grad(int64_t n, int64_t dim, int64_t ld, const double* x, const double* p,
                        double sigma, double* dx, double* dp, cudaStream_t s) {
  return launch_gaussnd_v(n, dim, ld, x, p, sigma, dx, dp, s, t_variant);
}

int gaussnd_set_variant(int v) {
  const int k = v % 100;
  if (v < 0 || v >= 200 || (k != 0 && k != 2 && k != 3 && k != 10))
    return fail(ADC_E_ARG, "gaussnd variant must be 0 (auto), 2, 3 or 10, + 100 for the static schedule");
  t_variant = v;
  return ADC_OK;
}

// ---- K2s: shared mean vector (SURVEY.md §8(e) "shared-p variant") -----------------
// Every point i calls gaussnd_grad_0_1(x[:, i], p, sigma, dim, dx[:, i], dp)
// with ONE mean vector p[dim] and ONE shared slot dp[dim] (the reference's
// race_check would flag dp, launch.cpp:217-224): the per-point arithmetic is
// K2's (same forward sum order, same scalar chain, same reverse order), dx is
// private (optional), and dp_d = sum_i (-_r6_{d,i}) is reduced in a FIXED
// order: per thread / tile a fixed order, tiles in order per CTA (a CTA walks
// tiles b, b + G, ... with G a function of n only), then the CTA partials in
// order, then dp[d] += total.  No atomics; the same bits on every run and
// device.  Three forms, by dims and layout (launch_gaussnd_shared_p): K2sr
// (<= 24 dims, a thread per point), the staged-tile form (<= 256 dims: 2-D
// TMA tile loads, or cp.async copies where a tensor map cannot describe the
// layout; 2-8 warps per tile), and K2s below (one warp per tile, LSU loads;
// above 256 dims and for the < 32-point tail).  With dx, all forms sum a
// point's forward in the same dim chunks, so dx does not depend on the form.
constexpr int64_t kSharedPMaxBlocks = 1184;
constexpr int64_t kSharedPSpan = 8;  // tiles per dp partial row (staged-tile form)
constexpr int64_t kSharedPRowsMaxDim = 24;  // K2sr below, the staged-tile forms above

template <int U, int V>
__global__ void __launch_bounds__(32) gaussnd_shared_p_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    int64_t n, int dim, int64_t ld, double t4, double r1, int dstage,
    double* __restrict__ partials, int dq) {
  // dq: the forward sum runs in chunks of dq dims combined in order, the
  // grouping of the staged-tile form's warps, so a point's bits do not
  // depend on which form its layout selects (dq >= dim: one chunk)
  extern __shared__ double smem[];
  double* dpart = smem;              // [dim]
  double* stage = smem + dim;        // [dstage][32]
  const int lane = threadIdx.x;
  for (int d = lane; d < dim; d += 32) dpart[d] = 0.0;
  __syncwarp();
  const int64_t ntiles = (n + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * 32 + lane;
    const bool valid = i < n;
    const double* xi = x + i;
    // ---- forward: U rows in flight, the next U rows prefetched into L2
    double t = 0.0, tc = 0.0;
    int left = dq;
    bool first = true;
    auto add = [&](double u) {
      tc = fadd(tc, fmul(u, u));  // t = t + _t1 (this chunk)
      if (--left == 0) {
        t = first ? tc : fadd(t, tc);
        first = false;
        tc = 0.0;
        left = dq;
      }
    };
    if (valid) {
      int d = 0;
      for (; d + U <= dim; d += U) {
        double xv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) xv[k] = ld_stream(xi + (int64_t)(d + k) * ld);
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int dn = d + U + k;
          if (dn < dim) prefetch_l2(xi + (int64_t)dn * ld);
          else if (dx != nullptr && dim - 1 - (dn - dim) >= 0)
            prefetch_l2(dx + i + (int64_t)(dim - 1 - (dn - dim)) * ld);  // first reverse rows
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const double u = fsub(xv[k], __ldg(p + d + k));  // _t0 = x[i] - p[i]
          if (d + k < dstage) stage[(d + k) * 32 + lane] = u;
          add(u);
        }
      }
      // the remainder in batches of 16, 8, 4, 2, 1 (row at a time: a round
      // trip each)
      auto frows = [&](auto kc) {
        constexpr int K = decltype(kc)::value;
        double xv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) xv[k] = ld_stream(xi + (int64_t)(d + k) * ld);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double u = fsub(xv[k], __ldg(p + d + k));
          if (d + k < dstage) stage[(d + k) * 32 + lane] = u;
          add(u);
        }
        d += K;
      };
      if (U > 16 && d + 16 <= dim) frows(std::integral_constant<int, 16>{});
      if (U > 8 && d + 8 <= dim) frows(std::integral_constant<int, 8>{});
      if (U > 4 && d + 4 <= dim) frows(std::integral_constant<int, 4>{});
      if (U > 2 && d + 2 <= dim) frows(std::integral_constant<int, 2>{});
      if (d < dim) frows(std::integral_constant<int, 1>{});
      if (left != dq) t = first ? tc : fadd(t, tc);  // the last, partial chunk
    }
    const double tt = fdiv(-t, t4);
    const double e = exp(tt);
    const double r2 = fadd(0.0, fmul(r1, e));
    const double r3 = fadd(0.0, fdiv(r2, t4));
    const double c = fadd(0.0, -r3);
    // ---- reverse (the generated loop order, d descending), V dims at a time
    // so V shuffle trees and dx read-modify-writes overlap; the remainder in
    // batches of 4, 2, 1
    auto rrows = [&](auto kc, int d) {
      constexpr int K = decltype(kc)::value;
      double v[K], a[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int dd = d - k;
        v[k] = 0.0;
        if (valid && dx != nullptr) a[k] = dx[i + (int64_t)dd * ld];
        // the next tile's row dim-1-dd into L2 (ascending over the sweep)
        const int64_t inext = i + (int64_t)gridDim.x * 32;
        if (inext < n) prefetch_l2(x + inext + (int64_t)(dim - 1 - dd) * ld);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int dd = d - k;
        if (valid) {
          const double u = dd < dstage ? stage[dd * 32 + lane]
                                       : fsub(ld_stream(xi + (int64_t)dd * ld), __ldg(p + dd));
          const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
          if (dx != nullptr) dx[i + (int64_t)dd * ld] = fadd(a[k], r6);  // _d_x[_i0] += _r6
          v[k] = -r6;                                                      // _d_p[_i0] += -_r6
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) dpart[d - k] = fadd(dpart[d - k], v[k]);
      }
    };
    int d = dim - 1;
    for (; d - (V - 1) >= 0; d -= V) rrows(std::integral_constant<int, V>{}, d);
    if (V > 4 && d - 3 >= 0) { rrows(std::integral_constant<int, 4>{}, d); d -= 4; }
    if (V > 2 && d - 1 >= 0) { rrows(std::integral_constant<int, 2>{}, d); d -= 2; }
    if (d >= 0) rrows(std::integral_constant<int, 1>{}, d);
    __syncwarp();
  }
  __syncwarp();
  for (int d = lane; d < dim; d += 32) partials[(int64_t)blockIdx.x * dim + d] = dpart[d];
}

// TMA-staged variant: one warp per CTA, two stage buffers; while a tile is
// computed from one buffer, the next tile's dim rows (256 B each, one bulk
// copy per row issued by the lanes) stream into the other, so every warp has
// a whole tile of x in flight.  u = x - p is formed from the staged x in both
// sweeps (the same bits as K2s).  The dp sum is transposed: lane l owns dims
// l, l + 32, ... and adds the tile's 32 points' -_r6 for them in a fixed
// rotated point order (l + s) % 32 (bank-conflict free), into registers — no
// cross-lane reductions per element.  dx (optional) stays per point.  Full
// 32-point tiles only; dim <= 32 * JMAX.
// ASYNC: the same kernel for layouts a tensor map cannot describe (odd ld,
// x not 16-byte aligned): each thread copies its rows' elements into the
// stage with 8-byte cp.async (LDGSTS), one commit group per tile, double
// buffered like the TMA form.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

template <int V, int JMAX, int NW, bool ASYNC = false>
__global__ void __launch_bounds__(32 * NW) gaussnd_shared_p_tma_kernel(
    const __grid_constant__ CUtensorMap tmap, const double* __restrict__ x,
    const double* __restrict__ p, double* __restrict__ dx, int64_t ntiles, int dim, int64_t ld,
    double t4, double r1, double* __restrict__ partials, unsigned long long* claim) {
  // NW warps share each staged tile: warp w sums the forward t over dims
  // [w dq, (w+1) dq) (the NW partials combined in warp order), does the dx
  // read-modify-write of those dims, and owns dims w 32 + lane + 32 NW j of
  // the transposed dp sum.  With one warp per SM sub-partition the tile's
  // dependent FP64 chains (100 adds of t, 32 of each dp owner) left the warp
  // waiting on fixed latency (ncu: issue active 38%, stall "wait" dominant).
  extern __shared__ __align__(128) double smem[];
  __shared__ int64_t s_span[2];
  double* buf0 = smem;                              // [dim][32]
  double* buf1 = smem + (size_t)dim * 32;           // [dim][32]
  double* cbuf = smem + (size_t)dim * 64;           // [NW][32]: each warp's copy of c
  double* tpart = cbuf + 32 * NW;                   // [NW][32]
  uint64_t* bar = reinterpret_cast<uint64_t*>(tpart + 32 * NW);  // 2 mbarriers
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t tile_bytes = (uint32_t)dim * 256u;
  // one 2-D TMA load per tile: box {32 points, dim rows} -> buf[dim][32]
  // (ASYNC: every thread's 8-byte copies, one commit group per call, empty
  // past the last tile so the wait below always counts the same groups)
  auto issue = [&](int64_t tile, int b) {
    double* buf = b ? buf1 : buf0;
    if (ASYNC) {
      if (tile < ntiles) {
        const double* src = x + tile * 32 + lane;
        for (int r = warp; r < dim; r += NW) cp_async8(buf + r * 32 + lane, src + (int64_t)r * ld);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
    if (tile >= ntiles) return;
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar[b], tile_bytes);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(buf)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((int)(tile * 32)), "r"(0),
          "r"(smem_u32(&bar[b]))
          : "memory");
    }
  };
  const int dq = (dim + NW - 1) / NW;
  const int f0 = min(dim, warp * dq), f1 = min(dim, f0 + dq);  // this warp's forward dims
  double acc[JMAX];
  double pj[JMAX];
#pragma unroll
  for (int j = 0; j < JMAX; ++j) {
    acc[j] = 0.0;
    const int d = warp * 32 + lane + 32 * NW * j;
    pj[j] = d < dim ? __ldg(p + d) : 0.0;
  }
  double* my_c = cbuf + warp * 32;
  uint32_t phase[2] = {0u, 0u};
  // Spans of kSharedPSpan consecutive tiles, each summed into its own dp
  // partial row partials[span] (the grouping is a function of n only, so the
  // bits do not depend on which CTA takes a span or when).  A CTA takes
  // spans in order from the claim counter (claim != nullptr: the spans in
  // flight stay neighbours) or grid-stride; s_span holds its current and
  // next span, refilled by thread 0 when it moves on (the barriers of the
  // tiles in between publish it).
  // SPANS (the cp.async form; measured: odd ld, 5M x 100 with dx 3.14 ->
  // 2.45 ms, dp only 1.48 -> 1.41): spans of consecutive tiles claimed in
  // order.  The TMA form keeps one row per CTA over tiles b, b + G, ...
  // (at any moment the CTAs' tiles are contiguous; with spans of 8
  // consecutive tiles per CTA its dx path measured slower: 10M x 100
  // 4.16 -> 5.25 ms).
  constexpr bool SPANS = ASYNC;
  const int64_t nspans = (ntiles + kSharedPSpan - 1) / kSharedPSpan;
  int64_t taken = 0;  // thread 0: spans taken so far (the grid-stride schedule)
  auto take = [&]() -> int64_t {
    return claim ? claim_next(claim) : (int64_t)blockIdx.x + (taken++) * gridDim.x;
  };
  if (SPANS && threadIdx.x == 0) {
    s_span[0] = take();
    s_span[1] = take();
  }
  __syncthreads();
  // tile of a (slot, index) position; past the last tile: ntiles (none).  A
  // position moves to the other slot only after all kSharedPSpan of this
  // one (the last, short span runs out into "none"), so the issue position,
  // two tiles ahead, enters a slot only after thread 0 refilled it.
  auto tile_of = [&](int slot, int idx) -> int64_t {
    if (!SPANS) {
      const int64_t t = (int64_t)blockIdx.x + (int64_t)idx * gridDim.x;
      return t < ntiles ? t : ntiles;
    }
    const int64_t t = s_span[slot] * kSharedPSpan + idx;
    return s_span[slot] < nspans && t < ntiles ? t : ntiles;
  };
  auto advance = [&](int& slot, int& idx) {
    if (++idx == kSharedPSpan && SPANS) {
      slot ^= 1;
      idx = 0;
    }
  };
  int pslot = 0, pidx = 0;  // the tile being computed
  int islot = 0, iidx = 0;  // the next tile to issue
  issue(tile_of(islot, iidx), 0);
  advance(islot, iidx);
  issue(tile_of(islot, iidx), 1);
  advance(islot, iidx);
  int64_t tile = tile_of(pslot, pidx);
  for (int k = 0; tile < ntiles; ++k) {
    const int b = k & 1;
    double* buf = b ? buf1 : buf0;
    if (ASYNC) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's group
      __syncthreads();                                       // every thread's copies
    } else {
      mbar_wait(&bar[b], phase[b]);
      phase[b] ^= 1u;
    }
    if (dx != nullptr && (!ASYNC || NW >= 8)) {
      // this tile's dx rows into L2 while the forward runs (the reverse's
      // read-modify-writes then wait on L2, not DRAM): one 256-byte bulk
      // prefetch per row.  Measured, ms (TMA form): 10M x 100 4.42 -> 4.17,
      // 27M x 37 4.33 -> 4.18, 5M x 200 5.14 -> 4.41; the cp.async form
      // gains at 8 warps (5M x 100 3.43 -> 3.10) and loses at 4 (5M x 37
      // 1.05 -> 1.33: its copies share the LSU path)
      for (int r = threadIdx.x; r < dim; r += 32 * NW)
        bulk_prefetch_l2(dx + tile * 32 + (int64_t)r * ld, 256);
    }
    const int64_t i = tile * 32 + lane;
    double t = 0.0;
    for (int d = f0; d < f1; ++d) {
      const double u = fsub(buf[d * 32 + lane], __ldg(p + d));  // _t0 = x[i] - p[i]
      t = fadd(t, fmul(u, u));                                 // t = t + _t1
    }
    if (NW > 1) {
      tpart[warp * 32 + lane] = t;
      __syncthreads();
      t = tpart[lane];
#pragma unroll
      for (int w = 1; w < NW; ++w) t = fadd(t, tpart[w * 32 + lane]);
    }
    const double tt = fdiv(-t, t4);
    const double e = exp(tt);
    const double r2 = fadd(0.0, fmul(r1, e));
    const double r3 = fadd(0.0, fdiv(r2, t4));
    const double c = fadd(0.0, -r3);
    my_c[lane] = c;
    if (dx != nullptr) {  // _d_x[_i0] += _r6 over this warp's dims (each slot once)
      // rows d, d-1, ..., d-K+1: K read-modify-writes in flight together
      auto rows = [&](auto kc, int d) {
        constexpr int K = decltype(kc)::value;
        double a[K];
#pragma unroll
        for (int q = 0; q < K; ++q) a[q] = dx[i + (int64_t)(d - q) * ld];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int dd = d - q;
          const double u = fsub(buf[dd * 32 + lane], __ldg(p + dd));
          dx[i + (int64_t)dd * ld] = fadd(a[q], fadd(fadd(0.0, fmul(c, u)), fmul(u, c)));
        }
      };
      int d = f1 - 1;
      for (; d - (V - 1) >= f0; d -= V) rows(std::integral_constant<int, V>{}, d);
      // the remainder in batches of 4, 2, 1 (row at a time: a round trip each)
      if (V > 4 && d - 3 >= f0) { rows(std::integral_constant<int, 4>{}, d); d -= 4; }
      if (V > 2 && d - 1 >= f0) { rows(std::integral_constant<int, 2>{}, d); d -= 2; }
      if (d >= f0) rows(std::integral_constant<int, 1>{}, d);
    }
    __syncwarp();  // my_c visible to the warp
    // _d_p[d] += -_r6 of every point of the tile
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      const int d = warp * 32 + lane + 32 * NW * j;
      if (32 * NW * j < dim && d < dim) {
        const double* row = buf + d * 32;
        double aj = acc[j];
        for (int s = 0; s < 32; ++s) {
          const int l = (lane + s) & 31;
          const double cl = my_c[l];
          const double u = fsub(row[l], pj[j]);
          aj = fadd(aj, -fadd(fadd(0.0, fmul(cl, u)), fmul(u, cl)));
        }
        acc[j] = aj;
      }
    }
    const int64_t span = SPANS ? s_span[pslot] : 0;
    const bool span_end = SPANS && (pidx == kSharedPSpan - 1 || tile == ntiles - 1);
    if (span_end) {  // the span's dp partial row; the next span starts from zero
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        const int d = warp * 32 + lane + 32 * NW * j;
        if (d < dim) partials[span * dim + d] = acc[j];
        acc[j] = 0.0;
      }
    }
    const int old_slot = pslot;
    advance(pslot, pidx);
    // every warp is done reading buf / its c / tpart (and this span's slot)
    // before they are refilled
    __syncthreads();
    if (span_end && threadIdx.x == 0 && pslot != old_slot)
      s_span[old_slot] = take();  // the span after next
    issue(tile_of(islot, iidx), b);
    advance(islot, iidx);
    tile = tile_of(pslot, pidx);
  }
  if (ASYNC) asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (!SPANS) {  // the CTA's dp partial row
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      const int d = warp * 32 + lane + 32 * NW * j;
      if (d < dim) partials[(int64_t)blockIdx.x * dim + d] = acc[j];
    }
  }
  if (claim && threadIdx.x == 0) claim_done(claim);
}

// K2sr: the shared-mean form for dims <= 24 (DIM at compile time).  A
// 32-point tile of so few rows is too little work per staged tile (the TMA
// form ran dim 8 at 1.7 TB/s), so here a thread owns single points: PPT
// points in flight per thread (PPT x DIM loads, each warp row access one
// 256 B segment), the forward sum and scalar chain per point as K2, dx per
// point (optional), and the point's -_r6 added to the thread's DIM
// accumulators.  Thread g walks points g, g + T, ... (T = grid threads, the
// grid a function of n only); the CTA combines its threads per dim with a
// fixed xor tree and then its 8 warps in order: deterministic.
template <int DIM, int PPT, bool DX>
__global__ void __launch_bounds__(256) gaussnd_shared_p_rows_kernel(
    const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ dx,
    int64_t n, int64_t ld, double t4, double r1, double* __restrict__ partials) {
  __shared__ double wsum[8][DIM];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t T = (int64_t)gridDim.x * 256;
  double pv[DIM], acc[DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    pv[d] = __ldg(p + d);
    acc[d] = 0.0;
  }
  for (int64_t i0 = (int64_t)blockIdx.x * 256 + threadIdx.x; i0 < n; i0 += T * PPT) {
    double xv[PPT][DIM];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int64_t i = i0 + q * T;
      if (i < n) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xv[q][d] = __ldg(x + i + d * ld);
      }
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int64_t i = i0 + q * T;
      if (i < n) {
        double t = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          xv[q][d] = fsub(xv[q][d], pv[d]);                // _t0 = x[i] - p[i]
          t = fadd(t, fmul(xv[q][d], xv[q][d]));           // t = t + _t1
        }
        const double e = exp(fdiv(-t, t4));
        const double c = fadd(0.0, -fadd(0.0, fdiv(fadd(0.0, fmul(r1, e)), t4)));
        double a[DIM];
        if (DX) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) a[d] = dx[i + d * ld];
        }
#pragma unroll
        for (int d = DIM - 1; d >= 0; --d) {
          const double u = xv[q][d];
          const double r6 = fadd(fadd(0.0, fmul(c, u)), fmul(u, c));
          if (DX) dx[i + d * ld] = fadd(a[d], r6);          // _d_x[_i0] += _r6
          acc[d] = fadd(acc[d], -r6);                         // _d_p[_i0] += -_r6
        }
      }
    }
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double v = acc[d];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wsum[warp][d] = v;
  }
  __syncthreads();
  if (threadIdx.x < DIM) {
    double v = wsum[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) v = fadd(v, wsum[w][threadIdx.x]);
    partials[(int64_t)blockIdx.x * DIM + threadIdx.x] = v;
  }
}

template <bool DX>
static void* shared_p_rows_fn(int dim) {
  switch (dim) {
#define ADCB_ROWS(D) \
    case D: return (void*)gaussnd_shared_p_rows_kernel<D, (32 / D > 16 ? 16 : (32 / D < 2 ? 2 : 32 / D)), DX>;
    ADCB_ROWS(1) ADCB_ROWS(2) ADCB_ROWS(3) ADCB_ROWS(4) ADCB_ROWS(5) ADCB_ROWS(6) ADCB_ROWS(7)
    ADCB_ROWS(8) ADCB_ROWS(9) ADCB_ROWS(10) ADCB_ROWS(11) ADCB_ROWS(12) ADCB_ROWS(13)
    ADCB_ROWS(14) ADCB_ROWS(15) ADCB_ROWS(16) ADCB_ROWS(17) ADCB_ROWS(18) ADCB_ROWS(19)
    ADCB_ROWS(20) ADCB_ROWS(21) ADCB_ROWS(22) ADCB_ROWS(23) ADCB_ROWS(24)
#undef ADCB_ROWS
    default: return nullptr;
  }
}

__global__ void gaussnd_shared_p_finish(const double* __restrict__ partials, int64_t nblocks,
                                        int dim, double* __restrict__ dp) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  double acc = 0.0;
  for (int64_t b = 0; b < nblocks; ++b) acc = fadd(acc, partials[b * dim + d]);
  dp[d] = fadd(dp[d], acc);
}

// The partial rows in groups of kFinishGroup, each summed in row order into
// w1[group] (many groups in parallel), then the groups in order into dp.
constexpr int64_t kFinishGroup = 64;

__global__ void gaussnd_shared_p_finish_groups(const double* __restrict__ partials, int64_t rows,
                                               int dim, double* __restrict__ w1) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  const int64_t groups = (rows + kFinishGroup - 1) / kFinishGroup;
  for (int64_t g = blockIdx.y; g < groups; g += gridDim.y) {
    const int64_t r1 = min(rows, (g + 1) * kFinishGroup);
    double acc = 0.0;
    for (int64_t r = g * kFinishGroup; r < r1; ++r) acc = fadd(acc, partials[r * dim + d]);
    w1[g * dim + d] = acc;
  }
}

// dp[d] += the fixed two-level sum of rows partial rows; the workspace past
// the rows (gaussnd_shared_p_ws_doubles) holds the group sums.
static int shared_p_finish(double* partials, int64_t rows, int64_t dim, double* dp,
                           cudaStream_t s) {
  const int64_t groups = (rows + kFinishGroup - 1) / kFinishGroup;
  double* w1 = partials + rows * dim;
  const unsigned gx = (unsigned)((dim + 127) / 128);
  const unsigned gy = (unsigned)std::min<int64_t>(groups, 65535);
  gaussnd_shared_p_finish_groups<<<dim3(gx, gy), 128, 0, s>>>(partials, rows, (int)dim, w1);
  gaussnd_shared_p_finish<<<gx, 128, 0, s>>>(w1, groups, (int)dim, dp);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

// 2-D tensor map over the SoA rows: inner dimension = points (contiguous),
// outer = dims (stride ld), box = {32 points, dim rows}.  The driver entry
// point is fetched through the runtime (no link-time libcuda dependency).
static int make_rows_tmap(CUtensorMap* m, const double* x, int64_t npts, int64_t dim, int64_t ld) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (encode == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        fn == nullptr) {
      cudaGetLastError();
      return ADC_E_CUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t gdim[2] = {(cuuint64_t)npts, (cuuint64_t)dim};
  const cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {32u, (cuuint32_t)dim};
  const cuuint32_t estride[2] = {1u, 1u};
  const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), gdim,
                            gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? ADC_OK : ADC_E_CUDA;
}

// Multi-rank shared mean vector: every rank's dp partial [world][dim] (an
// all-gather) is summed in rank order, dp[d] += (0 + part_0) + part_1 + ...,
// the same bits on every rank.
__global__ void gaussnd_shared_p_rank_sum(const double* __restrict__ parts, int world, int dim,
                                          double* __restrict__ dp) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  double acc = 0.0;
  for (int r = 0; r < world; ++r) acc = fadd(acc, parts[(size_t)r * dim + d]);
  dp[d] = fadd(dp[d], acc);
}

int gaussnd_shared_p_rank_sum_enqueue(const double* parts, int world, int64_t dim, double* dp,
                                      cudaStream_t s) {
  if (dim == 0) return ADC_OK;
  gaussnd_shared_p_rank_sum<<<(unsigned)((dim + 127) / 128), 128, 0, s>>>(parts, world, (int)dim,
                                                                         dp);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int64_t gaussnd_shared_p_blocks(int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>((n + 31) / 32, kSharedPMaxBlocks));
}

// Workspace (doubles) of launch_gaussnd_shared_p: the dp partial rows of any
// form (CTA rows, or one per span of tiles) plus the tail's row, then the
// finish's group sums.
int64_t gaussnd_shared_p_ws_doubles(int64_t n, int64_t dim) {
  const int64_t spans = (n / 32 + kSharedPSpan - 1) / kSharedPSpan;
  const int64_t rows = std::max(gaussnd_shared_p_blocks(n), spans) + 1;
  return (rows + (rows + kFinishGroup - 1) / kFinishGroup) * std::max<int64_t>(dim, 1);
}

int launch_gaussnd_shared_p(int64_t n, int64_t dim, int64_t ld, const double* x, const double* p,
                            double sigma, double* dx, double* dp, double* partials,
                            cudaStream_t s) {
  const double PI = 3.14159265358979323846;
  const double t3 = 2 * sigma;
  const double t4 = t3 * sigma;
  if (n > 0 && t4 == 0.0) return fail(ADC_E_EVAL, "division by zero");
  if (n == 0 || dim == 0) return ADC_OK;
  if (dim > (1 << 20)) return fail(ADC_E_ARG, "gaussnd: dim too large");
  double d_t9 = 0;
  d_t9 += (std::pow(2 * PI, -0.5) * std::pow(sigma, -0.5)) * 1.0;
  // K2sr up to 24 dims (measured against the staged-tile forms, ms, dp only /
  // with dx: 1.2e8 x 8 1.28 / 4.83 vs 4.48 / 8.39; 6e7 x 16 1.22 / 3.99 vs
  // 2.50 / 6.78; 4e7 x 24 1.32 / 4.21 vs 2.35 / 5.74; at 32 dims its
  // registers spill and the TMA form wins with dx, 4.81 vs 3.84)
  if (dim <= kSharedPRowsMaxDim) {
    const int64_t blocks = gaussnd_shared_p_blocks(n);
    void* fn = dx ? shared_p_rows_fn<true>((int)dim) : shared_p_rows_fn<false>((int)dim);
    void* args[] = {(void*)&x, (void*)&p, (void*)&dx, (void*)&n, (void*)&ld, (void*)&t4,
                    (void*)&d_t9, (void*)&partials};
    ADCB_CUDA(cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(256), args, 0, s));
    return shared_p_finish(partials, blocks, dim, dp, s);
  }
  // stage as many dims of u as fit next to dp's partials (<= 26 KB: 8 CTAs/SM)
  const size_t budget = 26 * 1024 + 1024;
  const size_t fixed = (size_t)dim * sizeof(double);
  int dstage = fixed >= budget ? 0 : (int)std::min<int64_t>(dim, (budget - fixed) / 256);
  const size_t smem = fixed + (size_t)dstage * 256;
  // measured best of U in {16, 32} x V in {4, 8}; below 32 dims both follow
  // the dims (a batch longer than the dims never runs).  Same bits for any
  // U, V (t in row order; one fixed shuffle tree per dim).
  auto k = dim >= 32 ? gaussnd_shared_p_kernel<32, 8>
         : dim >= 16 ? gaussnd_shared_p_kernel<16, 8>
         : dim >= 8  ? gaussnd_shared_p_kernel<8, 8>
         : dim >= 4  ? gaussnd_shared_p_kernel<4, 4>
                     : gaussnd_shared_p_kernel<2, 2>;
  if (smem > 48 * 1024)
    ADCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // Decomposition (a function of n only, so the bits do not depend on the
  // path or the device): the full 32-point tiles over `blocks` CTAs, the last
  // partial tile (if any) as one more block of partials, then a fixed-order
  // total per dim.
  const int64_t full = n / 32, rem = n % 32;
  const int64_t blocks = full > 0 ? gaussnd_shared_p_blocks(full * 32) : 0;
  // warps per staged tile of the TMA form by the dims (measured, ms, dp only
  // 10M x 100: 2.03 / 1.50 / 1.51 / 1.73 with 1 / 2 / 4 / 8 warps; 5M x 200
  // 2.99 / 1.99 / 1.52 / 1.53; with dx 10M x 100 7.48 / 5.10 / 4.75 with
  // 2 / 4 / 8, 27M x 37 5.50 / 4.72 / 6.93, 5M x 200 12.5 / 7.64 / 5.14).
  // K2s sums in the same chunks wherever the TMA form could run (dim <= 256).
  // With dx the chunking is the same in every form (the dx bits do not
  // depend on the layout); dp only, the cp.async form takes more warps
  // (measured at odd ld, ms: dim 100 3.56 / 2.84 / 2.99 with 2 / 4 / 8 warps,
  // dim 200 8.70 / 7.11 / 6.11).
  const bool aligned = ld % 2 == 0 && ((uintptr_t)x & 15) == 0;
  const int nw = dx ? (dim >= 64 ? 8 : 4)
                    : aligned ? (dim >= 128 ? 4 : 2) : (dim >= 128 ? 8 : 4);
  const int dq = dim <= 256 ? (int)((dim + nw - 1) / nw) : (int)dim;
  const size_t tma_smem = (size_t)dim * 64 * sizeof(double) + 64 * 8 * sizeof(double) +
                          2 * sizeof(uint64_t);
  // The staged-tile form: x streamed by 2-D tensor loads (TMA), or by 8-byte
  // cp.async copies where a tensor map cannot describe the layout (odd ld, x
  // not 16-byte aligned), NW warps per staged tile, dx (optional) per point.
  // Above 256 dims K2s.
  const bool tma = aligned && dim <= 256 && tma_smem <= 200 * 1024;
  int64_t rows = blocks;  // dp partial rows before the tail's
  if (full > 0) {
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    const bool tmap_ok = tma && make_rows_tmap(&tmap, x, full * 32, dim, ld) == ADC_OK;
    if (tmap_ok || (dim <= 256 && tma_smem <= 200 * 1024)) {
      auto kt = nw == 8 ? (tmap_ok ? gaussnd_shared_p_tma_kernel<8, 1, 8>
                                   : gaussnd_shared_p_tma_kernel<8, 1, 8, true>)
              : nw == 4 ? (tmap_ok ? gaussnd_shared_p_tma_kernel<8, 2, 4>
                                   : gaussnd_shared_p_tma_kernel<8, 2, 4, true>)
                        : (tmap_ok ? gaussnd_shared_p_tma_kernel<8, 2, 2>
                                   : gaussnd_shared_p_tma_kernel<8, 2, 2, true>);
      if (tma_smem > 48 * 1024)
        ADCB_CUDA(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tma_smem));
      // TMA form: one dp partial row per CTA (blocks, a function of n only);
      // cp.async form: one per span of kSharedPSpan tiles, claimed in order
      int64_t grid = blocks;
      unsigned long long* claim = nullptr;
      if (!tmap_ok) {
        const int64_t nspans = (full + kSharedPSpan - 1) / kSharedPSpan;
        int occ = 0;
        ADCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kt, 32 * nw, tma_smem));
        grid = std::min<int64_t>(nspans, (int64_t)std::max(1, occ) * sm_count());
        claim = grid < nspans ? claim_slot(s) : nullptr;
        rows = nspans;
      }
      kt<<<(unsigned)grid, 32 * nw, tma_smem, s>>>(tmap, x, p, dx, full, (int)dim, ld, t4, d_t9,
                                                  partials, claim);
    } else {
      k<<<(unsigned)blocks, 32, smem, s>>>(x, p, dx, full * 32, (int)dim, ld, t4, d_t9, dstage,
                                           partials, dq);
    }
    ADCB_CUDA(cudaGetLastError());
  }
  if (rem != 0) {
    const int64_t off = full * 32;
    k<<<1, 32, smem, s>>>(x + off, p, dx ? dx + off : nullptr, rem, (int)dim, ld, t4, d_t9, dstage,
                          partials + rows * dim, dq);
    ADCB_CUDA(cudaGetLastError());
  }
  return shared_p_finish(partials, rows + (rem != 0 ? 1 : 0), dim, dp, s);
}

}  // namespace adcb
