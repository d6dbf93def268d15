// K3/K4 — chi2 histogram-fit pass (FitEngine::chi2 / chi2_gradient,
// proj/src/fit.cpp:206-259) as ONE pass over the bins.
//
// Per bin j (centre x_j = lo + (j + 0.5) * width, fit.hpp:30-31) the model
// m_j and its parameter gradient dm_j/dq (the generated <model>_grad_1) are
// evaluated in registers and folded into
//   S += m; [c>0]: A1 += m; A2 += m*(m/c); C0 += c; G1 += dm; G2 += (m/c) dm
//   G0 += dm
// (record layout [S, A1, A2, C0, G0[np], G1[np], G2[np]]).  adc_chi2_finalize
// (chi2_host.cpp) turns the records into chi2 and its gradient with the exact
// algebra of fit.cpp:231-258 (see include/adc_cuda.h).
//
// Determinism: a tile of tile_bins bins is one CTA pass with a fixed
// in-thread order, a fixed shuffle tree and a fixed cross-warp tree; a chunk
// of chunk_tiles tiles is reduced by K4 in a fixed tree; chunks are reduced on
// the host in a fixed tree.  No atomics.  Tile and chunk boundaries depend only
// on `bins`, so any sharding of whole chunks over GPUs gives the same bits.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "chi2_internal.h"
#include "common.cuh"

namespace adcb {

constexpr int kTileThreads = 256;
constexpr int kChunkThreads = 256;

// Uniform data for one pass, staged in device memory so CUDA-graph replays
// pick up new parameters from a pinned host buffer.
struct QDev {
  double q[kMaxNp];
  double inv[kMaxNp];  // 1/q for width parameters (fast mode)
};

// ---- models ------------------------------------------------------------------
// gpoly (oracle/dsl/gpoly.dsl) and its generated gpoly_grad_1; gsum
// (fit.cpp:125-138) and gsum_grad_1.  FAST replaces the divisions by the
// width parameter with multiplies by its host-computed reciprocal.
struct GPoly {
  static constexpr int NP = 6;
  template <bool GRAD, bool FAST>
  __device__ static __forceinline__ void eval(double x, const QDev& Q, double& m, double* bg) {
    const double q0 = Q.q[0], q1 = Q.q[1], q2 = Q.q[2], q3 = Q.q[3], q4 = Q.q[4], q5 = Q.q[5];
    const double t0 = fsub(x, q1);                              // _t0 = x - q[1]
    const double z = FAST ? fmul(t0, Q.inv[2]) : fdiv(t0, q2);  // z = _t0 / q[2]
    const double t1 = fmul(-0.5, z);                            // _t1 = -0.5 * z
    const double t2 = fmul(t1, z);                              // _t2 = _t1 * z
    const double e = exp(t2);                                   // _t3 = exp(_t2)
    const double g = fmul(q0, e);                               // g = q[0] * _t3
    m = fadd(fadd(fadd(g, q3), fmul(q4, x)), fmul(fmul(q5, x), x));
    if constexpr (GRAD) {
      // gpoly_grad_1 reverse sweep with the unit seeds folded (0 + v terms
      // only normalise -0, which cannot change a sum).
      bg[5] = fmul(x, x);                     // _d_q[5] += (_r1*x)*x
      bg[4] = x;                              // _d_q[4] += _r4*x, _r4 = 1
      bg[3] = 1.0;                            // _d_q[3] += _r5
      bg[0] = e;                              // _d_q[0] += _r6*_t3
      const double r8 = fmul(q0, e);          // _r8 = (q[0]*_r6)*_q0
      const double d1 = fmul(r8, z);          // _d__t1 += _r8*z
      double dz = fmul(t1, r8);               // _d_z += _t1*_r8
      dz = fadd(dz, fmul(-0.5, d1));          // _d_z += -0.5*_r9
      const double r11 = FAST ? fmul(dz, Q.inv[2]) : fdiv(dz, q2);             // _r10/q[2]
      bg[2] = -(FAST ? fmul(fmul(dz, z), Q.inv[2]) : fdiv(fmul(dz, z), q2));  // -(_r10*_q1/q[2])
      bg[1] = -r11;                                                            // _d_q[1] += -_r11
    }
  }
};

template <int K>
struct GSum {
  static constexpr int NP = 3 * K;
  template <bool GRAD, bool FAST>
  __device__ static __forceinline__ void eval(double x, const QDev& Q, double& m, double* bg) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double amp = Q.q[3 * j], mu = Q.q[3 * j + 1], sg = Q.q[3 * j + 2];
      const double t0 = fsub(x, mu);                                   // _t0 = x - mu
      const double z = FAST ? fmul(t0, Q.inv[3 * j + 2]) : fdiv(t0, sg);  // z = _t0 / sg
      const double t1 = fmul(-0.5, z);                                 // _t1 = -0.5 * z
      const double t2 = fmul(t1, z);                                   // _t2 = _t1 * z
      const double e = exp(t2);                                        // _t3 = exp(_t2)
      acc = fadd(acc, fmul(amp, e));                                   // acc = acc + amp*_t3
      if constexpr (GRAD) {
        const double r3 = fmul(amp, e);        // _r3 = (amp*_r1)*_q0
        const double r4 = fmul(r3, z);         // _d__t1 += _r3*z
        double dz = fmul(t1, r3);              // _d_z += _t1*_r3
        dz = fadd(dz, fmul(-0.5, r4));         // _d_z += -0.5*_r4
        const double r6 = FAST ? fmul(dz, Q.inv[3 * j + 2]) : fdiv(dz, sg);
        bg[3 * j + 2] = -(FAST ? fmul(fmul(dz, z), Q.inv[3 * j + 2]) : fdiv(fmul(dz, z), sg));
        bg[3 * j + 1] = -r6;                   // _d_mu += -_r6
        bg[3 * j] = e;                         // _d_amp += _r1*_t3
      }
    }
    m = acc;
  }
};

// ---- K3: tile pass -------------------------------------------------------------
template <class M, bool GRAD, bool FAST, int BPT>
__global__ void __launch_bounds__(kTileThreads) chi2_tile_kernel(Chi2Pass P) {
  constexpr int NP = M::NP;
  constexpr int R = GRAD ? 4 + 3 * NP : 4;
  __shared__ QDev Q;
  __shared__ double red[kTileThreads / 32][R];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = P.qdev[threadIdx.x];
    Q.inv[threadIdx.x] = P.qdev[kMaxNp + threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t tile = P.tile_begin + blockIdx.x; tile < P.tile_end; tile += gridDim.x) {
    double acc[R];
#pragma unroll
    for (int v = 0; v < R; ++v) acc[v] = 0.0;
    const int64_t base = tile * (int64_t)(BPT * kTileThreads) + threadIdx.x;
#pragma unroll 2
    for (int k = 0; k < BPT; ++k) {
      const int64_t j = base + (int64_t)k * kTileThreads;
      if (j < P.bin_end) {
        const double c = ld_stream(P.counts + j);
        const double x = fadd(P.lo, fmul(fadd((double)j, 0.5), P.width));  // Histogram::center
        double m, bg[GRAD ? NP : 1];
        M::template eval<GRAD, FAST>(x, Q, m, bg);
        const bool pos = c > 0.0;
        const double ic = pos ? (FAST ? __drcp_rn(c) : 1.0) : 0.0;
        const double mc = pos ? (FAST ? m * ic : m / c) : 0.0;
        acc[0] += m;
        acc[1] += pos ? m : 0.0;
        acc[2] += m * mc;
        acc[3] += pos ? c : 0.0;
        if constexpr (GRAD) {
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            acc[4 + i] += bg[i];
            acc[4 + NP + i] += pos ? bg[i] : 0.0;
            acc[4 + 2 * NP + i] += mc * bg[i];
          }
        }
      }
    }
    // fixed shuffle tree, then fixed cross-warp tree
#pragma unroll
    for (int v = 0; v < R; ++v) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[v] += __shfl_down_sync(0xffffffffu, acc[v], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int v = 0; v < R; ++v) red[warp][v] = acc[v];
    }
    __syncthreads();
    for (int v = threadIdx.x; v < R; v += kTileThreads) {
      const double s01 = red[0][v] + red[1][v], s23 = red[2][v] + red[3][v];
      const double s45 = red[4][v] + red[5][v], s67 = red[6][v] + red[7][v];
      P.tile_ws[(tile - P.tile_begin) * R + v] = (s01 + s23) + (s45 + s67);
    }
    __syncthreads();
  }
}

// ---- K4: chunk reduce (fixed tree over the chunk's tiles) ---------------------
// One CTA per chunk; warp w owns record entries v = w, w+8, ...; lane l sums
// tiles l, l+32, l+64, l+96 pairwise, then a fixed shuffle tree.
__global__ void __launch_bounds__(kChunkThreads) chi2_chunk_kernel(
    const double* __restrict__ tile_ws, int64_t ntiles, int R, int chunk_tiles,
    double* __restrict__ records) {
  const int64_t chunk = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = chunk * chunk_tiles;
  for (int v = warp; v < R; v += kChunkThreads / 32) {
    double part[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int64_t t = t0 + lane + 32 * s;
      part[s] = (lane + 32 * s < chunk_tiles && t < ntiles) ? tile_ws[t * R + v] : 0.0;
    }
    double a = (part[0] + part[1]) + (part[2] + part[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_down_sync(0xffffffffu, a, off);
    if (lane == 0) records[chunk * R + v] = a;
  }
}

// ---- dispatch ----------------------------------------------------------------
template <class M, bool GRAD, bool FAST>
static void launch_tiles_t(const Chi2Pass& P, int bpt, int blocks, cudaStream_t s) {
  if (bpt == 32)
    chi2_tile_kernel<M, GRAD, FAST, 32><<<blocks, kTileThreads, 0, s>>>(P);
  else
    chi2_tile_kernel<M, GRAD, FAST, 4><<<blocks, kTileThreads, 0, s>>>(P);
}

template <class M>
static void launch_tiles_m(const Chi2Pass& P, bool grad, bool fast, int bpt, int blocks,
                           cudaStream_t s) {
  if (grad) {
    if (fast) launch_tiles_t<M, true, true>(P, bpt, blocks, s);
    else launch_tiles_t<M, true, false>(P, bpt, blocks, s);
  } else {
    if (fast) launch_tiles_t<M, false, true>(P, bpt, blocks, s);
    else launch_tiles_t<M, false, false>(P, bpt, blocks, s);
  }
}

int chi2_enqueue(const Chi2Pass& P, int model, int np, bool grad, bool fast, int bpt,
                 int64_t chunk_tiles, double* records, cudaStream_t s) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  const int R = grad ? 4 + 3 * np : 4;
  // Persistent grid: a few CTAs per SM, tiles grid-strided.
  const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)sm_count() * 4);
  if (model == ADC_MODEL_GPOLY) {
    launch_tiles_m<GPoly>(P, grad, fast, bpt, (int)blocks, s);
  } else {
    switch (np / 3) {
      case 1: launch_tiles_m<GSum<1>>(P, grad, fast, bpt, (int)blocks, s); break;
      case 2: launch_tiles_m<GSum<2>>(P, grad, fast, bpt, (int)blocks, s); break;
      case 3: launch_tiles_m<GSum<3>>(P, grad, fast, bpt, (int)blocks, s); break;
      case 4: launch_tiles_m<GSum<4>>(P, grad, fast, bpt, (int)blocks, s); break;
      case 8: launch_tiles_m<GSum<8>>(P, grad, fast, bpt, (int)blocks, s); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
  }
  ADCB_CUDA(cudaGetLastError());
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  chi2_chunk_kernel<<<(unsigned)nchunks, kChunkThreads, 0, s>>>(P.tile_ws, ntiles, R,
                                                               (int)chunk_tiles, records);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

void fill_qdev(int model, int np, const double* q, double* host_qdev) {
  std::memset(host_qdev, 0, sizeof(QDev));
  QDev* Q = reinterpret_cast<QDev*>(host_qdev);
  for (int i = 0; i < np; ++i) Q->q[i] = q[i];
  if (model == ADC_MODEL_GPOLY) {
    Q->inv[2] = 1.0 / q[2];
  } else {
    for (int j = 2; j < np; j += 3) Q->inv[j] = 1.0 / q[j];
  }
}

size_t qdev_bytes() { return sizeof(QDev); }

}  // namespace adcb
