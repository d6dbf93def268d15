// K3/K4 — chi2 histogram-fit pass (FitEngine::chi2 / chi2_gradient,
// proj/src/fit.cpp:206-259) as ONE pass over the bins.
//
// Per bin j (centre x_j = lo + (j + 0.5) * width, fit.hpp:30-31) the model
// m_j and its parameter gradient dm_j/dq (the generated <model>_grad_1) are
// evaluated in registers and folded into
//   S += m; [c>0]: A1 += m; A2 += m*(m/c); C0 += c; G1 += dm; G2 += (m/c) dm
//   G0 += dm
// (record layout [S, A1, A2, C0, G0[np], G1[np], G2[np]]).
// Everything that depends on the counts alone is computed once per plan
// (K0 chi2_inverse_kernel: ic_j = [c_j > 0] / c_j, IEEE-rounded; K3l
// chi2_lin_kernel: C0 and the linear parameters' G0/G1), so a pass streams
// ic (8 B/bin) and spends its FP64 work on the model and its gradient only.  adc_chi2_finalize
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
#include <type_traits>
#include <vector>

#include "chi2_internal.h"
#include "common.cuh"
#include "fastmath.cuh"
#include "peer.cuh"

namespace adcb {

constexpr int kTileThreads = 256;
constexpr int kChunkThreads = 1024;  // one warp per record entry: the grid is only nchunks CTAs

// Uniform data for one pass, staged in device memory so CUDA-graph replays
// pick up new parameters from a pinned host buffer.
struct QDev {
  double q[kMaxNp];
  double inv[kMaxNp];  // 1/q for width parameters (fast mode)
};
// GradientProvider::Numeric (fit.cpp:187-190 -> central_gradient,
// numdiff.cpp:38-87): per parameter the two probe values q_i +- h_i with
// h_i = cbrt(eps) max(1, |q_i|), their width reciprocals, 2h_i and 1/(2h_i).
// Stored right after QDev (fill_qdev), computed on the host with the same
// libm as the reference.
struct QNum {
  double qp[kMaxNp], qm[kMaxNp];
  double invp[kMaxNp], invm[kMaxNp];
  double h2[kMaxNp], rh2[kMaxNp];
};
static_assert(sizeof(QDev) + sizeof(QNum) == kQDoubles * sizeof(double), "QDev layout");

// ---- fast-mode math ----------------------------------------------------------
// exp_nonpos (fastmath.cuh): table-driven exp for the models' non-positive
// arguments, ~11 FP64 ops with its constants in uniform registers.

// ---- models ------------------------------------------------------------------
// gpoly (oracle/dsl/gpoly.dsl) and its generated gpoly_grad_1; gsum
// (fit.cpp:125-138) and gsum_grad_1.  FAST replaces the divisions by the
// width parameter with multiplies by its host-computed reciprocal.
struct GPoly {
  static constexpr int NP = 6;
  static constexpr int NG = 1;  // Gaussian factors exp(-z^2/2), z = (x - mu) / sigma
  // q[3..5] enter linearly: dm/dq = (1, x, x^2) does not depend on q, so their
  // G0 and G1 sums are the same for every pass of a fit (precomputed once).
  static constexpr int LIN0 = 3;
  __device__ static __forceinline__ void lin_basis(double x, double* phi) {
    phi[0] = 1.0;
    phi[1] = x;
    phi[2] = fmul(x, x);
  }
  struct Reg {  // uniform parameters, held in registers for the whole pass
    double q0, q1, q2, q3, q4, q5, inv2;
  };
  __device__ static __forceinline__ Reg load(const QDev& Q) {
    return Reg{Q.q[0], Q.q[1], Q.q[2], Q.q[3], Q.q[4], Q.q[5], Q.inv[2]};
  }
  // The parameter vector with q[i] replaced by v (inv = 1/v for the width).
  __device__ static __forceinline__ Reg with(Reg r, int i, double v, double inv) {
    switch (i) {
      case 0: r.q0 = v; break;
      case 1: r.q1 = v; break;
      case 2: r.q2 = v; r.inv2 = inv; break;
      case 3: r.q3 = v; break;
      case 4: r.q4 = v; break;
      default: r.q5 = v; break;
    }
    return r;
  }
  __device__ static __forceinline__ void gauss(const Reg& Q, int, double& mu, double& inv) {
    mu = Q.q1;
    inv = Q.inv2;
  }
  // Fast mode with the run recurrence (tile_bins REC): x, z and the Gaussian
  // factor e come from the thread's run (x = x0 + k Dx, z = z0 + k Dz with one
  // rounding each, e from the anchored product); the rest is eval's fast form.
  template <bool GRAD>
  __device__ static __forceinline__ void eval_rec(double x, const double* z, const double* e,
                                                  const Reg& Q, double& m, double* bg) {
    m = __fma_rn(Q.q0, e[0], __fma_rn(__fma_rn(Q.q5, x, Q.q4), x, Q.q3));
    if constexpr (GRAD) {
      bg[0] = e[0];
      bg[1] = fmul(e[0], z[0]);  // without the factor q[0] / q[2] (Derive)
      bg[2] = fmul(bg[1], z[0]);
      bg[3] = 1.0;
      bg[4] = x;
      bg[5] = fmul(x, x);
    }
  }
  template <bool GRAD, bool FAST>
  __device__ static __forceinline__ void eval(double x, const Reg& Q, const double* tab, double& m,
                                              double* bg, const double* erec = nullptr) {
    const double q0 = Q.q0, q1 = Q.q1, q2 = Q.q2, q3 = Q.q3, q4 = Q.q4, q5 = Q.q5;
    if constexpr (FAST) {
      // Fast modes: the same values with fewer operations.  The polynomial in
      // Horner form; in the reverse sweep _t1 = -0.5 z makes
      //   _d_z = _t1 _r8 - 0.5 (_r8 z) = -(_r8 z)
      // exactly (halving is exact), so with u = g z (g = _r8 = q0 _t3):
      //   _d_q[1] = -_r11 = u / q2,  _d_q[2] = -(_r10 _q1 / q2) = (u / q2) z.
      const double z = fmul(fsub(x, q1), Q.inv2);                 // z = (x - q[1]) / q[2]
      const double e = erec != nullptr ? erec[0]                  // _t3 (recurrence)
                                       : exp_nonpos(fmul(fmul(-0.5, z), z), tab);
      m = __fma_rn(q0, e, __fma_rn(__fma_rn(q5, x, q4), x, q3));
      if constexpr (GRAD) {
        // _d_q[1], _d_q[2] without their common factor q[0] / q[2] (the
        // chunk kernel multiplies the sums: Derive)
        bg[0] = e;
        bg[1] = fmul(e, z);
        bg[2] = fmul(bg[1], z);
        bg[3] = 1.0;
        bg[4] = x;
        bg[5] = fmul(x, x);
      }
      return;
    }
    const double t0 = fsub(x, q1);                              // _t0 = x - q[1]
    const double z = fdiv(t0, q2);                              // z = _t0 / q[2]
    const double t1 = fmul(-0.5, z);                            // _t1 = -0.5 * z
    double e;
    if (erec != nullptr) {
      e = erec[0];  // _t3 from the per-thread recurrence (tile_bins, REC)
    } else {
      const double t2 = fmul(t1, z);                            // _t2 = _t1 * z
      e = exp(t2);                                              // _t3 = exp(_t2)
    }
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
      const double r11 = fdiv(dz, q2);                  // _r11 = _r10 / q[2]
      bg[2] = -fdiv(fmul(dz, z), q2);                   // -(_r10*_q1/q[2])
      bg[1] = -r11;                                     // _d_q[1] += -_r11
    }
  }
};

template <int K>
struct GSum {
  static constexpr int NP = 3 * K;
  static constexpr int NG = K;
  static constexpr int LIN0 = NP;  // no q-independent gradient components
  __device__ static __forceinline__ void lin_basis(double, double*) {}
  struct Reg {
    double q[3 * K];
    double inv[K];
  };
  __device__ static __forceinline__ Reg load(const QDev& Q) {
    Reg r;
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) r.q[i] = Q.q[i];
#pragma unroll
    for (int j = 0; j < K; ++j) r.inv[j] = Q.inv[3 * j + 2];
    return r;
  }
  __device__ static __forceinline__ Reg with(Reg r, int i, double v, double inv) {
    r.q[i] = v;
    if (i % 3 == 2) r.inv[i / 3] = inv;
    return r;
  }
  __device__ static __forceinline__ void gauss(const Reg& Q, int j, double& mu, double& inv) {
    mu = Q.q[3 * j + 1];
    inv = Q.inv[j];
  }
  template <bool GRAD>
  __device__ static __forceinline__ void eval_rec(double x, const double* z, const double* e,
                                                  const Reg& Q, double& m, double* bg) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double amp = Q.q[3 * j];
      acc = __fma_rn(amp, e[j], acc);
      if constexpr (GRAD) {  // without the factor amp / sg (Derive)
        const double b1 = fmul(e[j], z[j]);
        bg[3 * j + 2] = fmul(b1, z[j]);
        bg[3 * j + 1] = b1;
        bg[3 * j] = e[j];
      }
    }
    m = acc;
  }
  template <bool GRAD, bool FAST>
  __device__ static __forceinline__ void eval(double x, const Reg& Q, const double* tab, double& m,
                                              double* bg, const double* erec = nullptr) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double amp = Q.q[3 * j], mu = Q.q[3 * j + 1], sg = Q.q[3 * j + 2];
      const double t0 = fsub(x, mu);                                   // _t0 = x - mu
      const double z = FAST ? fmul(t0, Q.inv[j]) : fdiv(t0, sg);  // z = _t0 / sg
      const double t1 = fmul(-0.5, z);                                 // _t1 = -0.5 * z
      double e;
      if (erec != nullptr) {
        e = erec[j];  // _t3 from the per-thread recurrence (tile_bins, REC)
      } else {
        const double t2 = fmul(t1, z);                                 // _t2 = _t1 * z
        e = FAST ? exp_nonpos(t2, tab) : exp(t2);                      // _t3 = exp(_t2)
      }
      acc = FAST ? __fma_rn(amp, e, acc) : fadd(acc, fmul(amp, e));    // acc = acc + amp*_t3
      if constexpr (GRAD && FAST) {
        // _d_z = _t1 _r3 - 0.5 (_r3 z) = -(_r3 z) exactly (see GPoly::eval);
        // the mu / sigma entries without their factor amp / sg (Derive)
        const double b1 = fmul(e, z);
        bg[3 * j + 2] = fmul(b1, z);           // -(_r5 _q1 / sg) * sg
        bg[3 * j + 1] = b1;                    // _d_mu += -_r6, * sg
        bg[3 * j] = e;                         // _d_amp += _r1*_t3
      } else if constexpr (GRAD) {
        const double r3 = fmul(amp, e);        // _r3 = (amp*_r1)*_q0
        const double r4 = fmul(r3, z);         // _d__t1 += _r3*z
        double dz = fmul(t1, r3);              // _d_z += _t1*_r3
        dz = FAST ? __fma_rn(-0.5, r4, dz) : fadd(dz, fmul(-0.5, r4));  // _d_z += -0.5*_r4
        const double r6 = FAST ? fmul(dz, Q.inv[j]) : fdiv(dz, sg);
        bg[3 * j + 2] = -(FAST ? fmul(fmul(dz, z), Q.inv[j]) : fdiv(fmul(dz, z), sg));
        bg[3 * j + 1] = -r6;                   // _d_mu += -_r6
        bg[3 * j] = e;                         // _d_amp += _r1*_t3
      }
    }
    m = acc;
  }
};

// ---- K3: tile pass -------------------------------------------------------------
// Per thread: bins base + k*256 (k < BPT) in increasing k, ic streamed
// through a PD-deep register ring (+ an L2 prefetch of the next tile), so the
// FP64 pipe is not left waiting on HBM.  Accumulation is branch-free: with
// w = [c > 0] = [ic > 0] and ic = [c > 0]/c,
//   S += m; A1 += w m; A2 += m (m ic); G0 += dm; G1 += w dm; G2 += (m ic) dm
// (C0 and the linear parameters' G0/G1 come from the once-per-plan K3l pass).
// Full tiles skip the per-bin bounds test.
constexpr int kPD = 4;
constexpr int kPrefetchRows = 16;  // L2 prefetch distance of the tile passes, in bin rows

// CTAs per SM the register budget is tuned for (spill-free at these counts).
// (measured on B200: 2 x 256 threads with 128 registers beats 3 x 256 with 80
// for the gpoly gradient pass, 0.503 vs 0.539 ms at 1e8 bins)
template <class M, bool GRAD>
constexpr int tile_min_blocks() {
  return M::NP <= 6 ? 2 : 1;
}

template <class M, bool GRAD, bool FAST>
struct BinTerm {
  double m, mc;
  bool empty;  // c == 0 (ic == +0.0: an integer test, not an FP64 compare)
  double bg[GRAD ? M::NP : 1];
};

__device__ __forceinline__ bool empty_bin(double ic) { return __double_as_longlong(ic) == 0; }

// Numeric provider: dm/dq_i = (m(q + h_i e_i) - m(q - h_i e_i)) / (2 h_i),
// two full model evaluations per parameter exactly as central_gradient
// (numdiff.cpp:62-79) runs the primal at the probes.  Each derivative is
// folded into G0/G1/G2 as soon as it is known (same per-entry expressions and
// bin order as bin_accumulate), so no per-bin gradient vector is held.
template <class M, bool FAST>
__device__ __forceinline__ void numeric_fold(double x, const typename M::Reg& QR, const QNum& N,
                                             const double* tab, bool empty, double mc,
                                             double* acc) {
  constexpr int NP = M::NP;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double mp, mm, dummy[1];
    M::template eval<false, FAST>(x, M::with(QR, i, N.qp[i], N.invp[i]), tab, mp, dummy);
    M::template eval<false, FAST>(x, M::with(QR, i, N.qm[i], N.invm[i]), tab, mm, dummy);
    const double d0 = fsub(mp, mm);
    const double d = FAST ? fmul(d0, N.rh2[i]) : fdiv(d0, N.h2[i]);
    acc[4 + i] += d;
    if (!empty) acc[4 + NP + i] += d;
    acc[4 + 2 * NP + i] = __fma_rn(mc, d, acc[4 + 2 * NP + i]);
  }
}

// jh = j + 0.5 exactly (j < 2^52), so x is bit-identical to Histogram::center.
// ic = [c > 0] / c from the plan's K0 pass (so ic > 0 exactly when c > 0).
template <class M, bool GRAD, bool FAST>
__device__ __forceinline__ void bin_term(const Chi2Pass& P, const typename M::Reg& QR,
                                         const double* tab, double jh, double ic,
                                         BinTerm<M, GRAD, FAST>& t,
                                         const double* erec = nullptr) {
  const double x = fadd(P.lo, fmul(jh, P.width));  // Histogram::center: lo + (j + 0.5) * width
  M::template eval<GRAD, FAST>(x, QR, tab, t.m, t.bg, erec);
  t.empty = empty_bin(ic);
  t.mc = t.m * ic;
}

// The [c > 0] sums are not accumulated per bin: a pass folds every bin into
// S and G0, and the record entries A1 = sum_{c>0} m and G1 = sum_{c>0} dm
// (nonlinear parameters) are S and G0 minus the same sums over the chunk's
// EMPTY bins, which a side pass (chi2_empty_kernel) evaluates from the plan's
// list of them (c = 0 is rare: 1% of the bins in the BASELINE histograms).
// The tile records carry copies (copy_source) and the chunk kernel subtracts
// the empty-bin sums (ZMerge).  No per-bin [c > 0] test, select or multiply.
// Fast AD gradient passes (DER) do not accumulate S and A2 at all: the models
// are sums of terms each linear in exactly one parameter of the set L (gpoly:
// q0 e + q3 + q4 x + q5 x^2; gsum: sum_k amp_k e_k), so
//   S = sum_{i in L} q_i G0_i,   A2 = sum_{i in L} q_i G2_i
// exactly (Euler's identity for m); the chunk kernel derives them (Derive).
template <class M, bool GRAD, bool FAST>
__device__ __forceinline__ void bin_accumulate(const BinTerm<M, GRAD, FAST>& t, double* acc) {
  constexpr int NP = M::NP;
  constexpr int LIN0 = M::LIN0;
  if constexpr (!(GRAD && FAST)) {
    acc[0] += t.m;
    acc[2] = __fma_rn(t.m, t.mc, acc[2]);
  }
  // acc[3] (C0) comes from the K3l pre-pass
  if constexpr (GRAD) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      if (i < LIN0) acc[4 + i] += t.bg[i];  // q-independent G0/G1 entries: lin pre-pass
      acc[4 + 2 * NP + i] = __fma_rn(t.mc, t.bg[i], acc[4 + 2 * NP + i]);
    }
  }
}

// Record entries a tile pass copies from another entry (A1 <- S; with the AD
// gradient the nonlinear G1 <- G0): the source's per-tile sum, bit for bit.
template <class M, bool GRAD, bool NUM>
__host__ __device__ constexpr int copy_source(int v) {
  constexpr int NP = M::NP;
  if (v == 1) return 0;
  if (GRAD && !NUM && v >= 4 + NP && v < 4 + NP + M::LIN0) return v - NP;
  return -1;
}

// ILP evaluates that many independent bins before folding any, giving the
// scheduler two dependency chains to interleave (the model's exp chain is
// ~15 dependent FP64 ops deep).  The accumulation order is unchanged.
// REC (gradient passes, precision mode 2): each thread's Gaussian factors
// e_k = exp(-z_k^2 / 2) over its run of bins z_k = z_0 + k D (D = 256 width /
// sigma, uniform) come from one anchor per tile instead of one exp per bin:
//   e_k = (e_0 A^k) B_k,  e_0 = exp(-z_0^2 / 2),  A = exp(-z_0 D),
//   B_k = exp(-(k D)^2 / 2)  (a per-pass table, uniform over threads),
// i.e. two multiplies per bin; the product's rounding error grows by about
// one ulp per bin (<= bpt + 2 ulp relative while e_0 is a normal number;
// below that the absolute error is < 1e-290).  Used when |D| bpt <= 1 (a
// run spans at most one sigma): then e_0 A^k = e_k / B_k <= e^(1/2), so the
// product cannot overflow; and when bpt >= 16 (shorter runs, e.g. the 4 bins
// per thread below ~600K bins, pay more for the two anchor exps than they
// save).
constexpr int kRecMaxBpt = 192;

template <class M, bool GRAD, bool FAST, bool CHECK, int ILP, bool NUM, bool REC = false>
__device__ __forceinline__ void tile_bins(const Chi2Pass& P, const typename M::Reg& QR,
                                          const double* tab, int64_t base, double* acc,
                                          const QNum* N, const double* rtab = nullptr,
                                          const double* rdl = nullptr) {
  constexpr int PD = kPD;  // ring depth (loads in flight per thread); P.bpt % 4 == 0
  const int BPT = P.bpt;
  constexpr int STEP = ILP <= PD ? ILP : PD;
  static_assert(PD % 4 == 0 && 4 % STEP == 0, "ring depth / step");
  double jh = fadd((double)base, 0.5);  // advanced by 256.0 per bin: exact integers + 0.5
  [[maybe_unused]] double rP[REC ? M::NG : 1], rA[REC ? M::NG : 1], rz0[REC ? M::NG : 1];
  [[maybe_unused]] double x0 = 0.0, kd = 0.0;
  if constexpr (REC) {
    x0 = fadd(P.lo, fmul(jh, P.width));
#pragma unroll
    for (int c = 0; c < M::NG; ++c) {
      double mu, inv;
      M::gauss(QR, c, mu, inv);
      rz0[c] = fmul(fsub(x0, mu), inv);  // the model's own z at bin 0
      rP[c] = exp_nonpos(fmul(fmul(-0.5, rz0[c]), rz0[c]), tab);
      rA[c] = exp(-fmul(rz0[c], rdl[c]));
    }
  }
  if constexpr (REC && !CHECK && !NUM && PD == 4) {
    // A full tile with the run recurrence (the default gradient and value
    // passes): the same bins and arithmetic as the general loop below, with
    // the index work hoisted.  Two register sets of 1/c values (blocks of 4
    // rows) alternate, so a block's loads land directly in the registers that
    // consume them (no ring copies); thread 0 keeps the CTA's rows 16 ahead
    // coming into L2 with one bulk prefetch (TMA unit) per 8 KB block, into
    // the CTA's next tile past this one's end.
    const int nblk = BPT / 4;
    const double* pn = P.icounts + base;
    const double dx = fmul(256.0, P.width);
    const int64_t tile_base = base - threadIdx.x;
    const double* pf = P.icounts + tile_base + (int64_t)kPrefetchRows * kTileThreads;
    const double* pf_end = P.icounts + tile_base + (int64_t)BPT * kTileThreads;
    const int64_t pf_shift = (int64_t)(gridDim.x - 1) * BPT * kTileThreads;
    const double* bin_end = P.icounts + P.bin_end;
    double ra[4], rb[4];
    auto load = [&](double* r, int blk) {
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = ld_stream(pn + ((int64_t)blk * 4 + u) * kTileThreads);
    };
    auto block = [&](const double* r, int blk) {
      if (threadIdx.x == 0) {
        if (pf >= pf_end && pf < pf_end + 4 * kTileThreads) pf += pf_shift;
        if (pf + 4 * kTileThreads <= bin_end) bulk_prefetch_l2(pf, 4 * kTileThreads * 8);
        pf += 4 * kTileThreads;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * blk + u;
        BinTerm<M, GRAD, FAST> t;
        double e[M::NG], z[M::NG];
        const double x = __fma_rn(kd, dx, x0);
#pragma unroll
        for (int g = 0; g < M::NG; ++g) {
          e[g] = fmul(rP[g], rtab[g * kRecMaxBpt + k]);
          rP[g] = fmul(rP[g], rA[g]);
          z[g] = __fma_rn(kd, rdl[g], rz0[g]);
        }
        M::template eval_rec<GRAD>(x, z, e, QR, t.m, t.bg);
        t.mc = t.m * r[u];
        bin_accumulate<M, GRAD, FAST>(t, acc);
        kd = fadd(kd, 1.0);
      }
    };
    load(ra, 0);
    if (nblk > 1) load(rb, 1);
    for (int b = 0; b < nblk; b += 2) {
      block(ra, b);
      if (b + 2 < nblk) load(ra, b + 2);
      if (b + 1 < nblk) {
        block(rb, b + 1);
        if (b + 3 < nblk) load(rb, b + 3);
      }
    }
  } else {
  double ring[PD];
#pragma unroll
  for (int k = 0; k < PD; ++k) {
    const int64_t j = base + (int64_t)k * kTileThreads;
    ring[k] = (k < BPT && (!CHECK || j < P.bin_end)) ? ld_stream(P.icounts + j) : 0.0;
  }
  // L2 prefetch kPrefetchRows bin rows ahead of the register ring: lanes 0-7
  // each take one 128-byte line of this warp's 4 x 256 bytes of that block
  // (past the tile's end: the same rows of the CTA's next tile), so the
  // ring's loads hit L2 instead of waiting on HBM.
  const int64_t tile_base = base - threadIdx.x;
  const int64_t next_base = tile_base + (int64_t)gridDim.x * BPT * kTileThreads;
  const int pl = threadIdx.x & 31;
  const int64_t poff = (int64_t)(pl >> 1) * kTileThreads + (threadIdx.x & ~31) + (pl & 1) * 16;
  for (int k0 = 0; k0 < BPT; k0 += PD) {
    if (pl < 8) {
      const int kp = k0 + kPrefetchRows;
      const int64_t pa = (kp < BPT ? tile_base + (int64_t)kp * kTileThreads
                                   : next_base + (int64_t)(kp - BPT) * kTileThreads) + poff;
      if (pa < P.bin_end) prefetch_l2(P.icounts + pa);
    }
#pragma unroll
    for (int kk = 0; kk < PD; kk += STEP) {
      if (PD > 4 && kk >= 4 && k0 + kk >= BPT) break;  // BPT % 4 == 0 (uniform)
      BinTerm<M, GRAD && !NUM, FAST> t[STEP];
      bool valid[STEP];
#pragma unroll
      for (int u = 0; u < STEP; ++u) {
        const int k = k0 + kk + u;
        const int64_t j = base + (int64_t)k * kTileThreads;
        const double c = ring[kk + u];
        const int64_t jn = j + (int64_t)PD * kTileThreads;
        ring[kk + u] = (k + PD < BPT && (!CHECK || jn < P.bin_end)) ? ld_stream(P.icounts + jn)
                                                                     : 0.0;
        valid[u] = !CHECK || j < P.bin_end;
        if constexpr (NUM) {
          // value terms, then the finite-difference gradient folded in place;
          // finite differences of a linear term are not exactly its basis, so
          // every G entry is accumulated here (no lin pre-pass)
          if (valid[u]) {
            BinTerm<M, false, FAST> tv;
            bin_term<M, false, FAST>(P, QR, tab, jh, c, tv);
            bin_accumulate<M, false, FAST>(tv, acc);
            numeric_fold<M, FAST>(fadd(P.lo, fmul(jh, P.width)), QR, *N, tab, tv.empty, tv.mc,
                                  acc);
          }
        } else if constexpr (REC) {
          if (valid[u]) {
            // bin k of the run: x = x0 + k (256 width), z = z0 + k D (one
            // rounding each; D = 256 width / sigma = rdl)
            double e[M::NG], z[M::NG];
            const double x = __fma_rn(kd, fmul(256.0, P.width), x0);
#pragma unroll
            for (int g = 0; g < M::NG; ++g) {
              e[g] = fmul(rP[g], rtab[g * kRecMaxBpt + k]);
              rP[g] = fmul(rP[g], rA[g]);
              z[g] = __fma_rn(kd, rdl[g], rz0[g]);
            }
            M::template eval_rec<GRAD>(x, z, e, QR, t[u].m, t[u].bg);
            t[u].mc = t[u].m * c;
          }
          kd = fadd(kd, 1.0);
        } else {
          if (valid[u]) bin_term<M, GRAD, FAST>(P, QR, tab, jh, c, t[u]);
        }
        jh = fadd(jh, (double)kTileThreads);
      }
      if constexpr (!NUM) {
#pragma unroll
        for (int u = 0; u < STEP; ++u)
          if (valid[u]) bin_accumulate<M, GRAD, FAST>(t[u], acc);
      }
    }
  }
  }  // the general loop
}

// Record entries a tile pass leaves at zero: C0 (always) and, for the AD
// gradient, the linear parameters' G0/G1 (all merged from the K3l pre-pass).
template <class M, bool GRAD, bool NUM, bool FAST>
__host__ __device__ constexpr bool pass_zero_entry(int v) {
  constexpr int NP = M::NP, L0 = M::LIN0;
  return v == 3 || (GRAD && FAST && !NUM && v <= 2) ||  // S, A1, A2 derived (DER)
         (GRAD && !NUM &&
          ((v >= 4 + L0 && v < 4 + NP) || (v >= 4 + NP + L0 && v < 4 + 2 * NP)));
}

template <class M, bool GRAD, bool FAST, int MINB = tile_min_blocks<M, GRAD>(),
          int ILP = 1, bool NUM = false, bool REC = false>
__global__ void __launch_bounds__(kTileThreads, MINB) chi2_tile_kernel(Chi2Pass P) {
  // batched passes (blockIdx.y = member): own parameters and tile records
  P.qdev += blockIdx.y * P.q_stride;
  P.tile_ws += blockIdx.y * P.ws_stride;
  constexpr int NP = M::NP;
  constexpr int R = GRAD ? 4 + 3 * NP : 4;
  __shared__ QDev Q;
  const QNum* Np = nullptr;
  if constexpr (NUM) {
    __shared__ QNum Ns;
    const double* src = P.qdev + 2 * kMaxNp;
    double* dst = reinterpret_cast<double*>(&Ns);
    for (int v = threadIdx.x; v < 6 * kMaxNp; v += kTileThreads) dst[v] = src[v];
    Np = &Ns;
  }
  __shared__ double red[kTileThreads / 32][R];
  __shared__ double tab[64];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = P.qdev[threadIdx.x];
    Q.inv[threadIdx.x] = P.qdev[kMaxNp + threadIdx.x];
  }
  if (threadIdx.x < 64) tab[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
  __syncwarp();  // reconverge (exp2's branches) before the CTA barrier (bar.sync is .aligned)
  __syncthreads();
  const typename M::Reg QR = M::load(Q);
  [[maybe_unused]] bool use_rec = false;
  __shared__ double rtab[REC ? M::NG * kRecMaxBpt : 1];
  __shared__ double rdl[REC ? M::NG : 1];
  if constexpr (REC) {
    // D per Gaussian factor and the B_k table (uniform; see tile_bins)
    use_rec = P.bpt >= 16 && P.bpt <= kRecMaxBpt;  // short runs: the anchors cost more
#pragma unroll
    for (int c = 0; c < M::NG; ++c) {
      double mu, inv;
      M::gauss(QR, c, mu, inv);
      const double dl = fmul((double)kTileThreads * P.width, inv);
      use_rec = use_rec && fabs(dl) * P.bpt <= 1.0;
      if (threadIdx.x == 0) rdl[c] = dl;
    }
    if (use_rec)
      for (int v = threadIdx.x; v < M::NG * P.bpt; v += kTileThreads) {
        const int c = v / P.bpt, k = v % P.bpt;
        double mu, inv;
        M::gauss(QR, c, mu, inv);
        const double kd = fmul((double)k, fmul((double)kTileThreads * P.width, inv));
        rtab[c * kRecMaxBpt + k] = exp(fmul(fmul(-0.5, kd), kd));
      }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int BPT = P.bpt;
  const int64_t TB = (int64_t)BPT * kTileThreads;
  for (int64_t tile = P.tile_begin + blockIdx.x; tile < P.tile_end; tile += gridDim.x) {
    const int64_t base = tile * TB + threadIdx.x;
    if (tile == P.tile_begin + blockIdx.x) {  // the first rows of the CTA's first tile
      const int pl = threadIdx.x & 31;
      if (pl < 8)
        for (int k = (pl >> 1); k < min(kPrefetchRows, BPT); k += 4) {
          const int64_t pa = tile * TB + (int64_t)k * kTileThreads + (threadIdx.x & ~31) +
                             (pl & 1) * 16;
          if (pa < P.bin_end) prefetch_l2(P.icounts + pa);
        }
    }
    double acc[R];
#pragma unroll
    for (int v = 0; v < R; ++v) acc[v] = 0.0;
    const bool full = (tile + 1) * TB <= P.bin_end;
    if (REC && use_rec) {
      if (full) tile_bins<M, GRAD, FAST, false, ILP, NUM, REC>(P, QR, tab, base, acc, Np, rtab, rdl);
      else tile_bins<M, GRAD, FAST, true, ILP, NUM, REC>(P, QR, tab, base, acc, Np, rtab, rdl);
    } else if (full) {
      tile_bins<M, GRAD, FAST, false, ILP, NUM>(P, QR, tab, base, acc, Np);
    } else {
      tile_bins<M, GRAD, FAST, true, ILP, NUM>(P, QR, tab, base, acc, Np);
    }
    // fixed shuffle tree, then fixed cross-warp tree; entries a pass never
    // touches (C0 and the linear G0/G1: the K3l pre-pass supplies them) are
    // exact zeros and skip the tree
#pragma unroll
    for (int v = 0; v < R; ++v) {
      if (!pass_zero_entry<M, GRAD, NUM, FAST>(v) && copy_source<M, GRAD, NUM>(v) < 0) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
          acc[v] += __shfl_down_sync(0xffffffffu, acc[v], off);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int v = 0; v < R; ++v)
        red[warp][v] = pass_zero_entry<M, GRAD, NUM, FAST>(v) ? 0.0 : acc[v];
    }
    __syncthreads();
    for (int v = threadIdx.x; v < R; v += kTileThreads) {
      const int cs = copy_source<M, GRAD, NUM>(v);
      const int u = cs >= 0 ? cs : v;
      const double s01 = red[0][u] + red[1][u], s23 = red[2][u] + red[3][u];
      const double s45 = red[4][u] + red[5][u], s67 = red[6][u] + red[7][u];
      P.tile_ws[(tile - P.tile_begin) * R + v] = (s01 + s23) + (s45 + s67);
    }
    __syncthreads();
  }
}

// ---- K3m: multi-candidate chi2 value pass (batched Armijo line search) ---------
// One sweep over the bins evaluates chi2 for up to kMultiMax parameter vectors
// (the line-search trials q - t g, t = 1, 1/2, ...).  blockIdx.y selects a
// group of kMultiGroup candidates.  Per candidate the per-thread order, the
// shuffle tree and the cross-warp tree are those of the single value pass, so
// every candidate's record is bit-identical to a separate chi2 pass.
// Record layout per tile / chunk: [C0, (S, A1, A2) x ncand].
constexpr int kMultiGroup = 8;



// candidates evaluated together per bin (independent chains), as registers allow
template <class M>
__host__ __device__ constexpr int multi_ilp() {
  return M::NP <= 6 ? 4 : M::NP <= 12 ? 2 : 1;
}

template <class M, bool REC = false>
__global__ void __launch_bounds__(kTileThreads, 2) chi2_multi_kernel(Chi2Pass P, int ncand) {
  constexpr int G = kMultiGroup, CG = multi_ilp<M>();
  if (P.ncand_dev != nullptr) ncand = *P.ncand_dev;  // set on the device (fit graph)
  if ((int)blockIdx.y * G >= ncand) return;           // uniform over the CTA
  __shared__ QDev Q[G];
  __shared__ double red[kTileThreads / 32][3 * G + 1];
  __shared__ double tab[64];
  const int g0 = blockIdx.y * G;
  const int ng = min(G, ncand - g0);
  for (int t = threadIdx.x; t < G * kMaxNp; t += kTileThreads) {
    const int c = t / kMaxNp, i = t % kMaxNp;
    const double* src = P.qdev + (size_t)(g0 + (c < ng ? c : 0)) * kQDoubles;
    Q[c].q[i] = src[i];
    Q[c].inv[i] = src[kMaxNp + i];
  }
  if (threadIdx.x < 64) tab[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
  // REC: per candidate the value pass's decision, D and B_k table (tile_bins)
  __shared__ double rtab[REC ? G * M::NG * kRecMaxBpt : 1];
  __shared__ double rdl[REC ? G * M::NG : 1];
  __shared__ bool ruse[REC ? G : 1];
  if constexpr (REC) {
    __syncthreads();
    if (threadIdx.x < G) {
      const typename M::Reg QR = M::load(Q[threadIdx.x]);
      bool use = P.bpt >= 16 && P.bpt <= kRecMaxBpt;
#pragma unroll
      for (int c = 0; c < M::NG; ++c) {
        double mu, inv;
        M::gauss(QR, c, mu, inv);
        const double dl = fmul((double)kTileThreads * P.width, inv);
        use = use && fabs(dl) * P.bpt <= 1.0;
        rdl[threadIdx.x * M::NG + c] = dl;
      }
      ruse[threadIdx.x] = use;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < G * M::NG * P.bpt; v += kTileThreads) {
      const int cg = v / P.bpt, k = v % P.bpt;  // cg = candidate * NG + factor
      if (ruse[cg / M::NG]) {
        const double kd = fmul((double)k, rdl[cg]);
        rtab[cg * kRecMaxBpt + k] = exp(fmul(fmul(-0.5, kd), kd));
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = 1 + 3 * ncand;
  const int BPT = P.bpt;
  const int64_t TB = (int64_t)BPT * kTileThreads;
  for (int64_t tile = P.tile_begin + blockIdx.x; tile < P.tile_end; tile += gridDim.x) {
    const int64_t base = tile * TB + threadIdx.x;
    // CG candidates at a time, bins inner: the CG model evaluations of a bin
    // are independent chains the scheduler interleaves, and the bin's centre
    // and 1/c are shared.  Per candidate the bin order, the accumulation
    // expressions and the trees are those of the single value pass
    // (tile_bins / bin_term / bin_accumulate), so each candidate's record is
    // bit-identical to a separate chi2 pass.
#pragma unroll
    for (int c0 = 0; c0 < G; c0 += CG) {
      if (c0 < ng) {
        typename M::Reg QR[CG];
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) QR[cc] = M::load(Q[c0 + cc]);
        double a0[CG], a2[CG];
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) a0[cc] = a2[cc] = 0.0;
        double jh = fadd((double)base, 0.5);
        [[maybe_unused]] double rP[REC ? CG * M::NG : 1], rA[REC ? CG * M::NG : 1],
            rz0[REC ? CG * M::NG : 1];
        [[maybe_unused]] double x0 = 0.0, kd = 0.0;
        if constexpr (REC) {  // the anchors of tile_bins, per candidate
          x0 = fadd(P.lo, fmul(jh, P.width));
#pragma unroll
          for (int cc = 0; cc < CG; ++cc)
#pragma unroll
            for (int c = 0; c < M::NG; ++c) {
              double mu, inv;
              M::gauss(QR[cc], c, mu, inv);
              const double z0 = fmul(fsub(x0, mu), inv);
              rz0[cc * M::NG + c] = z0;
              rP[cc * M::NG + c] = exp_nonpos(fmul(fmul(-0.5, z0), z0), tab);
              rA[cc * M::NG + c] = exp(-fmul(z0, rdl[(c0 + cc) * M::NG + c]));
            }
        }
        auto bin = [&](int k, double ic) {
          const double x = fadd(P.lo, fmul(jh, P.width));
          [[maybe_unused]] const double xr = REC ? __fma_rn(kd, fmul(256.0, P.width), x0) : 0.0;
#pragma unroll
          for (int cc = 0; cc < CG; ++cc) {
            double m, bg[1];
            if (REC && ruse[c0 + cc]) {  // tile_bins' REC arithmetic, per candidate
              double e[M::NG], z[M::NG];
#pragma unroll
              for (int c = 0; c < M::NG; ++c) {
                e[c] = fmul(rP[cc * M::NG + c], rtab[((c0 + cc) * M::NG + c) * kRecMaxBpt + k]);
                rP[cc * M::NG + c] = fmul(rP[cc * M::NG + c], rA[cc * M::NG + c]);
                z[c] = __fma_rn(kd, rdl[(c0 + cc) * M::NG + c], rz0[cc * M::NG + c]);
              }
              M::template eval_rec<false>(xr, z, e, QR[cc], m, bg);
            } else {
              M::template eval<false, true>(x, QR[cc], tab, m, bg);
            }
            const double mc = m * ic;
            a0[cc] += m;  // the value pass's bin_accumulate
            a2[cc] = __fma_rn(m, mc, a2[cc]);
          }
        };
        for (int k = 0; k < BPT; ++k) {
          const int64_t j = base + (int64_t)k * kTileThreads;
          if (j < P.bin_end) bin(k, ld_stream(P.icounts + j));
          jh = fadd(jh, (double)kTileThreads);
          if constexpr (REC) kd = fadd(kd, 1.0);
        }
        // this group's fixed shuffle trees (A1 is a copy of S: copy_source)
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            a0[cc] += __shfl_down_sync(0xffffffffu, a0[cc], off);
            a2[cc] += __shfl_down_sync(0xffffffffu, a2[cc], off);
          }
          if (lane == 0) {
            red[warp][3 * (c0 + cc)] = a0[cc];
            red[warp][3 * (c0 + cc) + 2] = a2[cc];
          }
        }
      }
    }
    if (lane == 0) red[warp][3 * G] = 0.0;  // C0: merged from the K3l pre-pass
    __syncthreads();
    for (int v = threadIdx.x; v < 3 * ng + 1; v += kTileThreads) {
      // C0 is the last local entry; a candidate's A1 is its S (copy_source)
      const int src = v < 3 * ng ? (v % 3 == 1 ? v - 1 : v) : 3 * G;
      const double s01 = red[0][src] + red[1][src], s23 = red[2][src] + red[3][src];
      const double s45 = red[4][src] + red[5][src], s67 = red[6][src] + red[7][src];
      const double val = (s01 + s23) + (s45 + s67);
      double* out = P.tile_ws + (tile - P.tile_begin) * R;
      if (v < 3 * ng) out[1 + 3 * g0 + v] = val;
      else if (blockIdx.y == 0) out[0] = val;
    }
    __syncthreads();
  }
}

// ---- K0: inverse counts (once per plan) -----------------------------------------
// ic_j = [c_j > 0] / c_j with an IEEE division: the faithful per-bin 1/c of
// the single-pass algebra, hoisted out of every pass (the histogram is fixed
// for the lifetime of a plan).
__global__ void __launch_bounds__(256) chi2_inverse_kernel(const double* __restrict__ counts,
                                                           double* __restrict__ ic, int64_t begin,
                                                           int64_t end) {
  for (int64_t j = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < end;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double c = ld_stream(counts + j);
    ic[j] = c > 0.0 ? fdiv(1.0, c) : 0.0;
  }
}

// ---- K3l: q-independent sums (once per plan) ------------------------------------
// C0 = sum [c_j > 0] c_j and, for the linear parameters, G0_i = sum phi_i(x_j),
// G1_i = sum [c_j > 0] phi_i(x_j), accumulated with exactly the per-thread order
// and trees of a pass, so merging them (chunk kernel) gives the same bits as
// accumulating them in every pass.  Record per tile / chunk:
// [G0_lin[L], G1_lin[L], C0].
template <class M>
__global__ void __launch_bounds__(kTileThreads) chi2_lin_kernel(Chi2Pass P) {
  constexpr int L = M::NP - M::LIN0;
  constexpr int RL = 2 * L + 1;
  __shared__ double red[kTileThreads / 32][RL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int BPT = P.bpt;
  const int64_t TB = (int64_t)BPT * kTileThreads;
  for (int64_t tile = P.tile_begin + blockIdx.x; tile < P.tile_end; tile += gridDim.x) {
    const int64_t base = tile * TB + threadIdx.x;
    double acc[RL];
#pragma unroll
    for (int v = 0; v < RL; ++v) acc[v] = 0.0;
    double jh = fadd((double)base, 0.5);
    for (int k = 0; k < BPT; ++k) {
      const int64_t j = base + (int64_t)k * kTileThreads;
      if (j < P.bin_end) {
        const double c = ld_stream(P.counts + j);
        const double x = fadd(P.lo, fmul(jh, P.width));
        const double w = c > 0.0 ? 1.0 : 0.0;
        double phi[L > 0 ? L : 1];
        M::lin_basis(x, phi);
#pragma unroll
        for (int i = 0; i < L; ++i) {
          acc[i] += phi[i];
          acc[L + i] = __fma_rn(w, phi[i], acc[L + i]);
        }
        acc[2 * L] += c > 0.0 ? c : 0.0;
      }
      jh = fadd(jh, (double)kTileThreads);
    }
#pragma unroll
    for (int v = 0; v < RL; ++v) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[v] += __shfl_down_sync(0xffffffffu, acc[v], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int v = 0; v < RL; ++v) red[warp][v] = acc[v];
    }
    __syncthreads();
    for (int v = threadIdx.x; v < RL; v += kTileThreads) {
      const double s01 = red[0][v] + red[1][v], s23 = red[2][v] + red[3][v];
      const double s45 = red[4][v] + red[5][v], s67 = red[6][v] + red[7][v];
      P.tile_ws[(tile - P.tile_begin) * RL + v] = (s01 + s23) + (s45 + s67);
    }
    __syncthreads();
  }
}

// ---- K0e: the empty bins of each chunk (once per plan) -------------------------
// Local chunk c covers bins [bin_begin + c cb, min(bin_begin + (c + 1) cb, bin_end)),
// cb = chunk_tiles * tile_bins.  One CTA per chunk.
constexpr int kEmptyThreads = 1024;

__device__ __forceinline__ void chunk_range(const Chi2Pass& P, int64_t chunk_tiles, int64_t c,
                                            int64_t& b0, int64_t& b1) {
  const int64_t tb = (int64_t)P.bpt * kTileThreads;
  const int64_t begin = P.tile_begin * tb;
  b0 = begin + c * chunk_tiles * tb;
  b1 = min(b0 + chunk_tiles * tb, P.bin_end);
}

// Section s of local chunk c (blockIdx = (c, s)): kEmptySections equal parts,
// so a chunk's list is built by that many CTAs (one CTA walking a 1 Mi-bin
// chunk in 1024-bin windows took 0.79 ms at 1e6 bins).
__device__ __forceinline__ void section_range(const Chi2Pass& P, int64_t chunk_tiles,
                                              int64_t& b0, int64_t& b1) {
  int64_t c0, c1;
  chunk_range(P, chunk_tiles, blockIdx.x, c0, c1);
  const int64_t len = (c1 - c0 + kEmptySections - 1) / kEmptySections;
  b0 = min(c1, c0 + (int64_t)blockIdx.y * len);
  b1 = min(c1, b0 + len);
}

__global__ void __launch_bounds__(kEmptyThreads) chi2_empty_count_kernel(Chi2Pass P,
                                                                         int64_t chunk_tiles,
                                                                         int64_t* counts) {
  int64_t b0, b1;
  section_range(P, chunk_tiles, b0, b1);
  unsigned n = 0;
  for (int64_t j = b0 + threadIdx.x; j < b1; j += kEmptyThreads) n += empty_bin(P.icounts[j]);
  __shared__ unsigned red[kEmptyThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) n += __shfl_down_sync(0xffffffffu, n, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kEmptyThreads / 32; ++w) t += red[w];
    counts[(int64_t)blockIdx.x * kEmptySections + blockIdx.y] = t;
  }
}

// Ordered compaction of a section: windows of 1024 x kEmptyRun bins, thread t
// owning the run of kEmptyRun consecutive bins at t kEmptyRun (its loads
// land in L1 lines its neighbours share); the runs' counts go through a
// warp scan and the warps' totals, then each thread writes its empty bins in
// order.  off[] = the sections' exclusive prefix in (chunk, section) order.
constexpr int kEmptyRun = 16;

__global__ void __launch_bounds__(kEmptyThreads) chi2_empty_fill_kernel(Chi2Pass P,
                                                                        int64_t chunk_tiles,
                                                                        const int64_t* off,
                                                                        int64_t* idx) {
  int64_t b0, b1;
  section_range(P, chunk_tiles, b0, b1);
  __shared__ unsigned wsum[kEmptyThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t base = off[(int64_t)blockIdx.x * kEmptySections + blockIdx.y];
  for (int64_t w0 = b0; w0 < b1; w0 += (int64_t)kEmptyThreads * kEmptyRun) {
    const int64_t j0 = w0 + (int64_t)threadIdx.x * kEmptyRun;
    unsigned mask = 0;
#pragma unroll
    for (int k = 0; k < kEmptyRun; ++k) {
      const int64_t j = j0 + k;
      if (j < b1 && empty_bin(P.icounts[j])) mask |= 1u << k;
    }
    const unsigned cnt = __popc(mask);
    unsigned incl = cnt;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned before = incl - cnt, total = 0;
    for (int w = 0; w < kEmptyThreads / 32; ++w) {
      before += w < warp ? wsum[w] : 0u;
      total += wsum[w];
    }
    int64_t o = base + before;
    while (mask) {
      const int k = __ffs(mask) - 1;
      idx[o++] = j0 + k;
      mask &= mask - 1;
    }
    base += total;
    __syncthreads();
  }
}

// ---- K3z: the model (and nonlinear gradient) sums over a chunk's empty bins -----
// One CTA per (local chunk, segment of its list, batch member / candidate);
// fixed per-thread order, shuffle tree and cross-warp tree.
// zws[y][chunk][seg][ZL]: [sum m, sum dm_i (i < ZL-1)]; the chunk kernel adds
// the segments in order (ZMerge).
// multi: blockIdx.y is a line-search candidate (q at qdev + y kQDoubles);
// otherwise a batch member (qdev + y q_stride).
template <class M, bool GRAD, bool FAST>
__global__ void __launch_bounds__(kTileThreads) chi2_empty_kernel(Chi2Pass P, int64_t nchunks,
                                                                  int nseg, bool multi) {
  constexpr int ZL = GRAD ? 1 + M::LIN0 : 1;
  const int y = blockIdx.y;
  if (multi && P.ncand_dev != nullptr && y >= *P.ncand_dev) return;  // uniform over the CTA
  const double* qd = P.qdev + (multi ? (int64_t)y * kQDoubles : y * P.q_stride);
  __shared__ QDev Q;
  __shared__ double tab[64];
  __shared__ double red[kTileThreads / 32][ZL];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = qd[threadIdx.x];
    Q.inv[threadIdx.x] = qd[kMaxNp + threadIdx.x];
  }
  if (threadIdx.x < 64) tab[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
  __syncwarp();
  __syncthreads();
  const typename M::Reg QR = M::load(Q);
  double acc[ZL];
#pragma unroll
  for (int v = 0; v < ZL; ++v) acc[v] = 0.0;
  const int64_t chunk = blockIdx.x / nseg, seg = blockIdx.x % nseg;
  const int64_t c0 = P.empty_off[chunk], c1 = P.empty_off[chunk + 1];
  const int64_t o0 = c0 + (c1 - c0) * seg / nseg, o1 = c0 + (c1 - c0) * (seg + 1) / nseg;
  for (int64_t t = o0 + threadIdx.x; t < o1; t += kTileThreads) {
    const double jh = fadd((double)P.empty_idx[t], 0.5);
    const double x = fadd(P.lo, fmul(jh, P.width));  // Histogram::center, as bin_term
    double m, bg[GRAD ? M::NP : 1];
    M::template eval<GRAD, FAST>(x, QR, tab, m, bg);
    acc[0] += m;
    if constexpr (GRAD) {
#pragma unroll
      for (int i = 0; i < M::LIN0; ++i) acc[1 + i] += bg[i];
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < ZL; ++v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[v] += __shfl_down_sync(0xffffffffu, acc[v], off);
    if (lane == 0) red[warp][v] = acc[v];
  }
  __syncthreads();
  if (threadIdx.x < ZL) {
    const int v = threadIdx.x;
    const double s01 = red[0][v] + red[1][v], s23 = red[2][v] + red[3][v];
    const double s45 = red[4][v] + red[5][v], s67 = red[6][v] + red[7][v];
    P.zws[(((int64_t)y * nchunks + chunk) * nseg + seg) * ZL + v] = (s01 + s23) + (s45 + s67);
  }
}

// Fast AD gradient passes: what the chunk kernel derives from the chunk's sums
// (bin_accumulate): the width-derivative entries (G0/G1/G2 of the parameters
// in `sc`) times 1/q[sinv] (the eval leaves that common factor out), then
// S = sum_{i in lin} q_i G0_i, A2 = sum_{i in lin} q_i G2_i, A1 = S - Z.
struct Derive {
  const double* qdev = nullptr;  // QDev of batch member blockIdx.y at qdev + y q_stride
  int64_t q_stride = 0;
  int np = 0, nl = 0, ns = 0;
  signed char lin[kMaxNp];
  signed char sc[kMaxNp], sq[kMaxNp], sinv[kMaxNp];  // entry sc times q[sq] / q[sinv]
};

template <class M>
Derive make_derive(const Chi2Pass& P) {
  Derive d;
  d.qdev = P.qdev;
  d.q_stride = P.q_stride;
  d.np = M::NP;
  if constexpr (std::is_same<M, GPoly>::value) {
    const signed char lin[] = {0, 3, 4, 5};
    for (signed char i : lin) d.lin[d.nl++] = i;
    d.sc[d.ns] = 1, d.sq[d.ns] = 0, d.sinv[d.ns++] = 2;
    d.sc[d.ns] = 2, d.sq[d.ns] = 0, d.sinv[d.ns++] = 2;
  } else {
    for (int j = 0; j < M::NG; ++j) {
      const signed char a = (signed char)(3 * j), w = (signed char)(3 * j + 2);
      d.lin[d.nl++] = a;
      d.sc[d.ns] = (signed char)(3 * j + 1), d.sq[d.ns] = a, d.sinv[d.ns++] = w;
      d.sc[d.ns] = w, d.sq[d.ns] = a, d.sinv[d.ns++] = w;
    }
  }
  return d;
}

// The chunk kernel's subtraction of the empty-bin sums (copy_source entries):
// single / batched passes: A1 (entry 1) -= z[0], G1 entries 4+NP+i -= z[1+i];
// multi records [C0, (S, A1, A2) x ncand]: candidate c's A1 -= z[c][chunk][0].
struct ZMerge {
  const double* z = nullptr;
  int zl = 0, np = 0, nseg = 1;
  bool multi = false;
  int64_t nchunks = 0;
};

// the empty-bin sum of entry k of member y: its segments added in order
__device__ __forceinline__ double zsum(const ZMerge& zm, int64_t y, int64_t chunk, int k) {
  const double* z = zm.z + ((y * zm.nchunks + chunk) * zm.nseg) * zm.zl + k;
  double s = z[0];
  for (int g = 1; g < zm.nseg; ++g) s = s + z[(int64_t)g * zm.zl];
  return s;
}

__device__ __forceinline__ double zmerge(const ZMerge& zm, int64_t chunk, int v, double a) {
  if (zm.z == nullptr) return a;
  if (zm.multi) {
    if (v >= 1 && (v - 1) % 3 == 1) return a - zsum(zm, (v - 1) / 3, chunk, 0);
    return a;
  }
  if (v == 1) return a - zsum(zm, blockIdx.y, chunk, 0);
  if (v >= 4 + zm.np && v < 4 + zm.np + zm.zl - 1)
    return a - zsum(zm, blockIdx.y, chunk, 1 + v - 4 - zm.np);
  return a;
}

// ---- K3r: the residual chi2 value (high-count histograms) -------------------------
// chi2 = sum_{c>0} (c - a m)^2 / c with a = E/S known from a first pass: the
// residual r is formed per bin, so nothing of magnitude E cancels (the single
// pass's C0 - 2a A1 + a^2 A2 loses ~eps * E).  Same bins, centres and fast /
// faithful model arithmetic as the value pass without the run recurrence, so
// S and the residuals see the same m.  One CTA per (local chunk, segment,
// candidate y); fixed per-thread order, shuffle tree and cross-warp tree into
// out[y][chunk][seg].
template <class M, bool FAST>
__global__ void __launch_bounds__(kTileThreads) chi2_resid_kernel(Chi2Pass P, int64_t chunk_bins,
                                                                  int64_t nchunks,
                                                                  const double* a_dev,
                                                                  bool multi, double* out) {
  const int y = blockIdx.y;
  const double* qd = P.qdev + (multi ? (int64_t)y * kQDoubles : y * P.q_stride);
  __shared__ QDev Q;
  __shared__ double tab[64];
  __shared__ double red[kTileThreads / 32];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = qd[threadIdx.x];
    Q.inv[threadIdx.x] = qd[kMaxNp + threadIdx.x];
  }
  if (threadIdx.x < 64) tab[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
  __syncwarp();
  __syncthreads();
  const typename M::Reg QR = M::load(Q);
  const double a = a_dev[y];
  const int64_t chunk = blockIdx.x / kResidSegs, seg = blockIdx.x % kResidSegs;
  const int64_t begin = P.tile_begin * (int64_t)P.bpt * kTileThreads;
  const int64_t c0 = begin + chunk * chunk_bins, c1 = min(c0 + chunk_bins, P.bin_end);
  const int64_t o0 = c0 + (c1 - c0) * seg / kResidSegs, o1 = c0 + (c1 - c0) * (seg + 1) / kResidSegs;
  double acc = 0.0;
  for (int64_t j = o0 + threadIdx.x; j < o1; j += kTileThreads) {
    const double x = fadd(P.lo, fmul(fadd((double)j, 0.5), P.width));
    double m, bg[1];
    M::template eval<false, FAST>(x, QR, tab, m, bg);
    const double r = P.counts[j] - a * m;  // [c > 0] via ic = 0 below
    acc += (r * r) * P.icounts[j];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0)
    out[((int64_t)y * nchunks + chunk) * kResidSegs + seg] =
        ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}

int chi2_resid_enqueue(const Chi2Pass& P, int model, int np, int prec, int64_t chunk_tiles,
                       const double* a_dev, int ny, bool multi, double* out, cudaStream_t s) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  const int64_t chunk_bins = chunk_tiles * (int64_t)P.bpt * kTileThreads;
  const dim3 grid((unsigned)(nchunks * kResidSegs), (unsigned)ny);
  auto go = [&](auto tag) {
    using M = decltype(tag);
    if (prec != 0)
      chi2_resid_kernel<M, true><<<grid, kTileThreads, 0, s>>>(P, chunk_bins, nchunks, a_dev, multi, out);
    else
      chi2_resid_kernel<M, false><<<grid, kTileThreads, 0, s>>>(P, chunk_bins, nchunks, a_dev, multi, out);
  };
  if (model == ADC_MODEL_GPOLY) {
    go(GPoly{});
  } else {
    switch (np / 3) {
      case 1: go(GSum<1>{}); break;
      case 2: go(GSum<2>{}); break;
      case 3: go(GSum<3>{}); break;
      case 4: go(GSum<4>{}); break;
      case 8: go(GSum<8>{}); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
  }
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

// ---- K4: chunk reduce (fixed tree over the chunk's tiles) ---------------------
// One CTA per chunk; warp w owns record entries v = w, w+8, ...; lane l sums
// tiles l, l+32, l+64, l+96 pairwise, then a fixed shuffle tree.
// lin (optional): per-chunk [G0_lin[L], G1_lin[L], C0] of the K3l pre-pass,
// merged into the record entries a pass leaves at zero (0 + v == v exactly):
// C0 at c0_pos, and (gradient passes of the AD provider, g0_pos >= 0) the
// linear G0 entries at g0_pos.. and G1 entries at g1_pos...
struct LinMerge {
  const double* lin = nullptr;
  int L = 0;
  int c0_pos = -1, g0_pos = -1, g1_pos = -1;
};

// pub (optional, the peer-memory transport): the kernel that reduces the
// chunks also publishes them — each CTA stores its record straight into every
// rank's receive slot as it is produced, and the last CTA to finish raises the
// flags, waits for every rank and compacts (peer.cuh): the reduction and the
// collective are one kernel.
__global__ void __launch_bounds__(kChunkThreads) chi2_chunk_kernel(
    const double* __restrict__ tile_ws, int64_t ntiles, int R, int chunk_tiles,
    double* __restrict__ records, LinMerge lm = LinMerge{}, PeerPublish pub = PeerPublish{},
    const int* ncand_dev = nullptr, int64_t ws_stride = 0, int64_t rec_stride = 0,
    ZMerge zm = ZMerge{}, Derive dv = Derive{}) {
  if (ncand_dev != nullptr) R = 1 + 3 * *ncand_dev;  // multi records sized on the device
  tile_ws += blockIdx.y * ws_stride;  // batched passes (blockIdx.y = member)
  records += blockIdx.y * rec_stride;
  const int64_t chunk = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = chunk * chunk_tiles;
  const bool publish = pub.peer_gather != nullptr;  // uniform over the grid
  __shared__ unsigned long long s_q;
  __shared__ bool s_last;
  __shared__ double srec[4 + 3 * kMaxNp];  // Derive: the chunk's record, staged
  if (publish) {
    if (threadIdx.x == 0) s_q = *pub.seq + 1;
    __syncthreads();
  }
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
    if (lm.lin != nullptr && lane == 0) {
      const int L = lm.L, RL = 2 * L + 1;
      const double* l = lm.lin + chunk * RL;
      if (v == lm.c0_pos) a = a + l[2 * L];
      else if (lm.g0_pos >= 0 && v >= lm.g0_pos && v < lm.g0_pos + L) a = a + l[v - lm.g0_pos];
      else if (lm.g1_pos >= 0 && v >= lm.g1_pos && v < lm.g1_pos + L) a = a + l[L + v - lm.g1_pos];
    }
    if (lane == 0) {
      a = zmerge(zm, chunk, v, a);
      if (dv.nl > 0) {
        srec[v] = a;
      } else {
        records[chunk * R + v] = a;
        if (publish)
          for (int r = 0; r < pub.world; ++r) peer_slot(pub, r, s_q)[chunk * R + v] = a;
      }
    }
  }
  if (dv.nl > 0) {  // uniform over the grid
    __syncthreads();
    if (threadIdx.x == 0) {
      const double* q = dv.qdev + blockIdx.y * dv.q_stride;  // QDev: q[kMaxNp], inv[kMaxNp]
      const int np = dv.np;
      for (int k = 0; k < dv.ns; ++k) {
        const double inv = q[dv.sq[k]] * q[kMaxNp + dv.sinv[k]];
        const int i = dv.sc[k];
        srec[4 + i] = srec[4 + i] * inv;
        srec[4 + np + i] = srec[4 + np + i] * inv;
        srec[4 + 2 * np + i] = srec[4 + 2 * np + i] * inv;
      }
      double S = 0.0, A2 = 0.0;
      for (int k = 0; k < dv.nl; ++k) {
        const int i = dv.lin[k];
        S = __fma_rn(q[i], srec[4 + i], S);
        A2 = __fma_rn(q[i], srec[4 + 2 * np + i], A2);
      }
      srec[0] = S;
      srec[1] = S + srec[1];  // the tile records' A1 is 0: minus the empty-bin sum
      srec[2] = A2;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < R; v += kChunkThreads) {
      records[chunk * R + v] = srec[v];
      if (publish)
        for (int r = 0; r < pub.world; ++r) peer_slot(pub, r, s_q)[chunk * R + v] = srec[v];
    }
  }
  if (publish) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(pub.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      if (threadIdx.x == 0) *pub.done = 0u;
      peer_signal_wait_compact(pub, s_q);
    }
  }
}

// ---- dispatch ----------------------------------------------------------------
template <class M, bool GRAD, bool FAST, bool REC = false>
static void launch_tiles_t(const Chi2Pass& P, dim3 blocks, cudaStream_t s) {
  constexpr int MB = tile_min_blocks<M, GRAD>();
  if constexpr (std::is_same<M, GPoly>::value && FAST) {
    // default: two bins evaluated before either is folded (measured 1.5% faster);
    // with REC one bin at a time (REC's extra live doubles push the two-bin
    // form into local memory).  The 1/c values come through a per-thread
    // register ring of streaming loads: 0.274 ms at 1e8 bins, vs 0.318 ms
    // staged through shared memory per warp by cp.async.bulk + mbarrier (the
    // stage bookkeeping costs issue slots the FP64 pipe needs)
    if (REC)
      chi2_tile_kernel<M, GRAD, FAST, MB, 1, false, REC><<<blocks, kTileThreads, 0, s>>>(P);
    else
      chi2_tile_kernel<M, GRAD, FAST, MB, 2, false, REC><<<blocks, kTileThreads, 0, s>>>(P);
    return;
  }
  chi2_tile_kernel<M, GRAD, FAST, MB, 1, false, REC><<<blocks, kTileThreads, 0, s>>>(P);
}

// prec: 0 faithful, 1 fast, 2 fast + the Gaussian-factor recurrence (every
// pass: gradient, value and the multi-candidate pass, which repeats the value
// pass's per-candidate decision and arithmetic)
template <class M>
static void launch_tiles_m(const Chi2Pass& P, bool grad, int prec, bool num, dim3 blocks,
                           cudaStream_t s) {
  constexpr int MB = tile_min_blocks<M, true>();
  const bool fast = prec != 0;
  if (grad && num) {  // GradientProvider::Numeric
    if (fast) chi2_tile_kernel<M, true, true, MB, 1, true><<<blocks, kTileThreads, 0, s>>>(P);
    else chi2_tile_kernel<M, true, false, MB, 1, true><<<blocks, kTileThreads, 0, s>>>(P);
    return;
  }
  if (grad) {
    // (REC holds two more doubles per Gaussian factor: models with <= 2
    // factors only, larger gsum spills; they run mode 1)
    if (prec == 2 && M::NG <= 2) launch_tiles_t<M, true, true, M::NG <= 2>(P, blocks, s);
    else if (fast) launch_tiles_t<M, true, true>(P, blocks, s);
    else launch_tiles_t<M, true, false>(P, blocks, s);
  } else {
    if (prec == 2 && M::NG <= 2) launch_tiles_t<M, false, true, M::NG <= 2>(P, blocks, s);
    else if (fast) launch_tiles_t<M, false, true>(P, blocks, s);
    else launch_tiles_t<M, false, false>(P, blocks, s);
  }
}

// K3z for a pass: grid (local chunks, ny).  Returns the ZMerge for its chunk kernel.
template <class M>
static void launch_empty_m(const Chi2Pass& P, bool grad, bool fast, int64_t nchunks, int nseg,
                           int ny, bool multi, cudaStream_t s) {
  const dim3 grid((unsigned)(nchunks * nseg), (unsigned)ny);
  if (grad) {
    if (fast)
      chi2_empty_kernel<M, true, true><<<grid, kTileThreads, 0, s>>>(P, nchunks, nseg, multi);
    else
      chi2_empty_kernel<M, true, false><<<grid, kTileThreads, 0, s>>>(P, nchunks, nseg, multi);
  } else {
    if (fast)
      chi2_empty_kernel<M, false, true><<<grid, kTileThreads, 0, s>>>(P, nchunks, nseg, multi);
    else
      chi2_empty_kernel<M, false, false><<<grid, kTileThreads, 0, s>>>(P, nchunks, nseg, multi);
  }
}

static int launch_empty(const Chi2Pass& P, int model, int np, bool grad, bool fast,
                        int64_t nchunks, int ny, bool multi, cudaStream_t s, ZMerge& zm) {
  if (P.empty_off == nullptr || P.zws == nullptr)
    return fail(ADC_E_ARG, "chi2 pass: the plan's empty-bin lists are not built");
  // a fixed number of segments per chunk list (not a function of the device
  // or the split, so the same sums on every rank and world size)
  const int nseg = kEmptySegs;
  zm.nseg = nseg;
  if (model == ADC_MODEL_GPOLY) {
    launch_empty_m<GPoly>(P, grad, fast, nchunks, nseg, ny, multi, s);
    zm.zl = grad ? 1 + GPoly::LIN0 : 1;
  } else {
    switch (np / 3) {
      case 1: launch_empty_m<GSum<1>>(P, grad, fast, nchunks, nseg, ny, multi, s); break;
      case 2: launch_empty_m<GSum<2>>(P, grad, fast, nchunks, nseg, ny, multi, s); break;
      case 3: launch_empty_m<GSum<3>>(P, grad, fast, nchunks, nseg, ny, multi, s); break;
      case 4: launch_empty_m<GSum<4>>(P, grad, fast, nchunks, nseg, ny, multi, s); break;
      case 8: launch_empty_m<GSum<8>>(P, grad, fast, nchunks, nseg, ny, multi, s); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
    zm.zl = grad ? 1 + np : 1;
  }
  ADCB_CUDA(cudaGetLastError());
  zm.z = P.zws;
  zm.np = np;
  zm.multi = multi;
  zm.nchunks = nchunks;
  return ADC_OK;
}

int chi2_enqueue(const Chi2Pass& P, int model, int np, bool grad, int prec,
                 int64_t chunk_tiles, double* records, cudaStream_t s, const double* lin,
                 bool numeric, const PeerPublish* pub, int nbatch, int64_t rec_stride) {

  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  const int R = grad ? 4 + 3 * np : 4;
  // Persistent grid: a few CTAs per SM, tiles grid-strided.
  // Persistent grid: as many CTAs as are resident (2 per SM for the small
  // models, see tile_min_blocks), tiles grid-strided.
  const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)sm_count() * (np <= 6 ? 2 : 1));
  const dim3 grid((unsigned)blocks, (unsigned)nbatch);
  // The empty-bin side pass (K3z) does not depend on the tile kernel: with the
  // plan's low-priority side stream it runs beside it (the block scheduler
  // places its CTAs as the tile kernel's retire in the last partial wave),
  // joined before the chunk kernel.
  const bool fork = P.side_stream != nullptr;
  if (fork) {
    ADCB_CUDA(cudaEventRecord(P.ev_fork, s));
    ADCB_CUDA(cudaStreamWaitEvent(P.side_stream, P.ev_fork, 0));
  }
  if (P.tk0) ADCB_CUDA(cudaEventRecord(P.tk0, s));
  if (model == ADC_MODEL_GPOLY) {
    launch_tiles_m<GPoly>(P, grad, prec, numeric, grid, s);
  } else {
    switch (np / 3) {
      case 1: launch_tiles_m<GSum<1>>(P, grad, prec, numeric, grid, s); break;
      case 2: launch_tiles_m<GSum<2>>(P, grad, prec, numeric, grid, s); break;
      case 3: launch_tiles_m<GSum<3>>(P, grad, prec, numeric, grid, s); break;
      case 4: launch_tiles_m<GSum<4>>(P, grad, prec, numeric, grid, s); break;
      case 8: launch_tiles_m<GSum<8>>(P, grad, prec, numeric, grid, s); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
  }
  ADCB_CUDA(cudaGetLastError());
  if (P.tk1) ADCB_CUDA(cudaEventRecord(P.tk1, s));
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  const int lin0 = model == ADC_MODEL_GPOLY ? GPoly::LIN0 : np;
  LinMerge lm;
  lm.lin = lin;
  lm.L = np - lin0;
  lm.c0_pos = 3;
  if (grad && !numeric && lm.L > 0) {  // finite differences of a linear term are not its basis
    lm.g0_pos = 4 + lin0;
    lm.g1_pos = 4 + np + lin0;
  }
  ZMerge zm;
  if (int rc = launch_empty(P, model, np, grad && !numeric, prec != 0, nchunks, nbatch, false,
                            fork ? P.side_stream : s, zm))
    return rc;
  if (fork) {
    ADCB_CUDA(cudaEventRecord(P.ev_join, P.side_stream));
    ADCB_CUDA(cudaStreamWaitEvent(s, P.ev_join, 0));
  }
  Derive dv;
  if (grad && !numeric && prec != 0) {
    if (model == ADC_MODEL_GPOLY) {
      dv = make_derive<GPoly>(P);
    } else {
      switch (np / 3) {
        case 1: dv = make_derive<GSum<1>>(P); break;
        case 2: dv = make_derive<GSum<2>>(P); break;
        case 3: dv = make_derive<GSum<3>>(P); break;
        case 4: dv = make_derive<GSum<4>>(P); break;
        case 8: dv = make_derive<GSum<8>>(P); break;
        default: return fail(ADC_E_ARG, "gsum: unsupported component count");
      }
    }
  }
  chi2_chunk_kernel<<<dim3((unsigned)nchunks, (unsigned)nbatch), kChunkThreads, 0, s>>>(
      P.tile_ws, ntiles, R, (int)chunk_tiles, records, lm, pub ? *pub : PeerPublish{}, nullptr,
      P.ws_stride, rec_stride, zm, dv);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int chi2_empty_count_enqueue(const Chi2Pass& P, int64_t chunk_tiles, int64_t* counts,
                             cudaStream_t s) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  chi2_empty_count_kernel<<<dim3((unsigned)nchunks, kEmptySections), kEmptyThreads, 0, s>>>(
      P, chunk_tiles, counts);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int chi2_empty_fill_enqueue(const Chi2Pass& P, int64_t chunk_tiles, const int64_t* off,
                            int64_t* idx, cudaStream_t s) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  chi2_empty_fill_kernel<<<dim3((unsigned)nchunks, kEmptySections), kEmptyThreads, 0, s>>>(
      P, chunk_tiles, off, idx);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int chi2_lin_count(int model, int np) {
  return model == ADC_MODEL_GPOLY ? GPoly::NP - GPoly::LIN0 : 0;
}

int chi2_lin_enqueue(const Chi2Pass& P, int model, int64_t chunk_tiles, double* lin_records,
                     double* icounts_local, cudaStream_t s) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  // K0 over this rank's bins (icounts_local = ic[bin_begin..bin_end))
  const int64_t bin_begin = P.tile_begin * (int64_t)P.bpt * kTileThreads;
  const int64_t nb = P.bin_end - bin_begin;
  const int64_t iblocks = std::min<int64_t>((nb + 255) / 256, (int64_t)sm_count() * 8);
  chi2_inverse_kernel<<<(unsigned)iblocks, 256, 0, s>>>(P.counts, icounts_local - bin_begin,
                                                        bin_begin, P.bin_end);
  ADCB_CUDA(cudaGetLastError());
  const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)sm_count() * 4);
  int RL = 1;
  if (model == ADC_MODEL_GPOLY) {
    chi2_lin_kernel<GPoly><<<(unsigned)blocks, kTileThreads, 0, s>>>(P);
    RL = 2 * (GPoly::NP - GPoly::LIN0) + 1;
  } else {
    chi2_lin_kernel<GSum<1>><<<(unsigned)blocks, kTileThreads, 0, s>>>(P);  // C0 only
  }
  ADCB_CUDA(cudaGetLastError());
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  chi2_chunk_kernel<<<(unsigned)nchunks, kChunkThreads, 0, s>>>(P.tile_ws, ntiles, RL,
                                                               (int)chunk_tiles, lin_records);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int chi2_multi_enqueue(const Chi2Pass& P, int model, int np, int ncand,
                       int64_t chunk_tiles, double* records, cudaStream_t s, const double* lin,
                       int prec) {
  const int64_t ntiles = P.tile_end - P.tile_begin;
  if (ntiles <= 0) return ADC_OK;
  if (ncand < 1 || ncand > kMultiMax) return fail(ADC_E_ARG, "chi2 multi: bad candidate count");
  const dim3 grid((unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * 2),
                  (unsigned)((ncand + kMultiGroup - 1) / kMultiGroup));
  auto go = [&](auto model_tag) {
    using M = decltype(model_tag);
    if constexpr (M::NG <= 2) {
      if (prec == 2) {
        chi2_multi_kernel<M, true><<<grid, kTileThreads, 0, s>>>(P, ncand);
        return;
      }
    }
    chi2_multi_kernel<M><<<grid, kTileThreads, 0, s>>>(P, ncand);
  };
  if (model == ADC_MODEL_GPOLY) {
    go(GPoly{});
  } else {
    switch (np / 3) {
      case 1: go(GSum<1>{}); break;
      case 2: go(GSum<2>{}); break;
      case 3: go(GSum<3>{}); break;
      case 4: go(GSum<4>{}); break;
      case 8: go(GSum<8>{}); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
  }
  ADCB_CUDA(cudaGetLastError());
  const int R = 1 + 3 * ncand;
  const int64_t nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
  LinMerge lm;
  lm.lin = lin;
  lm.L = chi2_lin_count(model, np);
  lm.c0_pos = 0;
  ZMerge zm;
  if (int rc = launch_empty(P, model, np, false, true, nchunks, ncand, true, s, zm)) return rc;
  chi2_chunk_kernel<<<(unsigned)nchunks, kChunkThreads, 0, s>>>(
      P.tile_ws, ntiles, R, (int)chunk_tiles, records, lm, PeerPublish{}, P.ncand_dev, 0, 0, zm);
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

void fill_qdev(int model, int np, const double* q, double* host_qdev) {
  std::memset(host_qdev, 0, sizeof(QDev) + sizeof(QNum));
  QDev* Q = reinterpret_cast<QDev*>(host_qdev);
  QNum* N = reinterpret_cast<QNum*>(host_qdev + 2 * kMaxNp);
  for (int i = 0; i < np; ++i) Q->q[i] = q[i];
  // numdiff.cpp:8-13 and 62-79: h = cbrt(eps) * max(1, |x|), probe = x + sign * h
  const double h0 = std::cbrt(2.220446049250313e-16);
  for (int i = 0; i < np; ++i) {
    const double h = h0 * std::max(1.0, std::fabs(q[i]));
    N->qp[i] = q[i] + 1.0 * h;
    N->qm[i] = q[i] + -1.0 * h;
    N->h2[i] = 2.0 * h;
    N->rh2[i] = 1.0 / N->h2[i];
  }
  auto width = [&](int j) {
    Q->inv[j] = 1.0 / q[j];
    N->invp[j] = 1.0 / N->qp[j];
    N->invm[j] = 1.0 / N->qm[j];
  };
  if (model == ADC_MODEL_GPOLY) {
    width(2);
  } else {
    for (int j = 2; j < np; j += 3) width(j);
  }
}

size_t qdev_bytes() { return sizeof(QDev) + sizeof(QNum); }


// ---- K6: on-device histogram sampling ---------------------
// The reference's sample_histogram (fit.cpp:70-104) draws events by rejection
// and cannot feed 1e8 bins.  Here each bin's count is drawn directly:
// c_j ~ Poisson(E m_j / S), S = sum_j m_j, with m the model at the truth
// parameters (the faithful per-bin arithmetic of the passes).  Randomness is
// counter-based (Philox4x32-10 keyed by the seed, counter = (bin, draw)), so
// the histogram is a pure function of (model, q, bins, range, E, seed): the
// same bits on any device, grid or world size.  Large means use Hörmann's
// transformed rejection (PTRS, 1993), small ones the multiplication method.
// S and the event total are reduced in a fixed order (no atomics).
namespace {
struct Philox {
  uint32_t k0, k1;
  __device__ __forceinline__ uint4 operator()(uint32_t c0, uint32_t c1, uint32_t c2,
                                              uint32_t c3) const {
    uint32_t a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
      const uint32_t n0 = hi1 ^ c1 ^ a, n2 = hi0 ^ c3 ^ b;
      c0 = n0;
      c1 = lo1;
      c2 = n2;
      c3 = lo0;
      a += 0x9E3779B9u;
      b += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
  }
};

// Two uniforms in (0, 1) from one Philox block (53-bit mantissas).
__device__ __forceinline__ double2 uniforms(const Philox& ph, uint64_t bin, uint32_t draw) {
  const uint4 r = ph((uint32_t)bin, (uint32_t)(bin >> 32), draw, 0x5EEDu);
  const uint64_t u0 = ((uint64_t)r.x << 21) ^ (r.y >> 11);
  const uint64_t u1 = ((uint64_t)r.z << 21) ^ (r.w >> 11);
  return make_double2(((double)(u0 & ((1ull << 53) - 1)) + 0.5) * 0x1.0p-53,
                      ((double)(u1 & ((1ull << 53) - 1)) + 0.5) * 0x1.0p-53);
}

__device__ double poisson(double lam, const Philox& ph, uint64_t bin) {
  uint32_t draw = 0;
  if (!(lam > 0.0)) return 0.0;
  if (lam < 10.0) {  // multiplication method
    const double L = exp(-lam);
    double p = 1.0, k = -1.0;
    for (;;) {
      const double2 u = uniforms(ph, bin, draw++);
      k += 1.0;
      p *= u.x;
      if (p <= L) return k;
      k += 1.0;
      p *= u.y;
      if (p <= L) return k;
    }
  }
  // PTRS (Hörmann 1993)
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double2 u2 = uniforms(ph, bin, draw++);
    const double U = u2.x - 0.5, V = u2.y;
    const double us = 0.5 - fabs(U);
    const double k = floor((2.0 * a / us + b) * U + lam + 0.43);
    if (us >= 0.07 && V <= vr) return k;
    if (k < 0.0 || (us < 0.013 && V > us)) continue;
    if (log(V) + log(inv_alpha) - log(a / (us * us) + b) <= -lam + k * loglam - lgamma(k + 1.0))
      return k;
  }
}

constexpr int kGenThreads = 256;
constexpr int64_t kGenTile = 16 * kGenThreads;  // bins per block, fixed

template <class M>
__global__ void __launch_bounds__(kGenThreads) sample_sum_kernel(Chi2Pass P, int64_t bins,
                                                                 double* partials) {
  __shared__ QDev Q;
  __shared__ double red[kGenThreads / 32];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = P.qdev[threadIdx.x];
    Q.inv[threadIdx.x] = P.qdev[kMaxNp + threadIdx.x];
  }
  __syncthreads();
  const typename M::Reg QR = M::load(Q);
  double acc = 0.0;
  for (int64_t j = blockIdx.x * kGenTile + threadIdx.x;
       j < min(bins, (int64_t)(blockIdx.x + 1) * kGenTile); j += kGenThreads) {
    const double x = fadd(P.lo, fmul(fadd((double)j, 0.5), P.width));
    double m, bg[1];
    M::template eval<false, false>(x, QR, nullptr, m, bg);
    acc += m;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0)
    partials[blockIdx.x] =
        ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}

// One CTA: fixed-order total of nblocks partials into *out.
__global__ void __launch_bounds__(kGenThreads) sample_total_kernel(const double* partials,
                                                                   int64_t nblocks, double* out) {
  __shared__ double red[kGenThreads / 32];
  double acc = 0.0;
  for (int64_t b = threadIdx.x; b < nblocks; b += kGenThreads) acc += partials[b];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0)
    *out = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}

template <class M>
__global__ void __launch_bounds__(kGenThreads) sample_counts_kernel(
    Chi2Pass P, int64_t bins, double events, const double* S, uint64_t seed, int64_t zero_every,
    double* counts, double* partials) {
  __shared__ QDev Q;
  __shared__ double red[kGenThreads / 32];
  if (threadIdx.x < kMaxNp) {
    Q.q[threadIdx.x] = P.qdev[threadIdx.x];
    Q.inv[threadIdx.x] = P.qdev[kMaxNp + threadIdx.x];
  }
  __syncthreads();
  const typename M::Reg QR = M::load(Q);
  const Philox ph{(uint32_t)seed, (uint32_t)(seed >> 32)};
  const double scale = events / *S;
  double acc = 0.0;
  for (int64_t j = blockIdx.x * kGenTile + threadIdx.x;
       j < min(bins, (int64_t)(blockIdx.x + 1) * kGenTile); j += kGenThreads) {
    const double x = fadd(P.lo, fmul(fadd((double)j, 0.5), P.width));
    double m, bg[1];
    M::template eval<false, false>(x, QR, nullptr, m, bg);
    double c = poisson(scale * m, ph, (uint64_t)j);
    if (zero_every > 0 && j % zero_every == 0) c = 0.0;
    counts[j] = c;
    acc += c;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0)
    partials[blockIdx.x] =
        ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}
}  // namespace

int histogram_sample_enqueue(int model, int np, const double* qdev, int64_t bins, double lo,
                             double width, double events, uint64_t seed, int64_t zero_every,
                             double* counts, double* ws, cudaStream_t s) {
  Chi2Pass P{};
  P.qdev = qdev;
  P.lo = lo;
  P.width = width;
  const int64_t nblocks = (bins + kGenTile - 1) / kGenTile;
  double* partials = ws;            // [nblocks]
  double* S = ws + nblocks;         // [1]
  double* total = ws + nblocks + 1; // [1]
  auto go = [&](auto tag) {
    using M = decltype(tag);
    sample_sum_kernel<M><<<(unsigned)nblocks, kGenThreads, 0, s>>>(P, bins, partials);
    sample_total_kernel<<<1, kGenThreads, 0, s>>>(partials, nblocks, S);
    sample_counts_kernel<M><<<(unsigned)nblocks, kGenThreads, 0, s>>>(
        P, bins, events, S, seed, zero_every, counts, partials);
    sample_total_kernel<<<1, kGenThreads, 0, s>>>(partials, nblocks, total);
  };
  if (model == ADC_MODEL_GPOLY) {
    go(GPoly{});
  } else {
    switch (np / 3) {
      case 1: go(GSum<1>{}); break;
      case 2: go(GSum<2>{}); break;
      case 3: go(GSum<3>{}); break;
      case 4: go(GSum<4>{}); break;
      case 8: go(GSum<8>{}); break;
      default: return fail(ADC_E_ARG, "gsum: unsupported component count");
    }
  }
  ADCB_CUDA(cudaGetLastError());
  return ADC_OK;
}

int64_t histogram_sample_ws_doubles(int64_t bins) { return (bins + kGenTile - 1) / kGenTile + 2; }

}  // namespace adcb
