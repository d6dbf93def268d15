// Internal interface between the chi2 kernels (chi2.cu) and the host side
// (chi2_host.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "peer.cuh"

namespace adcb {

constexpr int kMaxNp = 24;
constexpr int kQDoubles = 8 * kMaxNp;  // QDev (q, 1/q) + QNum (numeric probes), chi2.cu
constexpr int kMultiMax = 64;  // line-search candidates (or gradients) per multi pass
constexpr int kEmptySegs = 8;  // segments of each chunk's empty-bin list (side pass CTAs)
constexpr int kEmptySections = 64;  // CTAs building each chunk's list (once per plan)

struct Chi2Pass {
  const double* counts;   // full histogram, device (read by the once-per-plan passes)
  const double* icounts;  // [c > 0] / c per bin, same global indexing (read by every pass)
  const double* qdev;    // QDev (2 * kMaxNp doubles), device
  double* tile_ws;       // [tile_end - tile_begin][R]
  double lo, width;      // Histogram::center = lo + (j + 0.5) * width
  int64_t bin_end;       // one past the last bin this rank reads
  int bpt;               // bins per thread per tile (multiple of 4)
  int64_t tile_begin, tile_end;
  const int* ncand_dev = nullptr;  // multi pass: candidate count read on the device (fit graph)
  // batched passes (chi2_enqueue nbatch > 1): member b reads qdev + b q_stride
  // and writes its tile records at tile_ws + b ws_stride (doubles)
  int64_t q_stride = 0, ws_stride = 0;
  // the empty bins (c <= 0) of this rank's chunks, ascending, CSR by local
  // chunk (chi2_empty_*_enqueue); zws: their per-chunk model sums
  // (chi2_enqueue / chi2_multi_enqueue), kMultiMax x local chunks x (1 + kMaxNp)
  const int64_t* empty_idx = nullptr;
  const int64_t* empty_off = nullptr;
  double* zws = nullptr;
  // optional: a low-priority stream (and fork / join events) the side pass
  // runs on beside the tile kernel (chi2_enqueue)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // optional (adc_cuda_chi2_partials with kernel timing on): recorded around
  // the tile kernel on the pass stream
  cudaEvent_t tk0 = nullptr, tk1 = nullptr;
};

// lin: per-chunk q-independent basis sums from chi2_lin_enqueue (gradient
// passes of models with linear parameters; nullptr otherwise).
// numeric: GradientProvider::Numeric (central differences of the model).
// pub: publish the chunk records over peer memory from the chunk kernel.
int chi2_enqueue(const Chi2Pass& P, int model, int np, bool grad, int prec,
                 int64_t chunk_tiles, double* records, cudaStream_t s, const double* lin,
                 bool numeric = false, const PeerPublish* pub = nullptr, int nbatch = 1,
                 int64_t rec_stride = 0);
int chi2_lin_count(int model, int np);  // L: number of linear parameters
// Once per plan: ic = [c > 0]/c into icounts_local (this rank's bins, indexed
// from bin_begin), then [G0_lin[L], G1_lin[L], C0] per local chunk into
// lin_records (2L + 1 doubles each); uses P.tile_ws.
int chi2_lin_enqueue(const Chi2Pass& P, int model, int64_t chunk_tiles, double* lin_records,
                     double* icounts_local, cudaStream_t s);
// ncand: candidates; with P.ncand_dev set, ncand is the upper bound (grid)
// and the actual count is read on the device.
int chi2_multi_enqueue(const Chi2Pass& P, int model, int np, int ncand,
                       int64_t chunk_tiles, double* records, cudaStream_t s, const double* lin,
                       int prec);
// The empty-bin lists (once per plan, after chi2_lin_enqueue has written ic):
// per local chunk the number of bins with ic == +0 into counts[nchunks]; then,
// with off[nchunks + 1] its exclusive scan, their indices in ascending order.
int chi2_empty_count_enqueue(const Chi2Pass& P, int64_t chunk_tiles, int64_t* counts,
                             cudaStream_t s);
int chi2_empty_fill_enqueue(const Chi2Pass& P, int64_t chunk_tiles, const int64_t* off,
                            int64_t* idx, cudaStream_t s);
// K3r: the residual chi2 value of ny parameter vectors (qdev + y q_stride, or
// candidate y of a multi pass) with a_dev[y] = E / S_y: partial sums
// out[y][local chunk][kResidSegs] (fixed order).
constexpr int kResidSegs = 8;
int chi2_resid_enqueue(const Chi2Pass& P, int model, int np, int prec, int64_t chunk_tiles,
                       const double* a_dev, int ny, bool multi, double* out, cudaStream_t s);
void fill_qdev(int model, int np, const double* q, double* host_qdev);
size_t qdev_bytes();
// K6: counts[j] ~ Poisson(events m_j / sum m) (Philox, counter = bin), ws =
// histogram_sample_ws_doubles(bins) doubles; ws[nblocks + 1] = sum of counts.
int histogram_sample_enqueue(int model, int np, const double* qdev, int64_t bins, double lo,
                             double width, double events, uint64_t seed, int64_t zero_every,
                             double* counts, double* ws, cudaStream_t s);
int64_t histogram_sample_ws_doubles(int64_t bins);

}  // namespace adcb
