// Host side of the chi2 pass: tiling/sharding layout, the fixed-order final
// reduction + closed form (adc_chi2_finalize), the per-histogram plan (device
// workspace, pinned staging, one CUDA graph per pass kind) and the fit loop
// (FitEngine::fit, proj/src/fit.cpp:315-425).
//
// Compiled with -ffp-contract=off: every host-side double expression here is
// evaluated operation by operation, like the reference's fit.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "chi2_internal.h"
#include "comm_internal.h"
#include "fit_device.h"
#include "common.cuh"

using namespace adcb;

namespace {

constexpr int64_t kTileThreads = 256;
// counts per non-empty bin above which chi2 values take the residual pass:
// the single pass's relative error is ~5 eps kappa (K3)
constexpr double kResidKappa = 256.0;
constexpr int64_t kChunkBins = int64_t(1) << 20;  // large histograms: 1 Mi-bin chunks

// Bins per thread per tile.  Large histograms amortise the per-tile
// reduction over ~80-130 bins per thread and size the tile so the histogram
// is a whole number of waves of kWaveCtas resident CTAs (2 per SM x 148 SMs
// on a B200).  From 6 waves up the wave count is rounded up to a multiple of
// 8, so each rank of a 2-, 4- or 8-GPU split also gets (close to) whole
// waves: 1e8 bins -> 84 bins/thread, 4651 tiles = 15.7 waves on one GPU,
// 1.97 per rank on eight (128 bins/thread would be 10.3 and 1.25 -> 2 waves,
// a 38% loss at 8 GPUs).  Small histograms keep 4 bins per thread so there
// are enough tiles to fill the GPU.  A pure function of `bins` (not of the
// device or world size): the same layout everywhere, hence the same bits.
constexpr int64_t kWaveCtas = 296;
int bpt_for(int64_t bins) {
  const int64_t per_wave = kTileThreads * kWaveCtas;
  if (bins < per_wave * 8) return 4;  // < 606K bins: keep tiles small enough to fill the GPU
  int64_t waves = (bins + per_wave * 64) / (per_wave * 128);  // round(bins / (per_wave*128))
  if (waves < 1) waves = 1;
  if (waves >= 6) waves = (waves + 7) / 8 * 8;
  const int64_t bpt = (bins + per_wave * waves * 4 - 1) / (per_wave * waves * 4) * 4;
  return (int)std::max<int64_t>(4, bpt);
}
int64_t chunk_tiles_for(int64_t bins) {
  const int64_t tile = bpt_for(bins) * kTileThreads;
  if (bpt_for(bins) == 4) return 128;
  return std::max<int64_t>(1, std::min<int64_t>(128, (kChunkBins + tile / 2) / tile));
}

}  // namespace

extern "C" int adc_chi2_make_layout(int64_t bins, int32_t world, int32_t rank,
                                    adc_chi2_layout* out) {
  clear_error();
  if (out == nullptr) return fail(ADC_E_ARG, "layout: null output");
  if (bins <= 0) return fail(ADC_E_ARG, "histogram must have at least one bin");
  if (world <= 0 || rank < 0 || rank >= world) return fail(ADC_E_ARG, "bad rank/world");
  adc_chi2_layout L{};
  L.bins = bins;
  L.tile_bins = bpt_for(bins) * kTileThreads;
  L.chunk_tiles = chunk_tiles_for(bins);
  const int64_t ntiles = (bins + L.tile_bins - 1) / L.tile_bins;
  L.nchunks = (ntiles + L.chunk_tiles - 1) / L.chunk_tiles;
  L.chunk_begin = L.nchunks * rank / world;
  L.chunk_end = L.nchunks * (rank + 1) / world;
  const int64_t chunk_bins = L.tile_bins * L.chunk_tiles;
  L.bin_begin = std::min(bins, L.chunk_begin * chunk_bins);
  L.bin_end = std::min(bins, L.chunk_end * chunk_bins);
  *out = L;
  return ADC_OK;
}

extern "C" int32_t adc_chi2_record_len(int32_t np, int32_t want_grad) {
  return want_grad ? 4 + 3 * np : 4;
}

extern "C" int adc_chi2_finalize(int32_t np, double events, const double* records,
                                 int64_t nchunks, int32_t want_grad, double* grad, double* chi2) {
  clear_error();
  if (records == nullptr || nchunks <= 0) return fail(ADC_E_ARG, "finalize: no records");
  if (np <= 0 || np > kMaxNp) return fail(ADC_E_ARG, "finalize: bad parameter count");
  const int R = adc_chi2_record_len(np, want_grad);
  std::vector<double> r(records, records + nchunks * R);
  // Fixed pairwise tree over chunks (stride doubling), identical for any
  // sharding of the chunks over GPUs.
  for (int64_t s = 1; s < nchunks; s *= 2)
    for (int64_t i = 0; i + s < nchunks; i += 2 * s)
      for (int v = 0; v < R; ++v) r[i * R + v] = r[i * R + v] + r[(i + s) * R + v];
  const double S = r[0], A1 = r[1], A2 = r[2], C0 = r[3];
  const double a = events / S;  // chi2: scale = E/S (fit.cpp:214)
  if (chi2 != nullptr) {
    // sum_{c>0} (c - a m)^2 / c = C0 - 2a A1 + a^2 A2
    const double two_a = 2.0 * a;
    *chi2 = (C0 - two_a * A1) + (a * a) * A2;
  }
  if (want_grad && grad != nullptr) {
    // T = sum_{c>0} 2 r m / c = 2 A1 - 2a A2; s_coef = E/S^2 * T (fit.cpp:238-245)
    const double t_sum = 2.0 * A1 - (2.0 * a) * A2;
    const double s_coef = events / (S * S) * t_sum;
    // w_j = s_coef + [c>0](-2 r_j / c_j * E / S)  =>  sum_j w_j dm_j
    //     = s_coef G0 - 2a (G1 - a G2)          (fit.cpp:248-258)
    const double* G0 = &r[4];
    const double* G1 = &r[4 + np];
    const double* G2 = &r[4 + 2 * np];
    for (int i = 0; i < np; ++i) grad[i] = s_coef * G0[i] - (2.0 * a) * (G1[i] - a * G2[i]);
  }
  return ADC_OK;
}

// ---------------------------------------------------------------------------
struct adc_chi2_plan {
  int model = 0, np = 0;
  int64_t bins = 0;
  double lo = 0, hi = 0, events = 0, width = 0;
  const double* counts = nullptr;
  adc_chi2_layout L{};
  int world = 1, rank = 0;
  int64_t maxc = 1;  // max chunks per rank: the padded per-rank record stride
  int bpt = 4;
  int fast = 2;  // precision mode (adc_cuda_chi2_set_precision)
  int provider = ADC_PROVIDER_AD_REVERSE;  // of the gradient passes
  int device = 0;
  cudaStream_t stream = nullptr;       // plan-owned: graph replays
  cudaStream_t side = nullptr;         // plan-owned, lowest priority: the empty-bin side pass
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t tk0 = nullptr, tk1 = nullptr;  // adc_cuda_chi2_set_kernel_timing
  cudaStream_t user_stream = nullptr;  // caller's (0 = legacy default): adc_cuda_chi2_partials
  double* qdev = nullptr;
  double* tile_ws = nullptr;
  double* records = nullptr;  // [maxc][R] (gradient / value pass)
  double* h_q = nullptr;
  // [kind][fast], kind 0 = value, 1 = AD gradient, 2 = numeric gradient
  cudaGraphExec_t graph[3][3] = {};  // [value, AD gradient, numeric gradient][precision mode]
  bool warm[3][3] = {};              // eager pass before capture
  bool no_graph = false;  // the transport refused stream capture: enqueue directly
  // exchange / copy-back staging, sized once for the largest pass kind
  adc_comm* comm = nullptr;
  PeerExchange peer;          // ADC_COMM_PEER: IPC-shared receive buffers
  size_t xcount = 0;          // doubles per rank the staging holds
  double* gather = nullptr;   // device [world][xcount] (NCCL)
  double* h_send = nullptr;   // pinned [xcount]  (host transport / single device)
  double* h_gather = nullptr; // pinned [world][xcount]
  std::vector<double> full;   // compacted [nb][nchunks][R]
  // batched line search (adc_cuda_chi2_multi): lazily allocated
  double* qmulti = nullptr;     // device [kMultiMax][QDev]
  double* h_qmulti = nullptr;   // pinned
  double* tile_ws_multi = nullptr;
  double* records_multi = nullptr;  // [maxc][1 + 3 kMultiMax]
  int64_t multi_passes = 0;
  double* grad_multi_records = nullptr;  // [kMultiMax][maxc][R] (adc_cuda_chi2_gradient_multi)
  double* batch_ws = nullptr;            // [kMultiMax][local tiles][R] tile records of a batch
  // device-resident fit loop (fit_device.cu): one graph, a WHILE node around the iteration
  FitDevState* fit_st = nullptr;   // device
  FitDevState* h_fit_st = nullptr; // pinned
  double* fit_scratch = nullptr;
  int* ncand_dev = nullptr;
  cudaGraphExec_t fit_graph = nullptr;
  double* fit_trace = nullptr;  // device iterate trace of the fit loop
  double* fit_full = nullptr;    // compact all-rank records (sharded device loop)
  int64_t* fit_rbegin = nullptr; // [world + 1] first chunk of each rank
  int fit_trace_cap = 0;
  FitDevConst fit_const{};
  // q-independent basis sums of the linear parameters (chi2_lin_enqueue)
  double* lin = nullptr;      // per local chunk [G0_lin[L], G1_lin[L], C0]
  double* icounts = nullptr;  // [c > 0]/c for this rank's bins (from bin_begin)
  bool lin_ready = false;
  // high counts per bin (kappa = C0 / non-empty bins > kResidKappa, whole
  // histogram on one device): chi2 VALUES come from the residual pass (K3r)
  bool resid = false;
  double kappa = 0.0;
  double* resid_a = nullptr;    // device [kMultiMax]: E / S per candidate
  double* h_resid_a = nullptr;  // pinned
  double* resid_out = nullptr;  // device [kMultiMax][local chunks][kResidSegs]
  double* h_resid_out = nullptr;
  // the empty bins of this rank's chunks (CSR by local chunk) and the side
  // pass's per-chunk sums over them (chi2.cu K3z)
  int64_t* empty_idx = nullptr;
  int64_t empty_cap = 0;
  int64_t* empty_off = nullptr;  // [local chunks + 1]
  int64_t* empty_cnt = nullptr;  // [local chunks x kEmptySections + 1]: counts, then bases
  double* zws = nullptr;         // [kMultiMax][maxc][kEmptySegs][1 + kMaxNp]
};

namespace {

int check_domain(const adc_chi2_plan* P, const double* q, bool probes = false) {
  // Divisions by the width parameters are the interpreter's checked
  // divisions (eval.cpp:543) in gpoly/gsum and their gradients; the numeric
  // provider also evaluates the model at q_i +- h (numdiff.cpp:62-79).
  auto bad = [&](int j) {
    if (q[j] == 0.0) return true;
    if (!probes) return false;
    const double h = std::cbrt(2.220446049250313e-16) * std::max(1.0, std::fabs(q[j]));
    return q[j] + 1.0 * h == 0.0 || q[j] + -1.0 * h == 0.0;
  };
  if (P->model == ADC_MODEL_GPOLY) {
    if (bad(2)) return fail(ADC_E_EVAL, "division by zero");
  } else {
    for (int j = 2; j < P->np; j += 3)
      if (bad(j)) return fail(ADC_E_EVAL, "division by zero");
  }
  return ADC_OK;
}

bool numeric(const adc_chi2_plan* P) { return P->provider == ADC_PROVIDER_NUMERIC; }

Chi2Pass make_pass(const adc_chi2_plan* P) {
  Chi2Pass pass{};
  pass.counts = P->counts;
  pass.icounts = P->icounts - P->L.bin_begin;
  pass.qdev = P->qdev;
  pass.tile_ws = P->tile_ws;
  pass.lo = P->lo;
  pass.width = P->width;
  pass.bin_end = P->L.bin_end;
  pass.bpt = (int)(P->L.tile_bins / kTileThreads);
  pass.tile_begin = P->L.chunk_begin * P->L.chunk_tiles;
  pass.tile_end = (P->L.bin_end + P->L.tile_bins - 1) / P->L.tile_bins;
  if (pass.tile_end < pass.tile_begin) pass.tile_end = pass.tile_begin;
  pass.empty_idx = P->empty_idx;
  pass.empty_off = P->empty_off;
  pass.zws = P->zws;
  pass.side_stream = P->side;
  pass.ev_fork = P->ev_fork;
  pass.ev_join = P->ev_join;
  return pass;
}

int64_t local_chunks(const adc_chi2_plan* P) { return P->L.chunk_end - P->L.chunk_begin; }

bool sharded(const adc_chi2_plan* P) {
  return P->L.chunk_begin != 0 || P->L.chunk_end != P->L.nchunks;
}

int require_whole_or_comm(const adc_chi2_plan* P) {
  if (sharded(P) && P->comm == nullptr)
    return fail(ADC_E_ARG,
                "sharded plan: attach a communicator (adc_cuda_chi2_plan_set_comm) or use "
                "adc_cuda_chi2_partials + adc_chi2_finalize");
  return ADC_OK;
}

// ---- exchange -----------------------------------------------------------------
// A pass leaves nb blocks of records on the device, block b at
// dev + b * maxc * R, each holding this rank's local chunks (padded to maxc).
// collect_enqueue puts them (all ranks' for NCCL) into pinned host memory on
// stream s; after the stream is synchronised, collect_finish runs the host
// transport (if any) and compacts to P->full = [nb][nchunks][R] in global
// chunk order — the same bytes whatever the world size.
int collect_enqueue(adc_chi2_plan* P, const double* dev, int R, int nb, cudaStream_t s,
                    bool published = false) {
  const size_t count = (size_t)nb * P->maxc * R;
  if (count > P->xcount) return fail(ADC_E_ARG, "exchange staging too small");
  if (P->comm != nullptr && P->comm->kind == ADC_COMM_NCCL) {
    if (int rc = comm_allgather_enqueue(P->comm, dev, P->gather, count, s)) return rc;
    ADCB_CUDA(cudaMemcpyAsync(P->h_gather, P->gather, count * P->world * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
  } else if (P->comm != nullptr && P->comm->kind == ADC_COMM_PEER) {
    // publish into every rank's buffer over peer memory, signal, wait: no NCCL
    // (already done by the chunk kernel itself when `published`)
    if (!published)
      if (int rc = peer_exchange_enqueue(&P->peer, dev, count, s)) return rc;
    ADCB_CUDA(cudaMemcpyAsync(P->h_gather, P->peer.out, count * P->world * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
  } else {
    ADCB_CUDA(cudaMemcpyAsync(P->h_send, dev, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  return ADC_OK;
}

int collect_finish(adc_chi2_plan* P, int R, int nb, const double** out) {
  const size_t count = (size_t)nb * P->maxc * R;
  const double* src = P->h_gather;
  if (P->comm == nullptr) {
    src = P->h_send;  // world == 1: [nb][maxc = nchunks][R] is already compact
    *out = src;
    return ADC_OK;
  }
  if (P->comm->kind == ADC_COMM_HOST)
    if (int rc = comm_allgather_host(P->comm, P->h_send, P->h_gather, count)) return rc;
  const int64_t nchunks = P->L.nchunks;
  P->full.resize((size_t)nb * nchunks * R);
  for (int r = 0; r < P->world; ++r) {
    adc_chi2_layout Lr{};
    adc_chi2_make_layout(P->bins, P->world, r, &Lr);
    const int64_t nloc = Lr.chunk_end - Lr.chunk_begin;
    for (int b = 0; b < nb; ++b)
      std::memcpy(&P->full[((size_t)b * nchunks + Lr.chunk_begin) * R],
                  src + (size_t)r * count + (size_t)b * P->maxc * R, (size_t)nloc * R * sizeof(double));
  }
  *out = P->full.data();
  return ADC_OK;
}

// Once per plan: the linear parameters' q-independent G0/G1 chunk sums.
// Once per plan (and after adc_cuda_chi2_plan_refresh): everything that
// depends on the counts alone — ic = [c > 0]/c per bin, C0 and the linear
// parameters' G0/G1 per chunk.
void drop_graphs(adc_chi2_plan* P);

int ensure_lin(adc_chi2_plan* P, cudaStream_t s) {
  if (P->lin_ready) return ADC_OK;
  const int L = chi2_lin_count(P->model, P->np);
  const int64_t nrec = std::max<int64_t>(1, local_chunks(P));
  if (P->lin == nullptr)
    ADCB_CUDA(cudaMalloc(&P->lin, (size_t)nrec * (2 * L + 1) * sizeof(double)));
  if (int rc = chi2_lin_enqueue(make_pass(P), P->model, P->L.chunk_tiles, P->lin, P->icounts, s))
    return rc;
  // the empty-bin lists (ascending per chunk) for the passes' side pass
  if (P->empty_off == nullptr) {
    ADCB_CUDA(cudaMalloc(&P->empty_off, (size_t)(nrec + 1) * sizeof(int64_t)));
    ADCB_CUDA(cudaMalloc(&P->empty_cnt, ((size_t)nrec * kEmptySections + 1) * sizeof(int64_t)));
    ADCB_CUDA(cudaMalloc(&P->zws, (size_t)kMultiMax * P->maxc * kEmptySegs * (1 + kMaxNp) *
                                      sizeof(double)));
  }
  const int64_t nloc = local_chunks(P);
  // per (chunk, section) counts -> their exclusive prefix (the fill kernel's
  // bases, uploaded into empty_cnt) and the per-chunk offsets (empty_off)
  std::vector<int64_t> off((size_t)nloc + 1, 0);
  std::vector<int64_t> sec((size_t)nloc * kEmptySections + 1, 0);
  if (nloc > 0) {
    if (int rc = chi2_empty_count_enqueue(make_pass(P), P->L.chunk_tiles, P->empty_cnt, s))
      return rc;
    ADCB_CUDA(cudaMemcpyAsync(sec.data() + 1, P->empty_cnt,
                              (size_t)nloc * kEmptySections * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, s));
    ADCB_CUDA(cudaStreamSynchronize(s));
    for (size_t k = 1; k < sec.size(); ++k) sec[k] += sec[k - 1];
    for (int64_t c = 0; c <= nloc; ++c) off[c] = sec[(size_t)c * kEmptySections];
  }
  const int64_t total = std::max<int64_t>(1, off[nloc]);
  if (total > P->empty_cap) {  // (a refreshed histogram with more empty bins)
    if (P->empty_idx) {
      ADCB_CUDA(cudaStreamSynchronize(s));
      cudaFree(P->empty_idx);
      drop_graphs(P);  // captured passes hold the old list
      if (P->fit_graph) cudaGraphExecDestroy(P->fit_graph);
      P->fit_graph = nullptr;
    }
    P->empty_idx = nullptr;
    ADCB_CUDA(cudaMalloc(&P->empty_idx, (size_t)total * sizeof(int64_t)));
    P->empty_cap = total;
  }
  ADCB_CUDA(cudaMemcpyAsync(P->empty_off, off.data(), (size_t)(nloc + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
  if (nloc > 0) {
    ADCB_CUDA(cudaMemcpyAsync(P->empty_cnt, sec.data(), sec.size() * sizeof(int64_t),
                              cudaMemcpyHostToDevice, s));
    if (int rc = chi2_empty_fill_enqueue(make_pass(P), P->L.chunk_tiles, P->empty_cnt,
                                         P->empty_idx, s))
      return rc;
  }
  ADCB_CUDA(cudaStreamSynchronize(s));
  // counts per non-empty bin: C0 over this rank's chunks / non-empty bins
  if (!sharded(P) && nloc > 0) {
    std::vector<double> lin((size_t)nrec * (2 * L + 1));
    ADCB_CUDA(cudaMemcpy(lin.data(), P->lin, lin.size() * sizeof(double), cudaMemcpyDeviceToHost));
    double c0 = 0.0;
    for (int64_t c = 0; c < nloc; ++c) c0 += lin[(size_t)c * (2 * L + 1) + 2 * L];
    const double nonempty = (double)(P->L.bin_end - P->L.bin_begin) - (double)off[nloc];
    P->kappa = nonempty > 0 ? c0 / nonempty : 0.0;
    const bool resid = P->comm == nullptr && P->kappa > kResidKappa;
    if (resid && P->resid_a == nullptr) {
      ADCB_CUDA(cudaMalloc(&P->resid_a, kMultiMax * sizeof(double)));
      ADCB_CUDA(cudaMallocHost(&P->h_resid_a, kMultiMax * sizeof(double)));
      const size_t cnt = (size_t)kMultiMax * P->L.nchunks * kResidSegs;
      ADCB_CUDA(cudaMalloc(&P->resid_out, cnt * sizeof(double)));
      ADCB_CUDA(cudaMallocHost(&P->h_resid_out, cnt * sizeof(double)));
    }
    if (resid != P->resid) {
      P->resid = resid;
      drop_graphs(P);
      if (P->fit_graph) cudaGraphExecDestroy(P->fit_graph);
      P->fit_graph = nullptr;
    }
    // the residual pass evaluates m without the run recurrence: so do the
    // passes whose S it uses
    if (P->resid && P->fast == 2) P->fast = 1;
  }
  P->lin_ready = true;
  return ADC_OK;
}

// The sum over chunks of record entry v in adc_chi2_finalize's fixed
// pairwise tree (the same bits as the finalize's S when v = 0).
double chunk_tree_sum(const double* rec, int64_t nchunks, int R, int v) {
  std::vector<double> t((size_t)nchunks);
  for (int64_t c = 0; c < nchunks; ++c) t[c] = rec[c * R + v];
  for (int64_t s = 1; s < nchunks; s *= 2)
    for (int64_t i = 0; i + s < nchunks; i += 2 * s) t[i] = t[i] + t[i + s];
  return t[0];
}

// Residual chi2 values (K3r) of ncand parameter vectors already on the device
// (P->qdev for one, P->qmulti for a multi pass) given their S: sum (c-am)^2/c
// with a = E/S, reduced in fixed order (segments, then the chunk tree).
int resid_values(adc_chi2_plan* P, int ncand, const double* S, bool multi, double* chi2) {
  const int64_t nch = P->L.nchunks;  // whole-histogram plans only (resid)
  for (int k = 0; k < ncand; ++k) P->h_resid_a[k] = P->events / S[k];
  ADCB_CUDA(cudaMemcpyAsync(P->resid_a, P->h_resid_a, ncand * sizeof(double),
                            cudaMemcpyHostToDevice, P->stream));
  Chi2Pass pass = make_pass(P);
  if (multi) pass.qdev = P->qmulti;
  if (int rc = chi2_resid_enqueue(pass, P->model, P->np, P->fast, P->L.chunk_tiles, P->resid_a,
                                  ncand, multi, P->resid_out, P->stream))
    return rc;
  const size_t cnt = (size_t)ncand * nch * kResidSegs;
  ADCB_CUDA(cudaMemcpyAsync(P->h_resid_out, P->resid_out, cnt * sizeof(double),
                            cudaMemcpyDeviceToHost, P->stream));
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  std::vector<double> per((size_t)nch);
  for (int k = 0; k < ncand; ++k) {
    for (int64_t c = 0; c < nch; ++c) {
      const double* o = P->h_resid_out + ((size_t)k * nch + c) * kResidSegs;
      double v = o[0];
      for (int g = 1; g < kResidSegs; ++g) v = v + o[g];
      per[c] = v;
    }
    chi2[k] = chunk_tree_sum(per.data(), nch, 1, 0);
  }
  return ADC_OK;
}

// q upload + tile/chunk kernels + exchange / copy back, on P->stream.
int enqueue_pass(adc_chi2_plan* P, int grad) {
  ADCB_CUDA(cudaMemcpyAsync(P->qdev, P->h_q, qdev_bytes(), cudaMemcpyHostToDevice, P->stream));
  const int R = adc_chi2_record_len(P->np, grad);
  // peer transport: the chunk kernel publishes its records itself (fused
  // reduction + collective); a rank without chunks uses the exchange kernel
  const bool fuse = P->comm != nullptr && P->comm->kind == ADC_COMM_PEER && local_chunks(P) > 0;
  PeerPublish pub;
  if (fuse) pub = peer_publish_args(&P->peer, (size_t)P->maxc * R);
  if (int rc = chi2_enqueue(make_pass(P), P->model, P->np, grad != 0, P->fast,
                            P->L.chunk_tiles, P->records, P->stream, P->lin,
                            grad != 0 && numeric(P), fuse ? &pub : nullptr))
    return rc;
  return collect_enqueue(P, P->records, R, 1, P->stream, fuse);
}

int build_graph(adc_chi2_plan* P, int grad) {
  cudaGraph_t g = nullptr;
  ADCB_CUDA(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_pass(P, grad);
  cudaError_t e = cudaStreamEndCapture(P->stream, &g);
  if (rc != ADC_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&P->graph[grad ? 1 + numeric(P) : 0][P->fast], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  return ADC_OK;
}

void drop_graphs(adc_chi2_plan* P) {
  for (int g = 0; g < 3; ++g)
    for (int f = 0; f < 3; ++f) {
      if (P->graph[g][f]) cudaGraphExecDestroy(P->graph[g][f]);
      P->graph[g][f] = nullptr;
      P->warm[g][f] = false;
    }
}

// One pass (exchange included); returns the compacted records of all chunks.
// The first pass of a kind runs eagerly (NCCL sets up its buffers lazily,
// which must not happen under capture); later passes replay a CUDA graph.
int run_pass(adc_chi2_plan* P, const double* q, int grad, const double** rec) {
  if (int rc = require_whole_or_comm(P)) return rc;
  if (int rc = check_domain(P, q, grad && numeric(P))) return rc;
  ADCB_CUDA(cudaSetDevice(P->device));
  fill_qdev(P->model, P->np, q, P->h_q);
  if (int rc = ensure_lin(P, P->stream)) return rc;
  const int kind = grad ? 1 + numeric(P) : 0;
  if (!P->warm[kind][P->fast] || P->no_graph) {
    if (int rc = enqueue_pass(P, grad)) return rc;
    P->warm[kind][P->fast] = true;
  } else {
    if (P->graph[kind][P->fast] == nullptr) {
      if (int rc = build_graph(P, grad)) {
        // A transport that cannot be captured (an older NCCL) keeps working
        // with direct stream enqueues; anything else is an error.
        if (P->comm == nullptr || P->comm->kind != ADC_COMM_NCCL) return rc;
        cudaGetLastError();
        clear_error();
        P->no_graph = true;
        if (int rc2 = enqueue_pass(P, grad)) return rc2;
        ADCB_CUDA(cudaStreamSynchronize(P->stream));
        return collect_finish(P, adc_chi2_record_len(P->np, grad), 1, rec);
      }
    }
    ADCB_CUDA(cudaGraphLaunch(P->graph[kind][P->fast], P->stream));
  }
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  return collect_finish(P, adc_chi2_record_len(P->np, grad), 1, rec);
}

int alloc_staging(adc_chi2_plan* P) {
  if (P->h_send) cudaFreeHost(P->h_send);
  if (P->h_gather) cudaFreeHost(P->h_gather);
  if (P->gather) cudaFree(P->gather);
  P->h_send = P->h_gather = P->gather = nullptr;
  const size_t Rmax = (size_t)adc_chi2_record_len(P->np, 1);
  P->xcount = (size_t)P->maxc * std::max<size_t>(kMultiMax * Rmax, 1 + 3 * kMultiMax);
  const bool nccl = P->comm != nullptr && P->comm->kind == ADC_COMM_NCCL;
  ADCB_CUDA(cudaMallocHost(&P->h_send, P->xcount * sizeof(double)));
  ADCB_CUDA(cudaMallocHost(&P->h_gather, P->xcount * P->world * sizeof(double)));
  if (nccl) ADCB_CUDA(cudaMalloc(&P->gather, P->xcount * P->world * sizeof(double)));
  if (P->comm != nullptr && P->comm->kind == ADC_COMM_PEER) {
    if (int rc = peer_setup(P->comm, P->xcount, &P->peer)) return rc;
  } else {
    peer_release(&P->peer);
  }
  return ADC_OK;
}

}  // namespace

extern "C" int adc_cuda_chi2_plan_create(adc_chi2_plan** out, int32_t model, int32_t np,
                                         int64_t bins, double lo, double hi, double events,
                                         const double* counts, int32_t world, int32_t rank,
                                         void* stream) {
  clear_error();
  if (out == nullptr) return fail(ADC_E_ARG, "plan: null output");
  *out = nullptr;
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  if (model != ADC_MODEL_GSUM && model != ADC_MODEL_GPOLY) return fail(ADC_E_ARG, "unknown model");
  if (model == ADC_MODEL_GPOLY && np != 6) return fail(ADC_E_ARG, "gpoly has 6 parameters");
  if (model == ADC_MODEL_GSUM) {
    const int k = np / 3;
    if (np % 3 != 0 || !(k == 1 || k == 2 || k == 3 || k == 4 || k == 8))
      return fail(ADC_E_ARG, "gsum: parameter count must be 3K with K in {1,2,3,4,8}");
  }
  if (!(hi > lo)) return fail(ADC_E_EVAL, "degenerate histogram range");
  adc_chi2_plan* P = new (std::nothrow) adc_chi2_plan();
  if (P == nullptr) return fail(ADC_E_CUDA, "out of host memory");
  if (int rc = adc_chi2_make_layout(bins, world, rank, &P->L)) {
    delete P;
    return rc;
  }
  // A rank without bins (more ranks than chunks) never reads its counts: an
  // empty shard may come with a null pointer.
  if (counts == nullptr && P->L.bin_end > P->L.bin_begin) {
    delete P;
    return fail(ADC_E_ARG, "plan: null counts");
  }
  P->model = model;
  P->np = np;
  P->bins = bins;
  P->lo = lo;
  P->hi = hi;
  P->events = events;
  P->width = (hi - lo) / static_cast<double>(bins);  // Histogram::width (fit.hpp:30)
  P->counts = counts;
  P->world = world;
  P->rank = rank;
  P->maxc = std::max<int64_t>(1, (P->L.nchunks + world - 1) / world);
  P->bpt = bpt_for(bins);
  cudaGetDevice(&P->device);
  auto cleanup = [&](int rc) {
    adc_cuda_chi2_plan_destroy(P);
    return rc;
  };
  P->user_stream = static_cast<cudaStream_t>(stream);
  if (stream != nullptr) {
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaStreamSynchronize"));
  }
  const int64_t ntiles_local = std::max<int64_t>(
      1, (P->L.bin_end + P->L.tile_bins - 1) / P->L.tile_bins - P->L.chunk_begin * P->L.chunk_tiles);
  const int Rmax = adc_chi2_record_len(np, 1);
  cudaError_t e;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  // the pass stream at the highest priority, the side pass below it, so the
  // block scheduler fills SMs with tile CTAs first
  if ((e = cudaStreamCreateWithPriority(&P->stream, cudaStreamNonBlocking, prio_hi)) !=
          cudaSuccess ||
      (e = cudaStreamCreateWithPriority(&P->side, cudaStreamNonBlocking, prio_lo)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaMalloc(&P->qdev, qdev_bytes())) != cudaSuccess ||
      (e = cudaMalloc(&P->tile_ws, (size_t)ntiles_local * Rmax * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&P->records, (size_t)P->maxc * Rmax * sizeof(double))) != cudaSuccess ||
      (e = cudaMemset(P->records, 0, (size_t)P->maxc * Rmax * sizeof(double))) != cudaSuccess ||
      (e = cudaMallocHost(&P->h_q, qdev_bytes())) != cudaSuccess ||
      (e = cudaMalloc(&P->icounts, (size_t)std::max<int64_t>(1, P->L.bin_end - P->L.bin_begin) *
                                       sizeof(double))) != cudaSuccess)
    return cleanup(cuda_fail(e, "chi2 plan allocation"));
  if (int rc = alloc_staging(P)) return cleanup(rc);
  *out = P;
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_plan_create_sharded(adc_chi2_plan** out, int32_t model, int32_t np,
                                                 int64_t bins, double lo, double hi,
                                                 double events, const double* shard_counts,
                                                 adc_comm* comm, void* stream) {
  clear_error();
  if (out == nullptr) return fail(ADC_E_ARG, "plan: null output");
  *out = nullptr;
  if (comm == nullptr) return fail(ADC_E_ARG, "sharded plan: null communicator");
  adc_chi2_layout L{};
  if (int rc = adc_chi2_make_layout(bins, comm->world, comm->rank, &L)) return rc;
  if (shard_counts == nullptr && L.bin_end > L.bin_begin)
    return fail(ADC_E_ARG, "plan: null counts");
  // The kernels index counts by global bin number; the shard starts at bin_begin.
  const double* base = shard_counts == nullptr ? nullptr : shard_counts - L.bin_begin;
  if (int rc = adc_cuda_chi2_plan_create(out, model, np, bins, lo, hi, events, base, comm->world,
                                         comm->rank, stream))
    return rc;
  if (int rc = adc_cuda_chi2_plan_set_comm(*out, comm)) {
    adc_cuda_chi2_plan_destroy(*out);
    *out = nullptr;
    return rc;
  }
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_plan_set_comm(adc_chi2_plan* P, adc_comm* comm) {
  clear_error();
  if (P == nullptr) return fail(ADC_E_ARG, "null plan");
  if (comm != nullptr && (comm->world != P->world || comm->rank != P->rank))
    return fail(ADC_E_ARG, "communicator world/rank differ from the plan's");
  if (comm != nullptr && (comm->kind == ADC_COMM_NCCL || comm->kind == ADC_COMM_PEER) &&
      comm->device != P->device)
    return fail(ADC_E_ARG, "communicator is on another device than the plan");
  if (comm == nullptr && P->world > 1)
    return fail(ADC_E_ARG, "a sharded plan keeps its communicator");
  ADCB_CUDA(cudaSetDevice(P->device));
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  drop_graphs(P);
  P->comm = comm;
  return alloc_staging(P);
}

extern "C" int adc_cuda_chi2_plan_destroy(adc_chi2_plan* P) {
  if (P == nullptr) return ADC_OK;
  drop_graphs(P);
  if (P->qdev) cudaFree(P->qdev);
  if (P->tile_ws) cudaFree(P->tile_ws);
  if (P->records) cudaFree(P->records);
  if (P->h_q) cudaFreeHost(P->h_q);
  if (P->h_send) cudaFreeHost(P->h_send);
  if (P->h_gather) cudaFreeHost(P->h_gather);
  if (P->gather) cudaFree(P->gather);
  peer_release(&P->peer);
  if (P->qmulti) cudaFree(P->qmulti);
  if (P->h_qmulti) cudaFreeHost(P->h_qmulti);
  if (P->tile_ws_multi) cudaFree(P->tile_ws_multi);
  if (P->records_multi) cudaFree(P->records_multi);
  if (P->lin) cudaFree(P->lin);
  if (P->icounts) cudaFree(P->icounts);
  if (P->resid_a) cudaFree(P->resid_a);
  if (P->h_resid_a) cudaFreeHost(P->h_resid_a);
  if (P->resid_out) cudaFree(P->resid_out);
  if (P->h_resid_out) cudaFreeHost(P->h_resid_out);
  if (P->empty_idx) cudaFree(P->empty_idx);
  if (P->empty_off) cudaFree(P->empty_off);
  if (P->empty_cnt) cudaFree(P->empty_cnt);
  if (P->zws) cudaFree(P->zws);
  if (P->grad_multi_records) cudaFree(P->grad_multi_records);
  if (P->batch_ws) cudaFree(P->batch_ws);
  if (P->fit_graph) cudaGraphExecDestroy(P->fit_graph);
  if (P->fit_st) cudaFree(P->fit_st);
  if (P->h_fit_st) cudaFreeHost(P->h_fit_st);
  if (P->fit_scratch) cudaFree(P->fit_scratch);
  if (P->ncand_dev) cudaFree(P->ncand_dev);
  if (P->fit_trace) cudaFree(P->fit_trace);
  if (P->fit_full) cudaFree(P->fit_full);
  if (P->fit_rbegin) cudaFree(P->fit_rbegin);
  if (P->stream) cudaStreamDestroy(P->stream);
  if (P->side) cudaStreamDestroy(P->side);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join) cudaEventDestroy(P->ev_join);
  if (P->tk0) cudaEventDestroy(P->tk0);
  if (P->tk1) cudaEventDestroy(P->tk1);
  delete P;
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_plan_layout(const adc_chi2_plan* P, adc_chi2_layout* out) {
  clear_error();
  if (P == nullptr || out == nullptr) return fail(ADC_E_ARG, "null plan");
  *out = P->L;
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_set_precision(adc_chi2_plan* P, int32_t mode) {
  clear_error();
  if (P == nullptr || mode < 0 || mode > 2) return fail(ADC_E_ARG, "precision mode is 0, 1 or 2");
  P->fast = P->resid && mode == 2 ? 1 : mode;  // (residual-value plans: no run recurrence)
  if (P->fit_graph) {  // the device fit iteration graph holds the gradient pass
    cudaGraphExecDestroy(P->fit_graph);
    P->fit_graph = nullptr;
  }
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_plan_refresh(adc_chi2_plan* P) {
  clear_error();
  if (P == nullptr) return fail(ADC_E_ARG, "null plan");
  ADCB_CUDA(cudaSetDevice(P->device));
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  P->lin_ready = false;  // recomputed (1/c, C0, linear sums) before the next pass
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_set_provider(adc_chi2_plan* P, int32_t provider) {
  clear_error();
  if (P == nullptr || (provider != ADC_PROVIDER_AD_REVERSE && provider != ADC_PROVIDER_NUMERIC))
    return fail(ADC_E_ARG, "provider is ADC_PROVIDER_AD_REVERSE or ADC_PROVIDER_NUMERIC");
  P->provider = provider;
  return ADC_OK;
}

extern "C" double* adc_cuda_chi2_plan_records(adc_chi2_plan* P) {
  return P ? P->records : nullptr;
}

extern "C" int adc_cuda_chi2_partials(adc_chi2_plan* P, const double* q, int32_t want_grad,
                                      double* records_dev) {
  clear_error();
  if (P == nullptr || q == nullptr) return fail(ADC_E_ARG, "null argument");
  if (int rc = check_domain(P, q, want_grad && numeric(P))) return rc;
  ADCB_CUDA(cudaSetDevice(P->device));
  cudaStream_t s = P->user_stream;  // the caller's stream (0 = legacy default stream)
  // h_q may still be read by an in-flight copy of a previous pass
  ADCB_CUDA(cudaStreamSynchronize(s));
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  if (int rc = ensure_lin(P, s)) return rc;
  fill_qdev(P->model, P->np, q, P->h_q);
  ADCB_CUDA(cudaMemcpyAsync(P->qdev, P->h_q, qdev_bytes(), cudaMemcpyHostToDevice, s));
  Chi2Pass pass = make_pass(P);
  pass.tk0 = P->tk0;
  pass.tk1 = P->tk1;
  return chi2_enqueue(pass, P->model, P->np, want_grad != 0, P->fast,
                      P->L.chunk_tiles, records_dev ? records_dev : P->records, s, P->lin,
                      want_grad && numeric(P));
}

extern "C" int adc_cuda_chi2_value_mode(adc_chi2_plan* P, int32_t* residual, double* kappa) {
  clear_error();
  if (P == nullptr || residual == nullptr || kappa == nullptr) return fail(ADC_E_ARG, "null argument");
  ADCB_CUDA(cudaSetDevice(P->device));
  if (int rc = ensure_lin(P, P->stream)) return rc;
  *residual = P->resid ? 1 : 0;
  *kappa = P->kappa;
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_set_kernel_timing(adc_chi2_plan* P, int32_t on) {
  clear_error();
  if (P == nullptr) return fail(ADC_E_ARG, "null plan");
  ADCB_CUDA(cudaSetDevice(P->device));
  if (on && P->tk0 == nullptr) {
    ADCB_CUDA(cudaEventCreate(&P->tk0));
    ADCB_CUDA(cudaEventCreate(&P->tk1));
  } else if (!on && P->tk0 != nullptr) {
    cudaEventDestroy(P->tk0);
    cudaEventDestroy(P->tk1);
    P->tk0 = P->tk1 = nullptr;
  }
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_kernel_ms(adc_chi2_plan* P, float* ms) {
  clear_error();
  if (P == nullptr || ms == nullptr) return fail(ADC_E_ARG, "null argument");
  if (P->tk0 == nullptr) return fail(ADC_E_ARG, "kernel timing is off");
  ADCB_CUDA(cudaSetDevice(P->device));
  ADCB_CUDA(cudaEventSynchronize(P->tk1));
  ADCB_CUDA(cudaEventElapsedTime(ms, P->tk0, P->tk1));
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_gradient(adc_chi2_plan* P, const double* q, double* grad,
                                      double* chi2) {
  clear_error();
  if (P == nullptr || q == nullptr || grad == nullptr) return fail(ADC_E_ARG, "null argument");
  const double* rec = nullptr;
  if (int rc = run_pass(P, q, 1, &rec)) return rc;
  if (int rc = adc_chi2_finalize(P->np, P->events, rec, P->L.nchunks, 1, grad, chi2)) return rc;
  if (P->resid && chi2 != nullptr) {
    const double S = chunk_tree_sum(rec, P->L.nchunks, adc_chi2_record_len(P->np, 1), 0);
    return resid_values(P, 1, &S, false, chi2);
  }
  return ADC_OK;
}

extern "C" int adc_cuda_chi2(adc_chi2_plan* P, const double* q, double* chi2) {
  clear_error();
  if (P == nullptr || q == nullptr || chi2 == nullptr) return fail(ADC_E_ARG, "null argument");
  const double* rec = nullptr;
  if (int rc = run_pass(P, q, 0, &rec)) return rc;
  if (int rc = adc_chi2_finalize(P->np, P->events, rec, P->L.nchunks, 0, nullptr, chi2)) return rc;
  if (P->resid) {
    const double S = chunk_tree_sum(rec, P->L.nchunks, 4, 0);
    return resid_values(P, 1, &S, false, chi2);
  }
  return ADC_OK;
}

namespace {
int ensure_multi(adc_chi2_plan* P) {
  if (P->qmulti != nullptr) return ADC_OK;
  const size_t qb = qdev_bytes();
  const int Rm = 1 + 3 * kMultiMax;
  const int64_t ntiles_local = std::max<int64_t>(
      1, (P->L.bin_end + P->L.tile_bins - 1) / P->L.tile_bins - P->L.chunk_begin * P->L.chunk_tiles);
  ADCB_CUDA(cudaMalloc(&P->qmulti, qb * kMultiMax));
  ADCB_CUDA(cudaMallocHost(&P->h_qmulti, qb * kMultiMax));
  ADCB_CUDA(cudaMalloc(&P->tile_ws_multi, (size_t)ntiles_local * Rm * sizeof(double)));
  ADCB_CUDA(cudaMalloc(&P->records_multi, (size_t)P->maxc * Rm * sizeof(double)));
  ADCB_CUDA(cudaMemset(P->records_multi, 0, (size_t)P->maxc * Rm * sizeof(double)));
  return ADC_OK;
}

int64_t local_tiles(const adc_chi2_plan* P) {
  return std::max<int64_t>(
      1, (P->L.bin_end + P->L.tile_bins - 1) / P->L.tile_bins - P->L.chunk_begin * P->L.chunk_tiles);
}

// Up to kMultiMax gradient passes as ONE batched launch (blockIdx.y = member):
// member k reads the QDev row at qdev + k kQDoubles and leaves its chunk
// records at grad_multi_records + k maxc R — each identical to a single
// gradient pass (same tiles, same per-tile work, same trees).
int ensure_grad_batch(adc_chi2_plan* P) {  // outside any stream capture
  const int R = adc_chi2_record_len(P->np, 1);
  const size_t per = (size_t)P->maxc * R;
  if (P->grad_multi_records == nullptr) {
    ADCB_CUDA(cudaMalloc(&P->grad_multi_records, per * kMultiMax * sizeof(double)));
    ADCB_CUDA(cudaMemset(P->grad_multi_records, 0, per * kMultiMax * sizeof(double)));
  }
  if (P->batch_ws == nullptr)
    ADCB_CUDA(cudaMalloc(&P->batch_ws, (size_t)kMultiMax * local_tiles(P) * R * sizeof(double)));
  return ADC_OK;
}

int enqueue_grad_batch(adc_chi2_plan* P, const double* qdev, int nb, cudaStream_t s) {
  const int R = adc_chi2_record_len(P->np, 1);
  const size_t per = (size_t)P->maxc * R;
  if (P->grad_multi_records == nullptr || P->batch_ws == nullptr)
    return fail(ADC_E_ARG, "gradient batch buffers not allocated");
  Chi2Pass pass = make_pass(P);
  pass.qdev = qdev;
  pass.q_stride = kQDoubles;
  pass.tile_ws = P->batch_ws;
  pass.ws_stride = local_tiles(P) * R;
  return chi2_enqueue(pass, P->model, P->np, true, P->fast, P->L.chunk_tiles,
                      P->grad_multi_records, s, P->lin, numeric(P), nullptr, nb, (int64_t)per);
}
}  // namespace

extern "C" int adc_cuda_chi2_multi(adc_chi2_plan* P, const double* qs, int32_t ncand,
                                   double* chi2s) {
  clear_error();
  if (P == nullptr || qs == nullptr || chi2s == nullptr) return fail(ADC_E_ARG, "null argument");
  if (ncand < 1 || ncand > kMultiMax) return fail(ADC_E_ARG, "chi2 multi: 1..64 candidates");
  if (int rc = require_whole_or_comm(P)) return rc;
  for (int k = 0; k < ncand; ++k)
    if (int rc = check_domain(P, qs + (size_t)k * P->np)) return rc;
  ADCB_CUDA(cudaSetDevice(P->device));
  if (int rc = ensure_lin(P, P->stream)) return rc;
  if (int rc = ensure_multi(P)) return rc;
  const size_t qb = qdev_bytes();
  for (int k = 0; k < ncand; ++k)
    fill_qdev(P->model, P->np, qs + (size_t)k * P->np,
              reinterpret_cast<double*>(reinterpret_cast<char*>(P->h_qmulti) + k * qb));
  ADCB_CUDA(cudaMemcpyAsync(P->qmulti, P->h_qmulti, qb * ncand, cudaMemcpyHostToDevice, P->stream));
  Chi2Pass pass = make_pass(P);
  pass.qdev = P->qmulti;
  pass.tile_ws = P->tile_ws_multi;
  if (int rc = chi2_multi_enqueue(pass, P->model, P->np, ncand, P->L.chunk_tiles,
                                  P->records_multi, P->stream, P->lin, P->fast))
    return rc;
  const int R = 1 + 3 * ncand;
  if (int rc = collect_enqueue(P, P->records_multi, R, 1, P->stream)) return rc;
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  const double* rec = nullptr;
  if (int rc = collect_finish(P, R, 1, &rec)) return rc;
  ++P->multi_passes;
  // Per candidate: the same records a single value pass produces -> same finalize.
  std::vector<double> rec4((size_t)P->L.nchunks * 4);
  for (int k = 0; k < ncand; ++k) {
    for (int64_t c = 0; c < P->L.nchunks; ++c) {
      const double* r = rec + c * R;
      rec4[c * 4 + 0] = r[1 + 3 * k];
      rec4[c * 4 + 1] = r[2 + 3 * k];
      rec4[c * 4 + 2] = r[3 + 3 * k];
      rec4[c * 4 + 3] = r[0];
    }
    if (int rc = adc_chi2_finalize(P->np, P->events, rec4.data(), P->L.nchunks, 0, nullptr,
                                   chi2s + k))
      return rc;
  }
  if (P->resid) {
    std::vector<double> S((size_t)ncand);
    for (int k = 0; k < ncand; ++k) S[k] = chunk_tree_sum(rec, P->L.nchunks, R, 1 + 3 * k);
    return resid_values(P, ncand, S.data(), true, chi2s);
  }
  return ADC_OK;
}

extern "C" int adc_cuda_chi2_gradient_multi(adc_chi2_plan* P, const double* qs, int32_t ncand,
                                            double* grads) {
  clear_error();
  if (P == nullptr || qs == nullptr || grads == nullptr) return fail(ADC_E_ARG, "null argument");
  if (ncand < 1 || ncand > kMultiMax) return fail(ADC_E_ARG, "gradient multi: 1..64 candidates");
  if (int rc = require_whole_or_comm(P)) return rc;
  for (int k = 0; k < ncand; ++k)
    if (int rc = check_domain(P, qs + (size_t)k * P->np, numeric(P))) return rc;
  ADCB_CUDA(cudaSetDevice(P->device));
  if (int rc = ensure_lin(P, P->stream)) return rc;
  if (int rc = ensure_multi(P)) return rc;
  const size_t qb = qdev_bytes();
  const int R = adc_chi2_record_len(P->np, 1);
  for (int k = 0; k < ncand; ++k)
    fill_qdev(P->model, P->np, qs + (size_t)k * P->np,
              reinterpret_cast<double*>(reinterpret_cast<char*>(P->h_qmulti) + k * qb));
  ADCB_CUDA(cudaMemcpyAsync(P->qmulti, P->h_qmulti, qb * ncand, cudaMemcpyHostToDevice, P->stream));
  // ncand gradient passes as one batched launch (each member identical to
  // adc_cuda_chi2_gradient), one exchange / copy back and one synchronisation.
  if (int rc = ensure_grad_batch(P)) return rc;
  if (int rc = enqueue_grad_batch(P, P->qmulti, ncand, P->stream)) return rc;
  if (int rc = collect_enqueue(P, P->grad_multi_records, R, ncand, P->stream)) return rc;
  ADCB_CUDA(cudaStreamSynchronize(P->stream));
  const double* rec = nullptr;
  if (int rc = collect_finish(P, R, ncand, &rec)) return rc;
  for (int k = 0; k < ncand; ++k)
    if (int rc = adc_chi2_finalize(P->np, P->events, rec + (size_t)P->L.nchunks * R * k,
                                   P->L.nchunks, 1, grads + (size_t)k * P->np, nullptr))
      return rc;
  return ADC_OK;
}

// ---------------------------------------------------------------------------
// On-device histogram sampling (K6, chi2.cu).
extern "C" int adc_cuda_histogram_sample(int32_t model, int32_t np, const double* q, int64_t bins,
                                         double lo, double hi, double events, uint64_t seed,
                                         int64_t zero_every, double* counts, double* total,
                                         void* stream) {
  clear_error();
  if (q == nullptr || counts == nullptr) return fail(ADC_E_ARG, "null argument");
  if (bins <= 0) return fail(ADC_E_ARG, "histogram must have at least one bin");
  if (!(hi > lo)) return fail(ADC_E_EVAL, "degenerate histogram range");
  if (!(events > 0)) return fail(ADC_E_ARG, "events must be positive");
  if (model == ADC_MODEL_GPOLY ? np != 6 : (model != ADC_MODEL_GSUM || np % 3 != 0))
    return fail(ADC_E_ARG, "model / parameter count mismatch");
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<double> hq(qdev_bytes() / sizeof(double));
  fill_qdev(model, np, q, hq.data());
  double* qd = nullptr;
  double* ws = nullptr;
  const int64_t wsn = histogram_sample_ws_doubles(bins);
  ADCB_CUDA(ws_alloc((void**)&qd, qdev_bytes(), s));
  ADCB_CUDA(ws_alloc((void**)&ws, (size_t)wsn * sizeof(double), s));
  ADCB_CUDA(cudaMemcpyAsync(qd, hq.data(), qdev_bytes(), cudaMemcpyHostToDevice, s));
  int rc = histogram_sample_enqueue(model, np, qd, bins, lo, (hi - lo) / (double)bins, events,
                                    seed, zero_every, counts, ws, s);
  double tot = 0.0;
  if (rc == ADC_OK) {
    cudaError_t e = cudaMemcpyAsync(&tot, ws + wsn - 1, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "histogram sample");
  }
  cudaFreeAsync(qd, s);
  cudaFreeAsync(ws, s);
  if (rc == ADC_OK && total != nullptr) *total = tot;
  return rc;
}

// ---------------------------------------------------------------------------
// Fit loop: FitEngine::fit (fit.cpp:315-425), steepest descent with Armijo
// backtracking, generalised sigma clamp (fit.cpp:268-278 hard-codes every
// third index, which is only right for gsum), and the optional numeric-Hessian
// Newton step (fit.cpp:346-381, off by default).  On a sharded plan every rank
// runs this loop; the exchanged, fixed-order results are bitwise identical on
// all ranks, so every rank takes the same decisions and steps.
extern "C" void adc_fit_default_options(adc_fit_options* o) {
  o->budget = 400;
  o->grad_tol = 1e-6;
  o->chi2_rel_tol = 1e-12;
  o->sigma_min = 1e-3;
  o->armijo_c1 = 1e-4;
  o->trace_iterates = 0;
  o->use_hessian = 0;
  o->host_loop = 0;
}

namespace {
// (H + lambda I) d = g by Gaussian elimination with partial pivoting, the
// reference's damped solve (fit.cpp:282-311); false on a vanishing pivot.
bool damped_solve(std::vector<double> h, std::vector<double> g, double lambda, int n,
                  std::vector<double>& out) {
  for (int i = 0; i < n; ++i) h[(size_t)i * n + i] += lambda;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(h[(size_t)r * n + col]) > std::fabs(h[(size_t)piv * n + col])) piv = r;
    if (std::fabs(h[(size_t)piv * n + col]) < 1e-30) return false;
    if (piv != col) {
      for (int c = 0; c < n; ++c) std::swap(h[(size_t)piv * n + c], h[(size_t)col * n + c]);
      std::swap(g[piv], g[col]);
    }
    for (int r = col + 1; r < n; ++r) {
      const double f = h[(size_t)r * n + col] / h[(size_t)col * n + col];
      for (int c = col; c < n; ++c) h[(size_t)r * n + c] -= f * h[(size_t)col * n + c];
      g[r] -= f * g[col];
    }
  }
  out.assign(n, 0.0);
  for (int r = n - 1; r >= 0; --r) {
    double v = g[r];
    for (int c = r + 1; c < n; ++c) v -= h[(size_t)r * n + c] * out[c];
    out[r] = v / h[(size_t)r * n + r];
  }
  return true;
}
}  // namespace

namespace {
// Builds (once per plan and option set) the device-resident fit loop: ONE
// graph whose WHILE conditional node repeats the steepest-descent iteration
// body — QDev from the device parameters, the gradient pass, finalize +
// trials, the multi-candidate pass, selection, the loop bookkeeping — until
// the loop-control kernel clears the condition (converged, budget spent, or
// a line search that needs more trials than one batch).  No host round trip
// between iterations.
int build_fit_graph(adc_chi2_plan* P, const FitDevConst& c) {
  const int64_t nchunks = P->L.nchunks;
  const int Rmax = adc_chi2_record_len(P->np, 1);
  if (P->fit_st == nullptr) {
    ADCB_CUDA(cudaMalloc(&P->fit_st, sizeof(FitDevState)));
    ADCB_CUDA(cudaMallocHost(&P->h_fit_st, sizeof(FitDevState)));
    // finalize trees of the gradient, the 2 np Newton probes, the candidates
    const size_t scratch = std::max<size_t>((size_t)nchunks * Rmax * 2 * P->np,
                                            (size_t)kMultiMax * nchunks * 4);
    ADCB_CUDA(cudaMalloc(&P->fit_scratch, scratch * sizeof(double)));
    ADCB_CUDA(cudaMalloc(&P->ncand_dev, sizeof(int)));
  }
  const size_t per = (size_t)P->maxc * Rmax;
  if (c.newton)
    if (int rc = ensure_grad_batch(P)) return rc;
  // Sharded plan on the peer transport: every pass publishes its records to
  // all ranks over peer memory inside the loop body, and a compaction kernel
  // lays the exchanged blocks out as [nchunks][R] for the finalize kernels —
  // every rank runs the same loop on the same bits, no host in between.
  const bool peer = P->comm != nullptr && P->comm->kind == ADC_COMM_PEER;
  const int Rm = 1 + 3 * kMultiMax;
  if (peer && P->fit_full == nullptr) {
    const size_t full = std::max<size_t>((size_t)nchunks * Rmax * 2 * P->np, (size_t)nchunks * Rm);
    ADCB_CUDA(cudaMalloc(&P->fit_full, full * sizeof(double)));
    std::vector<int64_t> rb(P->world + 1);
    for (int r = 0; r < P->world; ++r) {
      adc_chi2_layout Lr{};
      adc_chi2_make_layout(P->bins, P->world, r, &Lr);
      rb[r] = Lr.chunk_begin;
    }
    rb[P->world] = nchunks;
    ADCB_CUDA(cudaMalloc(&P->fit_rbegin, rb.size() * sizeof(int64_t)));
    ADCB_CUDA(cudaMemcpy(P->fit_rbegin, rb.data(), rb.size() * sizeof(int64_t),
                         cudaMemcpyHostToDevice));
  }
  auto exchange = [&](const double* local, int nb, int R, bool published, const int* ndev,
                      cudaStream_t st) -> int {
    const size_t count = (size_t)nb * P->maxc * R;
    if (!published)
      if (int rc = peer_exchange_enqueue(&P->peer, local, count, st)) return rc;
    return fit_device_enqueue_compact(P->peer.out, count, P->world, P->fit_rbegin, nchunks, nb,
                                      P->maxc, R, ndev, P->fit_full, st);
  };
  if (P->fit_graph != nullptr && std::memcmp(&P->fit_const, &c, sizeof(c)) == 0) return ADC_OK;
  if (P->fit_graph) cudaGraphExecDestroy(P->fit_graph);
  P->fit_graph = nullptr;
  P->fit_const = c;
  if (int rc = ensure_lin(P, P->stream)) return rc;
  if (int rc = ensure_multi(P)) return rc;
  cudaStream_t s = P->stream;
  cudaGraph_t g = nullptr;
  ADCB_CUDA(cudaGraphCreate(&g, 0));
  auto fail_graph = [&](cudaError_t e, const char* what) {
    cudaGraphDestroy(g);
    return cuda_fail(e, what);
  };
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return fail_graph(e, "cudaGraphConditionalHandleCreate");
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = h;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  e = cudaGraphAddNode(&wnode, g, nullptr, 0, &wp);
  if (e != cudaSuccess) return fail_graph(e, "cudaGraphAddNode (while)");
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return fail_graph(e, "cudaStreamBeginCaptureToGraph (fit body)");
  int rc = fit_device_enqueue_qdev(P->fit_st, P->model, P->np, P->qdev,
                                   c.numeric ? c.cbrt_eps : 0.0, s);
  const bool fuse = peer && local_chunks(P) > 0;  // the chunk kernel publishes itself
  const double* grad_rec = peer ? P->fit_full : P->records;
  if (rc == ADC_OK) {
    PeerPublish pub;
    if (fuse) pub = peer_publish_args(&P->peer, (size_t)P->maxc * Rmax);
    rc = chi2_enqueue(make_pass(P), P->model, P->np, true, P->fast, P->L.chunk_tiles, P->records,
                      s, P->lin, numeric(P), fuse ? &pub : nullptr);
  }
  if (rc == ADC_OK && peer) rc = exchange(P->records, 1, Rmax, fuse, nullptr, s);
  if (rc == ADC_OK)
    rc = fit_device_enqueue_grad(P->fit_st, grad_rec, P->fit_scratch, nchunks, P->np, P->model,
                                 P->events, c, P->qmulti, P->ncand_dev, s);
  if (c.newton) {  // the 2 np probe gradient passes (one batch), Hessian + solve + trials
    if (rc == ADC_OK) rc = enqueue_grad_batch(P, P->qmulti, 2 * P->np, s);
    if (rc == ADC_OK && peer) rc = exchange(P->grad_multi_records, 2 * P->np, Rmax, false, nullptr, s);
    if (rc == ADC_OK)
      rc = fit_device_enqueue_newton(P->fit_st, peer ? P->fit_full : P->grad_multi_records,
                                     peer ? (size_t)nchunks * Rmax : per, P->fit_scratch, nchunks,
                                     P->np, P->model, P->events, c, P->qmulti, P->ncand_dev, s);
  }
  if (rc == ADC_OK) {
    Chi2Pass pass = make_pass(P);
    pass.qdev = P->qmulti;
    pass.tile_ws = P->tile_ws_multi;
    pass.ncand_dev = P->ncand_dev;
    rc = chi2_multi_enqueue(pass, P->model, P->np, kMultiMax, P->L.chunk_tiles, P->records_multi,
                            s, P->lin, P->fast);
  }
  if (rc == ADC_OK && peer) {
    // the multi records' stride is the device candidate count: exchange the
    // kMultiMax-sized block, compact with the device count
    const size_t count = (size_t)P->maxc * Rm;
    rc = peer_exchange_enqueue(&P->peer, P->records_multi, count, s);
    if (rc == ADC_OK)
      rc = fit_device_enqueue_compact(P->peer.out, count, P->world, P->fit_rbegin, nchunks, 1,
                                      P->maxc, Rm, P->ncand_dev, P->fit_full, s);
  }
  if (rc == ADC_OK)
    rc = fit_device_enqueue_accept(P->fit_st, peer ? P->fit_full : P->records_multi,
                                   P->fit_scratch, nchunks, P->events, c, s);
  if (rc == ADC_OK) rc = fit_device_enqueue_loop_ctl(P->fit_st, h, c, s);
  cudaGraph_t captured = nullptr;
  e = cudaStreamEndCapture(s, &captured);
  if (rc != ADC_OK) {
    cudaGraphDestroy(g);
    if (rc == ADC_E_CUDA) return fail(ADC_E_CUDA, "fit graph capture");
    return rc;
  }
  if (e != cudaSuccess) return fail_graph(e, "cudaStreamEndCapture (fit body)");
  e = cudaGraphInstantiate(&P->fit_graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate (fit loop)");
  return ADC_OK;
}
}  // namespace

extern "C" int adc_cuda_fit(adc_chi2_plan* P, double* params, const int32_t* clamp_idx,
                            int32_t nclamp, const adc_fit_options* opts, adc_fit_result* result,
                            double* iterates) {
  using clk = std::chrono::steady_clock;
  clear_error();
  if (P == nullptr || params == nullptr || opts == nullptr || result == nullptr)
    return fail(ADC_E_ARG, "null argument");
  const int np = P->np;
  auto clamp = [&](std::vector<double>& q) {
    int n = 0;
    for (int k = 0; k < nclamp; ++k) {
      const int i = clamp_idx[k];
      if (i >= 0 && i < np && q[i] < opts->sigma_min) {
        q[i] = opts->sigma_min;
        ++n;
      }
    }
    return n;
  };
  adc_fit_result res{};
  std::vector<double> q(params, params + np);
  res.sigma_clamps += clamp(q);
  int traced = 0;
  auto trace = [&](const std::vector<double>& v) {
    if (iterates != nullptr && traced < opts->trace_iterates) {
      std::memcpy(iterates + (size_t)traced * np, v.data(), np * sizeof(double));
      ++traced;
    }
  };
  double cur = 0.0;
  if (int rc = adc_cuda_chi2(P, q.data(), &cur)) return rc;
  ++res.chi2_evals;
  if (opts->trace_iterates > 0) trace(q);
  std::vector<double> g(np), trial(np);
  int first_batch = 32;  // line-search batch size, adapted per iteration
  // next batch = the last search's trial count + margin, in groups of 4 (the
  // multi pass's candidate group)
  const int margin = 4;
  // Device-resident loop (fit_device.cu): the fast passes on one device,
  // either gradient provider, steepest descent or the Newton option.
  // opts->host_loop keeps the host-driven loop (both give the same bits).
  const bool peer = P->comm != nullptr && P->comm->kind == ADC_COMM_PEER;
  // (residual-value plans keep the host loop: its value passes add K3r)
  const bool dev_mode = P->fast && (peer || (P->comm == nullptr && !sharded(P))) &&
                        nclamp <= kMaxNp && !opts->host_loop && !P->resid;
  if (dev_mode) {
    FitDevConst c{};
    c.grad_tol = opts->grad_tol;
    c.chi2_rel_tol = opts->chi2_rel_tol;
    c.sigma_min = opts->sigma_min;
    c.armijo_c1 = opts->armijo_c1;
    c.nclamp = nclamp;
    for (int k = 0; k < nclamp; ++k) c.clamp_idx[k] = clamp_idx[k];
    c.np = np;
    c.margin = margin;
    c.newton = opts->use_hessian ? 1 : 0;
    c.numeric = numeric(P) ? 1 : 0;  // part of the graph's key: the provider picks the kernel
    c.cbrt_eps = std::cbrt(2.220446049250313e-16);
    if (iterates != nullptr && opts->trace_iterates > 1) {
      if (P->fit_trace_cap < opts->trace_iterates) {
        if (P->fit_trace) cudaFree(P->fit_trace);
        P->fit_trace = nullptr;
        P->fit_trace_cap = 0;
        ADCB_CUDA(cudaMalloc(&P->fit_trace, (size_t)opts->trace_iterates * kMaxNp * sizeof(double)));
        P->fit_trace_cap = opts->trace_iterates;
      }
      c.trace = P->fit_trace;
      c.trace_cap = opts->trace_iterates;
    }
    if (int rc = build_fit_graph(P, c)) return rc;
    FitDevState& st = *P->h_fit_st;
    std::memset(&st, 0, sizeof(FitDevState));
    for (int i = 0; i < np; ++i) st.q[i] = q[i];
    st.cur = cur;
    st.first_batch = first_batch;
    st.budget = opts->budget;
    const uint64_t chi2_evals0 = res.chi2_evals;
    const int clamps0 = res.sigma_clamps;
    while (st.passes < st.budget) {
      // device loop: iterations until converged, budget spent or NeedHost
      ADCB_CUDA(cudaMemcpyAsync(P->fit_st, &st, sizeof(FitDevState), cudaMemcpyHostToDevice,
                                P->stream));
      ADCB_CUDA(cudaGraphLaunch(P->fit_graph, P->stream));
      ADCB_CUDA(cudaMemcpyAsync(&st, P->fit_st, sizeof(FitDevState), cudaMemcpyDeviceToHost,
                                P->stream));
      ADCB_CUDA(cudaStreamSynchronize(P->stream));
      q.assign(st.q, st.q + np);
      cur = st.cur;
      if (st.status == kFitConvergedGrad || st.status == kFitConvergedRelDec ||
          st.status == kFitConvergedNoStep) {
        res.converged = 1;
        break;
      }
      if (st.status != kFitNeedHost) break;  // running: the budget is spent
      // the first batch held no acceptable step: continue the same search
      // (t_next, t_next/2, ...) with host-driven batches, then hand the state
      // back to the device loop
      bool accepted = false;
      double next = cur;
      int tried = st.evals;
      std::vector<double> trials, tvals, c2s(kMultiMax);
      std::vector<int> cls;
      double t = st.t_next;
      while (t >= 1e-18 && !accepted) {
        trials.clear();
        tvals.clear();
        cls.clear();
        for (double tt = t; tt >= 1e-18 && (int)tvals.size() < kMultiMax; tt *= 0.5) {
          trial = q;
          const double* dir = c.newton ? st.dir : st.g;
          for (int i = 0; i < np; ++i) trial[i] -= tt * dir[i];
          cls.push_back(clamp(trial));
          trials.insert(trials.end(), trial.begin(), trial.end());
          tvals.push_back(tt);
        }
        if (tvals.empty()) break;
        if (int rc = adc_cuda_chi2_multi(P, trials.data(), (int32_t)tvals.size(), c2s.data()))
          return rc;
        for (size_t k = 0; k < tvals.size(); ++k) {
          ++st.evals_total;
          ++tried;
          if (c2s[k] <= cur - opts->armijo_c1 * tvals[k] * st.gd) {
            accepted = true;
            next = c2s[k];
            st.clamps_total += cls[k];
            trial.assign(trials.begin() + k * np, trials.begin() + (k + 1) * np);
            break;
          }
        }
        t = tvals.back() * 0.5;
      }
      if (!accepted) {
        res.converged = 1;
        break;
      }
      const double rel_dec = (cur - next) / std::max(1.0, std::fabs(cur));
      q = trial;
      cur = next;
      for (int i = 0; i < np; ++i) st.q[i] = q[i];
      st.cur = next;
      st.first_batch = std::min(kMultiMax, std::max(8, (tried + margin + 3) / 4 * 4));
      st.iters += 1;
      if (c.trace != nullptr && c.trace_cap > st.iters)
        ADCB_CUDA(cudaMemcpy(c.trace + (size_t)st.iters * np, q.data(), np * sizeof(double),
                             cudaMemcpyHostToDevice));
      if (rel_dec <= opts->chi2_rel_tol) {
        res.converged = 1;
        break;
      }
    }
    res.iterations = st.iters;
    res.gradient_evals = st.n_grad;
    res.gradient_ns = st.grad_ns;
    res.chi2_evals = chi2_evals0 + (uint64_t)st.evals_total;
    res.sigma_clamps = clamps0 + st.clamps_total;
    if (c.trace != nullptr) {
      const int rows = std::min(opts->trace_iterates, st.iters + 1);
      if (rows > 1)
        ADCB_CUDA(cudaMemcpy(iterates + np, c.trace + np, (size_t)(rows - 1) * np * sizeof(double),
                             cudaMemcpyDeviceToHost));
    }
    std::memcpy(params, q.data(), np * sizeof(double));
    res.chi2 = cur;
    *result = res;
    return ADC_OK;
  }
  for (int iter = 0; iter < opts->budget; ++iter) {
    auto t0 = clk::now();
    if (int rc = adc_cuda_chi2_gradient(P, q.data(), g.data(), nullptr)) return rc;
    res.gradient_ns += (uint64_t)std::chrono::nanoseconds(clk::now() - t0).count();
    ++res.gradient_evals;
    double gmax = 0.0;
    for (double v : g) gmax = std::max(gmax, std::fabs(v));
    if (gmax <= opts->grad_tol) {
      res.converged = 1;
      break;
    }
    std::vector<double> direction = g;
    if (opts->use_hessian) {
      // Central differences of the gradient, 2*np extra passes (fit.cpp:346-381).
      // All 2*np probes go to the device in one batch (adc_cuda_chi2_gradient_multi);
      // each probe's gradient is the one adc_cuda_chi2_gradient returns.
      std::vector<double> hess((size_t)np * np, 0.0), probes((size_t)2 * np * np),
          pg((size_t)2 * np * np), steps(np);
      for (int c = 0; c < np; ++c) {
        const double x = q[c];
        steps[c] = std::cbrt(2.220446049250313e-16) * std::max(1.0, std::fabs(x));
        for (int s2 = 0; s2 < 2; ++s2) {
          double* pr = &probes[(size_t)(2 * c + s2) * np];
          std::memcpy(pr, q.data(), np * sizeof(double));
          pr[c] = s2 == 0 ? x + steps[c] : x - steps[c];
        }
      }
      const auto h0 = clk::now();
      for (int b = 0; b < 2 * np; b += kMultiMax) {
        const int nb = std::min(kMultiMax, 2 * np - b);
        if (int rc = adc_cuda_chi2_gradient_multi(P, &probes[(size_t)b * np], nb,
                                                  &pg[(size_t)b * np]))
          return rc;
      }
      res.gradient_ns += (uint64_t)std::chrono::nanoseconds(clk::now() - h0).count();
      res.gradient_evals += 2 * np;
      for (int c = 0; c < np; ++c)
        for (int r = 0; r < np; ++r)
          hess[(size_t)r * np + c] =
              (pg[(size_t)(2 * c) * np + r] - pg[(size_t)(2 * c + 1) * np + r]) / (2.0 * steps[c]);
      double lambda = 0.0;
      bool ok = false;
      for (int attempt = 0; attempt < 10 && !ok; ++attempt) {
        ok = damped_solve(hess, g, lambda, np, direction);
        if (ok) {
          double descent = 0.0;
          for (int i = 0; i < np; ++i) descent += g[i] * direction[i];
          ok = descent > 0.0;
        }
        lambda = lambda == 0.0 ? 1e-6 : lambda * 10.0;
      }
      if (!ok) direction = g;  // steepest descent
    }
    double gd = 0.0;
    for (int i = 0; i < np; ++i) gd += g[i] * direction[i];
    double t = 1.0, next = 0.0;
    bool accepted = false;
    if (P->fast) {
      // Batched Armijo: the trials t = 1, 1/2, 1/4, ... of the sequential
      // search (fit.cpp:390-403) evaluated in batches, one pass each; the
      // first accepted one is taken, so the iterate is the same as the
      // sequential search's (each candidate's chi2 is bit-identical to a
      // single value pass).  The first batch of an iteration is sized from
      // the previous iteration's accepted trial (+8), so a typical search is
      // one pass; later batches take kMultiMax.
      std::vector<double> trials, tvals, c2s(kMultiMax);
      std::vector<int> cls;
      int want = first_batch, tried = 0;
      while (t >= 1e-18 && !accepted) {
        trials.clear();
        tvals.clear();
        cls.clear();
        for (double tt = t; tt >= 1e-18 && (int)tvals.size() < want; tt *= 0.5) {
          trial = q;
          for (int i = 0; i < np; ++i) trial[i] -= tt * direction[i];
          cls.push_back(clamp(trial));
          trials.insert(trials.end(), trial.begin(), trial.end());
          tvals.push_back(tt);
        }
        if (tvals.empty()) break;
        if (int rc = adc_cuda_chi2_multi(P, trials.data(), (int32_t)tvals.size(), c2s.data()))
          return rc;
        for (size_t k = 0; k < tvals.size(); ++k) {
          ++res.chi2_evals;
          ++tried;
          if (c2s[k] <= cur - opts->armijo_c1 * tvals[k] * gd) {
            accepted = true;
            next = c2s[k];
            res.sigma_clamps += cls[k];
            trial.assign(trials.begin() + k * np, trials.begin() + (k + 1) * np);
            break;
          }
        }
        t = tvals.back() * 0.5;
        want = kMultiMax;
      }
      if (accepted) first_batch = std::min(kMultiMax, std::max(8, (tried + margin + 3) / 4 * 4));
    } else {
      while (t >= 1e-18) {
        trial = q;
        for (int i = 0; i < np; ++i) trial[i] -= t * direction[i];
        const int cl = clamp(trial);
        double c2 = 0.0;
        if (int rc = adc_cuda_chi2(P, trial.data(), &c2)) return rc;
        ++res.chi2_evals;
        if (c2 <= cur - opts->armijo_c1 * t * gd) {
          accepted = true;
          next = c2;
          res.sigma_clamps += cl;
          break;
        }
        t *= 0.5;
      }
    }
    if (!accepted) {
      res.converged = 1;
      break;
    }
    const double rel_dec = (cur - next) / std::max(1.0, std::fabs(cur));
    q = trial;
    cur = next;
    ++res.iterations;
    if (opts->trace_iterates > res.iterations) trace(q);
    if (rel_dec <= opts->chi2_rel_tol) {
      res.converged = 1;
      break;
    }
  }
  std::memcpy(params, q.data(), np * sizeof(double));
  res.chi2 = cur;
  *result = res;
  return ADC_OK;
}

// ---- histogram ingest format (include/adc_cuda.h) ---------------------------------
namespace {
constexpr char kHistMagic[8] = {'A', 'D', 'C', 'H', 'I', 'S', 'T', '1'};
constexpr size_t kHistHeader = 8 + 8 + 3 * 8;
constexpr size_t kHistPiece = size_t(64) << 20;  // bytes per bounce-buffer piece

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

extern "C" int adc_histogram_write(const char* path, int64_t bins, double lo, double hi,
                                   double events, const double* counts) {
  clear_error();
  if (path == nullptr || counts == nullptr || bins <= 0) return fail(ADC_E_ARG, "histogram write: bad argument");
  FILE* f = std::fopen(path, "wb");
  if (f == nullptr) return fail(ADC_E_ARG, std::string("histogram write: cannot open ") + path);
  bool ok = std::fwrite(kHistMagic, 1, 8, f) == 8 && std::fwrite(&bins, 8, 1, f) == 1 &&
            std::fwrite(&lo, 8, 1, f) == 1 && std::fwrite(&hi, 8, 1, f) == 1 &&
            std::fwrite(&events, 8, 1, f) == 1;
  if (ok && !is_device_ptr(counts)) {
    ok = std::fwrite(counts, 8, (size_t)bins, f) == (size_t)bins;
  } else if (ok) {
    double* bounce = nullptr;
    if (cudaMallocHost(&bounce, kHistPiece) != cudaSuccess) {
      std::fclose(f);
      return cuda_fail(cudaGetLastError(), "histogram write: pinned buffer");
    }
    const size_t per = kHistPiece / 8;
    for (int64_t o = 0; ok && o < bins; o += (int64_t)per) {
      const size_t n = (size_t)std::min<int64_t>((int64_t)per, bins - o);
      ok = cudaMemcpy(bounce, counts + o, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess &&
           std::fwrite(bounce, 8, n, f) == n;
    }
    cudaFreeHost(bounce);
  }
  ok = std::fclose(f) == 0 && ok;
  return ok ? ADC_OK : fail(ADC_E_ARG, std::string("histogram write failed: ") + path);
}

extern "C" int adc_histogram_read_header(const char* path, int64_t* bins, double* lo, double* hi,
                                         double* events) {
  clear_error();
  if (path == nullptr || bins == nullptr || lo == nullptr || hi == nullptr || events == nullptr)
    return fail(ADC_E_ARG, "null argument");
  FILE* f = std::fopen(path, "rb");
  if (f == nullptr) return fail(ADC_E_ARG, std::string("histogram read: cannot open ") + path);
  char magic[8];
  const bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kHistMagic, 8) == 0 &&
                  std::fread(bins, 8, 1, f) == 1 && std::fread(lo, 8, 1, f) == 1 &&
                  std::fread(hi, 8, 1, f) == 1 && std::fread(events, 8, 1, f) == 1 && *bins > 0;
  std::fclose(f);
  return ok ? ADC_OK : fail(ADC_E_ARG, std::string("not an ADCHIST1 histogram file: ") + path);
}

extern "C" int adc_histogram_read_counts(const char* path, int64_t bins, double* counts) {
  clear_error();
  if (counts == nullptr) return fail(ADC_E_ARG, "null argument");
  int64_t fb = 0;
  double lo, hi, ev;
  if (int rc = adc_histogram_read_header(path, &fb, &lo, &hi, &ev)) return rc;
  if (fb != bins)
    return fail(ADC_E_ARG, "histogram read: file has " + std::to_string(fb) + " bins, not " +
                               std::to_string(bins));
  FILE* f = std::fopen(path, "rb");
  if (f == nullptr || std::fseek(f, (long)kHistHeader, SEEK_SET) != 0) {
    if (f) std::fclose(f);
    return fail(ADC_E_ARG, std::string("histogram read: cannot open ") + path);
  }
  bool ok = true;
  if (!is_device_ptr(counts)) {
    ok = std::fread(counts, 8, (size_t)bins, f) == (size_t)bins;
  } else {
    // two pinned pieces: the file read of one overlaps the H2D copy of the other
    double* bounce[2] = {nullptr, nullptr};
    cudaStream_t s = nullptr;
    if (cudaMallocHost(&bounce[0], kHistPiece) != cudaSuccess ||
        cudaMallocHost(&bounce[1], kHistPiece) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      if (bounce[0]) cudaFreeHost(bounce[0]);
      if (bounce[1]) cudaFreeHost(bounce[1]);
      std::fclose(f);
      return cuda_fail(cudaGetLastError(), "histogram read: pinned buffers");
    }
    cudaEvent_t done[2];
    cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
    const size_t per = kHistPiece / 8;
    int k = 0;
    for (int64_t o = 0; ok && o < bins; o += (int64_t)per, k ^= 1) {
      const size_t n = (size_t)std::min<int64_t>((int64_t)per, bins - o);
      ok = cudaEventSynchronize(done[k]) == cudaSuccess && std::fread(bounce[k], 8, n, f) == n &&
           cudaMemcpyAsync(counts + o, bounce[k], n * 8, cudaMemcpyHostToDevice, s) == cudaSuccess &&
           cudaEventRecord(done[k], s) == cudaSuccess;
    }
    ok = cudaStreamSynchronize(s) == cudaSuccess && ok;
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    cudaStreamDestroy(s);
    cudaFreeHost(bounce[0]);
    cudaFreeHost(bounce[1]);
  }
  std::fclose(f);
  return ok ? ADC_OK : fail(ADC_E_ARG, std::string("histogram read: short or unreadable file ") + path);
}
