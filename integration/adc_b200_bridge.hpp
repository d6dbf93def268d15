// adc_b200_bridge.hpp — the REFERENCE-SIDE binding: what a maintainer of the
// reference `adc` (arxiv/paper_2203_06139 artifact) adds so its own call sites
// run the hot path on a B200 through include/adc_cuda.h.  It is written against
// the reference's public headers (proj/include/adc/*.hpp) and is compiled here
// only by oracle/Makefile for the integration test (tests/test_bridge.py);
// INTEGRATION.md shows where it plugs in.
#pragma once

#include <string>

#include "adc/fit.hpp"
#include "adc/launch.hpp"

namespace adc::b200_bridge {

/// Same signature and contract as adc::launch (proj/include/adc/launch.hpp:66-67,
/// proj/src/launch.cpp:252-346).  Validation, the race_check refusal and buffer
/// binding are the reference's own.  A Listing-1 kernel calling a registered
/// generated gradient (printed-text fingerprint) runs its hand-written sm_100a
/// kernel; any other global kernel of the Program is lowered to CUDA by the
/// engine's generic JIT (adc_jit_*, NVRTC).  Either way it runs on the GPU —
/// there is no interpreter fallback; a module the JIT cannot lower throws.
/// LaunchStats.counts come from one interpreted active and idle thread, exact
/// for kernels whose op counts do not depend on the data.
LaunchStats launch(const Program& p, const std::string& kernel, const LaunchConfig& cfg,
                   BufferSet& buffers, const LaunchOptions& opts = {});

/// The FitEngine model source (fit.cpp:125-138 kModelSource); its generated
/// gradient is fingerprinted against the B200 registry before any pass.
void set_model_source(const std::string& source);

/// FitEngine::chi2_gradient / chi2 (fit.cpp:206-259) for the reference model
/// (gsum, fit.cpp:125-138) with the histogram on the GPU.  The model's
/// generated gradient text is checked against the B200 registry first; the
/// provider is the caller's (AdReverse: the generated gradient; Numeric:
/// central differences of the model, numdiff.cpp:38-87).
void chi2_gradient(const FitEngine& engine, const Histogram& h, const std::vector<double>& q,
                   std::vector<double>& out,
                   GradientProvider provider = GradientProvider::AdReverse);
double chi2(const FitEngine& engine, const Histogram& h, const std::vector<double>& q);

/// FitEngine::fit (fit.cpp:315-425) with every pass on the GPU (adc_cuda_fit:
/// batched Armijo trials, batched Hessian probes), the sigma clamp of
/// fit.cpp:268-278 and the reference's op-count metadata (one interpreted
/// model / model-gradient call at the middle bin, fit.cpp:324-325).
FitResult fit(const FitEngine& engine, const Histogram& h, GradientProvider provider,
              std::vector<double> init, const FitOptions& opts = {});

/// bench_scaling (fit.cpp:427-458), the paper's Fig. 2b: for each K, the
/// reference's own histogram (sample_histogram, default_truth, perturbed_init)
/// fitted with both providers on the GPU; same rows, so bench_csv /
/// bench_plot_table apply unchanged.
std::vector<BenchRow> bench_scaling(const BenchConfig& cfg);

}  // namespace adc::b200_bridge
