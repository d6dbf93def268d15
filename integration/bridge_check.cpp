// bridge_check — integration test of the reference-side binding
// (integration/adc_b200_bridge.cpp): the unmodified reference library
// (oracle/_ref/libadc.a) and its own public API, with adc::launch and
// FitEngine::chi2_gradient routed to the B200 through include/adc_cuda.h.
// Built by oracle/Makefile; run by tests/test_bridge.py.
//   bridge_check cpu   — error-contract checks that need no GPU
//   bridge_check gpu   — parity of the bridged calls against the reference's
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "adc/fit.hpp"
#include "adc/launch.hpp"
#include "adc/parser.hpp"
#include "adc/tooling.hpp"
#include "adc_b200_bridge.hpp"
#include "adc_cuda.h"
#include "corpus_embed.inc"

using namespace adc;

static int failures = 0;
#define EXPECT(cond, what)                                 \
  do {                                                     \
    if (!(cond)) {                                         \
      std::printf("FAIL %s\n", what);                      \
      ++failures;                                          \
    } else {                                               \
      std::printf("ok   %s\n", what);                      \
    }                                                      \
  } while (0)

static Program kernels_program() {
  Module m = parse_or_throw(kKernelsDsl);
  ensure_called_derivatives(m);
  return Program(std::move(m));
}

template <class F>
static std::string error_of(F&& f, ErrorKind* kind = nullptr) {
  try {
    f();
  } catch (const Error& e) {
    if (kind) *kind = e.kind();
    return e.what();
  }
  return "";
}

static double rel(double a, double b) {
  double s = std::max(std::fabs(a), std::fabs(b));
  return s == 0 ? 0 : std::fabs(a - b) / s;
}

static void cpu_checks(const Program& p, bool gpu) {
  // Refusal and binding errors are the reference's own, before any device use.
  BufferSet b;
  b.arrays["x"] = std::vector<double>(64, 0.5);
  b.arrays["p"] = std::vector<double>(64, 0.0);
  b.scalars["sigma"] = 1.0;
  b.arrays["dx"] = std::vector<double>(64, 0.0);
  b.arrays["dp"] = std::vector<double>(64, 0.0);
  b.arrays["dsigma"] = std::vector<double>(1, 0.0);
  ErrorKind k1{}, k2{};
  std::string r = error_of([&] { adc::launch(p, "compute_shared", {1, 64, 64}, b); }, &k1);
  std::string g = error_of([&] { b200_bridge::launch(p, "compute_shared", {1, 64, 64}, b); }, &k2);
  EXPECT(!r.empty() && r == g && k1 == k2 && k1 == ErrorKind::Launch,
         "hazardous compute_shared refused with the reference's message");
  BufferSet s = b;
  s.arrays["x"].resize(10);
  EXPECT(error_of([&] { adc::launch(p, "compute", {3, 256, 512}, s); }) ==
             error_of([&] { b200_bridge::launch(p, "compute", {3, 256, 512}, s); }),
         "short buffer: same message");
  s.arrays.erase("x");
  EXPECT(error_of([&] { b200_bridge::launch(p, "compute", {3, 256, 512}, s); }) ==
             "missing buffer 'x'",
         "missing buffer: same message");
  EXPECT(error_of([&] { b200_bridge::launch(p, "compute", {0, 256, 512}, b); }) ==
             error_of([&] { adc::launch(p, "compute", {0, 256, 512}, b); }),
         "bad LaunchConfig: same message");
  if (gpu)
    EXPECT(error_of([&] { b200_bridge::launch(p, "noop", {1, 1, 1}, b); }).empty(),
           "non-registered kernel (noop) runs through the JIT");
  else {
    int sms = 0, major = 0, minor = 0;
    const bool have_device = adc_cuda_device_info(&sms, &major, &minor) == 0;
    const std::string e = error_of([&] { b200_bridge::launch(p, "noop", {1, 1, 1}, b); });
    if (have_device)  // `cpu` mode on a GPU machine: the JIT simply runs it
      EXPECT(e.empty(), "non-registered kernel goes to the JIT (device present)");
    else
      EXPECT(e.find("no CUDA device") != std::string::npos,
             "non-registered kernel goes to the JIT: no device -> Error, no interpreter fallback");
  }
}

static void gpu_checks(const Program& p) {
  for (int64_t n : {512, 1000003}) {
    std::mt19937_64 rng(n == 512 ? 0x5EED : 7);
    std::vector<double> x(n), px(n), d0(n), e0(n);
    for (int64_t i = 0; i < n; ++i) {
      x[i] = std::uniform_real_distribution<double>(-3, 3)(rng);
      px[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
      d0[i] = n == 512 ? 0.0 : std::uniform_real_distribution<double>(-1, 1)(rng);
      e0[i] = n == 512 ? 0.0 : std::uniform_real_distribution<double>(-1, 1)(rng);
    }
    BufferSet ref, gpu;
    for (BufferSet* b : {&ref, &gpu}) {
      b->arrays["x"] = x;
      b->arrays["p"] = px;
      b->scalars["sigma"] = 1.3;
      b->arrays["dx"] = d0;
      b->arrays["dp"] = e0;
    }
    LaunchConfig cfg{n / 256 + 1, 256, n};
    LaunchStats rs = adc::launch(p, "compute", cfg, ref);
    LaunchStats gs = b200_bridge::launch(p, "compute", cfg, gpu);
    double worst = 0;
    size_t same = 0;
    for (int64_t i = 0; i < n; ++i) {
      for (const char* a : {"dx", "dp"}) {
        double r = ref.arrays[a][i], g = gpu.arrays[a][i];
        double scale = std::max({std::fabs(r), std::fabs(g), std::fabs(a[1] == 'x' ? d0[i] : e0[i])});
        worst = std::max(worst, scale == 0 ? 0 : std::fabs(r - g) / scale);
        same += r == g;
      }
    }
    std::printf("     n=%lld worst rel %.3g, bit-identical %.4f\n", (long long)n, worst,
                double(same) / (2.0 * n));
    EXPECT(worst <= 1e-12, "bridged launch matches adc::launch within 1e-12");
    EXPECT(rs.thread_statements == gs.thread_statements, "LaunchStats.thread_statements equal");
    EXPECT(rs.counts == gs.counts, "LaunchStats.counts (op counters) equal");
  }
  // compute_shared forced: the reference's sequential run vs the B200's
  // fixed-order reduction (test_launch.cpp:148-165 precedent: 1e-9).
  {
    const int64_t n = 100003;
    std::mt19937_64 rng(99);
    BufferSet ref, gpu;
    std::vector<double> x(n), px(n);
    for (int64_t i = 0; i < n; ++i) {
      x[i] = std::uniform_real_distribution<double>(-3, 3)(rng);
      px[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
    }
    for (BufferSet* b : {&ref, &gpu}) {
      b->arrays["x"] = x;
      b->arrays["p"] = px;
      b->scalars["sigma"] = 1.1;
      b->arrays["dx"] = std::vector<double>(n, 0.0);
      b->arrays["dp"] = std::vector<double>(n, 0.0);
      b->arrays["dsigma"] = std::vector<double>(1, 0.5);
    }
    LaunchOptions forced;
    forced.unsafe = true;
    forced.sequential = true;
    LaunchConfig cfg{n / 256 + 1, 256, n};
    LaunchStats rs = adc::launch(p, "compute_shared", cfg, ref, forced);
    LaunchStats gs = b200_bridge::launch(p, "compute_shared", cfg, gpu, forced);
    double worst = 0;
    for (int64_t i = 0; i < n; ++i)
      worst = std::max({worst, rel(ref.arrays["dx"][i], gpu.arrays["dx"][i]),
                        rel(ref.arrays["dp"][i], gpu.arrays["dp"][i])});
    const double ds = rel(ref.arrays["dsigma"][0], gpu.arrays["dsigma"][0]);
    std::printf("     compute_shared: dx/dp worst rel %.3g, dsigma rel %.3g\n", worst, ds);
    EXPECT(worst <= 1e-12 && ds <= 1e-9, "bridged forced compute_shared matches the reference");
    EXPECT(rs.counts == gs.counts, "compute_shared LaunchStats.counts equal");
  }
  // Generic JIT path through the bridge: corpus gradients the registry does
  // not hold, same inputs through adc::launch (sequential) and the bridge.
  {
    Module jm = parse_or_throw(kJitModuleDsl);
    ensure_called_derivatives(jm);
    Program jp(std::move(jm));
    for (const char* kern : {"k_rational", "k_branchy", "k_looped"}) {
      const int64_t n = 20001;
      std::mt19937_64 rng(5);
      BufferSet ref, gpu;
      std::vector<double> x(n), y(n);
      for (int64_t i = 0; i < n; ++i) {
        x[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
        y[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
      }
      for (BufferSet* b : {&ref, &gpu}) {
        b->arrays["x"] = x;
        b->arrays["dx"] = std::vector<double>(n, 0.0);
        if (std::string(kern) == "k_looped") {
          b->integers["n"] = 12;
        } else {
          b->arrays["y"] = y;
          b->arrays["dy"] = std::vector<double>(n, 0.0);
        }
      }
      LaunchOptions seq;
      seq.sequential = true;
      LaunchConfig cfg{n / 256 + 1, 256, n};
      LaunchStats rs = adc::launch(jp, kern, cfg, ref, seq);
      LaunchStats gs = b200_bridge::launch(jp, kern, cfg, gpu);
      double worst = 0;
      for (const auto& kv : ref.arrays)
        for (int64_t i = 0; i < n; ++i)
          worst = std::max(worst, rel(kv.second[i], gpu.arrays[kv.first][i]));
      std::printf("     JIT %s: worst rel %.3g\n", kern, worst);
      EXPECT(worst <= 1e-12, "bridged JIT launch matches adc::launch");
      EXPECT(rs.thread_statements == gs.thread_statements, "JIT LaunchStats.thread_statements");
      std::printf("     JIT %s: counts adds %llu/%llu muls %llu/%llu divs %llu/%llu pushes %llu/%llu\n",
                  kern, (unsigned long long)rs.counts.adds, (unsigned long long)gs.counts.adds,
                  (unsigned long long)rs.counts.muls, (unsigned long long)gs.counts.muls,
                  (unsigned long long)rs.counts.divs, (unsigned long long)gs.counts.divs,
                  (unsigned long long)rs.counts.tape_pushes,
                  (unsigned long long)gs.counts.tape_pushes);
      EXPECT(rs.counts == gs.counts, "JIT LaunchStats.counts (exact, data-dependent kernels too)");
    }
  }
  // FitEngine::fit through the bridge vs the reference's own fit (both providers).
  {
    b200_bridge::set_model_source(kGsumDsl);
    FitEngine eng;
    std::vector<double> truth = gauss_sum::default_truth(2, -5, 5);
    Histogram h = sample_histogram(truth, 200000, 1200, -5, 5, 11);
    std::vector<double> init = gauss_sum::perturbed_init(truth);
    FitOptions fo;
    fo.budget = 30;
    fo.trace_iterates = 8;
    for (GradientProvider prov : {GradientProvider::AdReverse, GradientProvider::Numeric}) {
      FitResult rr = eng.fit(h, prov, init, fo);
      FitResult gr = b200_bridge::fit(eng, h, prov, init, fo);
      double worst = 0;
      for (size_t k = 0; k < std::min(rr.iterates.size(), gr.iterates.size()); ++k)
        for (size_t i = 0; i < init.size(); ++i)
          worst = std::max(worst, rel(rr.iterates[k][i], gr.iterates[k][i]));
      std::printf("     fit %s: iterations %d/%d, chi2 rel %.3g, iterates worst rel %.3g\n",
                  provider_name(prov), rr.iterations, gr.iterations, rel(rr.chi2, gr.chi2), worst);
      const double tol = prov == GradientProvider::AdReverse ? 1e-9 : 1e-5;
      EXPECT(rr.iterations == gr.iterations && rr.iterates.size() == gr.iterates.size() &&
                 worst <= tol && rel(rr.chi2, gr.chi2) <= 1e-6 &&
                 rr.primal_call_counts == gr.primal_call_counts &&
                 rr.gradient_call_counts == gr.gradient_call_counts,
             "bridged FitEngine::fit matches the reference fit (iterates, counts)");
    }
    BenchConfig bc;
    bc.k_list = {1, 2};
    bc.bins = 2000;
    bc.events = 100000;
    bc.fit.budget = 20;
    std::vector<BenchRow> rows = b200_bridge::bench_scaling(bc);
    std::printf("%s", bench_csv(rows).c_str());
    EXPECT(rows.size() == 4 && rows[0].grad_evals > 0, "bridged bench_scaling produces the rows");
  }
  // FitEngine (gsum K=1, 2) chi2 and gradient on the GPU vs the reference engine.
  b200_bridge::set_model_source(kGsumDsl);
  FitEngine eng;
  for (int k : {1, 2}) {
    std::vector<double> truth = gauss_sum::default_truth(k, -5, 5);
    Histogram h = sample_histogram(truth, 100000, 1000, -5, 5, 42 + k);
    std::vector<double> q = gauss_sum::perturbed_init(truth);
    std::vector<double> gr, gg;
    eng.chi2_gradient(h, q, GradientProvider::AdReverse, gr);
    b200_bridge::chi2_gradient(eng, h, q, gg);
    double gmax = 0, worst = 0;
    for (double v : gr) gmax = std::max(gmax, std::fabs(v));
    for (size_t i = 0; i < q.size(); ++i) worst = std::max(worst, std::fabs(gr[i] - gg[i]) / gmax);
    double cr = eng.chi2(h, q), cg = b200_bridge::chi2(eng, h, q);
    std::printf("     gsum K=%d: gradient worst |diff|/max|g| %.3g, chi2 rel %.3g\n", k, worst,
                rel(cr, cg));
    EXPECT(worst <= 1e-11 && rel(cr, cg) <= 1e-12, "bridged FitEngine chi2/gradient match");
    // GradientProvider::Numeric through the bridge vs the reference's numeric provider
    std::vector<double> nr, ng;
    eng.chi2_gradient(h, q, GradientProvider::Numeric, nr);
    b200_bridge::chi2_gradient(eng, h, q, ng, GradientProvider::Numeric);
    double nw = 0;
    for (size_t i = 0; i < q.size(); ++i) nw = std::max(nw, std::fabs(nr[i] - ng[i]) / gmax);
    std::printf("     gsum K=%d numeric provider: worst |diff|/max|g| %.3g\n", k, nw);
    EXPECT(nw <= 1e-8, "bridged FitEngine numeric-provider gradient matches");
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  Program p = kernels_program();
  try {
    cpu_checks(p, mode == "gpu");
    if (mode == "gpu") gpu_checks(p);
  } catch (const Error& e) {
    std::printf("FAIL unexpected adc::Error: %s\n", e.what());
    ++failures;
  }
  std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
  return failures == 0 ? 0 : 1;
}
