// C++ mirror (include/adcx/adc_b200.hpp) check: compiles against the header,
// links libadc_b200.so, exercises the reference-shaped API.
//   cxx_api_check cpu — error contract without a GPU (no CPU fallback)
//   cxx_api_check gpu — Listing-1 launch, batched N-dim, FitEngine vs the C oracle
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>

#include "adcx/adc_b200.hpp"
#include "restate.h"

using namespace adc::b200;
static int failures = 0;
#define EXPECT(c, w)                   \
  do {                                 \
    std::printf("%s %s\n", (c) ? "ok  " : "FAIL", w); \
    if (!(c)) ++failures;              \
  } while (0)

template <class F>
static std::string err(F&& f, ErrorKind* k = nullptr) {
  try {
    f();
  } catch (const Error& e) {
    if (k) *k = e.kind();
    return e.what();
  }
  return "";
}

static double relmax(const std::vector<double>& a, const std::vector<double>& b) {
  double w = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    double s = std::max(std::fabs(a[i]), std::fabs(b[i]));
    if (s > 0) w = std::max(w, std::fabs(a[i] - b[i]) / s);
  }
  return w;
}

// Host all-gather between threads of one process (two ranks sharing one GPU).
struct ThreadGather {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, gen = 0;
  std::vector<std::vector<char>> slot;
  explicit ThreadGather(int w) : world(w), slot(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
struct RankCtx {
  ThreadGather* g;
  int rank;
};
static int thread_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  auto* c = static_cast<RankCtx*>(ctx);
  {
    std::lock_guard<std::mutex> lk(c->g->mu);
    c->g->slot[c->rank].assign(static_cast<const char*>(send), static_cast<const char*>(send) + bytes);
  }
  c->g->barrier();
  for (int r = 0; r < c->g->world; ++r)
    std::memcpy(static_cast<char*>(recv) + r * bytes, c->g->slot[r].data(), bytes);
  c->g->barrier();
  return 0;
}

int main(int argc, char** argv) {
  // "gpu-launch": the launch paths only (for compute-sanitizer's racecheck /
  // synccheck, which do not follow the fit's device-side graph loop)
  const bool launch_only = argc > 1 && std::string(argv[1]) == "gpu-launch";
  const bool gpu = argc > 1 && (std::string(argv[1]) == "gpu" || launch_only);
  BufferSet b;
  b.arrays["x"] = std::vector<double>(512, 0.5);
  b.arrays["p"] = std::vector<double>(512, 0.0);
  b.arrays["dx"] = std::vector<double>(512, 0.0);
  b.arrays["dp"] = std::vector<double>(512, 0.0);
  b.scalars["sigma"] = 1.3;
  ErrorKind k{};
  EXPECT(err([&] { launch("compute", {1, 256, 512}, b); }, &k) ==
                 "grid 1 x block 256 does not cover problem size 512" && k == ErrorKind::Launch,
         "LaunchConfig::validate message");
  EXPECT(err([&] { launch("compute_shared", {1, 64, 64}, b); }).find("launch refused") == 0,
         "hazard refusal");
  if (!gpu) {
    EXPECT(err([&] { launch("compute", {3, 256, 512}, b); }, &k).find("no CUDA device") !=
                   std::string::npos && k == ErrorKind::Cuda,
           "no GPU: Error(Cuda), no CPU fallback");
  } else {
    // Listing 1 at n = 512 (acceptance.cpp:160-211 analog) vs the oracle.
    const int64_t n = 100003;
    std::mt19937_64 rng(0x5EED);
    BufferSet h;
    for (const char* a : {"x", "p", "dx", "dp"}) h.arrays[a].resize(n);
    for (int64_t i = 0; i < n; ++i) {
      h.arrays["x"][i] = std::uniform_real_distribution<double>(-3, 3)(rng);
      h.arrays["p"][i] = std::uniform_real_distribution<double>(-2, 2)(rng);
    }
    h.scalars["sigma"] = 1.3;
    std::vector<double> ox(n, 0.0), op(n, 0.0);
    rs_gauss_grad_batch(h.arrays["x"].data(), h.arrays["p"].data(), 1.3, ox.data(), op.data(), n);
    LaunchStats st = launch("compute", {n / 256 + 1, 256, n}, h);
    EXPECT(relmax(h.arrays["dx"], ox) <= 1e-12 && relmax(h.arrays["dp"], op) <= 1e-12,
           "launch(compute) matches the oracle within 1e-12");
    EXPECT(st.thread_statements.size() == size_t((n / 256 + 1) * 256) &&
               st.thread_statements[0] == 3 && st.thread_statements.back() == 2,
           "LaunchStats shape");
    // Batched N-dim.
    const int64_t dim = 37, m = 1001;
    std::vector<double> X(dim * m), P(dim * m), DX(dim * m, 0.0), DP(dim * m, 0.0);
    for (auto& v : P) v = std::uniform_real_distribution<double>(-2, 2)(rng);
    for (size_t i = 0; i < X.size(); ++i) X[i] = P[i] + 0.1 * std::normal_distribution<double>()(rng);
    std::vector<double> RX(dim * m, 0.0), RP(dim * m, 0.0);
    rs_gaussnd_grad_batch(X.data(), P.data(), 1.3, dim, m, m, RX.data(), RP.data());
    launch_batch_gaussnd(m, dim, X, P, 1.3, DX, DP);
    EXPECT(relmax(DX, RX) <= 1e-12 && relmax(DP, RP) <= 1e-12, "launch_batch_gaussnd matches");
    // Thread safety (the reference's launch is safe from several threads on
    // distinct buffer sets): 4 threads, each its own buffers,
    // each calling the host pipeline 3 times (the per-device staging lock
    // serialises them) and the multi-GPU form; every thread's result is
    // bit-identical to the sequential one.
    {
      const int T = 4;
      std::vector<std::vector<double>> tdx(T, std::vector<double>(dim * m, 0.0)),
          tdp(T, std::vector<double>(dim * m, 0.0));
      std::vector<double> sdx(dim * m, 0.0), sdp(dim * m, 0.0);
      for (int k = 0; k < 3; ++k) launch_batch_gaussnd(m, dim, X, P, 1.3, sdx, sdp);
      launch_batch_gaussnd(m, dim, X, P, 1.3, sdx, sdp, std::vector<int32_t>{0});
      std::vector<std::string> terr(T);
      std::vector<std::thread> tt;
      for (int t = 0; t < T; ++t)
        tt.emplace_back([&, t] {
          try {
            for (int k = 0; k < 3; ++k) launch_batch_gaussnd(m, dim, X, P, 1.3, tdx[t], tdp[t]);
            launch_batch_gaussnd(m, dim, X, P, 1.3, tdx[t], tdp[t], std::vector<int32_t>{0});
          } catch (const std::exception& ex) {
            terr[t] = ex.what();
          }
        });
      for (auto& t : tt) t.join();
      bool same = true;
      for (int t = 0; t < T; ++t)
        same = same && terr[t].empty() &&
               std::memcmp(tdx[t].data(), sdx.data(), sdx.size() * sizeof(double)) == 0 &&
               std::memcmp(tdp[t].data(), sdp.data(), sdp.size() * sizeof(double)) == 0;
      EXPECT(same, "4 threads on distinct buffers: bitwise equal to the sequential calls");
      ErrorKind ek{};
      EXPECT(err([&] { launch_batch_gaussnd(m, dim, X, P, 1.3, sdx, sdp,
                                            std::vector<int32_t>{0, 0}); }, &ek)
                     .find("device listed twice") != std::string::npos && ek == ErrorKind::Arg,
             "multi-GPU form: a device listed twice is Error(Arg)");
      EXPECT(err([&] { launch_batch_gaussnd(m, dim, X, P, 1.3, sdx, sdp,
                                            std::vector<int32_t>{0, 4096}); })
                     .find("does not exist") != std::string::npos,
             "multi-GPU form: a missing device is refused");
    }
    if (launch_only) {
      std::printf("%d failure(s)\n", failures);
      return failures ? 1 : 0;
    }
    // FitEngine gsum K=1 over a 4000-bin histogram vs the compensated oracle.
    Histogram hist;
    hist.bins = 4000;
    hist.lo = -5;
    hist.hi = 5;
    hist.counts.resize(hist.bins);
    double tot = 0;
    for (int j = 0; j < hist.bins; ++j) {
      double x = hist.center(j);
      hist.counts[j] = j % 100 == 0 ? 0.0 : std::round(200 * std::exp(-0.5 * x * x / 2.25));
      tot += hist.counts[j];
    }
    hist.events = (uint64_t)tot;
    std::vector<double> q = {0.8, 0.3, 1.2}, g, ref(3), scale(3);
    FitEngine eng("gsum", 3);
    eng.chi2_gradient(hist, q, g);
    rs_chi2_gradient_compensated(RS_MODEL_GSUM, hist.counts.data(), hist.bins, -5, 5, tot,
                                 q.data(), 3, ref.data(), scale.data());
    bool okg = true;
    for (int i = 0; i < 3; ++i) okg = okg && std::fabs(g[i] - ref[i]) <= 1e-12 * scale[i];
    EXPECT(okg, "FitEngine::chi2_gradient within 1e-12 * sum|terms|");
    const double c0 = eng.chi2(hist, q);
    FitResult r = eng.fit(hist, q, FitOptions{});
    std::printf("     fit: %d iterations, chi2 %.6g -> %.6g, mu %.4f sigma %.4f\n", r.iterations, c0,
                r.chi2, r.params[1], r.params[2]);
    EXPECT(r.chi2 < c0 && std::fabs(r.params[1]) < 0.05 && std::fabs(r.params[2] - 1.5) < 0.05,
           "FitEngine::fit recovers mu and sigma (test_fit.cpp:81-93 bounds)");

    // Multi-GPU API: a 3-chunk gpoly histogram sharded over 2 ranks (threads
    // sharing this GPU, host transport) and over NCCL at world size 1: the
    // gradient and the whole fit are bitwise those of the single engine.
    Histogram big;
    big.bins = 3 * (1 << 20) + 77;
    big.lo = -5;
    big.hi = 5;
    big.counts.resize(big.bins);
    double tb = 0;
    for (int j = 0; j < big.bins; ++j) {
      const double x = big.center(j);
      big.counts[j] = j % 100 == 0 ? 0.0 : std::round(150 * std::exp(-0.5 * x * x / 2.25) + 20 - x);
      tb += big.counts[j];
    }
    big.events = (uint64_t)tb;
    const std::vector<double> qp = {120.0, 0.3, 1.2, 25.0, -0.5, 0.01};
    FitOptions fo;
    fo.budget = 8;
    std::vector<double> g1;
    FitEngine single("gpoly", 6);
    single.chi2_gradient(big, qp, g1);
    const FitResult f1 = single.fit(big, qp, fo);
    ThreadGather tg(2);
    std::vector<std::vector<double>> gr(2);
    std::vector<FitResult> fr(2);
    std::vector<std::string> errs(2);
    std::vector<std::thread> th;
    for (int rank = 0; rank < 2; ++rank)
      th.emplace_back([&, rank] {
        try {
          RankCtx ctx{&tg, rank};
          Comm comm = Comm::host(2, rank, thread_allgather, &ctx);
          FitEngine e("gpoly", 6, &comm);
          e.chi2_gradient(big, qp, gr[rank]);
          fr[rank] = e.fit(big, qp, fo);
        } catch (const std::exception& ex) {
          errs[rank] = ex.what();
        }
      });
    for (auto& t : th) t.join();
    bool same = errs[0].empty() && errs[1].empty();
    for (int rank = 0; rank < 2 && same; ++rank)
      same = std::memcmp(gr[rank].data(), g1.data(), 6 * sizeof(double)) == 0 &&
             std::memcmp(fr[rank].params.data(), f1.params.data(), 6 * sizeof(double)) == 0 &&
             fr[rank].iterations == f1.iterations && fr[rank].chi2 == f1.chi2;
    if (!errs[0].empty()) std::printf("     rank 0: %s\n", errs[0].c_str());
    EXPECT(same, "2 ranks (host transport): gradient and fit bitwise equal to one engine");
    std::string nerr;
    std::vector<double> gn;
    try {
      Comm nc = Comm::nccl(1, 0, Comm::unique_id());
      FitEngine e("gpoly", 6, &nc);
      e.chi2_gradient(big, qp, gn);
      e.chi2_gradient(big, qp, gn);  // graph replay with the NCCL all-gather inside
    } catch (const std::exception& ex) {
      nerr = ex.what();
    }
    if (!nerr.empty()) std::printf("     nccl: %s\n", nerr.c_str());
    EXPECT(nerr.empty() && std::memcmp(gn.data(), g1.data(), 6 * sizeof(double)) == 0,
           "NCCL communicator (world 1): gradient bitwise equal to one engine");
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
