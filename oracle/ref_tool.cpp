// ref_tool — TEST INFRASTRUCTURE (oracle).  Drives the UNMODIFIED reference
// library (oracle/_ref/libadc.a, built from /root/reference/proj/src by
// oracle/Makefile) through its own public API to
//   * print the generated gradients the B200 kernels transcribe,
//   * produce golden input/output vectors for the parity tests,
//   * time the reference CPU path on the host cores (bench.py --impl reference
//     and the cpu_baseline leg).
// Only tests/, __graft_entry__.smoke() and bench.py's reference legs run it.
//
// Binary I/O: raw little-endian float64 arrays, concatenated, sizes given on
// the command line.  Timing and summaries are printed as one JSON line.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "adc/eval.hpp"
#include "adc/fit.hpp"
#include "adc/launch.hpp"
#include "adc/numdiff.hpp"
#include "adc/parser.hpp"
#include "adc/printer.hpp"
#include "adc/tooling.hpp"
#include "adc/transform.hpp"

#include "corpus_embed.inc"

using namespace adc;
using clk = std::chrono::steady_clock;

namespace {

[[noreturn]] void die(const std::string& m) {
  std::fprintf(stderr, "ref_tool: %s\n", m.c_str());
  std::exit(2);
}

std::vector<double> read_f64(const std::string& path, size_t count) {
  std::ifstream in(path, std::ios::binary);
  if (!in) die("cannot open " + path);
  std::vector<double> v(count);
  in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(count * 8));
  if (static_cast<size_t>(in.gcount()) != count * 8) die("short read from " + path);
  return v;
}

void write_f64(std::ofstream& out, const std::vector<double>& v) {
  out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// Module holding the named DSL plus every derivative its calls reference
// (tooling.cpp:103-119), exactly as the CLI's load_and_derive does.
Module load_named(const std::string& name) {
  const char* src = nullptr;
  if (name == "kernels") src = kKernelsDsl;
  else if (name == "gsum") src = kGsumDsl;
  else if (name == "gaussnd") src = kGaussndDsl;
  else if (name == "gpoly") src = kGpolyDsl;
  else die("unknown module " + name);
  Module m = parse_or_throw(src);
  ensure_called_derivatives(m);
  return m;
}

// Adds `<fn>_grad...` for the requested parameters (reverse.cpp:703-725).
std::string add_gradient(Module& m, const std::string& fn, const std::vector<std::string>& wrt) {
  const FunctionDef* f = m.find(fn);
  if (f == nullptr) die("no function " + fn);
  std::string name = gradient_name(*f, wrt);
  if (m.find(name) == nullptr) {
    AdjointProgram g = differentiate_gradient(*f, wrt);
    m.functions.push_back(std::move(g.derived));
  }
  return name;
}

unsigned default_workers() {
  unsigned w = std::thread::hardware_concurrency();
  return w == 0 ? 1 : w;
}

// ---------------------------------------------------------------------------
// print <module> <fn> <wrt...>   — the generated gradient text.
int cmd_print(int argc, char** argv) {
  if (argc < 4) die("print <module> <fn> <wrt...>");
  Module m = load_named(argv[1]);
  std::vector<std::string> wrt(argv + 3, argv + argc);
  std::string name = add_gradient(m, argv[2], wrt);
  std::cout << print(*m.find(name));
  return 0;
}

// golden-check — the printed gauss_grad_0_1 must equal the reference's frozen
// golden text (proj/tests/golden/gauss_grad_0_1.golden, compared byte-for-byte
// as test_reverse.cpp:62-67 does).
int cmd_golden_check(int, char**) {
  Module m = load_named("kernels");
  const FunctionDef* g = m.find("gauss_grad_0_1");
  if (g == nullptr) die("gauss_grad_0_1 not derived");
  std::string text = print(*g);
  bool ok = text == std::string(kGaussGradGolden);
  std::printf("{\"golden_match\": %s}\n", ok ? "true" : "false");
  return ok ? 0 : 1;
}


// ---------------------------------------------------------------------------
// gauss1d <n> <seed> <sigma> <block> <out.bin> [workers]
//   Criterion-5 style fixture (acceptance.cpp:160-211): x~U(-3,3), p~U(-2,2)
//   drawn from mt19937_64(seed) through uniform_real_distribution in the same
//   order as PointSampler (support.hpp:36-43); runs adc::launch(prog,"compute",
//   {n/block+1, block, n}) and the plain sequential Program::eval loop.
//   Writes x, p, dx, dp.
int cmd_gauss1d(int argc, char** argv) {
  if (argc < 6) die("gauss1d <n> <seed> <sigma> <block> <out> [workers]");
  const int64_t n = std::atoll(argv[1]);
  const uint64_t seed = std::strtoull(argv[2], nullptr, 0);
  const double sigma = std::atof(argv[3]);
  const int64_t block = std::atoll(argv[4]);
  const unsigned workers = argc > 6 ? static_cast<unsigned>(std::atoi(argv[6])) : 0;
  std::mt19937_64 rng(seed);
  std::vector<double> x(n), px(n);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = std::uniform_real_distribution<double>(-3, 3)(rng);
    px[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
  }
  Program prog(load_named("kernels"));
  LaunchConfig cfg{n / block + 1, block, n};
  std::vector<double> dx_seq(n, 0.0), dp_seq(n, 0.0);
  {
    ArgPack args;
    args.add_array(x).add_array(px).add_real(sigma).add_array(dx_seq).add_array(dp_seq);
    for (int64_t g = 0; g < cfg.grid_dim * cfg.block_dim; ++g) {
      EvalOptions o;
      o.has_thread_ctx = true;
      o.block_idx = g / cfg.block_dim;
      o.block_dim = cfg.block_dim;
      o.thread_idx = g % cfg.block_dim;
      o.problem_n = n;
      prog.eval("compute", args, o);
    }
  }
  BufferSet b;
  b.arrays["x"] = x;
  b.arrays["p"] = px;
  b.scalars["sigma"] = sigma;
  b.arrays["dx"] = std::vector<double>(n, 0.0);
  b.arrays["dp"] = std::vector<double>(n, 0.0);
  LaunchOptions lo;
  lo.workers = workers;
  auto t0 = clk::now();
  LaunchStats st = launch(prog, "compute", cfg, b, lo);
  double sec = secs(t0, clk::now());
  int64_t active = 0, idle = 0;
  for (uint32_t c : st.thread_statements) (c == 3 ? active : idle) += 1;
  bool same = b.arrays["dx"] == dx_seq && b.arrays["dp"] == dp_seq;
  std::ofstream out(argv[5], std::ios::binary);
  write_f64(out, x);
  write_f64(out, px);
  write_f64(out, b.arrays["dx"]);
  write_f64(out, b.arrays["dp"]);
  std::printf("{\"n\": %lld, \"grid\": %lld, \"block\": %lld, \"active\": %lld, \"idle\": %lld, "
              "\"launch_equals_sequential\": %s, \"seconds\": %.6f, \"workers\": %u}\n",
              (long long)n, (long long)cfg.grid_dim, (long long)block, (long long)active,
              (long long)idle, same ? "true" : "false", sec,
              workers ? workers : default_workers());
  return same ? 0 : 1;
}

// gauss1d-in <n> <sigma> <block> <in.bin> <out.bin> [workers] [repeats]
//   in = x, p, dx0, dp0 (n each); out = dx, dp after one adc::launch.
//   Used for parity at arbitrary sizes and as the timed reference arm.
int cmd_gauss1d_in(int argc, char** argv) {
  if (argc < 6) die("gauss1d-in <n> <sigma> <block> <in> <out> [workers] [repeats]");
  const int64_t n = std::atoll(argv[1]);
  const double sigma = std::atof(argv[2]);
  const int64_t block = std::atoll(argv[3]);
  const unsigned workers = argc > 6 ? static_cast<unsigned>(std::atoi(argv[6])) : 0;
  const int repeats = argc > 7 ? std::max(1, std::atoi(argv[7])) : 1;
  std::vector<double> all = read_f64(argv[4], static_cast<size_t>(4 * n));
  Program prog(load_named("kernels"));
  LaunchConfig cfg{n / block + 1, block, n};
  BufferSet b;
  b.arrays["x"].assign(all.begin(), all.begin() + n);
  b.arrays["p"].assign(all.begin() + n, all.begin() + 2 * n);
  b.scalars["sigma"] = sigma;
  LaunchOptions lo;
  lo.workers = workers;
  std::vector<double> times;
  for (int r = 0; r < repeats; ++r) {
    b.arrays["dx"].assign(all.begin() + 2 * n, all.begin() + 3 * n);
    b.arrays["dp"].assign(all.begin() + 3 * n, all.begin() + 4 * n);
    auto t0 = clk::now();
    launch(prog, "compute", cfg, b, lo);
    times.push_back(secs(t0, clk::now()));
  }
  std::ofstream out(argv[5], std::ios::binary);
  write_f64(out, b.arrays["dx"]);
  write_f64(out, b.arrays["dp"]);
  std::sort(times.begin(), times.end());
  std::printf("{\"n\": %lld, \"seconds_median\": %.6f, \"seconds_min\": %.6f, \"workers\": %u}\n",
              (long long)n, times[times.size() / 2], times[0], workers ? workers : default_workers());
  return 0;
}

// gauss-shared-in <n> <sigma> <block> <in.bin> <out.bin>
//   Listing-1's hazardous twin `compute_shared` (kernels.dsl:16-21): every
//   thread accumulates into the one-element slot dsigma.  The default launch
//   must refuse (launch.cpp:261-267); the forced sequential launch
//   (LaunchOptions{unsafe, sequential}, test_launch.cpp:148-153) gives the
//   point-order sum.  in = x, p, dx0, dp0 (n each) + dsigma0; out = dx, dp, dsigma.
int cmd_gauss_shared_in(int argc, char** argv) {
  if (argc < 6) die("gauss-shared-in <n> <sigma> <block> <in> <out>");
  const int64_t n = std::atoll(argv[1]);
  const double sigma = std::atof(argv[2]);
  const int64_t block = std::atoll(argv[3]);
  std::vector<double> all = read_f64(argv[4], static_cast<size_t>(4 * n + 1));
  Program prog(load_named("kernels"));
  LaunchConfig cfg{n / block + 1, block, n};
  BufferSet b;
  b.arrays["x"].assign(all.begin(), all.begin() + n);
  b.arrays["p"].assign(all.begin() + n, all.begin() + 2 * n);
  b.arrays["dx"].assign(all.begin() + 2 * n, all.begin() + 3 * n);
  b.arrays["dp"].assign(all.begin() + 3 * n, all.begin() + 4 * n);
  b.arrays["dsigma"].assign(1, all[4 * n]);
  b.scalars["sigma"] = sigma;
  bool refused = false;
  try {
    launch(prog, "compute_shared", cfg, b);
  } catch (const Error& e) {
    refused = e.kind() == ErrorKind::Launch;
  }
  LaunchOptions lo;
  lo.unsafe = true;
  lo.sequential = true;
  launch(prog, "compute_shared", cfg, b, lo);
  std::ofstream out(argv[5], std::ios::binary);
  write_f64(out, b.arrays["dx"]);
  write_f64(out, b.arrays["dp"]);
  write_f64(out, b.arrays["dsigma"]);
  std::printf("{\"n\": %lld, \"refused_by_default\": %s}\n", (long long)n,
              refused ? "true" : "false");
  return refused ? 0 : 1;
}

// print-forward <module> <fn> <wrt>   — differentiate_forward(fn, wrt) text
// (forward-over-reverse when fn is a generated gradient, hessian.cpp:31).
int cmd_print_forward(int argc, char** argv) {
  if (argc < 4) die("print-forward <module> <fn> <wrt>");
  Module m = load_named(argv[1]);
  const FunctionDef* f = m.find(argv[2]);
  if (f == nullptr) die(std::string("no function ") + argv[2]);
  TangentProgram t = differentiate_forward(*f, argv[3]);
  std::cout << print(t.derived);
  return 0;
}

// launch-file <module.dsl> <kernel> <n> <block> <in.bin> <out.bin> <module_out.txt> [unsafe]
//   Any Listing-style kernel of a DSL module (the generic-lowering parity
//   fixture): parse, ensure_called_derivatives (tooling.cpp:103-119), then
//   adc::launch on the kernel's parameters read in order from in.bin:
//   real[] -> [len, values...], real -> [value], integer -> [value] (as f64).
//   out = every real[] parameter after the launch, in order;
//   module_out = print(module) — the text the B200 JIT consumes.
int cmd_launch_file(int argc, char** argv) {
  if (argc < 8) die("launch-file <dsl> <kernel> <n> <block> <in> <out> <module_out> [unsafe]");
  std::ifstream f(argv[1]);
  if (!f) die(std::string("cannot open ") + argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  Module m = parse_or_throw(ss.str());
  ensure_called_derivatives(m);
  const std::string text = print(m);
  Program prog(std::move(m));
  const FunctionDef* k = prog.module().find(argv[2]);
  if (k == nullptr) die(std::string("no kernel ") + argv[2]);
  const int64_t n = std::atoll(argv[3]);
  const int64_t block = std::atoll(argv[4]);
  std::ifstream in(argv[5], std::ios::binary | std::ios::ate);
  const size_t bytes = static_cast<size_t>(in.tellg());
  std::vector<double> raw = read_f64(argv[5], bytes / 8);
  size_t pos = 0;
  BufferSet b;
  for (const auto& prm : k->params) {
    if (prm.type == ValType::RealArray) {
      const size_t len = static_cast<size_t>(raw.at(pos++));
      b.arrays[prm.name].assign(raw.begin() + pos, raw.begin() + pos + len);
      pos += len;
    } else if (prm.type == ValType::Real) {
      b.scalars[prm.name] = raw.at(pos++);
    } else {
      b.integers[prm.name] = static_cast<int64_t>(raw.at(pos++));
    }
  }
  // unsafe: forced hazardous launch, sequential; sequential: one worker (an
  // Eval error thrown on a pool worker terminates the process, so error
  // cases run sequentially to surface the reference's message).
  LaunchOptions lo;
  const std::string mode = argc > 8 ? argv[8] : "";
  if (mode == "unsafe") lo.unsafe = true;
  if (mode == "unsafe" || mode == "sequential") lo.sequential = true;
  std::string err;
  LaunchStats st;
  try {
    st = launch(prog, argv[2], LaunchConfig{n / block + 1, block, n}, b, lo);
  } catch (const Error& e) {
    err = e.what();
  }
  std::ofstream out(argv[6], std::ios::binary);
  for (const auto& prm : k->params)
    if (prm.type == ValType::RealArray) write_f64(out, b.arrays[prm.name]);
  std::ofstream mo(argv[7]);
  mo << text;
  // LaunchStats (launch.hpp:58-61): the OpCounters summed over all threads
  // and every thread's kernel-frame statement count
  const OpCounters& c = st.counts;
  std::printf("{\"n\": %lld, \"error\": \"%s\", \"counts\": [%llu, %llu, %llu, %llu, %llu, "
              "%llu, %llu], \"stm\": [",
              (long long)n, err.c_str(), (unsigned long long)c.adds, (unsigned long long)c.muls,
              (unsigned long long)c.divs, (unsigned long long)c.intrinsics,
              (unsigned long long)c.comparisons, (unsigned long long)c.tape_pushes,
              (unsigned long long)c.tape_pops);
  for (size_t i = 0; i < st.thread_statements.size(); ++i)
    std::printf("%s%u", i ? ", " : "", (unsigned)st.thread_statements[i]);
  std::printf("]}\n");
  return 0;
}

// gaussnd-shared-p-in <dim> <n> <sigma> <in.bin> <out.bin>
//   The shared-mean form: every point runs Program::eval("gaussnd_grad_0_1")
//   with the same p vector and the same dp slot (ArgPack holds raw pointers,
//   eval.hpp:36-61), points in order on one thread.  in = x (SoA dim x n),
//   p (dim), dx0 (SoA), dp0 (dim); out = dx (SoA), dp (dim).
int cmd_gaussnd_shared_p_in(int argc, char** argv) {
  if (argc < 6) die("gaussnd-shared-p-in <dim> <n> <sigma> <in> <out>");
  const int64_t dim = std::atoll(argv[1]);
  const int64_t n = std::atoll(argv[2]);
  const double sigma = std::atof(argv[3]);
  const size_t tot = static_cast<size_t>(dim * n);
  std::vector<double> all = read_f64(argv[4], 2 * tot + 2 * static_cast<size_t>(dim));
  const double* X = all.data();
  std::vector<double> p(all.begin() + tot, all.begin() + tot + dim);
  std::vector<double> DX(all.begin() + tot + dim, all.begin() + 2 * tot + dim);
  std::vector<double> dp(all.begin() + 2 * tot + dim, all.end());
  Module m = load_named("gaussnd");
  add_gradient(m, "gaussnd", {"x", "p"});
  Program prog(std::move(m));
  std::vector<double> x(dim), dx(dim);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t d = 0; d < dim; ++d) {
      x[d] = X[d * n + i];
      dx[d] = DX[d * n + i];
    }
    ArgPack a;
    a.add_array(x).add_array(p).add_real(sigma).add_int(dim).add_array(dx).add_array(dp);
    prog.eval("gaussnd_grad_0_1", a);
    for (int64_t d = 0; d < dim; ++d) DX[d * n + i] = dx[d];
  }
  std::ofstream out(argv[5], std::ios::binary);
  write_f64(out, DX);
  write_f64(out, dp);
  std::printf("{\"dim\": %lld, \"n\": %lld}\n", (long long)dim, (long long)n);
  return 0;
}

// gaussnd-in <dim> <n> <sigma> <in.bin> <out.bin> [workers]
//   in = x, p, dx0, dp0 in structure-of-arrays layout ([d*n + i]); each point
//   is gathered into contiguous rows and run through
//   Program::eval("gaussnd_grad_0_1") on an nproc thread pool (Program is
//   immutable and safe for concurrent eval, eval.hpp:86-88).  out = dx, dp (SoA).
int cmd_gaussnd_in(int argc, char** argv) {
  if (argc < 6) die("gaussnd-in <dim> <n> <sigma> <in> <out> [workers]");
  const int64_t dim = std::atoll(argv[1]);
  const int64_t n = std::atoll(argv[2]);
  const double sigma = std::atof(argv[3]);
  unsigned workers = argc > 6 ? static_cast<unsigned>(std::atoi(argv[6])) : 0;
  if (workers == 0) workers = default_workers();
  const size_t tot = static_cast<size_t>(dim * n);
  std::vector<double> all = read_f64(argv[4], 4 * tot);
  const double* X = all.data();
  const double* P = X + tot;
  std::vector<double> DX(all.begin() + 2 * tot, all.begin() + 3 * tot);
  std::vector<double> DP(all.begin() + 3 * tot, all.begin() + 4 * tot);
  Module m = load_named("gaussnd");
  add_gradient(m, "gaussnd", {"x", "p"});
  Program prog(std::move(m));
  std::atomic<int64_t> next{0};
  auto body = [&]() {
    std::vector<double> x(dim), p(dim), dx(dim), dp(dim);
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      for (int64_t d = 0; d < dim; ++d) {
        x[d] = X[d * n + i];
        p[d] = P[d * n + i];
        dx[d] = DX[d * n + i];
        dp[d] = DP[d * n + i];
      }
      ArgPack a;
      a.add_array(x).add_array(p).add_real(sigma).add_int(dim).add_array(dx).add_array(dp);
      prog.eval("gaussnd_grad_0_1", a);
      for (int64_t d = 0; d < dim; ++d) {
        DX[d * n + i] = dx[d];
        DP[d * n + i] = dp[d];
      }
    }
  };
  auto t0 = clk::now();
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < workers; ++w) pool.emplace_back(body);
  for (auto& t : pool) t.join();
  double sec = secs(t0, clk::now());
  std::ofstream out(argv[5], std::ios::binary);
  write_f64(out, DX);
  write_f64(out, DP);
  std::printf("{\"dim\": %lld, \"n\": %lld, \"seconds\": %.6f, \"workers\": %u}\n",
              (long long)dim, (long long)n, sec, workers);
  return 0;
}

// ---------------------------------------------------------------------------
// χ² over a model-parameterised engine.  For gsum this is the unmodified
// FitEngine (fit.cpp); for any other model the same formulas
// (fit.cpp:206-259, 268-278, 315-425) are evaluated over the reference
// Program running that model and its generated gradient.  `clamp` lists the
// parameter indices the σ clamp applies to (fit.cpp:268-278 hard-codes every
// third index, which is right for gsum only).
struct ModelEngine {
  std::string model;
  std::string grad;
  Program prog;
  std::vector<int> clamp_idx;
  bool numeric = false;  // GradientProvider::Numeric: central_gradient (fit.cpp:187-190)

  ModelEngine(const std::string& name, Module m, std::string g, std::vector<int> clamp)
      : model(name), grad(std::move(g)), prog(std::move(m)), clamp_idx(std::move(clamp)) {}

  ArgPack pack(double x, const std::vector<double>& q) const {
    ArgPack a;
    a.add_real(x);
    a.add_array(const_cast<double*>(q.data()), static_cast<int64_t>(q.size()));
    a.add_int(static_cast<int64_t>(q.size()) / 3);
    return a;
  }
  double eval_model(double x, const std::vector<double>& q) const {
    ArgPack a = pack(x, q);
    return *prog.eval(model, a).value;
  }
  void eval_grad(double x, const std::vector<double>& q, std::vector<double>& out) const {
    if (numeric) {  // FitEngine::model_gradient, GradientProvider::Numeric branch
      ArgPack a = pack(x, q);
      CentralGradient g = central_gradient(prog, model, a, {"q"});
      out = std::move(g.values);
      return;
    }
    out.assign(q.size(), 0.0);
    ArgPack a = pack(x, q);
    a.add_array(out.data(), static_cast<int64_t>(out.size()));
    prog.eval(grad, a);
  }
  double chi2(const Histogram& h, const std::vector<double>& q) const {
    double s = 0.0;
    std::vector<double> m(static_cast<size_t>(h.bins));
    for (int j = 0; j < h.bins; ++j) {
      m[j] = eval_model(h.center(j), q);
      s += m[j];
    }
    double sum = 0.0;
    const double scale = static_cast<double>(h.events) / s;
    for (int j = 0; j < h.bins; ++j) {
      double c = h.counts[j];
      if (c <= 0.0) continue;
      double r = c - scale * m[j];
      sum += r * r / c;
    }
    return sum;
  }
  void chi2_gradient(const Histogram& h, const std::vector<double>& q,
                     std::vector<double>& out) const {
    const size_t np = q.size();
    out.assign(np, 0.0);
    const double events = static_cast<double>(h.events);
    std::vector<double> m(static_cast<size_t>(h.bins));
    double s = 0.0;
    for (int j = 0; j < h.bins; ++j) {
      m[j] = eval_model(h.center(j), q);
      s += m[j];
    }
    double t_sum = 0.0;
    for (int j = 0; j < h.bins; ++j) {
      double c = h.counts[j];
      if (c <= 0.0) continue;
      double r = c - events * m[j] / s;
      t_sum += 2.0 * r * m[j] / c;
    }
    const double s_coef = events / (s * s) * t_sum;
    std::vector<double> bg(np);
    for (int j = 0; j < h.bins; ++j) {
      double c = h.counts[j];
      double w = s_coef;
      if (c > 0.0) {
        double r = c - events * m[j] / s;
        w += -2.0 * r / c * events / s;
      }
      if (w == 0.0) continue;
      eval_grad(h.center(j), q, bg);
      for (size_t i = 0; i < np; ++i) out[i] += w * bg[i];
    }
  }
  int clamp(std::vector<double>& q, double sigma_min) const {
    int n = 0;
    for (int i : clamp_idx)
      if (static_cast<size_t>(i) < q.size() && q[i] < sigma_min) {
        q[i] = sigma_min;
        ++n;
      }
    return n;
  }
  // (H + lambda I) d = g, Gaussian elimination with partial pivoting
  // (the algorithm of fit.cpp:282-311).
  static bool damped(std::vector<double> hm, std::vector<double> g, double lambda, int n,
                     std::vector<double>& out) {
    for (int i = 0; i < n; ++i) hm[i * n + i] += lambda;
    for (int col = 0; col < n; ++col) {
      int piv = col;
      for (int r = col + 1; r < n; ++r)
        if (std::fabs(hm[r * n + col]) > std::fabs(hm[piv * n + col])) piv = r;
      if (std::fabs(hm[piv * n + col]) < 1e-30) return false;
      if (piv != col) {
        for (int c = 0; c < n; ++c) std::swap(hm[piv * n + c], hm[col * n + c]);
        std::swap(g[piv], g[col]);
      }
      for (int r = col + 1; r < n; ++r) {
        double f = hm[r * n + col] / hm[col * n + col];
        for (int c = col; c < n; ++c) hm[r * n + c] -= f * hm[col * n + c];
        g[r] -= f * g[col];
      }
    }
    out.assign(n, 0.0);
    for (int r = n - 1; r >= 0; --r) {
      double v = g[r];
      for (int c = r + 1; c < n; ++c) v -= hm[r * n + c] * out[c];
      out[r] = v / hm[r * n + r];
    }
    return true;
  }

  // Steepest descent or the numeric-Hessian Newton step + Armijo
  // backtracking, fit.cpp:315-425.
  FitResult fit(const Histogram& h, std::vector<double> q, const FitOptions& o) const {
    FitResult res;
    res.sigma_clamps += clamp(q, o.sigma_min);
    const size_t np = q.size();
    double cur = chi2(h, q);
    if (o.trace_iterates > 0) res.iterates.push_back(q);
    std::vector<double> g(np);
    for (int iter = 0; iter < o.budget; ++iter) {
      chi2_gradient(h, q, g);
      ++res.gradient_evals;
      double gmax = 0.0;
      for (double v : g) gmax = std::max(gmax, std::fabs(v));
      if (gmax <= o.grad_tol) {
        res.converged = true;
        break;
      }
      std::vector<double> direction = g;
      if (o.use_hessian) {
        const int n = static_cast<int>(np);
        std::vector<double> hess(np * np, 0.0), gp(np), gm(np), probe = q;
        for (int c = 0; c < n; ++c) {
          double x = probe[c];
          double step = std::cbrt(2.220446049250313e-16) * std::max(1.0, std::fabs(x));
          probe[c] = x + step;
          chi2_gradient(h, probe, gp);
          probe[c] = x - step;
          chi2_gradient(h, probe, gm);
          res.gradient_evals += 2;
          probe[c] = x;
          for (int r = 0; r < n; ++r) hess[r * n + c] = (gp[r] - gm[r]) / (2.0 * step);
        }
        double lambda = 0.0;
        bool ok = false;
        for (int attempt = 0; attempt < 10 && !ok; ++attempt) {
          ok = damped(hess, g, lambda, n, direction);
          if (ok) {
            double descent = 0.0;
            for (size_t i = 0; i < np; ++i) descent += g[i] * direction[i];
            ok = descent > 0.0;
          }
          lambda = lambda == 0.0 ? 1e-6 : lambda * 10.0;
        }
        if (!ok) direction = g;
      }
      double gd = 0.0;
      for (size_t i = 0; i < np; ++i) gd += g[i] * direction[i];
      double t = 1.0, next = 0.0;
      bool accepted = false;
      std::vector<double> cand;
      while (t >= 1e-18) {
        std::vector<double> trial = q;
        for (size_t i = 0; i < np; ++i) trial[i] -= t * direction[i];
        int cl = clamp(trial, o.sigma_min);
        double c2 = chi2(h, trial);
        if (c2 <= cur - o.armijo_c1 * t * gd) {
          accepted = true;
          next = c2;
          cand = std::move(trial);
          res.sigma_clamps += cl;
          break;
        }
        t *= 0.5;
      }
      if (!accepted) {
        res.converged = true;
        break;
      }
      double rel_dec = (cur - next) / std::max(1.0, std::fabs(cur));
      q = std::move(cand);
      cur = next;
      ++res.iterations;
      if (o.trace_iterates > res.iterations) res.iterates.push_back(q);
      if (rel_dec <= o.chi2_rel_tol) {
        res.converged = true;
        break;
      }
    }
    res.params = std::move(q);
    res.chi2 = cur;
    return res;
  }
};

// "<model>" or "<model>:numeric" (the GradientProvider).
GradientProvider split_provider(std::string& model) {
  const auto colon = model.find(':');
  if (colon == std::string::npos) return GradientProvider::AdReverse;
  const std::string p = model.substr(colon + 1);
  model = model.substr(0, colon);
  if (p != "numeric") die("unknown provider '" + p + "'");
  return GradientProvider::Numeric;
}

ModelEngine make_engine(std::string model) {
  const GradientProvider prov = split_provider(model);
  Module m = load_named(model);
  std::string g = add_gradient(m, model, {"q"});
  std::vector<int> clamp;
  if (model == "gsum") {
    for (int i = 2; i < 64; i += 3) clamp.push_back(i);
  } else {
    clamp = {2};  // gpoly: only q[2] is a width
  }
  ModelEngine e(model, std::move(m), g, clamp);
  e.numeric = prov == GradientProvider::Numeric;
  return e;
}

Histogram read_hist(int64_t bins, double lo, double hi, const std::string& path) {
  Histogram h;
  h.bins = static_cast<int>(bins);
  h.lo = lo;
  h.hi = hi;
  h.counts = read_f64(path, static_cast<size_t>(bins));
  double tot = 0;
  for (double c : h.counts) tot += c;
  h.events = static_cast<uint64_t>(tot);
  return h;
}

// chi2-in <model> <bins> <lo> <hi> <counts.bin> <out.bin> <repeats> q...
//   out = [chi2, grad[np]].  events = Σ counts (the reference sampler
//   guarantees this, fit.cpp:88,94-102).  For gsum the result also comes from
//   the unmodified adc::FitEngine and both must agree bitwise.
int cmd_chi2_in(int argc, char** argv) {
  if (argc < 8) die("chi2-in <model> <bins> <lo> <hi> <counts> <out> <repeats> q...");
  std::string model = argv[1];
  Histogram h = read_hist(std::atoll(argv[2]), std::atof(argv[3]), std::atof(argv[4]), argv[5]);
  const int repeats = std::max(1, std::atoi(argv[7]));
  std::vector<double> q;
  for (int i = 8; i < argc; ++i) q.push_back(std::atof(argv[i]));
  ModelEngine eng = make_engine(model);
  const GradientProvider prov = split_provider(model);
  std::vector<double> g;
  double c2 = 0;
  std::vector<double> tg, tc;
  for (int r = 0; r < repeats; ++r) {
    auto t0 = clk::now();
    eng.chi2_gradient(h, q, g);
    auto t1 = clk::now();
    c2 = eng.chi2(h, q);
    auto t2 = clk::now();
    tg.push_back(secs(t0, t1));
    tc.push_back(secs(t1, t2));
  }
  bool engine_match = true;
  if (model == "gsum") {
    FitEngine fe;
    std::vector<double> g2;
    fe.chi2_gradient(h, q, prov, g2);
    engine_match = g2 == g && fe.chi2(h, q) == c2;
  }
  std::ofstream out(argv[6], std::ios::binary);
  std::vector<double> res{c2};
  res.insert(res.end(), g.begin(), g.end());
  write_f64(out, res);
  std::sort(tg.begin(), tg.end());
  std::sort(tc.begin(), tc.end());
  std::printf("{\"bins\": %d, \"events\": %llu, \"grad_seconds\": %.6f, \"chi2_seconds\": %.6f, "
              "\"fitengine_match\": %s}\n",
              h.bins, (unsigned long long)h.events, tg[tg.size() / 2], tc[tc.size() / 2],
              engine_match ? "true" : "false");
  return engine_match ? 0 : 1;
}

// chi2-file <model> <hist.adchist> <out.bin> q...  — the reference's chi2 and
// chi2_gradient (the FitEngine formula over the reference Program) of a
// histogram in the engine's ingest format (include/adc_cuda.h "ADCHIST1"),
// read here independently of the product.  out = [chi2, grad[np]].
int cmd_chi2_file(int argc, char** argv) {
  if (argc < 4) die("chi2-file <model> <hist.adchist> <out> q...");
  std::string model = argv[1];
  std::ifstream in(argv[2], std::ios::binary);
  if (!in) die(std::string("cannot open ") + argv[2]);
  char magic[8];
  int64_t bins = 0;
  double lo = 0, hi = 0, events = 0;
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(&bins), 8);
  in.read(reinterpret_cast<char*>(&lo), 8);
  in.read(reinterpret_cast<char*>(&hi), 8);
  in.read(reinterpret_cast<char*>(&events), 8);
  if (!in || std::memcmp(magic, "ADCHIST1", 8) != 0 || bins <= 0) die("not an ADCHIST1 file");
  Histogram h;
  h.bins = static_cast<int>(bins);
  h.lo = lo;
  h.hi = hi;
  h.events = static_cast<uint64_t>(events);
  h.counts.resize(bins);
  in.read(reinterpret_cast<char*>(h.counts.data()), bins * 8);
  if (!in) die("short histogram file");
  std::vector<double> q;
  for (int i = 4; i < argc; ++i) q.push_back(std::atof(argv[i]));
  ModelEngine eng = make_engine(model);
  std::vector<double> g;
  eng.chi2_gradient(h, q, g);
  std::vector<double> res{eng.chi2(h, q)};
  res.insert(res.end(), g.begin(), g.end());
  std::ofstream out(argv[3], std::ios::binary);
  write_f64(out, res);
  std::printf("{\"bins\": %lld, \"events\": %.17g}\n", (long long)bins, events);
  return 0;
}

// fit-in <model> <bins> <lo> <hi> <counts.bin> <out.bin> <trace> <budget[:hess]> q...
//   out = [chi2, iterations, gradient_evals, converged, sigma_clamps,
//          params[np], iterates[trace x np] (zero padded)].
int cmd_fit_in(int argc, char** argv) {
  if (argc < 9) die("fit-in <model> <bins> <lo> <hi> <counts> <out> <trace> <budget> q...");
  std::string model = argv[1];
  Histogram h = read_hist(std::atoll(argv[2]), std::atof(argv[3]), std::atof(argv[4]), argv[5]);
  FitOptions o;
  o.trace_iterates = std::atoi(argv[7]);
  o.budget = std::atoi(argv[8]);
  o.use_hessian = std::strstr(argv[8], ":hess") != nullptr;
  std::vector<double> q;
  for (int i = 9; i < argc; ++i) q.push_back(std::atof(argv[i]));
  ModelEngine eng = make_engine(model);
  const GradientProvider prov = split_provider(model);
  auto t0 = clk::now();
  FitResult r = eng.fit(h, q, o);
  double sec = secs(t0, clk::now());
  bool engine_match = true;
  if (model == "gsum") {
    FitEngine fe;
    FitResult r2 = fe.fit(h, prov, q, o);
    engine_match = r2.params == r.params && r2.iterates == r.iterates && r2.chi2 == r.chi2 &&
                   r2.iterations == r.iterations;
  }
  std::vector<double> res{r.chi2, double(r.iterations), double(r.gradient_evals),
                          r.converged ? 1.0 : 0.0, double(r.sigma_clamps)};
  res.insert(res.end(), r.params.begin(), r.params.end());
  for (int k = 0; k < o.trace_iterates; ++k) {
    if (static_cast<size_t>(k) < r.iterates.size())
      res.insert(res.end(), r.iterates[k].begin(), r.iterates[k].end());
    else
      res.insert(res.end(), q.size(), 0.0);
  }
  std::ofstream out(argv[6], std::ios::binary);
  write_f64(out, res);
  std::printf("{\"iterations\": %d, \"converged\": %s, \"seconds\": %.6f, "
              "\"fitengine_match\": %s}\n",
              r.iterations, r.converged ? "true" : "false", sec, engine_match ? "true" : "false");
  return engine_match ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Timed reference arms (bench.py --impl reference and the cpu_baseline leg).
// Inputs are drawn here from mt19937_64 in the per-point layout the reference
// evaluates; `total` evaluations cycle over `unique` points so the sample's
// memory stays bounded while its CPU time scales.

// gaussnd-bench <dim> <unique> <total> <sigma> <seed> [workers]
int cmd_gaussnd_bench(int argc, char** argv) {
  if (argc < 6) die("gaussnd-bench <dim> <unique> <total> <sigma> <seed> [workers]");
  const int64_t dim = std::atoll(argv[1]);
  const int64_t uniq = std::atoll(argv[2]);
  const int64_t total = std::atoll(argv[3]);
  const double sigma = std::atof(argv[4]);
  const uint64_t seed = std::strtoull(argv[5], nullptr, 0);
  unsigned workers = argc > 6 ? static_cast<unsigned>(std::atoi(argv[6])) : 0;
  if (workers == 0) workers = default_workers();
  const double spread = dim <= 100 ? 0.1 : 0.03;
  std::mt19937_64 rng(seed);
  std::vector<double> X(uniq * dim), P(uniq * dim);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (int64_t k = 0; k < uniq * dim; ++k) {
    P[k] = std::uniform_real_distribution<double>(-2, 2)(rng);
    X[k] = P[k] + spread * nd(rng);
  }
  Module m = load_named("gaussnd");
  add_gradient(m, "gaussnd", {"x", "p"});
  Program prog(std::move(m));
  std::atomic<int64_t> next{0};
  std::vector<double> checksum(workers, 0.0);
  auto body = [&](unsigned w) {
    std::vector<double> dx(dim), dp(dim);
    for (;;) {
      int64_t g = next.fetch_add(1);
      if (g >= total) break;
      const int64_t i = g % uniq;
      std::fill(dx.begin(), dx.end(), 0.0);
      std::fill(dp.begin(), dp.end(), 0.0);
      ArgPack a;
      a.add_array(&X[i * dim], dim).add_array(&P[i * dim], dim).add_real(sigma).add_int(dim);
      a.add_array(dx).add_array(dp);
      prog.eval("gaussnd_grad_0_1", a);
      checksum[w] += dx[0];
    }
  };
  auto t0 = clk::now();
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < workers; ++w) pool.emplace_back(body, w);
  for (auto& t : pool) t.join();
  double sec = secs(t0, clk::now());
  double cs = 0;
  for (double c : checksum) cs += c;
  std::printf("{\"dim\": %lld, \"points\": %lld, \"unique\": %lld, \"seconds\": %.6f, "
              "\"workers\": %u, \"checksum\": %.17g}\n",
              (long long)dim, (long long)total, (long long)uniq, sec, workers, cs);
  return 0;
}

// gauss1d-bench <n> <seed> [workers]  — adc::launch(compute) over n points.
int cmd_gauss1d_bench(int argc, char** argv) {
  if (argc < 3) die("gauss1d-bench <n> <seed> [workers]");
  const int64_t n = std::atoll(argv[1]);
  const uint64_t seed = std::strtoull(argv[2], nullptr, 0);
  const unsigned workers = argc > 3 ? static_cast<unsigned>(std::atoi(argv[3])) : 0;
  std::mt19937_64 rng(seed);
  BufferSet b;
  auto& x = b.arrays["x"];
  auto& p = b.arrays["p"];
  x.resize(n);
  p.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = std::uniform_real_distribution<double>(-3, 3)(rng);
    p[i] = std::uniform_real_distribution<double>(-2, 2)(rng);
  }
  b.arrays["dx"].assign(n, 0.0);
  b.arrays["dp"].assign(n, 0.0);
  b.scalars["sigma"] = 1.3;
  Program prog(load_named("kernels"));
  LaunchOptions lo;
  lo.workers = workers;
  auto t0 = clk::now();
  launch(prog, "compute", {n / 256 + 1, 256, n}, b, lo);
  double sec = secs(t0, clk::now());
  std::printf("{\"points\": %lld, \"seconds\": %.6f, \"workers\": %u}\n", (long long)n, sec,
              workers ? workers : default_workers());
  return 0;
}

// chi2-bench <model> <bins> <passes> q...  — single-threaded, as the
// reference's chi2_gradient is (fit.cpp:224-259); Poisson-free synthetic
// counts (the pass cost does not depend on the values).
int cmd_chi2_bench(int argc, char** argv) {
  if (argc < 4) die("chi2-bench <model> <bins> <passes> q...");
  std::string model = argv[1];
  const int64_t bins = std::atoll(argv[2]);
  const int passes = std::max(1, std::atoi(argv[3]));
  std::vector<double> q;
  for (int i = 4; i < argc; ++i) q.push_back(std::atof(argv[i]));
  Histogram h;
  h.bins = static_cast<int>(bins);
  h.lo = -5.0;
  h.hi = 5.0;
  h.counts.resize(bins);
  std::mt19937_64 rng(42);
  double tot = 0;
  for (int64_t j = 0; j < bins; ++j) {
    h.counts[j] = (j % 100 == 0) ? 0.0 : double(50 + rng() % 100);
    tot += h.counts[j];
  }
  h.events = static_cast<uint64_t>(tot);
  ModelEngine eng = make_engine(model);
  std::vector<double> g;
  auto t0 = clk::now();
  for (int r = 0; r < passes; ++r) eng.chi2_gradient(h, q, g);
  double sec = secs(t0, clk::now());
  std::printf("{\"bins\": %lld, \"passes\": %d, \"seconds\": %.6f, \"workers\": 1, "
              "\"g0\": %.17g}\n", (long long)bins, passes, sec, g.empty() ? 0.0 : g[0]);
  return 0;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) die("usage: ref_tool <command> ...");
  std::string cmd = argv[1];
  try {
    if (cmd == "print") return cmd_print(argc - 1, argv + 1);
    if (cmd == "golden-check") return cmd_golden_check(argc - 1, argv + 1);
    if (cmd == "gauss1d") return cmd_gauss1d(argc - 1, argv + 1);
    if (cmd == "gauss1d-in") return cmd_gauss1d_in(argc - 1, argv + 1);
    if (cmd == "gaussnd-in") return cmd_gaussnd_in(argc - 1, argv + 1);
    if (cmd == "gaussnd-shared-p-in") return cmd_gaussnd_shared_p_in(argc - 1, argv + 1);
    if (cmd == "gauss-shared-in") return cmd_gauss_shared_in(argc - 1, argv + 1);
    if (cmd == "launch-file") return cmd_launch_file(argc - 1, argv + 1);
    if (cmd == "print-forward") return cmd_print_forward(argc - 1, argv + 1);
    if (cmd == "chi2-in") return cmd_chi2_in(argc - 1, argv + 1);
    if (cmd == "fit-in") return cmd_fit_in(argc - 1, argv + 1);
    if (cmd == "gaussnd-bench") return cmd_gaussnd_bench(argc - 1, argv + 1);
    if (cmd == "gauss1d-bench") return cmd_gauss1d_bench(argc - 1, argv + 1);
    if (cmd == "chi2-bench") return cmd_chi2_bench(argc - 1, argv + 1);
    if (cmd == "chi2-file") return cmd_chi2_file(argc - 1, argv + 1);
  } catch (const Error& e) {
    std::fprintf(stderr, "ref_tool: adc::Error(kind=%d): %s\n", static_cast<int>(e.kind()),
                 e.what());
    return 3;
  }
  die("unknown command " + cmd);
}
