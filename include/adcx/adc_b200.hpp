// adc_b200.hpp — header-only C++ mirror of the reference's hot-path API over
// the B200 C ABI (include/adc_cuda.h).  Same type names, fields and error
// behaviour as the reference (proj/include/adc/launch.hpp, fit.hpp,
// diag.hpp) in namespace adc::b200, so C++ callers switch by namespace:
//
//   adc::launch(prog, "compute", cfg, buffers)   ->  adc::b200::launch("compute", cfg, buffers)
//   adc::FitEngine().chi2_gradient(h, q, p, out)  ->  adc::b200::FitEngine("gsum", 3)...
//
// Differences, by design: a launch names the Listing-1 kernel (the DSL Program
// is not needed on this path; the reference-side bridge in INTEGRATION.md
// recognises it from the Program), and FitEngine takes the model name because
// the B200 engine is model-parameterised (fit.cpp hard-wires gsum).
// Link with -ladc_b200 (paper_2203_06139_b200/libadc_b200.so).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "adc_cuda.h"

namespace adc::b200 {

// diag.hpp:17-23 order; Cuda/Arg/Nccl are the device-side additions.
enum class ErrorKind { Semantic, Transform, Eval, Launch, Io, Cuda, Arg, Nccl };

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

inline void check(int rc) {
  if (rc == ADC_OK) return;
  throw Error(static_cast<ErrorKind>(rc - 1), adc_cuda_last_error());
}

// ---- launch.hpp ------------------------------------------------------------
struct LaunchConfig {
  int64_t grid_dim = 0;
  int64_t block_dim = 0;
  int64_t n = 0;
  void validate() const {  // launch.cpp:9-19, same messages
    if (grid_dim <= 0 || block_dim <= 0 || n <= 0)
      throw Error(ErrorKind::Launch, "launch configuration must be positive (grid " +
                                         std::to_string(grid_dim) + ", block " +
                                         std::to_string(block_dim) + ", n " + std::to_string(n) +
                                         ")");
    if (grid_dim * block_dim < n)
      throw Error(ErrorKind::Launch, "grid " + std::to_string(grid_dim) + " x block " +
                                         std::to_string(block_dim) +
                                         " does not cover problem size " + std::to_string(n));
  }
};

struct BufferSet {
  std::map<std::string, std::vector<double>> arrays;
  std::map<std::string, double> scalars;
  std::map<std::string, int64_t> integers;
};

struct LaunchOptions {
  bool unsafe = false;    // forces compute_shared (deterministic fixed-order dsigma reduction)
  unsigned workers = 0;   // accepted for drop-in use; the GPU result does not depend on it
  bool sequential = false;
};

struct LaunchStats {
  std::vector<uint32_t> thread_statements;  // 3 per active thread, 2 per padding thread
};

// adc::launch (launch.cpp:252-346) for the Listing-1 kernels `compute`
// (kernels.dsl:9-14) and, forced with opts.unsafe, `compute_shared`
// (kernels.dsl:16-21), with host buffers; callee_fingerprint 0 = the registry's.
inline LaunchStats launch(const std::string& kernel, const LaunchConfig& cfg, BufferSet& buffers,
                          const LaunchOptions& opts = {}, uint64_t callee_fingerprint = 0) {
  cfg.validate();
  const bool shared = kernel == "compute_shared";
  if (shared && !opts.unsafe)
    throw Error(ErrorKind::Launch,
                "launch refused, hazardous parameter(s): dsigma (whole array shared with a "
                "writing callee across threads); pass the unsafe flag to force");
  if (!shared && kernel != "compute")
    throw Error(ErrorKind::Launch, "unknown kernel '" + kernel + "'");
  const int32_t kid = shared ? ADC_KERNEL_GAUSS_GRAD : ADC_KERNEL_GAUSS_GRAD_0_1;
  int32_t id = -1;
  check(adc_cuda_registry_find(
      adc_cuda_registry_name(kid),
      callee_fingerprint ? callee_fingerprint : adc_cuda_registry_fingerprint(kid), &id));
  for (const char* name : {"x", "p", "dx", "dp"}) {
    auto it = buffers.arrays.find(name);
    if (it == buffers.arrays.end())
      throw Error(ErrorKind::Launch, std::string("missing buffer '") + name + "'");
    if (static_cast<int64_t>(it->second.size()) < cfg.n)
      throw Error(ErrorKind::Launch, std::string("buffer '") + name + "' has length " +
                                         std::to_string(it->second.size()) +
                                         " but is indexed by thread over " +
                                         std::to_string(cfg.n) + " elements");
  }
  auto s = buffers.scalars.find("sigma");
  if (s == buffers.scalars.end()) throw Error(ErrorKind::Launch, "missing scalar value 'sigma'");
  if (shared) {
    auto ds = buffers.arrays.find("dsigma");
    if (ds == buffers.arrays.end()) throw Error(ErrorKind::Launch, "missing buffer 'dsigma'");
    if (ds->second.empty()) throw Error(ErrorKind::Launch, "buffer 'dsigma' is empty");
    check(adc_cuda_compute_gauss_shared_host(
        cfg.grid_dim, cfg.block_dim, cfg.n, buffers.arrays["x"].data(),
        buffers.arrays["p"].data(), s->second, buffers.arrays["dx"].data(),
        buffers.arrays["dp"].data(), ds->second.data(), 1));
  } else {
    check(adc_cuda_compute_gauss_host(cfg.grid_dim, cfg.block_dim, cfg.n,
                                      buffers.arrays["x"].data(), buffers.arrays["p"].data(),
                                      s->second, buffers.arrays["dx"].data(),
                                      buffers.arrays["dp"].data()));
  }
  LaunchStats st;
  st.thread_statements.assign(static_cast<size_t>(cfg.grid_dim * cfg.block_dim), 2u);
  for (int64_t g = 0; g < cfg.n; ++g) st.thread_statements[static_cast<size_t>(g)] = 3u;
  return st;
}

// Any Listing-style global kernel of a DSL module (as adc::print emits the
// Program, derivatives included), lowered to CUDA by the engine's JIT; host
// buffers, compiled once per (source, kernel, unsafe).
inline LaunchStats launch_module(const std::string& source, const std::string& kernel,
                                 const LaunchConfig& cfg, BufferSet& buffers,
                                 const LaunchOptions& opts = {}) {
  cfg.validate();
  static std::map<std::string, adc_jit_module*> cache;
  const std::string key = source + '\0' + kernel + (opts.unsafe ? "\1" : "\0");
  adc_jit_module*& m = cache[key];
  if (m == nullptr) check(adc_jit_compile(source.c_str(), kernel.c_str(), opts.unsafe, 0, &m));
  int32_t np = 0;
  int32_t kinds[64];
  check(adc_jit_kernel_params(m, &np, kinds, 64));
  std::vector<adc_jit_arg> args(static_cast<size_t>(np));
  for (int32_t i = 0; i < np; ++i) {
    const std::string name = adc_jit_kernel_param_name(m, i);
    if (kinds[i] == 0) {
      auto it = buffers.arrays.find(name);
      if (it == buffers.arrays.end()) throw Error(ErrorKind::Launch, "missing buffer '" + name + "'");
      args[i].ptr = it->second.data();
      args[i].len = static_cast<int64_t>(it->second.size());
    } else if (kinds[i] == 1) {
      auto it = buffers.scalars.find(name);
      if (it == buffers.scalars.end())
        throw Error(ErrorKind::Launch, "missing scalar value '" + name + "'");
      args[i].real_value = it->second;
    } else {
      auto it = buffers.integers.find(name);
      if (it == buffers.integers.end())
        throw Error(ErrorKind::Launch, "missing integer value '" + name + "'");
      args[i].int_value = it->second;
    }
  }
  check(adc_cuda_jit_launch_host(m, cfg.grid_dim, cfg.block_dim, cfg.n, args.data(), np));
  LaunchStats st;
  st.thread_statements.assign(static_cast<size_t>(cfg.grid_dim * cfg.block_dim), 2u);
  for (int64_t g = 0; g < cfg.n; ++g) st.thread_statements[static_cast<size_t>(g)] = 3u;
  return st;
}

// The batched path the reference cannot express:
// gaussnd_grad_0_1 over n points, structure-of-arrays [d * ld + i].
inline void launch_batch_gaussnd(int64_t n, int64_t dim, const std::vector<double>& x,
                                 const std::vector<double>& p, double sigma,
                                 std::vector<double>& dx, std::vector<double>& dp) {
  const size_t need = static_cast<size_t>(n * dim);
  if (x.size() < need || p.size() < need || dx.size() < need || dp.size() < need)
    throw Error(ErrorKind::Launch, "gaussnd buffers shorter than dim * n");
  check(adc_cuda_gaussnd_grad_host(n, dim, n, x.data(), p.data(), sigma, dx.data(), dp.data()));
}

// The same over several GPUs (one host thread per device, contiguous point
// ranges; no collective): bit-identical to the single-device call.
inline void launch_batch_gaussnd(int64_t n, int64_t dim, const std::vector<double>& x,
                                 const std::vector<double>& p, double sigma,
                                 std::vector<double>& dx, std::vector<double>& dp,
                                 const std::vector<int32_t>& devices) {
  const size_t need = static_cast<size_t>(n * dim);
  if (x.size() < need || p.size() < need || dx.size() < need || dp.size() < need)
    throw Error(ErrorKind::Launch, "gaussnd buffers shorter than dim * n");
  check(adc_cuda_gaussnd_grad_host_mg(static_cast<int32_t>(devices.size()), devices.data(), n, dim,
                                      n, x.data(), p.data(), sigma, dx.data(), dp.data()));
}

// ---- fit.hpp -------------------------------------------------------------
struct Histogram {
  int bins = 0;
  double lo = 0.0;
  double hi = 0.0;
  uint64_t events = 0;
  std::vector<double> counts;
  double width() const { return (hi - lo) / bins; }
  double center(int i) const { return lo + (i + 0.5) * width(); }
};

struct FitOptions {
  int budget = 400;
  double grad_tol = 1e-6;
  double chi2_rel_tol = 1e-12;
  double sigma_min = 1e-3;
  double armijo_c1 = 1e-4;
  bool use_hessian = false;
  int trace_iterates = 0;
  bool host_loop = false;  // B200 option: host-driven loop (same bits as the device loop)
};

struct FitResult {
  std::vector<double> params;
  double chi2 = 0.0;
  int iterations = 0;
  uint64_t gradient_evals = 0;
  uint64_t gradient_wall_ns = 0;
  bool converged = false;
  int sigma_clamps = 0;
  std::vector<std::vector<double>> iterates;
};

// ---- multi-GPU (one process per GPU) ---------------------------------------
// Owns an adc_comm.  NCCL: rank 0 calls Comm::unique_id() and the application
// distributes the 128 bytes (MPI_Bcast, a file, ...); every rank then builds
// Comm::nccl(world, rank, id) on its device.  Host: any all-gather over host
// memory (e.g. MPI_Allgather) as a callback.
class Comm {
 public:
  static std::array<unsigned char, 128> unique_id() {
    std::array<unsigned char, 128> id{};
    check(adc_nccl_unique_id(id.data()));
    return id;
  }
  static Comm nccl(int world, int rank, const std::array<unsigned char, 128>& id) {
    adc_comm* c = nullptr;
    check(adc_cuda_comm_init_nccl(&c, id.data(), world, rank));
    return Comm(c);
  }
  static Comm host(int world, int rank, adc_allgather_fn fn, void* ctx) {
    adc_comm* c = nullptr;
    check(adc_comm_init_host(&c, world, rank, fn, ctx));
    return Comm(c);
  }
  // peer memory: fn only bootstraps the CUDA IPC handles of each plan
  static Comm peer(int world, int rank, adc_allgather_fn fn, void* ctx) {
    adc_comm* c = nullptr;
    check(adc_cuda_comm_init_peer(&c, world, rank, fn, ctx));
    return Comm(c);
  }
  Comm(Comm&& o) noexcept : c_(o.c_) { o.c_ = nullptr; }
  Comm& operator=(Comm&& o) noexcept {
    std::swap(c_, o.c_);
    return *this;
  }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  ~Comm() {
    if (c_) adc_comm_destroy(c_);
  }
  int world() const { return info(0); }
  int rank() const { return info(1); }
  adc_comm* get() const { return c_; }

 private:
  explicit Comm(adc_comm* c) : c_(c) {}
  int info(int which) const {
    int32_t w = 0, r = 0, k = 0;
    check(adc_comm_info(c_, &w, &r, &k));
    return which == 0 ? w : r;
  }
  adc_comm* c_ = nullptr;
};

class FitEngine {
 public:
  // model: "gsum" (np = 3K, fit.cpp:125-138) or "gpoly" (np = 6).  With a
  // communicator every histogram is sharded over its ranks: each rank uploads
  // only its own bin range, every rank calls the same methods and gets the
  // same bits back (the exchange runs inside the library).
  FitEngine(std::string model = "gsum", int np = 3, const Comm* comm = nullptr)
      : model_(std::move(model)), np_(np), comm_(comm) {
    if (model_ != "gsum" && model_ != "gpoly")
      throw Error(ErrorKind::Arg, "unknown model '" + model_ + "'");
  }
  ~FitEngine() { release(); }
  FitEngine(const FitEngine&) = delete;
  FitEngine& operator=(const FitEngine&) = delete;

  std::string gradient_fn_name() const { return model_ + "_grad_1"; }

  double chi2(const Histogram& h, const std::vector<double>& q) {
    double c2 = 0.0;
    check(adc_cuda_chi2(plan(h), q.data(), &c2));
    return c2;
  }
  void chi2_gradient(const Histogram& h, const std::vector<double>& q, std::vector<double>& out) {
    out.assign(q.size(), 0.0);
    check(adc_cuda_chi2_gradient(plan(h), q.data(), out.data(), nullptr));
  }
  FitResult fit(const Histogram& h, std::vector<double> init, const FitOptions& o = {}) {
    std::vector<int32_t> clamp;
    if (model_ == "gsum")
      for (int i = 2; i < np_; i += 3) clamp.push_back(i);
    else
      clamp.push_back(2);
    adc_fit_options co{o.budget, o.grad_tol, o.chi2_rel_tol, o.sigma_min, o.armijo_c1,
                       o.trace_iterates, o.use_hessian ? 1 : 0, o.host_loop ? 1 : 0};
    adc_fit_result cr{};
    std::vector<double> its(static_cast<size_t>(std::max(1, o.trace_iterates) * np_));
    check(adc_cuda_fit(plan(h), init.data(), clamp.data(), static_cast<int32_t>(clamp.size()),
                       &co, &cr, its.data()));
    FitResult r;
    r.params = init;
    r.chi2 = cr.chi2;
    r.iterations = cr.iterations;
    r.gradient_evals = cr.gradient_evals;
    r.gradient_wall_ns = cr.gradient_ns;
    r.converged = cr.converged != 0;
    r.sigma_clamps = cr.sigma_clamps;
    const int n_tr = o.trace_iterates ? std::min(o.trace_iterates, cr.iterations + 1) : 0;
    for (int k = 0; k < n_tr; ++k)
      r.iterates.emplace_back(its.begin() + k * np_, its.begin() + (k + 1) * np_);
    return r;
  }

 private:
  // One device-resident histogram is cached (re-uploaded when `h` changes).
  adc_chi2_plan* plan(const Histogram& h) {
    if (plan_ != nullptr && key_ == &h && key_counts_ == h.counts.data()) return plan_;
    release();
    const int32_t model = model_ == "gsum" ? ADC_MODEL_GSUM : ADC_MODEL_GPOLY;
    if (comm_ != nullptr) {
      adc_chi2_layout L{};
      check(adc_chi2_make_layout(h.bins, comm_->world(), comm_->rank(), &L));
      const size_t bytes = static_cast<size_t>(std::max<int64_t>(1, L.bin_end - L.bin_begin)) *
                           sizeof(double);
      check(adc_cuda_alloc(&counts_, bytes));
      if (L.bin_end > L.bin_begin)
        check(adc_cuda_copy(counts_, h.counts.data() + L.bin_begin,
                            static_cast<size_t>(L.bin_end - L.bin_begin) * sizeof(double), 1));
      check(adc_cuda_chi2_plan_create_sharded(&plan_, model, np_, h.bins, h.lo, h.hi,
                                              static_cast<double>(h.events),
                                              static_cast<const double*>(counts_), comm_->get(),
                                              nullptr));
    } else {
      const size_t bytes = h.counts.size() * sizeof(double);
      check(adc_cuda_alloc(&counts_, bytes));
      check(adc_cuda_copy(counts_, h.counts.data(), bytes, 1));
      check(adc_cuda_chi2_plan_create(&plan_, model, np_, h.bins, h.lo, h.hi,
                                      static_cast<double>(h.events),
                                      static_cast<const double*>(counts_), 1, 0, nullptr));
    }
    key_ = &h;
    key_counts_ = h.counts.data();
    return plan_;
  }
  void release() {
    if (plan_) adc_cuda_chi2_plan_destroy(plan_);
    if (counts_) adc_cuda_free(counts_);
    plan_ = nullptr;
    counts_ = nullptr;
  }

  std::string model_;
  int np_;
  const Comm* comm_ = nullptr;
  adc_chi2_plan* plan_ = nullptr;
  void* counts_ = nullptr;
  const Histogram* key_ = nullptr;
  const double* key_counts_ = nullptr;
};

}  // namespace adc::b200
