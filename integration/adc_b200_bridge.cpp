// Reference-side binding (see adc_b200_bridge.hpp).  Uses only the reference's
// public API plus the C ABI of include/adc_cuda.h.
#include "adc_b200_bridge.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "adc/parser.hpp"
#include "adc/printer.hpp"
#include "adc/transform.hpp"
#include "adc_cuda.h"

namespace adc::b200_bridge {
namespace {

[[noreturn]] void rethrow(int rc) {
  // adc_status 1..5 == ErrorKind + 1 (include/adc_cuda.h)
  ErrorKind k = rc >= 1 && rc <= 5 ? static_cast<ErrorKind>(rc - 1) : ErrorKind::Launch;
  throw Error(k, std::string("B200: ") + adc_cuda_last_error());
}
void check(int rc) {
  if (rc != ADC_OK) rethrow(rc);
}

uint64_t fingerprint(const FunctionDef& f) {
  const std::string text = print(f);
  return adc_cuda_fingerprint(text.data(), text.size());
}

bool is_var(const Expr& e, const char* name) {
  return e.kind == ExprKind::VarRef && e.name == name;
}

// The Listing-1 shape (kernels.dsl:9-14):
//   integer i = blockIdx * blockDim + threadIdx;  if (i < N) { grad(args...); }
struct Listing1 {
  std::string thread_var;
  const Stmt* call = nullptr;
};

bool match_listing1(const FunctionDef& k, Listing1& out) {
  if (k.body.size() != 2) return false;
  const Stmt& d = *k.body[0];
  if (d.kind != StmtKind::VarDecl || d.decl_type != ValType::Integer || !d.expr) return false;
  const Expr& e = *d.expr;
  if (e.kind != ExprKind::Binary || e.op != BinOp::Add) return false;
  const Expr& mul = *e.args[0];
  if (mul.kind != ExprKind::Binary || mul.op != BinOp::Mul || !is_var(*mul.args[0], "blockIdx") ||
      !is_var(*mul.args[1], "blockDim") || !is_var(*e.args[1], "threadIdx"))
    return false;
  const Stmt& g = *k.body[1];
  if (g.kind != StmtKind::If || !g.else_block.empty() || g.then_block.size() != 1) return false;
  const Expr& c = *g.expr;
  if (c.kind != ExprKind::Compare || c.cmp != CmpOp::Lt || !is_var(*c.args[0], d.target.c_str()) ||
      !is_var(*c.args[1], "N"))
    return false;
  const Stmt& call = *g.then_block[0];
  if (call.kind != StmtKind::CallStmt) return false;
  out.thread_var = d.target;
  out.call = &call;
  return true;
}

// Per-thread interpreter counters for one active and one idle thread of the
// kernel (ops are data-independent for these gradients), so LaunchStats.counts
// matches the reference's sum over threads without interpreting every point.
void analytic_counts(const Program& p, const std::string& kernel, const FunctionDef& k,
                     const LaunchConfig& cfg, const BufferSet& buffers, LaunchStats& st) {
  std::vector<std::vector<double>> scratch;
  scratch.reserve(k.params.size());
  ArgPack args;
  for (const auto& prm : k.params) {
    if (prm.type == ValType::RealArray) {
      scratch.emplace_back(1, buffers.arrays.at(prm.name)[0]);
      args.add_array(scratch.back());
    } else if (prm.type == ValType::Real) {
      args.add_real(buffers.scalars.at(prm.name));
    } else {
      args.add_int(buffers.integers.at(prm.name));
    }
  }
  EvalOptions o;
  o.has_thread_ctx = true;
  o.block_dim = cfg.block_dim;
  o.problem_n = cfg.n;
  o.block_idx = 0;
  o.thread_idx = 0;
  EvalResult active = p.eval(kernel, args, o);
  const int64_t total = cfg.grid_dim * cfg.block_dim;
  EvalResult idle{};
  if (total > cfg.n) {
    o.block_idx = cfg.n / cfg.block_dim;
    o.thread_idx = cfg.n % cfg.block_dim;
    idle = p.eval(kernel, args, o);
  }
  auto scale = [](const OpCounters& c, uint64_t n) {
    OpCounters r;
    r.adds = c.adds * n;
    r.muls = c.muls * n;
    r.divs = c.divs * n;
    r.intrinsics = c.intrinsics * n;
    r.comparisons = c.comparisons * n;
    r.tape_pushes = c.tape_pushes * n;
    r.tape_pops = c.tape_pops * n;
    return r;
  };
  st.counts = scale(active.counts, static_cast<uint64_t>(cfg.n));
  st.counts += scale(idle.counts, static_cast<uint64_t>(total - cfg.n));
  st.thread_statements.assign(static_cast<size_t>(total),
                              static_cast<uint32_t>(idle.top_statements));
  for (int64_t g = 0; g < cfg.n; ++g)
    st.thread_statements[static_cast<size_t>(g)] = static_cast<uint32_t>(active.top_statements);
}

// The generic path: the whole module as the reference prints it, lowered to
// CUDA and compiled with NVRTC by the engine (adc_jit_*), cached per
// (module text, kernel, unsafe).
LaunchStats launch_jit(const Program& p, const std::string& kernel, const FunctionDef& k,
                       const LaunchConfig& cfg, BufferSet& buffers, const LaunchOptions& opts) {
  static std::mutex mu;
  static std::map<std::string, adc_jit_module*> cache;
  const std::string text = print(p.module());
  const std::string key = text + '\0' + kernel + (opts.unsafe ? "\1" : "\0");
  adc_jit_module* m = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      m = it->second;
    } else {
      check(adc_jit_compile(text.c_str(), kernel.c_str(), opts.unsafe ? 1 : 0, 0, &m));
      cache[key] = m;
    }
  }
  std::vector<adc_jit_arg> args(k.params.size());
  for (size_t i = 0; i < k.params.size(); ++i) {
    const Param& prm = k.params[i];
    if (prm.type == ValType::RealArray) {
      std::vector<double>& v = buffers.arrays.at(prm.name);
      args[i].ptr = v.data();
      args[i].len = static_cast<int64_t>(v.size());
    } else if (prm.type == ValType::Real) {
      args[i].real_value = buffers.scalars.at(prm.name);
    } else {
      args[i].int_value = buffers.integers.at(prm.name);
    }
  }
  // the counting variant: the reference's LaunchStats exactly (OpCounters
  // summed over all threads, every thread's kernel-frame statements), for any
  // kernel — data-dependent branches and loops included
  LaunchStats st;
  const int64_t total = cfg.grid_dim * cfg.block_dim;
  st.thread_statements.assign(static_cast<size_t>(total), 0u);
  uint64_t c[7] = {0, 0, 0, 0, 0, 0, 0};
  check(adc_cuda_jit_launch_counted_host(m, cfg.grid_dim, cfg.block_dim, cfg.n, args.data(),
                                         static_cast<int32_t>(args.size()), c,
                                         st.thread_statements.data()));
  st.counts.adds = c[0];
  st.counts.muls = c[1];
  st.counts.divs = c[2];
  st.counts.intrinsics = c[3];
  st.counts.comparisons = c[4];
  st.counts.tape_pushes = c[5];
  st.counts.tape_pops = c[6];
  return st;
}

}  // namespace

LaunchStats launch(const Program& p, const std::string& kernel, const LaunchConfig& cfg,
                   BufferSet& buffers, const LaunchOptions& opts) {
  // launch.cpp:254-267 — validation and the hazard gate, unchanged.
  cfg.validate();
  const FunctionDef* k = p.module().find(kernel);
  if (k == nullptr) throw Error(ErrorKind::Launch, "unknown kernel '" + kernel + "'");
  if (!k->qualifiers.global)
    throw Error(ErrorKind::Launch, "'" + kernel + "' is not a global kernel");
  AccessReport report = race_check(p.module(), kernel);
  if (report.has_hazard() && !opts.unsafe) {
    std::string msg = "launch refused, hazardous parameter(s):";
    for (const auto& e : report.entries)
      if (e.access == Access::SharedWriteHazard) msg += " " + e.param + " (" + e.note + ")";
    msg += "; pass the unsafe flag to force";
    throw Error(ErrorKind::Launch, msg);
  }
  // launch.cpp:271-303 — buffer binding and length validation, unchanged.
  for (const auto& param : k->params) {
    if (param.type == ValType::RealArray) {
      auto it = buffers.arrays.find(param.name);
      if (it == buffers.arrays.end())
        throw Error(ErrorKind::Launch, "missing buffer '" + param.name + "'");
      const AccessReport::Entry* e = report.find(param.name);
      if (e != nullptr && e->indexed_by_thread && static_cast<int64_t>(it->second.size()) < cfg.n)
        throw Error(ErrorKind::Launch, "buffer '" + param.name + "' has length " +
                                           std::to_string(it->second.size()) +
                                           " but is indexed by thread over " +
                                           std::to_string(cfg.n) + " elements");
    } else if (param.type == ValType::Real) {
      if (!buffers.scalars.count(param.name))
        throw Error(ErrorKind::Launch, "missing scalar value '" + param.name + "'");
    } else if (!buffers.integers.count(param.name)) {
      throw Error(ErrorKind::Launch, "missing integer value '" + param.name + "'");
    }
  }
  // Kernel shape + registry lookup by the callee's printed text: the
  // hand-written kernels.  Everything else is lowered by the generic JIT.
  Listing1 l1;
  const FunctionDef* callee =
      match_listing1(*k, l1) ? p.module().find(l1.call->callee) : nullptr;
  int32_t id = -1;
  const bool registered =
      callee != nullptr &&
      adc_cuda_registry_find(callee->name.c_str(), fingerprint(*callee), &id) == ADC_OK;
  const size_t nargs = registered ? l1.call->call_args.size() : 0;
  // gauss_grad_0_1(x[i], p[i], sigma, dx[i], dp[i]) (compute), or the forced
  // hazardous gauss_grad(x[i], p[i], sigma, dx[i], dp[i], dsigma)
  // (compute_shared): only the shared slot may be a whole array.
  const bool shared = registered && id == ADC_KERNEL_GAUSS_GRAD && nargs == 6;
  const bool plain = registered && id == ADC_KERNEL_GAUSS_GRAD_0_1 && nargs == 5 &&
                     !report.has_hazard();
  if (!plain && !shared) return launch_jit(p, kernel, *k, cfg, buffers, opts);
  std::vector<double*> arr;
  double sigma = 0.0;
  for (size_t a = 0; a < 5; ++a) {
    const Expr& e = *l1.call->call_args[a];
    if (a == 2) {
      if (e.kind != ExprKind::VarRef) throw Error(ErrorKind::Launch, "unsupported sigma argument");
      sigma = buffers.scalars.at(e.name);
      continue;
    }
    if (e.kind != ExprKind::Index || !is_var(*e.args[0], l1.thread_var.c_str()))
      throw Error(ErrorKind::Launch, "unsupported argument shape for the B200 kernel");
    arr.push_back(buffers.arrays.at(e.name).data());
  }
  LaunchStats st;
  analytic_counts(p, kernel, *k, cfg, buffers, st);
  if (shared) {
    const Expr& e = *l1.call->call_args[5];
    if (e.kind != ExprKind::VarRef) throw Error(ErrorKind::Launch, "unsupported dsigma argument");
    std::vector<double>& ds = buffers.arrays.at(e.name);
    if (ds.empty()) throw Error(ErrorKind::Launch, "buffer '" + e.name + "' is empty");
    check(adc_cuda_compute_gauss_shared_host(cfg.grid_dim, cfg.block_dim, cfg.n, arr[0], arr[1],
                                             sigma, arr[2], arr[3], ds.data(), 1));
  } else {
    check(adc_cuda_compute_gauss_host(cfg.grid_dim, cfg.block_dim, cfg.n, arr[0], arr[1], sigma,
                                      arr[2], arr[3]));
  }
  return st;
}

// ---------------------------------------------------------------------------
namespace {
struct DevHist {
  const Histogram* key = nullptr;
  void* counts = nullptr;
  adc_chi2_plan* plan = nullptr;
  int np = 0;
  ~DevHist() {
    if (plan) adc_cuda_chi2_plan_destroy(plan);
    if (counts) adc_cuda_free(counts);
  }
};
thread_local DevHist t_hist;
std::string t_model_source;

adc_chi2_plan* plan_for(const FitEngine& engine, const Histogram& h, size_t np) {
  // The engine's generated gradient must be the registered one.
  if (t_model_source.empty())
    throw Error(ErrorKind::Launch, "B200: set_model_source() was not called");
  Module m = parse_or_throw(t_model_source);
  AdjointProgram g = differentiate_gradient(*m.find("gsum"), {"q"});
  int32_t id = -1;
  check(adc_cuda_registry_find(engine.gradient_fn_name().c_str(), fingerprint(g.derived), &id));
  if (t_hist.key == &h && t_hist.np == static_cast<int>(np)) return t_hist.plan;
  t_hist.~DevHist();
  new (&t_hist) DevHist();
  const size_t bytes = h.counts.size() * sizeof(double);
  check(adc_cuda_alloc(&t_hist.counts, bytes));
  check(adc_cuda_copy(t_hist.counts, h.counts.data(), bytes, 1));
  check(adc_cuda_chi2_plan_create(&t_hist.plan, ADC_MODEL_GSUM, static_cast<int32_t>(np), h.bins,
                                  h.lo, h.hi, static_cast<double>(h.events),
                                  static_cast<const double*>(t_hist.counts), 1, 0, nullptr));
  t_hist.key = &h;
  t_hist.np = static_cast<int>(np);
  return t_hist.plan;
}
}  // namespace

void set_model_source(const std::string& source) { t_model_source = source; }

void chi2_gradient(const FitEngine& engine, const Histogram& h, const std::vector<double>& q,
                   std::vector<double>& out, GradientProvider provider) {
  out.assign(q.size(), 0.0);
  adc_chi2_plan* plan = plan_for(engine, h, q.size());
  check(adc_cuda_chi2_set_provider(plan, provider == GradientProvider::Numeric
                                             ? ADC_PROVIDER_NUMERIC
                                             : ADC_PROVIDER_AD_REVERSE));
  check(adc_cuda_chi2_gradient(plan, q.data(), out.data(), nullptr));
}

FitResult fit(const FitEngine& engine, const Histogram& h, GradientProvider provider,
              std::vector<double> init, const FitOptions& opts) {
  const size_t np = init.size();
  adc_chi2_plan* plan = plan_for(engine, h, np);
  check(adc_cuda_chi2_set_provider(plan, provider == GradientProvider::Numeric
                                             ? ADC_PROVIDER_NUMERIC
                                             : ADC_PROVIDER_AD_REVERSE));
  std::vector<int32_t> clamp;  // clamp_sigmas: every third coordinate (fit.cpp:268-278)
  for (size_t i = 2; i < np; i += 3) clamp.push_back(static_cast<int32_t>(i));
  FitResult r;
  {  // op-count metadata at the clamped start, as fit.cpp:324-325
    std::vector<double> q0 = init;
    for (int32_t i : clamp)
      if (q0[static_cast<size_t>(i)] < opts.sigma_min) q0[static_cast<size_t>(i)] = opts.sigma_min;
    r.primal_call_counts = engine.model_counts(h.center(h.bins / 2), q0);
    r.gradient_call_counts = engine.model_gradient_counts(h.center(h.bins / 2), q0, provider);
  }
  adc_fit_options o;
  adc_fit_default_options(&o);
  o.budget = opts.budget;
  o.grad_tol = opts.grad_tol;
  o.chi2_rel_tol = opts.chi2_rel_tol;
  o.sigma_min = opts.sigma_min;
  o.armijo_c1 = opts.armijo_c1;
  o.trace_iterates = opts.trace_iterates;
  o.use_hessian = opts.use_hessian ? 1 : 0;
  adc_fit_result res{};
  std::vector<double> its(static_cast<size_t>(std::max(1, opts.trace_iterates)) * np);
  check(adc_cuda_fit(plan, init.data(), clamp.data(), static_cast<int32_t>(clamp.size()), &o,
                     &res, its.data()));
  r.params = init;
  r.chi2 = res.chi2;
  r.iterations = res.iterations;
  r.gradient_evals = res.gradient_evals;
  r.gradient_wall_ns = res.gradient_ns;
  r.converged = res.converged != 0;
  r.sigma_clamps = res.sigma_clamps;
  const int n_tr = opts.trace_iterates ? std::min(opts.trace_iterates, res.iterations + 1) : 0;
  for (int k = 0; k < n_tr; ++k)
    r.iterates.emplace_back(its.begin() + static_cast<long>(k * np),
                            its.begin() + static_cast<long>((k + 1) * np));
  return r;
}

std::vector<BenchRow> bench_scaling(const BenchConfig& cfg) {
  if (cfg.k_list.empty()) throw Error(ErrorKind::Eval, "empty K list");
  FitEngine engine;
  std::vector<BenchRow> rows;
  for (int k : cfg.k_list) {
    std::vector<double> truth = gauss_sum::default_truth(k, cfg.lo, cfg.hi);
    Histogram h = sample_histogram(truth, cfg.events, cfg.bins, cfg.lo, cfg.hi,
                                   cfg.seed + static_cast<uint64_t>(k));
    std::vector<double> init = gauss_sum::perturbed_init(truth);
    for (GradientProvider provider : {GradientProvider::AdReverse, GradientProvider::Numeric}) {
      std::vector<uint64_t> walls;
      FitResult last;
      for (int rep = 0; rep < std::max(1, cfg.repeats); ++rep) {
        last = fit(engine, h, provider, init, cfg.fit);
        walls.push_back(last.gradient_wall_ns);
      }
      std::sort(walls.begin(), walls.end());
      BenchRow row;
      row.k = k;
      row.params = 3 * k;
      row.provider = provider;
      row.median_wall_ns = walls[walls.size() / 2];
      row.grad_evals = last.gradient_evals;
      row.primal_opcount = last.primal_call_counts.total();
      row.grad_opcount = last.gradient_call_counts.total();
      row.converged = last.converged;
      row.final_params = last.params;
      rows.push_back(std::move(row));
    }
  }
  return rows;
}

double chi2(const FitEngine& engine, const Histogram& h, const std::vector<double>& q) {
  double c2 = 0.0;
  check(adc_cuda_chi2(plan_for(engine, h, q.size()), q.data(), &c2));
  return c2;
}

}  // namespace adc::b200_bridge
