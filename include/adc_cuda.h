/* adc_cuda.h — C ABI of the B200-native batched reverse-mode gradient engine.
 *
 * Drop-in boundary for the reference `adc` (arxiv/paper_2203_06139 artifact)
 * hot path.  The reference exposes a C++ API only (no FFI); the entry points
 * below are what its C++ call sites bind when the B200 backend is enabled
 * (INTEGRATION.md shows the bridge a maintainer adds to launch.cpp / fit.cpp).
 * Plain pointers and sizes, no torch or C++ types, stream-ordered, never
 * throws.  Every function returns an adc_status; on failure the thread-local
 * message is available from adc_cuda_last_error().
 *
 * There is NO CPU fallback: without a CUDA device every compute entry point
 * returns ADC_E_CUDA.
 */
#ifndef ADC_CUDA_H
#define ADC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADC_CUDA_ABI_VERSION 1

/* Status codes.  1..5 mirror adc::ErrorKind in declaration order
 * (proj/include/adc/diag.hpp:17-23) so the C++ bridge maps them back to
 * adc::Error(kind, message) one-to-one. */
typedef enum adc_status {
  ADC_OK = 0,
  ADC_E_SEMANTIC = 1,  /* ErrorKind::Semantic */
  ADC_E_TRANSFORM = 2, /* ErrorKind::Transform */
  ADC_E_EVAL = 3,      /* ErrorKind::Eval: domain errors (division by zero, ...) */
  ADC_E_LAUNCH = 4,    /* ErrorKind::Launch: config, refusal, buffer binding */
  ADC_E_IO = 5,        /* ErrorKind::Io */
  ADC_E_CUDA = 6,      /* CUDA runtime failure / no device */
  ADC_E_ARG = 7,       /* invalid argument to the C ABI itself */
  ADC_E_NCCL = 8       /* NCCL failure in the multi-GPU exchange */
} adc_status;

int adc_cuda_abi_version(void);
/* Thread-local text of the last failure on this thread ("" if none). */
const char* adc_cuda_last_error(void);
/* Device query: SM count and compute capability of the current device. */
int adc_cuda_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* Device memory and ordering helpers for C / C++ callers without a CUDA
 * runtime of their own (the C++ mirror in include/adcx/adc_b200.hpp).
 * kind: 1 = host->device, 2 = device->host, 3 = device->device. */
int adc_cuda_alloc(void** ptr, size_t bytes);
int adc_cuda_free(void* ptr);
int adc_cuda_copy(void* dst, const void* src, size_t bytes, int32_t kind);
int adc_cuda_synchronize(void);

/* ---------------------------------------------------------------------------
 * Kernel registry.  Each hand-written kernel implements exactly one generated
 * gradient; it is keyed by the gradient's name (gradient_name,
 * linearize.cpp:243-258) and the FNV-1a-64 fingerprint of its printed text
 * (adc::print(FunctionDef), printer.hpp:13).  A miss is ADC_E_LAUNCH —
 * there is no interpreter fallback.
 */
uint64_t adc_cuda_fingerprint(const char* text, size_t len);
int adc_cuda_registry_find(const char* gradient_name, uint64_t fingerprint, int32_t* kernel_id);
int32_t adc_cuda_registry_size(void);
const char* adc_cuda_registry_name(int32_t kernel_id);
uint64_t adc_cuda_registry_fingerprint(int32_t kernel_id);

enum {
  ADC_KERNEL_GAUSS_GRAD_0_1 = 0,   /* proj/tests/golden/gauss_grad_0_1.golden */
  ADC_KERNEL_GAUSSND_GRAD_0_1 = 1, /* oracle/dsl/gaussnd.dsl, wrt {x, p} */
  ADC_KERNEL_GSUM_GRAD_1 = 2,      /* fit.cpp:125-138 model, wrt {q} */
  ADC_KERNEL_GPOLY_GRAD_1 = 3,     /* oracle/dsl/gpoly.dsl, wrt {q} */
  ADC_KERNEL_GAUSS_GRAD = 4        /* kernels.dsl gauss, wrt {x, p, sigma} (compute_shared) */
};

/* ---------------------------------------------------------------------------
 * Listing-1 kernel `compute` (proj/corpus/kernels.dsl:9-14) launched as
 * adc::launch(prog, "compute", {grid_dim, block_dim, n}, buffers)
 * (proj/src/launch.cpp:252-346): for every global index g < n,
 *   gauss_grad_0_1(x[g], p[g], sigma, dx[g], dp[g])
 * accumulating into dx/dp (slots are += only, never assigned).
 * Validates like LaunchConfig::validate (launch.cpp:9-19).  Device pointers.
 * sigma == 0 is the interpreter's "division by zero" (ADC_E_EVAL). */
int adc_cuda_compute_gauss(int64_t grid_dim, int64_t block_dim, int64_t n, const double* x,
                           const double* p, double sigma, double* dx, double* dp, void* stream);

/* Same, host buffers: copies in, runs, copies dx/dp back, chunked over two
 * streams so PCIe traffic overlaps the kernel.  Synchronous. */
int adc_cuda_compute_gauss_host(int64_t grid_dim, int64_t block_dim, int64_t n, const double* x,
                                const double* p, double sigma, double* dx, double* dp);

/* Listing-1's hazardous twin `compute_shared` (proj/corpus/kernels.dsl:16-21):
 * every thread calls gauss_grad(x[i], p[i], sigma, dx[i], dp[i], dsigma), so all
 * threads accumulate into the one-element slot dsigma.  The reference's
 * race_check flags dsigma and launch refuses (launch.cpp:261-267, same
 * message, ADC_E_LAUNCH) unless `unsafe`; forced, the reference uses CAS
 * atomics in an unspecified order (eval.cpp:414-423).  Here the forced run is
 * DETERMINISTIC: dx, dp private as in `compute`, the sigma contributions summed
 * in a fixed order (per thread in point order, fixed CTA tree, one fixed final
 * tree) and added to dsigma[0] once.  Same bits on every run and device. */
int adc_cuda_compute_gauss_shared(int64_t grid_dim, int64_t block_dim, int64_t n,
                                  const double* x, const double* p, double sigma, double* dx,
                                  double* dp, double* dsigma, int32_t unsafe, void* stream);
int adc_cuda_compute_gauss_shared_host(int64_t grid_dim, int64_t block_dim, int64_t n,
                                       const double* x, const double* p, double sigma, double* dx,
                                       double* dp, double* dsigma, int32_t unsafe);
/* Over ranks: each rank launches over its own n points; every rank's dsigma
 * partial is all-gathered through `comm` and added in rank order (the same
 * dsigma bits on every rank; world 1 = the single-device result). */
typedef struct adc_comm adc_comm;
int adc_cuda_compute_gauss_shared_comm(int64_t grid_dim, int64_t block_dim, int64_t n,
                                       const double* x, const double* p, double sigma, double* dx,
                                       double* dp, double* dsigma, int32_t unsafe, adc_comm* comm,
                                       void* stream);

/* ---------------------------------------------------------------------------
 * Batched N-dim Gaussian gradient gaussnd_grad_0_1(x, p, sigma, dim, dx, dp)
 * over n independent points.  Structure-of-arrays: coordinate d of point i is
 * at [d * ld + i] (ld >= n) in x, p, dx, dp.  Slots accumulate.  Device
 * pointers, stream-ordered. */
int adc_cuda_gaussnd_grad(int64_t n, int64_t dim, int64_t ld, const double* x, const double* p,
                          double sigma, double* dx, double* dp, void* stream);
/* Host-buffer variant (pinned memory recommended); synchronous, pipelined. */
int adc_cuda_gaussnd_grad_host(int64_t n, int64_t dim, int64_t ld, const double* x,
                               const double* p, double sigma, double* dx, double* dp);
/* Multi-GPU host-buffer form (north_star (4); replaces the reference's
 * data-parallel split of one batch over its worker threads, launch.cpp:305-343):
 * the n points are split into ndev contiguous ranges of whole 64-point tiles
 * and one host thread per device runs the host pipeline on its range, so
 * every device's PCIe link carries its share of the copies at once.  No
 * collective: points are independent, so every output is bit-identical to
 * the single-device call.  devices: ndev distinct device ordinals, or NULL
 * for 0..ndev-1.  Synchronous; safe to call from several threads. */
int adc_cuda_gaussnd_grad_host_mg(int32_t ndev, const int32_t* devices, int64_t n, int64_t dim,
                                  int64_t ld, const double* x, const double* p, double sigma,
                                  double* dx, double* dp);
int adc_cuda_compute_gauss_host_mg(int32_t ndev, const int32_t* devices, int64_t grid_dim,
                                   int64_t block_dim, int64_t n, const double* x, const double* p,
                                   double sigma, double* dx, double* dp);
/* Shared mean vector: every point i runs
 * gaussnd_grad_0_1(x[:, i], p, sigma, dim, dx[:, i], dp) with ONE p[dim] and
 * ONE shared slot dp[dim] — a shared-write hazard the reference refuses
 * (launch.cpp:217-224, same message) unless `unsafe`.  Forced, dx[:, i]
 * accumulates privately (dx may be NULL) and dp[d] += sum_i -_r6_{d,i} is
 * reduced in a fixed order (no atomics; the same bits on every run and
 * device).  Device pointers, stream-ordered. */
int adc_cuda_gaussnd_grad_shared_p(int64_t n, int64_t dim, int64_t ld, const double* x,
                                   const double* p, double sigma, double* dx, double* dp,
                                   int32_t unsafe, void* stream);
/* The same over the points of several ranks (the shared-p
 * variant's one all-reduce of dp[dim]): each rank passes its own n points and
 * the same p; every rank's dp partial (its points in the single-device fixed
 * order) is all-gathered through `comm` (NCCL, or the host / peer transport's
 * all-gather callback) and summed in rank order, so every rank ends with the
 * same dp bits; at world 1 the result is the single-device one bit for bit. */
int adc_cuda_gaussnd_grad_shared_p_comm(int64_t n, int64_t dim, int64_t ld, const double* x,
                                        const double* p, double sigma, double* dx, double* dp,
                                        int32_t unsafe, adc_comm* comm, void* stream);
/* Kernel selection for the calling thread (parity tests): 0 = auto,
 * 2 = dims over the warps of a 32-point tile, 3 = one warp per 32-point tile
 * (reference summation order), 10 = two points per lane (double2); + 100 runs
 * the same kernel on the static grid-stride schedule instead of claimed
 * spans (same bits). */
int adc_cuda_gaussnd_set_variant(int32_t variant);

/* ---------------------------------------------------------------------------
 * Generic lowering: a DSL module as the reference prints it
 * (adc::print(Module): a Listing-style `global` kernel plus the generated
 * gradients it calls, e.g. after ensure_called_derivatives) is translated to
 * CUDA C++ and compiled for sm_100a with NVRTC.  Each real op is one IEEE
 * double op in source order, value/control tapes are per call frame in
 * thread-private memory (tape_capacity entries each; 0 = 256), and the
 * interpreter's domain errors (eval.cpp) come back as ADC_E_EVAL.
 * adc_jit_* need no device (parse, hazard check, emission, NVRTC);
 * adc_cuda_jit_* launch.  A kernel with a shared-write hazard
 * (launch.cpp:261-267) is refused with the reference's message unless
 * `unsafe`, which turns indexed += into atomic adds (order unspecified, as
 * the reference's forced parallel mode). */
typedef struct adc_jit_module adc_jit_module;
/* One kernel parameter: real[] -> ptr + len (elements), real -> real_value,
 * integer -> int_value.  Device pointers for adc_cuda_jit_launch, host
 * pointers (copied in and back) for adc_cuda_jit_launch_host. */
typedef struct adc_jit_arg {
  double* ptr;
  int64_t len;
  double real_value;
  int64_t int_value;
} adc_jit_arg;
int adc_jit_compile(const char* module_source, const char* kernel, int32_t unsafe,
                    int32_t tape_capacity, adc_jit_module** out);
int adc_jit_destroy(adc_jit_module* module);
/* kinds[i]: 0 = real[], 1 = real, 2 = integer (kernel parameter order). */
int adc_jit_kernel_params(const adc_jit_module* module, int32_t* nparams, int32_t* kinds,
                          int32_t cap);
const char* adc_jit_kernel_param_name(const adc_jit_module* module, int32_t index);
const char* adc_jit_cuda_source(const adc_jit_module* module);
/* Tape elimination: where every tape push/pop sits
 * at a compile-time depth, launches run a static-tape variant whose entries
 * are locals (registers) instead of the per-frame tape arrays — for kernels
 * with integer parameters specialised per tuple of integer arguments (loops
 * with those trip counts unrolled), built by NVRTC on first use.  Same
 * operations in the same order: the same bits.  This returns the CUDA source
 * of the variant a launch with these integer arguments (kernel parameter
 * order, integers only) uses, or *cuda_source = NULL when it runs the
 * dynamic-tape kernel (adc_jit_cuda_source). */
int adc_jit_static_variant(adc_jit_module* module, const int64_t* int_args, int32_t nint,
                           const char** cuda_source);
size_t adc_jit_cubin_size(const adc_jit_module* module);
/* LaunchConfig semantics (launch.cpp:9-19): grid x block threads, the
 * kernel's own `i < N` guard idles the padding.  Synchronous on `stream`. */
int adc_cuda_jit_launch(adc_jit_module* module, int64_t grid_dim, int64_t block_dim, int64_t n,
                        const adc_jit_arg* args, int32_t nargs, void* stream);
int adc_cuda_jit_launch_host(adc_jit_module* module, int64_t grid_dim, int64_t block_dim,
                             int64_t n, const adc_jit_arg* args, int32_t nargs);
/* The same launch with the reference's LaunchStats (launch.hpp:58-61): the
 * counting variant of the kernel (built on first use) adds every operation
 * the interpreter counts (eval.cpp: adds incl. unary minus and compound +=,
 * muls, divs, intrinsics, if-comparisons, tape pushes and pops) into
 * counts[7] = {adds, muls, divs, intrinsics, comparisons, tape_pushes,
 * tape_pops} summed over all grid x block threads, and writes each thread's
 * kernel-frame statement count to thread_statements[grid x block] (device
 * memory for the device form, host memory for _host; may be NULL). */
int adc_cuda_jit_launch_counted(adc_jit_module* module, int64_t grid_dim, int64_t block_dim,
                                int64_t n, const adc_jit_arg* args, int32_t nargs, void* stream,
                                uint64_t* counts, uint32_t* thread_statements);
int adc_cuda_jit_launch_counted_host(adc_jit_module* module, int64_t grid_dim,
                                     int64_t block_dim, int64_t n, const adc_jit_arg* args,
                                     int32_t nargs, uint64_t* counts,
                                     uint32_t* thread_statements);

/* ---------------------------------------------------------------------------
 * chi2 histogram fit (FitEngine::chi2 / chi2_gradient, proj/src/fit.cpp:206-259)
 * for model-parameterised histograms.
 *
 * One pass over the bins accumulates, per fixed-size chunk of bins,
 *   [S, A1, A2, C0, G0[np], G1[np], G2[np]]     (value-only: [S, A1, A2, C0])
 * with S = sum m_j, A1 = sum_{c>0} m_j, A2 = sum_{c>0} m_j^2/c_j,
 * C0 = sum_{c>0} c_j, G0 = sum grad m_j, G1 = sum_{c>0} grad m_j,
 * G2 = sum_{c>0} (m_j/c_j) grad m_j, reduced in a FIXED order (no atomics).
 * adc_chi2_finalize turns the chunk records into chi2 and its gradient:
 *   a = E/S, chi2 = C0 - 2a A1 + a^2 A2, T = 2 A1 - 2a A2,
 *   grad = (E/S^2) T G0 - 2a G1 + 2a^2 G2
 * which is exact algebra on fit.cpp:231-258.  Chunk boundaries are the same
 * for every world size, so the result is bitwise independent of the number
 * of GPUs the chunks were computed on.
 */
enum { ADC_MODEL_GSUM = 0, ADC_MODEL_GPOLY = 1 };

typedef struct adc_chi2_layout {
  int64_t bins;
  int64_t tile_bins;   /* bins per tile (one CTA pass, fixed in-tile order) */
  int64_t chunk_tiles; /* tiles per chunk (fixed tree) */
  int64_t nchunks;     /* chunks over the whole histogram */
  int64_t chunk_begin; /* this rank's chunk range [chunk_begin, chunk_end) */
  int64_t chunk_end;
  int64_t bin_begin; /* this rank's bin range */
  int64_t bin_end;
} adc_chi2_layout;

/* Host-only (no device needed): the tiling and this rank's shard. */
int adc_chi2_make_layout(int64_t bins, int32_t world, int32_t rank, adc_chi2_layout* out);
/* Doubles per chunk record: 4 + 3*np (gradient) or 4 (value only). */
int32_t adc_chi2_record_len(int32_t np, int32_t want_grad);
/* Host-only: fixed-order tree over nchunks records, then the closed form
 * above.  grad may be NULL when want_grad == 0. */
int adc_chi2_finalize(int32_t np, double events, const double* records, int64_t nchunks,
                      int32_t want_grad, double* grad, double* chi2);

typedef struct adc_chi2_plan adc_chi2_plan;
/* counts: DEVICE pointer to the full histogram (float64[bins]); only this
 * rank's bin range is read.  The plan owns its workspace, a CUDA graph per
 * pass kind and a pinned result buffer.  What depends on the counts alone
 * (1/c per bin, 8 B/bin of device memory, and the q-independent chunk sums)
 * is computed once, before the first pass: call adc_cuda_chi2_plan_refresh
 * after changing the counts in place. */
int adc_cuda_chi2_plan_create(adc_chi2_plan** plan, int32_t model, int32_t np, int64_t bins,
                              double lo, double hi, double events, const double* counts,
                              int32_t world, int32_t rank, void* stream);
int adc_cuda_chi2_plan_destroy(adc_chi2_plan* plan);
int adc_cuda_chi2_plan_refresh(adc_chi2_plan* plan);
int adc_cuda_chi2_plan_layout(const adc_chi2_plan* plan, adc_chi2_layout* out);
/* Enqueue this rank's pass: chunk records for [chunk_begin, chunk_end) are
 * written to records_dev + (chunk - chunk_begin) * record_len (device
 * pointer; NULL = the plan's own buffer, readable via
 * adc_cuda_chi2_plan_records).  Stream-ordered, asynchronous. */
/* chi2 values of high-count histograms.  The single pass forms chi2 as
 * C0 - 2a A1 + a^2 A2 from sums of magnitude E (events), so its relative
 * rounding error is ~5 eps kappa, kappa = C0 / non-empty bins (the counts
 * per bin).  A whole-histogram plan with kappa > 256 computes every chi2
 * VALUE it returns (adc_cuda_chi2, _multi, the gradient's chi2 output, the
 * fit's line search) as sum (c - a m)^2 / c directly in a second pass (K3r)
 * with a = E/S from the first; its passes then run precision mode 1 (the
 * residual pass and the S it uses see the same m) and the fit runs its host
 * loop.  *residual = 1 in that mode; *kappa = C0 / non-empty bins. */
int adc_cuda_chi2_value_mode(adc_chi2_plan* plan, int32_t* residual, double* kappa);
/* Measurement hook: with timing on, adc_cuda_chi2_partials records CUDA
 * events around the pass's tile kernel (the dominant one) on its stream;
 * adc_cuda_chi2_kernel_ms waits for and returns the last such duration. */
int adc_cuda_chi2_set_kernel_timing(adc_chi2_plan* plan, int32_t on);
int adc_cuda_chi2_kernel_ms(adc_chi2_plan* plan, float* ms);
int adc_cuda_chi2_partials(adc_chi2_plan* plan, const double* q, int32_t want_grad,
                           double* records_dev);
double* adc_cuda_chi2_plan_records(adc_chi2_plan* plan);
/* Pass + exchange + finalize, synchronous: whole-histogram plans, or sharded
 * plans with a communicator attached (adc_cuda_chi2_plan_set_comm).
 * FitEngine::chi2_gradient(h, q, AdReverse, out) and FitEngine::chi2(h, q). */
int adc_cuda_chi2_gradient(adc_chi2_plan* plan, const double* q, double* grad, double* chi2);
int adc_cuda_chi2(adc_chi2_plan* plan, const double* q, double* chi2);
/* chi2 of ncand (<= 64) parameter vectors qs[ncand][np] in ONE pass over the
 * bins (fast mode): each result is bit-identical to adc_cuda_chi2 on that
 * vector.  The fit loop uses it to evaluate the Armijo trials t = 1, 1/2, ...
 * of fit.cpp:390-403 in batches.  Sharded plans need a communicator. */
int adc_cuda_chi2_multi(adc_chi2_plan* plan, const double* qs, int32_t ncand, double* chi2s);
/* Gradients (and nothing else) of ncand (<= 64) parameter vectors: ncand
 * ordinary gradient passes enqueued back to back, one copy back, one sync;
 * each result equals adc_cuda_chi2_gradient on that vector.  Used for the
 * 2*np central-difference probes of the Newton option.  Sharded plans need a
 * communicator. */
int adc_cuda_chi2_gradient_multi(adc_chi2_plan* plan, const double* qs, int32_t ncand,
                                 double* grads);
/* adc::GradientProvider (proj/include/adc/fit.hpp:52) of the gradient passes
 * (chi2_gradient, the fit loop and its Hessian probes):
 * ADC_PROVIDER_AD_REVERSE (default) = the generated <model>_grad_1;
 * ADC_PROVIDER_NUMERIC = central differences of the model over q per bin,
 * h_i = cbrt(eps) max(1, |q_i|), two model evaluations per parameter
 * (FitEngine::model_gradient, fit.cpp:187-190 -> numdiff.cpp:38-87). */
enum { ADC_PROVIDER_AD_REVERSE = 0, ADC_PROVIDER_NUMERIC = 1 };
int adc_cuda_chi2_set_provider(adc_chi2_plan* plan, int32_t provider);
/* Selects per-bin arithmetic: 0 = faithful (IEEE divisions exactly as the
 * generated code), 1 = fast (reciprocal multiplies, table-driven exp; within
 * the reduction tolerance), 2 = fast, and every pass (gradient, value,
 * batched line search) evaluates each thread's run of Gaussian factors
 * exp(-z^2/2) by an anchored product recurrence (two multiplies per bin,
 * <= bpt + 2 ulp; models with <= 2 Gaussian factors, runs of >= 16 bins that
 * span at most one sigma).  Default 2. */
int adc_cuda_chi2_set_precision(adc_chi2_plan* plan, int32_t mode);

/* ---------------------------------------------------------------------------
 * Multi-GPU exchange.  One process per GPU; each rank's plan
 * covers a contiguous range of whole chunks (adc_chi2_make_layout) and the one
 * exchange step of every pass is an all-gather of the chunk records (<= 32 KB
 * at 1e8 bins), after which every rank runs the same fixed-order finalize.
 * The result is therefore bitwise identical on every rank and for every world
 * size.  With a communicator attached, every plan entry point below
 * (adc_cuda_chi2, _gradient, _multi, _gradient_multi, adc_cuda_fit) works on
 * a sharded plan exactly as on a whole-histogram plan.
 *
 * Three transports (the third, peer memory, is declared below):
 *  - NCCL (the product path on NVLink/NVSwitch): ncclAllGather enqueued on the
 *    plan's stream right after the chunk kernel, captured into the same CUDA
 *    graph as the pass.  Rank 0 calls adc_nccl_unique_id and the caller
 *    distributes the 128 bytes (MPI, torch.distributed, a file, ...).
 *  - host callback: the caller's own all-gather over host memory (MPI_Allgather,
 *    gloo, ...): fn(ctx, send, recv, bytes) must place every rank's `bytes`
 *    bytes at recv + rank * bytes and return 0.  Used to run several ranks on
 *    one GPU in tests.
 * (adc_comm is declared above, with adc_cuda_gaussnd_grad_shared_p_comm.)
 */
typedef int (*adc_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);
enum { ADC_COMM_NCCL = 1, ADC_COMM_HOST = 2, ADC_COMM_PEER = 3 };
int adc_nccl_unique_id(unsigned char id[128]);
/* Collective over the world: every rank calls it with the same id, on the
 * device it will run its plan on (the current device). */
int adc_cuda_comm_init_nccl(adc_comm** comm, const unsigned char id[128], int32_t world,
                            int32_t rank);
int adc_comm_init_host(adc_comm** comm, int32_t world, int32_t rank, adc_allgather_fn fn,
                       void* ctx);
/* Peer memory (no NCCL on the pass path): each plan's receive buffer is
 * exported with CUDA IPC and opened by every rank (the bootstrap all-gather
 * `fn` exchanges the 64-byte handles once, when a plan attaches the comm).
 * A pass then publishes its chunk records straight into every peer's buffer
 * from the GPU (NVLink stores), raises a system-scope flag per peer and
 * waits for every peer's flag — one small kernel after the chunk kernel,
 * captured in the pass's CUDA graph.  All ranks must live on one node (on
 * distinct GPUs, or sharing one).  The wait for the peers' flags is bounded:
 * after ADC_PEER_TIMEOUT_S seconds (environment, default 120, 0 = unbounded)
 * the kernel traps and the call fails with ADC_E_CUDA (the CUDA context of
 * that process is lost) instead of spinning on the GPU forever. */
int adc_cuda_comm_init_peer(adc_comm** comm, int32_t world, int32_t rank, adc_allgather_fn fn,
                            void* ctx);
int adc_comm_destroy(adc_comm* comm);
int adc_comm_info(const adc_comm* comm, int32_t* world, int32_t* rank, int32_t* kind);
/* Attaches comm (NULL detaches) to a plan created with the same world/rank.
 * The plan does not own the communicator. */
int adc_cuda_chi2_plan_set_comm(adc_chi2_plan* plan, adc_comm* comm);
/* One call for a rank that holds only its own shard: world/rank come from
 * comm, shard_counts is a DEVICE pointer to counts[bin_begin, bin_end) of the
 * layout adc_chi2_make_layout(bins, world, rank) gives, and comm is attached.
 * A rank the layout gives no bins (more ranks than chunks) may pass NULL. */
int adc_cuda_chi2_plan_create_sharded(adc_chi2_plan** plan, int32_t model, int32_t np,
                                      int64_t bins, double lo, double hi, double events,
                                      const double* shard_counts, adc_comm* comm, void* stream);

/* On-device histogram sampling (the reference's
 * sample_histogram, fit.cpp:70-104, draws events by rejection and cannot feed
 * 1e8 bins): counts_dev[j] ~ Poisson(events * m_j / sum_k m_k) with m the
 * model at q (faithful per-bin arithmetic), every zero_every-th bin forced to
 * 0 (0 = none).  Counter-based Philox4x32-10 keyed by seed: the histogram is a
 * pure function of the arguments on any device.  *total = sum of the counts
 * (the Histogram's `events`, as the reference sampler guarantees).
 * Synchronous on `stream`. */
int adc_cuda_histogram_sample(int32_t model, int32_t np, const double* q, int64_t bins, double lo,
                              double hi, double events, uint64_t seed, int64_t zero_every,
                              double* counts_dev, double* total, void* stream);

/* Histogram ingest format (the reference's Histogram, fit.hpp:23-34, on
 * disk; shared with the oracle's readers): little-endian
 *   char magic[8] = "ADCHIST1"; int64 bins; double lo, hi, events;
 *   double counts[bins].
 * adc_histogram_write takes host or device counts (copied through a pinned
 * bounce buffer in 64 MiB pieces); adc_histogram_read_header fills the
 * scalars; adc_histogram_read_counts reads the counts into host or device
 * memory (device: pinned pieces, H2D overlapped with the file reads).
 * Errors: ADC_E_ARG (bad magic, short file, bins mismatch). */
int adc_histogram_write(const char* path, int64_t bins, double lo, double hi, double events,
                        const double* counts);
int adc_histogram_read_header(const char* path, int64_t* bins, double* lo, double* hi,
                              double* events);
int adc_histogram_read_counts(const char* path, int64_t bins, double* counts);

/* ---------------------------------------------------------------------------
 * Fit loop (FitEngine::fit, proj/src/fit.cpp:315-425: steepest descent or the
 * optional damped Newton step from a central-difference Hessian of the
 * gradient, Armijo backtracking, sigma clamp) driven on the host over the
 * device passes.
 * clamp_idx lists the parameters the sigma clamp applies to (fit.cpp:268-278
 * hard-codes every third index; gsum passes 2,5,8,..., gpoly passes 2). */
typedef struct adc_fit_options {
  int32_t budget;        /* 400 */
  double grad_tol;       /* 1e-6 */
  double chi2_rel_tol;   /* 1e-12 */
  double sigma_min;      /* 1e-3 */
  double armijo_c1;      /* 1e-4 */
  int32_t trace_iterates;
  int32_t use_hessian;   /* 0; Newton step from a numeric Hessian of the gradient (fit.cpp:346-381) */
  int32_t host_loop;     /* 0: the device-resident loop where the plan allows it; 1: the
                            host-driven loop over graph-replayed passes (the same bits) */
} adc_fit_options;

typedef struct adc_fit_result {
  double chi2;
  int32_t iterations;
  int32_t converged;
  int32_t sigma_clamps;
  uint64_t gradient_evals;
  uint64_t chi2_evals;
  uint64_t gradient_ns; /* time in gradient passes (fit.cpp:332-336): host wall clock in
                           the host loop, the device's %globaltimer in the device loop */
} adc_fit_result;

void adc_fit_default_options(adc_fit_options* o);
/* params: in = init (np), out = final.  iterates: trace_iterates * np doubles
 * (or NULL).  Single device, or every rank of a sharded plan with a
 * communicator attached (all ranks take the same steps).  With the fast
 * passes (precision mode >= 1) on one device or over the peer transport, the
 * whole loop runs on the device: one CUDA graph whose WHILE node repeats the
 * iteration (gradient pass, finalize, Newton probes and solve when
 * use_hessian, batched Armijo trials, selection, bookkeeping); the host only
 * continues a line search that needs more trials than one batch.  NCCL and
 * host-callback plans, and mode 0, run the same passes from a host loop.
 * Both loops give the same bits. */
int adc_cuda_fit(adc_chi2_plan* plan, double* params, const int32_t* clamp_idx, int32_t nclamp,
                 const adc_fit_options* opts, adc_fit_result* result, double* iterates);

#ifdef __cplusplus
}
#endif
#endif /* ADC_CUDA_H */
