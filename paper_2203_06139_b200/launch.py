"""Host-side mirror of the reference batch-dispatch API (proj/include/adc/launch.hpp)
over the B200 C ABI.

    cfg = LaunchConfig(n // 256 + 1, 256, n)
    buffers = BufferSet(arrays={"x": x, "p": p, "dx": dx, "dp": dp}, scalars={"sigma": 1.3})
    stats = launch("compute", cfg, buffers)          # adc::launch(prog, "compute", cfg, buffers)

Arrays may be numpy float64 arrays (host: the call copies in and out) or
torch float64 CUDA tensors (device: stream-ordered, no copies).  The kernel
is the Listing-1 `compute` (proj/corpus/kernels.dsl:9-14) whose callee is
looked up in the kernel registry by the gradient's name and fingerprint.

launch_batch is the NEW batched path for multi-dimensional per-point
gradients (the reference cannot express it safely): one
point per column of structure-of-arrays buffers.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict

import numpy as np

from ._capi import AdcError, check, dptr, lib

# The Listing-1 kernel signature (kernels.dsl:9) and the race_check verdict of
# the reference for it (launch.cpp:112-240; test_launch.cpp:60-65).
COMPUTE_PARAMS = (("x", "real[]"), ("p", "real[]"), ("sigma", "real"), ("dx", "real[]"),
                  ("dp", "real[]"))
COMPUTE_ACCESS = {"x": "shared-read", "p": "shared-read", "sigma": "shared-read",
                  "dx": "private-per-thread", "dp": "private-per-thread"}
COMPUTE_SHARED_HAZARD = {"dsigma": "whole array shared with a writing callee across threads"}


@dataclass
class LaunchConfig:
    """launch.hpp:15-21."""
    grid_dim: int = 0
    block_dim: int = 0
    n: int = 0

    def validate(self):
        """LaunchConfig::validate (launch.cpp:9-19), same messages."""
        if self.grid_dim <= 0 or self.block_dim <= 0 or self.n <= 0:
            raise AdcError("Launch", f"launch configuration must be positive (grid {self.grid_dim}"
                                     f", block {self.block_dim}, n {self.n})")
        if self.grid_dim * self.block_dim < self.n:
            raise AdcError("Launch", f"grid {self.grid_dim} x block {self.block_dim} does not "
                                     f"cover problem size {self.n}")


@dataclass
class BufferSet:
    """launch.hpp:46-50."""
    arrays: Dict[str, object] = field(default_factory=dict)
    scalars: Dict[str, float] = field(default_factory=dict)
    integers: Dict[str, int] = field(default_factory=dict)


@dataclass
class LaunchOptions:
    """launch.hpp:52-56.  `workers` and `sequential` have no meaning on the GPU
    (the result is identical for any of them) and are accepted for drop-in use."""
    unsafe: bool = False
    workers: int = 0
    sequential: bool = False


@dataclass
class LaunchStats:
    """launch.hpp:58-61.  Registered (hand-written) kernels: thread_statements
    is the Listing-1 shape's — 3 kernel-frame statements for g < n, 2 for the
    padding threads (test_launch.cpp:119-128), materialised on first access.
    JIT launches with counts=True carry the exact per-thread statements and
    the OpCounters sums (`counts`: adds, muls, divs, intrinsics, comparisons,
    tape_pushes, tape_pops) from the counting variant of the kernel."""
    active: int
    idle: int
    counts: dict | None = None
    statements: np.ndarray | None = None

    @property
    def thread_statements(self) -> np.ndarray:
        if self.statements is not None:
            return self.statements
        ts = np.full(self.active + self.idle, 2, dtype=np.uint32)
        ts[:self.active] = 3
        return ts


_FP = None
_FOUND = {}


def _fingerprints():
    """The registry's own (name -> fingerprint) table (include/adc_cuda.h);
    the registry is compiled in, so it is read once."""
    global _FP
    if _FP is None:
        _FP = {lib.adc_cuda_registry_name(i).decode(): lib.adc_cuda_registry_fingerprint(i)
               for i in range(lib.adc_cuda_registry_size())}
    return _FP


def registry_find(name: str, fingerprint: int) -> int:
    key = (name, fingerprint)
    if key in _FOUND:  # hits only: a miss always goes to the library (and raises)
        return _FOUND[key]
    import ctypes
    kid = ctypes.c_int32(-1)
    check(lib.adc_cuda_registry_find(name.encode(), fingerprint, ctypes.byref(kid)))
    _FOUND[key] = kid.value
    return kid.value


def printed_function(module: str, fn: str) -> str:
    """The text of function `fn` as adc::print emits it, cut out of a printed
    module (functions are separated by one blank line)."""
    for head in ("device host void ", "device host real ", "host void ", "device void "):
        i = module.find(head + fn + "(")
        if i >= 0:
            break
    else:
        raise AdcError("Launch", f"function '{fn}' not found in the module text")
    k = module.find("\n}\n", i)
    if k < 0:
        raise AdcError("Launch", f"function '{fn}' is not terminated in the module text")
    return module[i:k + 3]


def fingerprint_of(text: str) -> int:
    """FNV-1a-64 of a printed generated gradient: the registry key the
    reference-side bridge computes from adc::print(FunctionDef)."""
    b = text.encode()
    return int(lib.adc_cuda_fingerprint(b, len(b)))


def _callee_fingerprint(callee: str, fingerprint: int | None, module: str | None) -> int:
    """Registry key of the called gradient.  With the Program's printed text
    (`module`), the fingerprint is computed from the gradient actually printed
    there, so a changed generator output is a registry miss (an
    Error(Launch)), as in the reference-side bridge.  Without it the caller
    vouches for the gradient by name and the registry's own fingerprint is
    used."""
    if fingerprint is not None:
        return fingerprint
    if module is not None:
        return fingerprint_of(printed_function(module, callee))
    return _fingerprints()[callee]


def _is_torch(a) -> bool:
    return hasattr(a, "is_cuda")


def _check_residency(arrays, what="buffers"):
    """All device buffers are float64 CUDA tensors on ONE device, or all are
    host float64 arrays: a host pointer never reaches a kernel."""
    arrays = [a for a in arrays if a is not None]
    dev = {_is_torch(a) and a.is_cuda for a in arrays}
    if len(dev) != 1:
        raise AdcError("Launch", f"{what}: mix of device (CUDA tensor) and host buffers")
    if dev.pop():
        devices = {a.device for a in arrays}
        if len(devices) != 1:
            raise AdcError("Launch", f"{what}: CUDA tensors on different devices {sorted(map(str, devices))}")
        return next(iter(devices))
    for a in arrays:
        if _is_torch(a):
            raise AdcError("Launch", f"{what}: CPU torch tensors are not accepted; pass numpy arrays")
    return None


class _on_device:
    """Runs the C call with the buffers' device current (the C ABI launches on
    the calling thread's current device)."""

    def __init__(self, device):
        self.device = device
        self.ctx = None

    def __enter__(self):
        if self.device is not None:
            import torch
            self.ctx = torch.cuda.device(self.device)
            self.ctx.__enter__()

    def __exit__(self, *a):
        if self.ctx is not None:
            self.ctx.__exit__(*a)


def _stream_of(a):
    import torch
    return torch.cuda.current_stream(a.device).cuda_stream


def launch(kernel: str, cfg: LaunchConfig, buffers: BufferSet,
           opts: LaunchOptions | None = None, callee_fingerprint: int | None = None,
           module: str | None = None, counts: bool = False, comm=None,
           devices=None) -> LaunchStats:
    """adc::launch (launch.cpp:252-346) for the Listing-1 kernels of kernels.dsl:
    `compute` (private slots) and `compute_shared` (the shared dsigma slot:
    refused unless opts.unsafe, then reduced in a fixed order, deterministic),
    on their hand-written kernels.  With `module` (the Program's text as
    adc::print emits it), any other global kernel goes through the generic
    JIT (jit.py).  `compute_shared` with `comm` (device buffers): each rank
    launches over its own points and the dsigma partials are summed over
    ranks in rank order (the same dsigma on every rank).  `compute` with host
    buffers and `devices` (device ordinals): the points are split over those
    GPUs, one host thread each (adc_cuda_compute_gauss_host_mg)."""
    opts = opts or LaunchOptions()
    if module is not None and kernel not in ("compute", "compute_shared"):
        from .jit import launch_module
        return launch_module(module, kernel, cfg, buffers, opts, counts=counts)
    cfg.validate()
    shared = kernel == "compute_shared"
    if shared:
        # race_check reports dsigma as a shared-write hazard (launch.cpp:261-267).
        if not opts.unsafe:
            raise AdcError("Launch", "launch refused, hazardous parameter(s): dsigma (whole array "
                                     "shared with a writing callee across threads); pass the "
                                     "unsafe flag to force")
    elif kernel != "compute":
        raise AdcError("Launch", f"unknown kernel '{kernel}'")
    callee = "gauss_grad" if shared else "gauss_grad_0_1"
    registry_find(callee, _callee_fingerprint(callee, callee_fingerprint, module))
    arrs = {}
    for name, typ in COMPUTE_PARAMS:
        if typ == "real[]":
            if name not in buffers.arrays:
                raise AdcError("Launch", f"missing buffer '{name}'")
            a = buffers.arrays[name]
            ln = a.numel() if _is_torch(a) else a.size
            if ln < cfg.n:  # every array of `compute` is indexed by the thread (launch.cpp:279-284)
                raise AdcError("Launch", f"buffer '{name}' has length {ln} but is indexed by thread"
                                         f" over {cfg.n} elements")
            arrs[name] = a
        elif name not in buffers.scalars:
            raise AdcError("Launch", f"missing scalar value '{name}'")
    sigma = float(buffers.scalars["sigma"])
    x, p, dx, dp = (arrs[k] for k in ("x", "p", "dx", "dp"))
    device = _check_residency((x, p, dx, dp) + ((buffers.arrays.get("dsigma"),) if shared else ()))
    for a in (x, p, dx, dp):
        if _is_torch(x):
            if not (_is_torch(a) and a.is_cuda and a.is_contiguous()) or \
                    str(a.dtype) != "torch.float64":
                raise AdcError("Launch", "device buffers must be contiguous float64 CUDA tensors")
        elif _is_torch(a) or a.dtype != np.float64 or not a.flags.c_contiguous:
            raise AdcError("Launch", "host buffers must be contiguous float64 arrays")
    with _on_device(device):
        return _launch_compute(cfg, buffers, shared, x, p, dx, dp, sigma, comm, devices)


def _launch_compute(cfg, buffers, shared, x, p, dx, dp, sigma, comm, devices):
    if shared:
        if "dsigma" not in buffers.arrays:
            raise AdcError("Launch", "missing buffer 'dsigma'")
        ds = buffers.arrays["dsigma"]
        if (ds.numel() if _is_torch(ds) else ds.size) < 1:
            raise AdcError("Launch", "buffer 'dsigma' is empty")
        if comm is not None:
            if not _is_torch(x):
                raise AdcError("Launch", "compute_shared over ranks takes device buffers")
            check(lib.adc_cuda_compute_gauss_shared_comm(
                cfg.grid_dim, cfg.block_dim, cfg.n, dptr(x), dptr(p), sigma, dptr(dx), dptr(dp),
                dptr(ds), 1, comm._p, _stream_of(x)))
        elif _is_torch(x):
            check(lib.adc_cuda_compute_gauss_shared(cfg.grid_dim, cfg.block_dim, cfg.n, dptr(x),
                                                    dptr(p), sigma, dptr(dx), dptr(dp), dptr(ds),
                                                    1, _stream_of(x)))
        else:
            check(lib.adc_cuda_compute_gauss_shared_host(cfg.grid_dim, cfg.block_dim, cfg.n,
                                                         dptr(x), dptr(p), sigma, dptr(dx),
                                                         dptr(dp), dptr(ds), 1))
        return LaunchStats(active=cfg.n, idle=cfg.grid_dim * cfg.block_dim - cfg.n)
    if _is_torch(x):
        check(lib.adc_cuda_compute_gauss(cfg.grid_dim, cfg.block_dim, cfg.n, dptr(x), dptr(p),
                                         sigma, dptr(dx), dptr(dp), _stream_of(x)))
    elif devices is not None:
        import ctypes
        devs = (ctypes.c_int32 * len(devices))(*devices)
        check(lib.adc_cuda_compute_gauss_host_mg(len(devices), devs, cfg.grid_dim, cfg.block_dim,
                                                 cfg.n, dptr(x), dptr(p), sigma, dptr(dx),
                                                 dptr(dp)))
    else:
        check(lib.adc_cuda_compute_gauss_host(cfg.grid_dim, cfg.block_dim, cfg.n, dptr(x),
                                              dptr(p), sigma, dptr(dx), dptr(dp)))
    return LaunchStats(active=cfg.n, idle=cfg.grid_dim * cfg.block_dim - cfg.n)


def _soa_ld(arrays, ld):
    """Leading dimension (elements between dims) shared by the SoA buffers:
    each must be (dim, n) float64 with unit point stride and the same row
    stride (views with a row stride > n, e.g. x[:, a:b], are fine)."""
    strides = set()
    for a in arrays:
        if a is None:
            continue
        if _is_torch(a):
            if str(a.dtype) != "torch.float64" or a.dim() != 2 or (a.shape[1] > 1 and a.stride(1) != 1):
                raise AdcError("Launch", "SoA buffers must be float64 (dim, n) with unit point stride")
            strides.add(a.stride(0))
        else:
            if a.dtype != np.float64 or a.ndim != 2 or (a.shape[1] > 1 and a.strides[1] != 8):
                raise AdcError("Launch", "SoA buffers must be float64 (dim, n) with unit point stride")
            strides.add(a.strides[0] // 8)
    if len(strides) != 1:
        raise AdcError("Launch", "SoA buffers must share one row stride")
    stride = strides.pop()
    if ld is not None and ld != stride:
        raise AdcError("Launch", f"ld {ld} differs from the buffers' row stride {stride}")
    return stride


def launch_batch(grad_fn: str, x, p, sigma: float, dx, dp, ld: int | None = None,
                 callee_fingerprint: int | None = None, module: str | None = None,
                 devices=None):
    """Batched per-point gradient over structure-of-arrays buffers of shape
    (dim, n): gaussnd_grad_0_1(x[:, i], p[:, i], sigma, dim, dx[:, i], dp[:, i])
    for every point i, accumulating into dx, dp.  Host buffers with `devices`
    (a list of device ordinals): the points are split over those GPUs, one
    host thread each (adc_cuda_gaussnd_grad_host_mg), the same bits as one
    device."""
    if grad_fn != "gaussnd_grad_0_1":
        raise AdcError("Launch", f"no B200 kernel registered for '{grad_fn}'")
    registry_find(grad_fn, _callee_fingerprint(grad_fn, callee_fingerprint, module))
    device = _check_residency((x, p, dx, dp))
    if len(x.shape) != 2:
        raise AdcError("Launch", "SoA buffers must be float64 (dim, n) with unit point stride")
    dim, n = x.shape
    for name, a in (("p", p), ("dx", dx), ("dp", dp)):
        if tuple(a.shape) != (dim, n):  # launch.cpp:279-284: no buffer may be shorter
            raise AdcError("Launch", f"buffer '{name}' has shape {tuple(a.shape)} but the points are "
                                     f"x's ({dim}, {n})")
    ld = _soa_ld((x, p, dx, dp), ld)
    with _on_device(device):
        if device is not None:
            check(lib.adc_cuda_gaussnd_grad(n, dim, ld, dptr(x), dptr(p), float(sigma), dptr(dx),
                                            dptr(dp), _stream_of(x)))
        elif devices is not None:
            import ctypes
            devs = (ctypes.c_int32 * len(devices))(*devices)
            check(lib.adc_cuda_gaussnd_grad_host_mg(len(devices), devs, n, dim, ld, dptr(x),
                                                    dptr(p), float(sigma), dptr(dx), dptr(dp)))
        else:
            check(lib.adc_cuda_gaussnd_grad_host(n, dim, ld, dptr(x), dptr(p), float(sigma),
                                                 dptr(dx), dptr(dp)))


def launch_batch_shared_p(grad_fn: str, x, p, sigma: float, dx, dp,
                          opts: LaunchOptions | None = None, ld: int | None = None,
                          callee_fingerprint: int | None = None, comm=None,
                          module: str | None = None):
    """The shared-mean batched path: for every point i,
    gaussnd_grad_0_1(x[:, i], p, sigma, dim, dx[:, i], dp) with ONE p (dim,)
    and ONE shared slot dp (dim,) — refused as a shared-write hazard unless
    opts.unsafe; forced, dp is reduced in a fixed order (deterministic).  dx
    may be None.  Device (CUDA tensor) buffers.  With `comm` (a Comm), x / dx
    hold this rank's points and every rank's dp partial is all-gathered and
    summed in rank order: the same dp on every rank."""
    opts = opts or LaunchOptions()
    if grad_fn != "gaussnd_grad_0_1":
        raise AdcError("Launch", f"no B200 kernel registered for '{grad_fn}'")
    registry_find(grad_fn, _callee_fingerprint(grad_fn, callee_fingerprint, module))
    if not _is_torch(x):
        raise AdcError("Launch", "launch_batch_shared_p takes device (CUDA tensor) buffers")
    device = _check_residency((x, p, dx, dp))
    if len(x.shape) != 2:
        raise AdcError("Launch", "SoA buffers must be float64 (dim, n) with unit point stride")
    dim, n = x.shape
    if dx is not None and tuple(dx.shape) != (dim, n):
        raise AdcError("Launch", f"buffer 'dx' has shape {tuple(dx.shape)} but the points are "
                                 f"x's ({dim}, {n})")
    for name, a in (("p", p), ("dp", dp)):
        if str(a.dtype) != "torch.float64" or not a.is_contiguous() or a.numel() < dim:
            raise AdcError("Launch", f"buffer '{name}' must be a contiguous float64 vector of at "
                                     f"least dim = {dim} elements (has {a.numel()})")
    ld = _soa_ld((x, dx), ld)
    with _on_device(device):
        _shared_p_call(n, dim, ld, x, p, sigma, dx, dp, opts, comm)


def _shared_p_call(n, dim, ld, x, p, sigma, dx, dp, opts, comm):
    if comm is not None:
        check(lib.adc_cuda_gaussnd_grad_shared_p_comm(
            n, dim, ld, dptr(x), dptr(p), float(sigma), dptr(dx) if dx is not None else None,
            dptr(dp), 1 if opts.unsafe else 0, comm._p, _stream_of(x)))
        return
    check(lib.adc_cuda_gaussnd_grad_shared_p(n, dim, ld, dptr(x), dptr(p), float(sigma),
                                             dptr(dx) if dx is not None else None, dptr(dp),
                                             1 if opts.unsafe else 0, _stream_of(x)))


def set_gaussnd_variant(v: int):
    check(lib.adc_cuda_gaussnd_set_variant(v))
