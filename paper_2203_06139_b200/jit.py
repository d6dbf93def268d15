"""Generic lowering of DSL kernels (include/adc_cuda.h, adc_jit_*): a module as
the reference prints it (adc::print(Module) after ensure_called_derivatives:
the Listing-style `global` kernel plus the generated gradients it calls) is
translated to CUDA C++ and compiled for sm_100a with NVRTC, then launched with
adc::launch's semantics (launch.cpp:252-346).

    mod = JitModule(module_text, "k_rational")
    mod.launch(LaunchConfig(n // 256 + 1, 256, n), BufferSet(arrays={...}))

Arrays may be numpy float64 arrays (host: copied in and back) or float64
CUDA tensors (device, in place).  A kernel with a shared-write hazard is
refused with the reference's message unless opts.unsafe.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Tuple

import numpy as np

from ._capi import AdcError, JitArg, check, lib
from .launch import BufferSet, LaunchConfig, LaunchOptions, LaunchStats

KINDS = {0: "real[]", 1: "real", 2: "integer"}


class JitModule:
    def __init__(self, module_source: str, kernel: str, unsafe: bool = False,
                 tape_capacity: int = 0):
        self.kernel = kernel
        self._p = ctypes.c_void_p()
        check(lib.adc_jit_compile(module_source.encode(), kernel.encode(), 1 if unsafe else 0,
                                  int(tape_capacity), ctypes.byref(self._p)))
        n = ctypes.c_int32()
        kinds = (ctypes.c_int32 * 64)()
        check(lib.adc_jit_kernel_params(self._p, ctypes.byref(n), kinds, 64))
        self.params = [(lib.adc_jit_kernel_param_name(self._p, i).decode(), KINDS[kinds[i]])
                       for i in range(n.value)]

    @property
    def cuda_source(self) -> str:
        return lib.adc_jit_cuda_source(self._p).decode()

    def static_source(self, integers=()):
        """CUDA source of the static-tape variant a launch with these integer
        arguments (kernel parameter order) runs, or None when it runs the
        dynamic-tape kernel (tape entries in thread-private arrays)."""
        vals = (ctypes.c_int64 * max(1, len(integers)))(*[int(v) for v in integers])
        out = ctypes.c_char_p()
        check(lib.adc_jit_static_variant(self._p, vals, len(integers), ctypes.byref(out)))
        return out.value.decode() if out.value is not None else None

    @property
    def cubin_size(self) -> int:
        return lib.adc_jit_cubin_size(self._p)

    COUNT_FIELDS = ("adds", "muls", "divs", "intrinsics", "comparisons", "tape_pushes",
                    "tape_pops")

    def launch(self, cfg: LaunchConfig, buffers: BufferSet, counts: bool = False) -> LaunchStats:
        """adc::launch over this module's kernel.  counts=True runs the
        counting variant and returns the reference's LaunchStats exactly
        (OpCounters sums and every thread's kernel-frame statements)."""
        cfg.validate()
        args = (JitArg * max(1, len(self.params)))()
        device = None
        for i, (name, kind) in enumerate(self.params):
            if kind == "real[]":
                if name not in buffers.arrays:
                    raise AdcError("Launch", f"missing buffer '{name}'")
                a = buffers.arrays[name]
                is_dev = hasattr(a, "is_cuda")
                if device is None:
                    device = is_dev
                elif device != is_dev:
                    raise AdcError("Launch", "mixing host and device buffers")
                if is_dev:
                    if not (a.is_cuda and a.is_contiguous()) or str(a.dtype) != "torch.float64":
                        raise AdcError("Launch", "device buffers must be contiguous float64 CUDA "
                                                 "tensors")
                    args[i].ptr, args[i].len = a.data_ptr(), a.numel()
                else:
                    if a.dtype != np.float64 or not a.flags.c_contiguous:
                        raise AdcError("Launch", "host buffers must be contiguous float64 arrays")
                    args[i].ptr, args[i].len = a.ctypes.data, a.size
            elif kind == "real":
                if name not in buffers.scalars:
                    raise AdcError("Launch", f"missing scalar value '{name}'")
                args[i].real_value = float(buffers.scalars[name])
            else:
                if name not in buffers.integers:
                    raise AdcError("Launch", f"missing integer value '{name}'")
                args[i].int_value = int(buffers.integers[name])
        total = cfg.grid_dim * cfg.block_dim
        if counts:
            c = (ctypes.c_uint64 * 7)()
            if device:
                import torch
                stm = torch.zeros(total, dtype=torch.int32, device="cuda")
                stream = torch.cuda.current_stream().cuda_stream
                check(lib.adc_cuda_jit_launch_counted(
                    self._p, cfg.grid_dim, cfg.block_dim, cfg.n, args, len(self.params),
                    ctypes.c_void_p(stream), c, ctypes.c_void_p(stm.data_ptr())))
                stm = stm.cpu().numpy().view(np.uint32)
            else:
                stm = np.zeros(total, dtype=np.uint32)
                check(lib.adc_cuda_jit_launch_counted_host(
                    self._p, cfg.grid_dim, cfg.block_dim, cfg.n, args, len(self.params), c,
                    stm.ctypes.data_as(ctypes.c_void_p)))
            return LaunchStats(active=cfg.n, idle=total - cfg.n,
                               counts=dict(zip(self.COUNT_FIELDS, (int(v) for v in c))),
                               statements=stm)
        if device:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
            check(lib.adc_cuda_jit_launch(self._p, cfg.grid_dim, cfg.block_dim, cfg.n, args,
                                          len(self.params), ctypes.c_void_p(stream)))
        else:
            check(lib.adc_cuda_jit_launch_host(self._p, cfg.grid_dim, cfg.block_dim, cfg.n, args,
                                               len(self.params)))
        return LaunchStats(active=cfg.n, idle=total - cfg.n)

    def close(self):
        if self._p:
            lib.adc_jit_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: Dict[Tuple[str, str, bool, int], JitModule] = {}


def launch_module(module_source: str, kernel: str, cfg: LaunchConfig, buffers: BufferSet,
                  opts: LaunchOptions | None = None, tape_capacity: int = 0,
                  counts: bool = False) -> LaunchStats:
    """adc::launch(Program(module), kernel, cfg, buffers, opts) through the JIT;
    compiled modules are cached per (source, kernel, unsafe, tape capacity).
    counts=True returns the exact LaunchStats (see JitModule.launch)."""
    opts = opts or LaunchOptions()
    key = (module_source, kernel, bool(opts.unsafe), int(tape_capacity))
    mod = _cache.get(key)
    if mod is None:
        mod = JitModule(module_source, kernel, opts.unsafe, tape_capacity)
        _cache[key] = mod
    return mod.launch(cfg, buffers, counts)
