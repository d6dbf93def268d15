"""B200-native batched reverse-mode gradient engine (arxiv/paper_2203_06139 hot path).

The compute path is libadc_b200.so (hand-written sm_100a CUDA behind the C ABI
of include/adc_cuda.h); this package is the host-side mirror of the
reference's launch/fit interfaces over that ABI.  Importing it without the
built library raises: there is no CPU fallback.
"""
from ._capi import AdcError, LIB_PATH, lib  # noqa: F401
from .launch import (BufferSet, LaunchConfig, LaunchOptions, LaunchStats, launch,  # noqa: F401
                     launch_batch, launch_batch_shared_p, registry_find)
from .comm import Comm  # noqa: F401
from .jit import JitModule, launch_module  # noqa: F401
from .fit import (Chi2Plan, FitEngine, FitOptions, FitResult, GradientProvider,  # noqa: F401
                  Histogram, bench_csv, bench_scaling, chi2_layout,
                  default_truth, finalize, perturbed_init, record_len, sample_histogram)

__all__ = [
    "AdcError", "BufferSet", "Comm", "JitModule", "launch_module", "LaunchConfig", "LaunchOptions", "LaunchStats", "launch",
    "launch_batch", "launch_batch_shared_p", "registry_find", "Chi2Plan", "FitEngine", "FitOptions", "FitResult",
    "GradientProvider", "Histogram", "bench_csv", "bench_scaling", "chi2_layout",
    "default_truth", "perturbed_init", "sample_histogram", "finalize", "record_len",
]
