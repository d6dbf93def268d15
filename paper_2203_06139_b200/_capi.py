"""ctypes binding of the C ABI in include/adc_cuda.h (libadc_b200.so, in-tree).

The product path: every compute call goes to the CUDA library.  If the
library is missing this module raises at import — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libadc_b200.so")

# adc_status codes; 1..5 mirror adc::ErrorKind (proj/include/adc/diag.hpp:17-23).
ERROR_KINDS = {1: "Semantic", 2: "Transform", 3: "Eval", 4: "Launch", 5: "Io", 6: "Cuda", 7: "Arg",
               8: "Nccl"}
COMM_NCCL, COMM_HOST, COMM_PEER = 1, 2, 3
# int (*adc_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t)
MODEL_IDS = {"gsum": 0, "gpoly": 1}


class AdcError(RuntimeError):
    """Mirror of adc::Error (diag.hpp:29-37): one exception type with a kind."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


class Chi2Layout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "bins", "tile_bins", "chunk_tiles", "nchunks", "chunk_begin", "chunk_end", "bin_begin",
        "bin_end")]


class JitArg(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("len", ctypes.c_int64), ("real_value", ctypes.c_double),
                ("int_value", ctypes.c_int64)]


class FitOptions(ctypes.Structure):
    _fields_ = [("budget", ctypes.c_int32), ("grad_tol", ctypes.c_double),
                ("chi2_rel_tol", ctypes.c_double), ("sigma_min", ctypes.c_double),
                ("armijo_c1", ctypes.c_double), ("trace_iterates", ctypes.c_int32),
                ("use_hessian", ctypes.c_int32), ("host_loop", ctypes.c_int32)]


class FitResultC(ctypes.Structure):
    _fields_ = [("chi2", ctypes.c_double), ("iterations", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("sigma_clamps", ctypes.c_int32),
                ("gradient_evals", ctypes.c_uint64), ("chi2_evals", ctypes.c_uint64),
                ("gradient_ns", ctypes.c_uint64)]


_D = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p
_I64, _I32, _DBL = ctypes.c_int64, ctypes.c_int32, ctypes.c_double

# name -> (restype, argtypes); every symbol declared in include/adc_cuda.h.
SIGNATURES = {
    "adc_cuda_abi_version": (ctypes.c_int, []),
    "adc_cuda_last_error": (ctypes.c_char_p, []),
    "adc_cuda_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)] * 3),
    "adc_cuda_alloc": (ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_size_t]),
    "adc_cuda_free": (ctypes.c_int, [_VP]),
    "adc_cuda_copy": (ctypes.c_int, [_VP, _VP, ctypes.c_size_t, _I32]),
    "adc_cuda_synchronize": (ctypes.c_int, []),
    "adc_cuda_fingerprint": (ctypes.c_uint64, [ctypes.c_char_p, ctypes.c_size_t]),
    "adc_cuda_registry_find": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint64,
                                              ctypes.POINTER(_I32)]),
    "adc_cuda_registry_size": (_I32, []),
    "adc_cuda_registry_name": (ctypes.c_char_p, [_I32]),
    "adc_cuda_registry_fingerprint": (ctypes.c_uint64, [_I32]),
    "adc_cuda_compute_gauss": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP, _VP]),
    "adc_cuda_compute_gauss_host": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP]),
    "adc_cuda_compute_gauss_shared": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP,
                                                     _VP, _I32, _VP]),
    "adc_cuda_compute_gauss_shared_host": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP,
                                                          _VP, _VP, _I32]),
    "adc_cuda_gaussnd_grad": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP, _VP]),
    "adc_cuda_gaussnd_grad_host": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP]),
    "adc_cuda_gaussnd_grad_host_mg": (ctypes.c_int, [_I32, _VP, _I64, _I64, _I64, _VP, _VP, _DBL,
                                                      _VP, _VP]),
    "adc_cuda_compute_gauss_host_mg": (ctypes.c_int, [_I32, _VP, _I64, _I64, _I64, _VP, _VP, _DBL,
                                                       _VP, _VP]),
    "adc_cuda_gaussnd_set_variant": (ctypes.c_int, [_I32]),
    "adc_cuda_gaussnd_grad_shared_p": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP, _VP,
                                                      _I32, _VP]),
    "adc_cuda_gaussnd_grad_shared_p_comm": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP,
                                                           _VP, _I32, _VP, _VP]),
    "adc_cuda_compute_gauss_shared_comm": (ctypes.c_int, [_I64, _I64, _I64, _VP, _VP, _DBL, _VP,
                                                          _VP, _VP, _I32, _VP, _VP]),
    "adc_chi2_make_layout": (ctypes.c_int, [_I64, _I32, _I32, ctypes.POINTER(Chi2Layout)]),
    "adc_chi2_record_len": (_I32, [_I32, _I32]),
    "adc_chi2_finalize": (ctypes.c_int, [_I32, _DBL, _D, _I64, _I32, _D, _D]),
    "adc_cuda_chi2_plan_create": (ctypes.c_int, [ctypes.POINTER(_VP), _I32, _I32, _I64, _DBL,
                                                 _DBL, _DBL, _VP, _I32, _I32, _VP]),
    "adc_cuda_chi2_plan_destroy": (ctypes.c_int, [_VP]),
    "adc_cuda_chi2_plan_refresh": (ctypes.c_int, [_VP]),
    "adc_cuda_chi2_plan_layout": (ctypes.c_int, [_VP, ctypes.POINTER(Chi2Layout)]),
    "adc_cuda_chi2_partials": (ctypes.c_int, [_VP, _D, _I32, _VP]),
    "adc_cuda_chi2_set_kernel_timing": (ctypes.c_int, [_VP, _I32]),
    "adc_histogram_write": (ctypes.c_int, [ctypes.c_char_p, _I64, _DBL, _DBL, _DBL, _VP]),
    "adc_histogram_read_header": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_I64),
                                                 ctypes.POINTER(_DBL), ctypes.POINTER(_DBL),
                                                 ctypes.POINTER(_DBL)]),
    "adc_histogram_read_counts": (ctypes.c_int, [ctypes.c_char_p, _I64, _VP]),
    "adc_cuda_chi2_value_mode": (ctypes.c_int, [_VP, ctypes.POINTER(_I32),
                                                ctypes.POINTER(ctypes.c_double)]),
    "adc_cuda_chi2_kernel_ms": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_float)]),
    "adc_cuda_chi2_plan_records": (_VP, [_VP]),
    "adc_cuda_chi2_gradient": (ctypes.c_int, [_VP, _D, _D, _D]),
    "adc_cuda_chi2": (ctypes.c_int, [_VP, _D, _D]),
    "adc_cuda_chi2_multi": (ctypes.c_int, [_VP, _D, _I32, _D]),
    "adc_cuda_chi2_gradient_multi": (ctypes.c_int, [_VP, _D, _I32, _D]),
    "adc_cuda_chi2_set_precision": (ctypes.c_int, [_VP, _I32]),
    "adc_cuda_chi2_set_provider": (ctypes.c_int, [_VP, _I32]),
    "adc_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "adc_cuda_comm_init_nccl": (ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_char_p, _I32, _I32]),
    "adc_comm_init_host": (ctypes.c_int, [ctypes.POINTER(_VP), _I32, _I32, ALLGATHER_FN, _VP]),
    "adc_cuda_comm_init_peer": (ctypes.c_int, [ctypes.POINTER(_VP), _I32, _I32, ALLGATHER_FN, _VP]),
    "adc_comm_destroy": (ctypes.c_int, [_VP]),
    "adc_comm_info": (ctypes.c_int, [_VP, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                     ctypes.POINTER(_I32)]),
    "adc_cuda_chi2_plan_set_comm": (ctypes.c_int, [_VP, _VP]),
    "adc_cuda_chi2_plan_create_sharded": (ctypes.c_int, [ctypes.POINTER(_VP), _I32, _I32, _I64,
                                                         _DBL, _DBL, _DBL, _VP, _VP, _VP]),
    "adc_jit_compile": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _I32, _I32,
                                       ctypes.POINTER(_VP)]),
    "adc_jit_destroy": (ctypes.c_int, [_VP]),
    "adc_jit_kernel_params": (ctypes.c_int, [_VP, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                             _I32]),
    "adc_jit_kernel_param_name": (ctypes.c_char_p, [_VP, _I32]),
    "adc_jit_cuda_source": (ctypes.c_char_p, [_VP]),
    "adc_jit_static_variant": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                                              ctypes.POINTER(ctypes.c_char_p)]),
    "adc_jit_cubin_size": (ctypes.c_size_t, [_VP]),
    "adc_cuda_jit_launch": (ctypes.c_int, [_VP, _I64, _I64, _I64, ctypes.POINTER(JitArg), _I32,
                                           _VP]),
    "adc_cuda_jit_launch_host": (ctypes.c_int, [_VP, _I64, _I64, _I64, ctypes.POINTER(JitArg),
                                                _I32]),
    "adc_cuda_jit_launch_counted": (ctypes.c_int, [_VP, _I64, _I64, _I64, ctypes.POINTER(JitArg),
                                                   _I32, _VP, ctypes.POINTER(ctypes.c_uint64),
                                                   _VP]),
    "adc_cuda_jit_launch_counted_host": (ctypes.c_int, [_VP, _I64, _I64, _I64,
                                                        ctypes.POINTER(JitArg), _I32,
                                                        ctypes.POINTER(ctypes.c_uint64), _VP]),
    "adc_cuda_histogram_sample": (ctypes.c_int, [_I32, _I32, _D, _I64, _DBL, _DBL, _DBL,
                                                 ctypes.c_uint64, _I64, _VP, _D, _VP]),
    "adc_fit_default_options": (None, [ctypes.POINTER(FitOptions)]),
    "adc_cuda_fit": (ctypes.c_int, [_VP, _D, ctypes.POINTER(_I32), _I32,
                                    ctypes.POINTER(FitOptions), ctypes.POINTER(FitResultC), _D]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (make -C paper_2203_06139_b200/csrc). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int):
    if rc != 0:
        msg = lib.adc_cuda_last_error().decode()
        raise AdcError(ERROR_KINDS.get(rc, str(rc)), msg)


def dptr(a) -> ctypes.c_void_p:
    """Pointer of a torch tensor (device or host) or a numpy array."""
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


def dbl_array(values):
    arr = (ctypes.c_double * len(values))(*[float(v) for v in values])
    return arr
