"""Generic lowering, host side (no device): every corpus kernel of the golden
module parses, passes the hazard gate exactly as the reference's race_check
does, is emitted as IEEE-exact CUDA and compiles for sm_100a with NVRTC."""
import numpy as np
import pytest

from conftest import golden

import paper_2203_06139_b200 as adc  # noqa: E402

G = golden("jit_cases.npz")
MODULE = str(G["module"])
CASES = ["gauss", "rational", "branchy", "poly", "looped", "gsum", "sumn", "hess"]


@pytest.mark.parametrize("key", CASES)
def test_corpus_kernel_compiles_for_sm100a(key):
    unsafe = str(G[f"{key}_mode"]) == "unsafe"
    m = adc.JitModule(MODULE, str(G[f"{key}_kernel"]), unsafe=unsafe)
    assert m.cubin_size > 1000
    src = m.cuda_source
    # one IEEE op per DSL op, no contraction: only the _rn intrinsics do arithmetic
    assert "__dadd_rn" in src or "__dmul_rn" in src
    assert "__fma" not in src and "fma(" not in src
    if unsafe:
        assert "adc_st_add_atomic(" in src


@pytest.mark.parametrize("key", ["gsum", "sumn"])
def test_hazard_refused_with_reference_message(key):
    with pytest.raises(adc.AdcError) as e:
        adc.JitModule(MODULE, str(G[f"{key}_kernel"]))
    assert e.value.kind == "Launch"
    assert str(e.value) == str(G[f"{key}_refused"])


def test_params_and_kinds():
    m = adc.JitModule(MODULE, "k_looped")
    assert m.params == [("x", "real[]"), ("n", "integer"), ("dx", "real[]")]


@pytest.mark.parametrize("src,kind", [
    ("global void k(real[] x) { integer i = blockIdx * blockDim + threadIdx; if (i < N) { "
     "nothere(x[i]); } }", "Semantic"),
    ("global void k(real[] x) { x[0] += $; }", "Semantic"),
    ("device host real f(real x) { return y; }\nglobal void k() { }", "Semantic"),
])
def test_bad_modules_are_semantic_errors(src, kind):
    with pytest.raises(adc.AdcError) as e:
        adc.JitModule(src, "k")
    assert e.value.kind == kind


def test_unknown_and_non_global_kernels():
    with pytest.raises(adc.AdcError) as e:
        adc.JitModule(MODULE, "nope")
    assert e.value.kind == "Launch" and "unknown kernel" in str(e.value)
    with pytest.raises(adc.AdcError) as e:
        adc.JitModule(MODULE, "rational_grad")
    assert "not a global kernel" in str(e.value)


def test_launch_without_device_has_no_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except ImportError:
        pass
    m = adc.JitModule(MODULE, "k_poly")
    n = 8
    bufs = adc.BufferSet(arrays={k: np.zeros(n) for k in ("x", "y", "dx", "dy")})
    with pytest.raises(adc.AdcError) as e:
        m.launch(adc.LaunchConfig(1, 8, n), bufs)
    assert e.value.kind == "Cuda"


def test_dsl_names_that_clash_with_cuda_or_emitter_names():
    # DSL identifiers are prefixed in the emitted CUDA: names like tape, ctx,
    # cp, double or threadIdx-lookalikes cannot collide with the emitter's own.
    src = """device host void f_grad(real tape, real ctx, integer cp, real[] _d_tape, real[] double) {
  real tp = 0;
  __push(tp);
  tp = tape * ctx;
  _d_tape[0] += ctx;
  double[0] += tape * cp;
  tp = __pop();
}
global void k(real[] x, real[] y, real[] dx, real[] dy) {
  integer i = blockIdx * blockDim + threadIdx;
  if (i < N) {
    f_grad(x[i], y[i], 3, dx[i], dy[i]);
  }
}
"""
    m = adc.JitModule(src, "k")
    assert m.cubin_size > 0 and "v_double" in m.cuda_source


def _fn_body(src, prefix):
    """The definition text of the first device function whose name starts with prefix."""
    i = src.index("__device__ void " + prefix)
    i = src.index("{", src.index(")", i))
    j = src.index("\n}\n", i)
    return src[i:j]


def test_static_tape_straight_line_and_branches():
    """Tape elimination: branchy_grad's value and control
    tapes sit at compile-time depths (both branches push one of each), so the
    launch variant keeps them in locals — no per-frame tape arrays."""
    m = adc.JitModule(MODULE, "k_branchy")
    src = m.static_source()
    assert src is not None
    body = _fn_body(src, "fn_branchy_grad_s")
    assert "_tv0 = v__ret0;" in body and "v__ret0 = _tv0;" in body
    assert "_tc0 = (long long)1;" in body and "long long v__c0 = _tc0;" in body
    assert "adc_push" not in body and "adc_pop" not in body and "tape[" not in body


def test_static_tape_unrolls_constant_trip_counts():
    """looped_grad pushes a data-dependent 1 or 2 values per iteration; with
    the trip count n a specialised integer argument the loop is unrolled and
    every push gets its own slot (2 per iteration, the branches padded), the
    reverse loop reads them back in mirrored order.  Division by the literal 2
    is the exact multiply by 0.5."""
    m = adc.JitModule(MODULE, "k_looped")
    body = _fn_body(m.static_source([10]), "fn_looped_grad_s")
    assert "adc_push" not in body and "adc_pop" not in body and "tape[" not in body
    assert body.count("_tc") and "double _tv19 = 0.0;" in body and "_tv20" not in body
    assert "__dmul_rn(v_s, 0.5)" in body and "adc_div(v_s" not in body
    # beyond the static slot bound (300 iterations) the dynamic tape stays
    assert m.static_source([300]) is None
    # kernels without integer parameters need no specialisation
    assert adc.JitModule(MODULE, "k_rational").static_source() is not None


def test_static_tape_falls_back_on_pop_underflow():
    src = ("device host void f(real x, real[] _d_x) {\n  real a = __pop();\n  _d_x[0] += a;\n}\n"
           "global void k(real[] x, real[] dx) {\n  integer i = blockIdx * blockDim + threadIdx;\n"
           "  if (i < N) {\n    f(x[i], dx[i]);\n  }\n}\n")
    m = adc.JitModule(src, "k")
    s = m.static_source()
    # the kernel frame is static, the callee keeps the dynamic tape (its run-time
    # underflow error is the interpreter's)
    assert s is not None and "adc_pop(tape, tp, ctx)" in s


def test_vector_listing1_kernel_is_emitted():
    """Listing-1 kernels (one call of a slot-only gradient at the thread
    index) get a vector form — two points per thread, 16-byte accesses —
    through a register-slot variant of the gradient; the others do not."""
    m = adc.JitModule(MODULE, "k_rational")
    src = m.static_source()
    assert "adc_kernel_k_rational_v2" in src and "double& c_v__d_x" in src
    looped = adc.JitModule(MODULE, "k_looped").static_source([10])
    assert "adc_kernel_k_looped_v2" in looped
    # a whole-array slot (sumn_grad(x, n, dx)) is not a Listing-1 slot call
    sumn = adc.JitModule(MODULE, "k_sumn", unsafe=True).static_source([64])
    assert sumn is None or "k_sumn_v2" not in sumn
