"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/ref_tool,
built by `make -C oracle` from /root/reference/proj/src).  Run here, in the
container that has /root/reference; the committed .npz files are what the
tests read (the GPU box has no /root/reference).

    python tests/golden/make_golden.py

Every fixture stores the inputs and the reference outputs side by side.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2203_06139_b200 import synth  # noqa: E402

TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
OUT = os.path.dirname(os.path.abspath(__file__))


def run(*args):
    r = subprocess.run([TOOL, *map(str, args)], check=True, capture_output=True, text=True)
    return json.loads(r.stdout.strip().splitlines()[-1]) if r.stdout.strip().startswith("{") else r.stdout


def f64(path, count):
    a = np.fromfile(path, dtype="<f8")
    assert a.size == count, (path, a.size, count)
    return a


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def main():
    tmp = tempfile.mkdtemp()
    ti, to = os.path.join(tmp, "in.bin"), os.path.join(tmp, "out.bin")
    # Fingerprints (FNV-1a 64) of the printed generated gradients: the B200
    # kernel registry is keyed by them (include/adc_cuda.h).  Only the hashes
    # are committed, not the generated text.
    assert run("golden-check")["golden_match"]
    fps = {}
    for mod, fn, wrt in (("kernels", "gauss", ("x", "p")), ("kernels", "gauss", ("x", "p", "sigma")),
                         ("gaussnd", "gaussnd", ("x", "p")),
                         ("gpoly", "gpoly", ("q",)), ("gsum", "gsum", ("q",))):
        text = run("print", mod, fn, *wrt)
        name = text.split("(")[0].split()[-1]
        fps[name] = f"0x{fnv1a64(text.encode()):016x}"
    with open(os.path.join(OUT, "gradient_fingerprints.json"), "w") as fh:
        json.dump(fps, fh, indent=1, sort_keys=True)
        fh.write("\n")

    # Listing 1 / criterion 5: N=512, seed 0x5EED, sigma 1.3, grid 3 x 256.
    meta = run("gauss1d", 512, "0x5EED", 1.3, 256, to)
    a = f64(to, 4 * 512).reshape(4, 512)
    np.savez(os.path.join(OUT, "gauss1d_n512.npz"), x=a[0], p=a[1], dx=a[2], dp=a[3], sigma=1.3,
             grid=meta["grid"], block=256, active=meta["active"], idle=meta["idle"])

    # KAT gauss(1,0,1) (test_reverse.cpp:69-82) + ragged accumulate case.
    cases = {}
    rng = np.random.Generator(np.random.PCG64(7))
    for name, n, sigma, block, x, p, dx0, dp0 in (
        ("kat", 1, 1.0, 1, np.array([1.0]), np.array([0.0]), np.zeros(1), np.zeros(1)),
        ("accum300", 300, 0.7, 128, rng.uniform(-3, 3, 300), rng.uniform(-2, 2, 300),
         rng.standard_normal(300), rng.standard_normal(300)),
        ("edges", 6, 1.3, 32, np.array([0.0, -0.0, 1e-300, 5.0, -40.0, 2.0]),
         np.array([0.0, 0.0, 0.0, -5.0, 40.0, 2.0]), np.array([-0.0, 0.0, 1.0, 0.0, 0.0, -0.0]),
         np.zeros(6)),
    ):
        np.concatenate([x, p, dx0, dp0]).astype("<f8").tofile(ti)
        run("gauss1d-in", n, sigma, block, ti, to)
        o = f64(to, 2 * n).reshape(2, n)
        cases[name] = dict(x=x, p=p, dx0=dx0, dp0=dp0, dx=o[0], dp=o[1], sigma=sigma, block=block)
    np.savez(os.path.join(OUT, "gauss1d_cases.npz"),
             **{f"{k}_{f}": v for k, d in cases.items() for f, v in d.items()})

    # compute_shared (kernels.dsl:16-21): refused by default, forced sequential
    # point-order accumulation into the shared dsigma slot.
    sh = {}
    for name, n, sigma, block, seed in (("n100", 100, 1.3, 32, 21), ("n4097", 4097, 0.9, 256, 22)):
        r = np.random.Generator(np.random.PCG64(seed))
        x, p = r.uniform(-3, 3, n), r.uniform(-2, 2, n)
        dx0, dp0, ds0 = r.standard_normal(n), r.standard_normal(n), np.array([0.25])
        np.concatenate([x, p, dx0, dp0, ds0]).astype("<f8").tofile(ti)
        meta = run("gauss-shared-in", n, sigma, block, ti, to)
        assert meta["refused_by_default"]
        o = f64(to, 2 * n + 1)
        sh.update({f"{name}_x": x, f"{name}_p": p, f"{name}_dx0": dx0, f"{name}_dp0": dp0,
                   f"{name}_dsigma0": ds0, f"{name}_dx": o[:n], f"{name}_dp": o[n:2 * n],
                   f"{name}_dsigma": o[2 * n:], f"{name}_sigma": sigma, f"{name}_block": block})
    np.savez(os.path.join(OUT, "gauss_shared_cases.npz"), **sh)

    # Generic lowering: Listing-style kernels (oracle/dsl/jit_kernels.dsl) over
    # the reference corpus gradients, run by the reference's own adc::launch;
    # the printed module (what the B200 JIT consumes) is stored with them.
    corpus = "/root/reference/proj/corpus"
    dsl = os.path.join(tmp, "jit.dsl")
    with open(dsl, "w") as fh:
        for name in ("gauss", "rational", "branchy", "poly", "looped", "gsum", "sumn"):
            fh.write(open(os.path.join(corpus, name + ".dsl")).read() + "\n")
        fh.write(open(os.path.join(ROOT, "oracle", "dsl", "jit_kernels.dsl")).read())
    r = np.random.Generator(np.random.PCG64(77))
    n = 1000
    ji, module_text = {}, None
    cases = (
        ("gauss", "k_gauss", n, [r.uniform(-3, 3, n), r.uniform(-2, 2, n), 1.3,
                                 r.standard_normal(n), r.standard_normal(n)], ""),
        ("rational", "k_rational", n, [r.uniform(-2, 2, n), r.uniform(-2, 2, n), np.zeros(n),
                                      np.zeros(n)], ""),
        ("branchy", "k_branchy", n, [r.uniform(-4, 4, n), r.uniform(-4, 4, n), np.zeros(n),
                                    r.standard_normal(n)], ""),
        ("poly", "k_poly", n, [r.uniform(-2, 2, n), r.uniform(-2, 2, n), np.zeros(n),
                              np.zeros(n)], ""),
        ("looped", "k_looped", n, [r.uniform(-2, 3, n), 10, np.zeros(n)], ""),
        ("gsum", "k_gsum", 500, [r.uniform(-5, 5, 500), np.array([1.0, 0.0, 1.5, 0.5, 1.0, 0.7]),
                                 2, np.zeros(6)], "unsafe"),
        ("sumn", "k_sumn", 200, [r.uniform(-1, 1, 64), 64, np.zeros(64)], "unsafe"),
        ("hess", "k_hess", n, [r.uniform(-3, 3, n), r.uniform(-2, 2, n), 1.3, np.zeros(n),
                               np.zeros(n), np.zeros(n), np.zeros(n)], ""),
        ("gauss_div0", "k_gauss", 64, [np.ones(64), np.zeros(64), 0.0, np.zeros(64),
                                       np.zeros(64)], "sequential"),
        ("iovf", "k_iovf", 64, [np.ones(64), 3037000500, np.zeros(64)], "sequential"),
        # deeper than the JIT's default 256-entry tapes: the host path grows them
        ("looped_deep", "k_looped", 300, [r.uniform(-2, 3, 300), 300, np.zeros(300)], ""),
    )
    for key, kern, nn, params, mode in cases:
        flat = []
        for v in params:
            if isinstance(v, np.ndarray):
                flat += [float(v.size)] + list(v)
            else:
                flat.append(float(v))
        np.array(flat, dtype="<f8").tofile(ti)
        mod = os.path.join(tmp, "module.txt")
        meta = run("launch-file", dsl, kern, nn, 256, ti, to, mod, *([mode] if mode else []))
        text = open(mod).read()
        assert module_text in (None, text)
        module_text = text
        arrays = [v for v in params if isinstance(v, np.ndarray)]
        o = f64(to, sum(a.size for a in arrays))
        outs, off = [], 0
        for a in arrays:
            outs.append(o[off:off + a.size])
            off += a.size
        ji[f"{key}_kernel"] = kern
        ji[f"{key}_n"] = nn
        ji[f"{key}_mode"] = mode
        ji[f"{key}_error"] = meta["error"]
        # LaunchStats: OpCounters over all threads (adds, muls, divs, intrinsics,
        # comparisons, tape_pushes, tape_pops) and per-thread statements
        ji[f"{key}_counts"] = np.array(meta["counts"], dtype=np.int64)
        ji[f"{key}_stm"] = np.array(meta["stm"], dtype=np.uint32)
        ji[f"{key}_nparams"] = len(params)
        for i, v in enumerate(params):
            ji[f"{key}_in{i}"] = np.asarray(v, dtype=np.float64)
        for i, v in enumerate(outs):
            ji[f"{key}_out{i}"] = v
    # the reference's refusal of the hazardous kernels (no unsafe flag)
    for key in ("gsum", "sumn"):
        flat = []
        for v in [ji[f"{key}_in{i}"] for i in range(ji[f"{key}_nparams"])]:
            flat += [float(v.size)] + list(v) if v.ndim else [float(v)]
        np.array(flat, dtype="<f8").tofile(ti)
        meta = run("launch-file", dsl, ji[f"{key}_kernel"], ji[f"{key}_n"], 256, ti, to,
                   os.path.join(tmp, "m2.txt"))
        ji[f"{key}_refused"] = meta["error"]
    ji["module"] = module_text
    np.savez(os.path.join(OUT, "jit_cases.npz"), **ji)

    # N-dim Gaussian, SoA layout, nonzero initial slots (accumulate semantics).
    nd = {}
    for dim, n, seed in ((100, 64, 11), (1000, 8, 12), (1, 33, 13), (37, 70, 14), (128, 40, 15),
                         (129, 5, 16)):
        x, p = synth.points_nd(dim, n, seed=seed)
        r = np.random.Generator(np.random.PCG64(seed + 100))
        dx0 = r.standard_normal((dim, n)) * 1e-3
        dp0 = r.standard_normal((dim, n)) * 1e-3
        sigma = 1.3
        np.concatenate([x.ravel(), p.ravel(), dx0.ravel(), dp0.ravel()]).astype("<f8").tofile(ti)
        run("gaussnd-in", dim, n, sigma, ti, to)
        o = f64(to, 2 * dim * n).reshape(2, dim, n)
        key = f"d{dim}_n{n}"
        nd.update({f"{key}_x": x, f"{key}_p": p, f"{key}_dx0": dx0, f"{key}_dp0": dp0,
                   f"{key}_dx": o[0], f"{key}_dp": o[1], f"{key}_sigma": sigma})
    np.savez(os.path.join(OUT, "gaussnd_cases.npz"), **nd)

    # Shared mean vector: one p, one dp slot for every point (points in order).
    sp = {}
    for dim, n, seed in ((100, 64, 31), (37, 150, 32), (1, 40, 33), (300, 33, 34)):
        x, _ = synth.points_nd(dim, n, seed=seed)
        r = np.random.Generator(np.random.PCG64(seed + 200))
        p = r.uniform(-2, 2, dim)
        x = p[:, None] + 0.1 * r.standard_normal((dim, n))
        dx0 = r.standard_normal((dim, n)) * 1e-3
        dp0 = r.standard_normal(dim) * 1e-3
        np.concatenate([x.ravel(), p, dx0.ravel(), dp0]).astype("<f8").tofile(ti)
        run("gaussnd-shared-p-in", dim, n, 1.3, ti, to)
        o = f64(to, dim * n + dim)
        key = f"d{dim}_n{n}"
        sp.update({f"{key}_x": x, f"{key}_p": p, f"{key}_dx0": dx0, f"{key}_dp0": dp0,
                   f"{key}_dx": o[:dim * n].reshape(dim, n), f"{key}_dp": o[dim * n:]})
    np.savez(os.path.join(OUT, "gaussnd_shared_p_cases.npz"), **sp)

    # chi2 value + gradient (fit.cpp:206-259) for gpoly and gsum K=1,2.
    ch = {}
    for key, model, bins, events, qtrue, q in (
        ("gpoly_b2000", "gpoly", 2000, 1e6, synth.GPOLY_TRUTH, synth.GPOLY_INIT),
        ("gsum1_b1000", "gsum", 1000, 1e5, (1.0, 0.0, 1.5), (0.8, 0.3, 1.2)),
        ("gsum2_b1500", "gsum", 1500, 2e5, (1.0, -5 / 3, 1.5, 1.0, 5 / 3, 1.0),
         (0.8, -1.3666666666666667, 1.2, 0.8, 1.9666666666666668, 0.8)),
    ):
        counts, ev = synth.histogram(bins, -5.0, 5.0, events, model, qtrue, seed=bins)
        counts.astype("<f8").tofile(ti)
        meta = run("chi2-in", model, bins, -5.0, 5.0, ti, to, 1, *[repr(float(v)) for v in q])
        assert meta["fitengine_match"]
        o = f64(to, 1 + len(q))
        ch.update({f"{key}_counts": counts, f"{key}_q": np.array(q, dtype=np.float64),
                   f"{key}_chi2": o[0], f"{key}_grad": o[1:], f"{key}_events": ev,
                   f"{key}_model": model})
    np.savez(os.path.join(OUT, "chi2_cases.npz"), **ch)

    # GradientProvider::Numeric (fit.cpp:187-190 -> central_gradient,
    # numdiff.cpp:38-87): chi2 gradient and a short fit, per model.
    nu = {}
    for key, model, bins, events, qtrue, q in (
        ("gpoly_b2000", "gpoly", 2000, 1e6, synth.GPOLY_TRUTH, synth.GPOLY_INIT),
        ("gsum1_b1000", "gsum", 1000, 1e5, (1.0, 0.0, 1.5), (0.8, 0.3, 1.2)),
        ("gsum2_b1500", "gsum", 1500, 2e5, (1.0, -5 / 3, 1.5, 1.0, 5 / 3, 1.0),
         (0.8, -1.3666666666666667, 1.2, 0.8, 1.9666666666666668, 0.8)),
    ):
        counts, ev = synth.histogram(bins, -5.0, 5.0, events, model, qtrue, seed=bins)
        counts.astype("<f8").tofile(ti)
        meta = run("chi2-in", model + ":numeric", bins, -5.0, 5.0, ti, to, 1,
                   *[repr(float(v)) for v in q])
        assert meta["fitengine_match"]
        o = f64(to, 1 + len(q))
        nu.update({f"{key}_counts": counts, f"{key}_q": np.array(q, dtype=np.float64),
                   f"{key}_grad": o[1:], f"{key}_events": ev, f"{key}_model": model})
        meta = run("fit-in", model + ":numeric", bins, -5.0, 5.0, ti, to, 10, "12",
                   *[repr(float(v)) for v in q])
        assert meta["fitengine_match"]
        np_ = len(q)
        o = f64(to, 5 + np_ + 10 * np_)
        nu.update({f"{key}_fit_chi2": o[0], f"{key}_fit_iterations": o[1],
                   f"{key}_fit_params": o[5:5 + np_],
                   f"{key}_fit_iterates": o[5 + np_:].reshape(10, np_)})
    np.savez(os.path.join(OUT, "chi2_numeric_cases.npz"), **nu)

    # Fit loop iterates (fit.cpp:315-425), trace 10, budget 12.
    fi = {}
    for key, model, bins, events, qtrue, q, budget in (
        ("gpoly_b400", "gpoly", 400, 2e5, synth.GPOLY_TRUTH, synth.GPOLY_INIT, "12"),
        ("gsum1_b300", "gsum", 300, 1e5, (1.0, 0.0, 1.5), (0.8, 0.3, 1.2), "12"),
        ("gpoly_b400_hess", "gpoly", 400, 2e5, synth.GPOLY_TRUTH, synth.GPOLY_INIT, "12:hess"),
        ("gsum1_b300_hess", "gsum", 300, 1e5, (1.0, 0.0, 1.5), (0.8, 0.3, 1.2), "12:hess"),
    ):
        counts, ev = synth.histogram(bins, -5.0, 5.0, events, model, qtrue, seed=bins + 1)
        counts.astype("<f8").tofile(ti)
        meta = run("fit-in", model, bins, -5.0, 5.0, ti, to, 10, budget,
                   *[repr(float(v)) for v in q])
        assert meta["fitengine_match"]
        np_ = len(q)
        o = f64(to, 5 + np_ + 10 * np_)
        fi.update({f"{key}_counts": counts, f"{key}_init": np.array(q, dtype=np.float64),
                   f"{key}_chi2": o[0], f"{key}_iterations": o[1], f"{key}_gradient_evals": o[2],
                   f"{key}_converged": o[3], f"{key}_sigma_clamps": o[4],
                   f"{key}_params": o[5:5 + np_], f"{key}_iterates": o[5 + np_:].reshape(10, np_),
                   f"{key}_model": model, f"{key}_hessian": budget.endswith(":hess")})
    np.savez(os.path.join(OUT, "fit_cases.npz"), **fi)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
