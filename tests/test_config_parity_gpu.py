"""Parity at the BASELINE.json configs' own sizes (VERDICT r01 "next" item 1).

* C1 (configs[0]): the GPU fp64 B-CoMM fit, 200 iterations on the exact C1
  problem, against the COMPILED REFERENCE's own 200-iteration run stored in
  tests/golden/c1_bcomm.npz (tests/golden/make_golden.py) -- 1e-10.
* C2 (configs[1], 512^3, R=32, J-CoMM L=5, 100 outer, every beta): the fp32
  streaming build (tcgen05 contraction, bf16 hi/lo P~/Q~ planes) against the
  fp64 validation build on the same device-resident data -- factors 1e-4,
  every trace row 1e-5 (north star; rel_err of reference
  tests/test_support.hpp:17-19).  The fp64 build is itself pinned to the
  oracle at small sizes (test_cp_gpu.py) and, at full size, by:
* a short-horizon check: ONE J-CoMM outer iteration at full C2 size from an
  identical state, GPU (fp64 and fp32) vs oracle/_ref (the compiled unmodified
  reference, cp.cpp:271-298) -- separates kernel bugs from accumulated drift.
* C5 (configs[4], 256^4, R=64, beta=0.5, J-CoMM L=5, 50 outer): fp32 vs fp64.
* C3 (configs[2], Tucker 256^3, core 16^3, beta in {0.5, 1}, B-CoMM and
  J-CoMM L=3, 100 iterations): fp32 vs fp64.
"""
import os
import sys
import threading

import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def rel_model(a, b):
    return max(O.rel_err(x, y) for x, y in zip(a, b))


def rel_trace(a, b):
    assert len(a) == len(b)
    return max(O.rel_err(np.array([r.loss]), np.array([s.loss])) for r, s in zip(a, b))


def report(tag, **kv):
    print(f"[parity] {tag} " + " ".join(f"{k}={v:.3e}" if isinstance(v, float) else f"{k}={v}"
                                        for k, v in kv.items()), flush=True)


# ---------------------------------------------------------------------------- C1

def test_c1_full_vs_reference_golden():
    import datagen as D
    g = np.load(os.path.join(HERE, "golden", "c1_bcomm.npz"))
    x, init = D.c1_problem(0)
    res = ntf.bcomm_fit(x, init, ntf.FitConfig(beta=1.0, rank=10, max_iters=200, precision="f64"))
    ef = rel_model(res.model, [g[f"c1_f{n}"] for n in range(3)])
    et = O.rel_err(np.array([t.loss for t in res.trace]), g["c1_trace"])
    report("C1 bcomm fp64 200 it vs reference", factors=ef, trace=et)
    assert len(res.trace) == 201
    assert ef < 1e-10 and et < 1e-10


# ---------------------------------------------------------------------------- C2

C2_DIMS = (512, 512, 512)


@pytest.fixture(scope="module")
def c2_data():
    from paper_2602_14683_b200 import io as nio
    x = nio.generate_cp_gamma(C2_DIMS, 32, seed=0)
    init = nio.cp_factors(C2_DIMS, 32, seed=1, which="init")
    yield x, init
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_c2_full_f32_vs_f64(c2_data, beta):
    x, init = c2_data
    ctx = ntf.Context(0)
    out = {}
    for prec in ("f64", "f32"):
        cfg = ntf.FitConfig(beta=beta, rank=32, inner_steps=5, max_iters=100, precision=prec)
        out[prec] = ntf.jcomm_fit(x, init, cfg, ctx=ctx)
        ctx.trim()
    ef = rel_model(out["f32"].model, out["f64"].model)
    et = rel_trace(out["f32"].trace, out["f64"].trace)
    report(f"C2 beta={beta} f32 vs f64 100 outer", factors=ef, trace=et,
           loss=out["f64"].trace[-1].loss)
    assert len(out["f32"].trace) == 101
    assert ef < 1e-4 and et < 1e-5


def test_c2_one_outer_vs_reference(c2_data):
    """One full-size J-CoMM outer iteration per beta, GPU vs oracle/_ref."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    x, init = c2_data
    xh = x.double().cpu().numpy()
    betas = [0.0, 0.5, 1.0, 1.5]
    ref = {}

    def run(b):
        f, _, tl = R.cp_fit("jcomm", xh, init, b, max_iters=1, inner_steps=5)
        ref[b] = (f, tl)

    th = [threading.Thread(target=run, args=(b,)) for b in betas]
    for t in th:
        t.start()
    got = {}
    ctx = ntf.Context(0)
    for b in betas:  # GPU runs overlap the CPU reference threads (ctypes drops the GIL)
        for prec in ("f64", "f32"):
            got[(b, prec)] = ntf.jcomm_fit(x, init, ntf.FitConfig(beta=b, rank=32, inner_steps=5, max_iters=1,
                                                                  precision=prec), ctx=ctx)
    for t in th:
        t.join()
    for b in betas:
        f, tl = ref[b]
        for prec, (tf, tt) in (("f64", (1e-10, 1e-10)), ("f32", (1e-4, 1e-5))):
            g = got[(b, prec)]
            ef = rel_model(g.model, f)
            et = O.rel_err(np.array([t.loss for t in g.trace]), tl)
            report(f"C2 beta={b} {prec} 1 outer vs oracle/_ref", factors=ef, trace=et)
            assert ef < tf and et < tt, (b, prec, ef, et)


# ---------------------------------------------------------------------------- C5

def test_c5_full_f32_vs_f64():
    from paper_2602_14683_b200 import io as nio
    dims = (256,) * 4
    iters = int(os.environ.get("NTFG_C5_PARITY_ITERS", "50"))
    x = nio.generate_cp_gamma(dims, 64, seed=0)
    init = nio.cp_factors(dims, 64, seed=1, which="init")
    ctx = ntf.Context(0)
    out = {}
    import time
    for prec in ("f32", "f64"):
        t0 = time.perf_counter()
        cfg = ntf.FitConfig(beta=0.5, rank=64, inner_steps=5, max_iters=iters, precision=prec)
        out[prec] = ntf.jcomm_fit(x, init, cfg, ctx=ctx)
        ctx.trim()
        torch.cuda.empty_cache()
        report(f"C5 {prec} fit", seconds=time.perf_counter() - t0)
    del x
    torch.cuda.empty_cache()
    ef = rel_model(out["f32"].model, out["f64"].model)
    et = rel_trace(out["f32"].trace, out["f64"].trace)
    report(f"C5 f32 vs f64 {iters} outer", factors=ef, trace=et, loss=out["f64"].trace[-1].loss)
    assert ef < 1e-4 and et < 1e-5


# ---------------------------------------------------------------------------- C3

def c3_problem(seed=0, dims=(256, 256, 256), ranks=(16, 16, 16)):
    """configs[2]: core, factors ~ U[0,1); X = Tucker reconstruction * Gamma(10, 0.1);
    init U[0.1, 1.1).  Generated on the device with seeded torch generators."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    core = torch.rand(ranks, generator=g, dtype=torch.float64)
    fs = [torch.rand(d, j, generator=g, dtype=torch.float64) for d, j in zip(dims, ranks)]
    dev = torch.device("cuda", 0)
    x = torch.einsum("abc,ia,jb,kc->ijk", core.to(dev), fs[0].to(dev), fs[1].to(dev), fs[2].to(dev))
    gc = torch.Generator(device=dev).manual_seed(seed + 7)
    noise = torch._standard_gamma(torch.full(dims, 10.0, device=dev, dtype=torch.float64), generator=gc) * 0.1
    x = (x * noise).float().contiguous()
    rng = np.random.default_rng(seed + 1)
    icore = 0.1 + rng.random(ranks)
    ifs = [0.1 + rng.random((d, j)) for d, j in zip(dims, ranks)]
    return x, (icore, ifs)


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_c3_full_f32_vs_f64(algo, beta):
    x, init = c3_problem(0)
    fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    ctx = ntf.Context(0)
    out = {}
    for prec in ("f64", "f32"):
        cfg = ntf.FitConfig(beta=beta, ranks=[16, 16, 16], inner_steps=3, max_iters=100, precision=prec)
        out[prec] = fit(x, init, cfg, ctx=ctx)
    (c32, f32), (c64, f64) = out["f32"].model, out["f64"].model
    ef = max(O.rel_err(c32, c64), rel_model(f32, f64))
    et = rel_trace(out["f32"].trace, out["f64"].trace)
    report(f"C3 tucker {algo} beta={beta} f32 vs f64 100 it", factors=ef, trace=et,
           s_f32=out["f32"].trace[-1].time_s, s_f64=out["f64"].trace[-1].time_s)
    assert ef < 1e-4 and et < 1e-5
