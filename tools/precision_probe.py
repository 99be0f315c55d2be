"""Precision probe (perf/numerics experiment, not a test): fp32 vs fp64 drift
and fp64 sensitivity to a 1e-9 perturbation of the init, per iteration count."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2602_14683_b200 as ntf
from paper_2602_14683_b200 import io as nio
from oracle import ntf_oracle as O


def rel_model(a, b):
    return max(O.rel_err(x, y) for x, y in zip(a, b))


def per_factor(a, b):
    return " ".join(f"{O.rel_err(x, y):.1e}" for x, y in zip(a, b))


def run(tag, dims, rank, betas, iters_list, inner=5):
    x = nio.generate_cp_gamma(dims, rank, seed=0)
    init = nio.cp_factors(dims, rank, seed=1, which="init")
    rng = np.random.default_rng(7)
    pert = [a * (1 + 1e-9 * rng.standard_normal(a.shape)) for a in init]
    ctx = ntf.Context(0)
    for beta in betas:
        for it in iters_list:
            t0 = time.perf_counter()
            r64 = ntf.jcomm_fit(x, init, ntf.FitConfig(beta=beta, rank=rank, inner_steps=inner, max_iters=it), ctx=ctx)
            ctx.trim()
            r64p = ntf.jcomm_fit(x, pert, ntf.FitConfig(beta=beta, rank=rank, inner_steps=inner, max_iters=it), ctx=ctx)
            ctx.trim()
            r32 = ntf.jcomm_fit(x, init, ntf.FitConfig(beta=beta, rank=rank, inner_steps=inner, max_iters=it,
                                                       precision="f32"), ctx=ctx)
            ctx.trim()
            tr = lambda r: np.array([t.loss for t in r.trace])
            print(f"{tag} beta={beta} it={it}: f32-f64 factors {rel_model(r32.model, r64.model):.2e} "
                  f"[{per_factor(r32.model, r64.model)}] trace {O.rel_err(tr(r32), tr(r64)):.2e} | "
                  f"pert1e-9 factors {rel_model(r64p.model, r64.model):.2e} trace {O.rel_err(tr(r64p), tr(r64)):.2e} "
                  f"| loss {r64.trace[-1].loss:.6f} ({time.perf_counter()-t0:.1f}s)", flush=True)
    del x
    torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if which == "c2q":  # quick: beta 1 and 0.5, 10 and 100 outer
        run("C2", (512,) * 3, 32, [1.0, 0.5], [10, 100])
    elif which == "c5q":
        run("C5", (256,) * 4, 64, [0.5], [3])
    elif which == "c2":
        run("C2", (512,) * 3, 32, [1.0, 0.5, 0.0, 1.5], [1, 2, 5, 10, 20, 50, 100])
    elif which == "c5":
        run("C5", (256,) * 4, 64, [0.5], [1, 2, 3, 5])
