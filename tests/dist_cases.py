"""Cases of the data-parallel engine tests (shared by tests/dist_worker.py and
tests/test_dist_gpu.py).  Seeded, small, every beta; CP B-CoMM / J-CoMM with
and without BMMe extrapolation, one fp32 tensor-core shape; Tucker B-CoMM /
J-CoMM."""
import numpy as np

import paper_2602_14683_b200 as ntf


def _cfg(algo, **kw):
    c = ntf.FitConfig(**kw)
    c.algo = algo
    return c


def _cp(dims, rank, seed):
    rng = np.random.default_rng(seed)
    truth = [rng.random((d, rank)) for d in dims]
    x = np.einsum("ir,jr,kr->ijk", *truth) * rng.gamma(10.0, 0.1, size=dims)
    init = [0.1 + rng.random((d, rank)) for d in dims]
    return x, init


def _tucker(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.random(ranks)
    fs = [rng.random((d, j)) for d, j in zip(dims, ranks)]
    x = np.einsum("abc,ia,jb,kc->ijk", core, *fs) * rng.gamma(10.0, 0.1, size=dims)
    return x, (0.1 + rng.random(ranks), [0.1 + rng.random((d, j)) for d, j in zip(dims, ranks)])


def cases():
    out = {}
    x, init = _cp((24, 20, 16), 5, 11)
    for algo in ("bcomm", "jcomm"):
        for beta in (0.0, 0.5, 1.0, 1.5):
            out[f"cp_{algo}_{beta}"] = (x, init, _cfg(algo, beta=beta, rank=5, max_iters=6, inner_steps=3), "cp")
        out[f"cp_{algo}_extrap"] = (x, init, _cfg(algo, beta=0.5, rank=5, max_iters=6, inner_steps=3,
                                                  extrapolate=True, extrap_cap=5.0), "cp")
    x4, init4 = _cp((10, 9, 8), 4, 12)
    out["cp_jcomm_order3_odd"] = (x4, init4, _cfg("jcomm", beta=1.0, rank=4, max_iters=5, inner_steps=2), "cp")
    # fp32 streaming build with the tcgen05 contraction (K % 128 == 0)
    xt, initt = _cp((32, 16, 128), 8, 13)
    out["cp_jcomm_f32_tc"] = (xt.astype(np.float32).astype(np.float64), initt,
                              _cfg("jcomm", beta=0.5, rank=8, max_iters=4, inner_steps=3, precision="f32"), "cp")
    xk, initk = _tucker((18, 14, 12), (3, 4, 2), 14)
    for algo in ("bcomm", "jcomm"):
        for beta in (0.5, 1.0):
            out[f"tk_{algo}_{beta}"] = (xk, initk, _cfg(algo, beta=beta, ranks=[3, 4, 2], max_iters=5,
                                                        inner_steps=2), "tucker")
    out["tk_bcomm_extrap"] = (xk, initk, _cfg("bcomm", beta=0.5, ranks=[3, 4, 2], max_iters=5, extrapolate=True,
                                              extrap_cap=5.0), "tucker")
    # sparse COO (beta = 1): nonzeros partitioned by mode-0 index ranges
    rng = np.random.default_rng(15)
    cd = (20, 9, 12, 15)
    nnz = 2500
    idx = np.stack([rng.integers(0, d, size=nnz) for d in cd], axis=1).astype(np.int32)
    idx[1::7] = idx[0::7][: len(idx[1::7])]  # duplicates (accumulate on ingestion)
    val = rng.geometric(0.5, size=nnz).astype(np.float64)
    cinit = [0.1 + rng.random((d, 4)) for d in cd]
    for algo in ("bcomm", "jcomm"):
        out[f"coo_{algo}"] = ((idx, val, cd), cinit, _cfg(algo, beta=1.0, rank=4, max_iters=5, inner_steps=3), "coo")
    out["coo_jcomm_extrap"] = ((idx, val, cd), cinit, _cfg("jcomm", beta=1.0, rank=4, max_iters=5, inner_steps=2,
                                                           extrapolate=True, extrap_cap=5.0), "coo")
    return out
